"""Interleaved A/B of the router forms (CUDA-core fp64 DFMA, FP64 tensor-core DMMA, bf16
tensor-core with the guard band and fp64 fix-up) at C2 and C3 shapes, CUDA-event timed on the
launching stream, plus an identity check of their routing (indices, counts, weights, l_aux)."""
import os
import sys

sys.path.insert(0, ".")
import torch

import paper_2304_11414_b200 as P
from paper_2304_11414_b200 import _ops

dev = torch.device("cuda", 0)
for name, h, e, k in (("C2", 4096, 8, 2), ("C3", 8192, 16, 2)):
    n = 16384
    x = P.Rng(1, 99).normal_tensor((n, h), dtype=torch.bfloat16, device=dev)
    wg = P.GateParams.init(h, e, P.Rng(0).spawn(1), device=dev).wg.detach()
    res = {}
    outs = {}
    for rep in range(6):
        for mode in ("dfma", "dmma", "tc"):
            os.environ["PPMOE_ROUTER"] = mode
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                rt = _ops.route(x, wg, k)
            b.record()
            torch.cuda.synchronize()
            if rep > 0:
                res.setdefault(mode, []).append(a.elapsed_time(b) / 20)
            outs[mode] = rt
    med = {m: sorted(v)[len(v) // 2] * 1e3 for m, v in res.items()}
    same = all(torch.equal(getattr(outs["dfma"], f), getattr(outs[m], f)) for f in ("idx", "top1_counts")
               for m in outs)
    wdiff = max(float((outs["dfma"].w - outs[m].w).abs().max()) for m in outs)
    ldiff = max(float((outs["dfma"].l_aux - outs[m].l_aux).abs().max()) for m in outs)
    bytes_ = n * h * 2 + h * e * 4 + n * k * 8
    fix = int(outs["tc"].fixups[0]) if outs["tc"].fixups is not None else -1
    print(f"{name}: tensor-core router re-routed {fix} of {n} tokens in fp64")
    print(f"{name}: router us/call {med}  HBM frac (6528.7 GB/s): "
          f"{ {m: round(bytes_ / (v * 1e-6) / 6528.7e9, 3) for m, v in med.items()} }  idx equal {same}  max|dw| {wdiff:.2e}  max|dl_aux| {ldiff:.2e}")
