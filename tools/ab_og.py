"""Dev tool: owner-gather combine timings (forward form, backward form with the gate term)
at a given shape on one GPU, through the public layer call (the two launches of a step).
usage: python tools/ab_og.py H E [k] (env knobs apply: PPMOE_OG16_U, PPMOE_OG8_U, PPMOE_OG8_CTAS, PPMOE_OG_CTAS)"""
import sys

sys.path.insert(0, ".")
import torch

import paper_2304_11414_b200 as P
from paper_2304_11414_b200 import _ops

h, E = int(sys.argv[1]), int(sys.argv[2])
k = int(sys.argv[3]) if len(sys.argv) > 3 else 2
n = 16384
dev = torch.device("cuda", 0)
x = P.Rng(1, 99).normal_tensor((n, h), dtype=torch.bfloat16, device=dev)
wg = P.GateParams.init(h, E, P.Rng(0).spawn(1), device=dev).wg.detach()
rt = _ops.route(x, wg, k)
pl = _ops.plan(rt.idx, rt.w, E)
rows_cap = _ops.local_rows_cap(n, k, E, pl.capacity)
rows = torch.randn(rows_cap, h, device=dev).bfloat16()
dl = torch.randn(n, E, device=dev) * 1e-3
st = _ops.ExpertFwdState(0, E, rows_cap, pl.seg, None, None, None, None, None, rows)
out = torch.empty(n, h, device=dev, dtype=torch.bfloat16)
for name, args in (("fwd", (rt.w, None, None)), ("bwd+gate", (None, dl, wg))):
    for _ in range(3):
        _ops.local_combine(rows, st, pl, rt.idx, args[0], out, args[1], args[2])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        _ops.local_combine(rows, st, pl, rt.idx, args[0], out, args[1], args[2])
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    nbytes = (int(pl.kept.sum()) + n) * h * 2 + (n * E * 4 if args[1] is not None else 0)
    print(f"h={h} E={E} k={k} {name}: {us:.1f} us, {nbytes / us / 1e6:.2f} TB/s ({nbytes / us / 1e6 / 6.5287:.2f} of HBM)")
