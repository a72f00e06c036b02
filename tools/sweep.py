"""PPMoE vs all-to-all expert-parallel MoE sweep (BASELINE.json configs[4]): tokens 4K-64K,
experts 8/16/32, the GPUs of this torchrun job (1/2/4/8).  h=4096, ffn=16384, top-2, bf16,
random-init weights, N(0,1) tokens.  One JSON line per (tokens, experts) on rank 0 with
both layers' fwd+bwd tokens/s (device time, max over ranks).

usage: python -m torch.distributed.run --nproc-per-node N tools/sweep.py [--tokens ...] [--experts ...]
       (or plain `python tools/sweep.py` for one GPU)
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import paper_2304_11414_b200 as P


def timed(fn, steps, warmup, dev, distributed):
    for _ in range(warmup):
        fn()
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / steps], device=dev, dtype=torch.float64)
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, nargs="+", default=[4096, 8192, 16384, 32768, 65536])
    ap.add_argument("--experts", type=int, nargs="+", default=[8, 16, 32])
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--top-k", type=int, default=2)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    distributed = ws > 1
    if distributed:
        dist.init_process_group("nccl", device_id=dev)
    world = P.World(1, ws, distributed=distributed)
    group = P.ProcessGroup(P.EP, tuple(range(ws)))
    h, k = a.hidden, a.top_k
    for E in a.experts:
        if E % ws:
            continue
        el = E // ws
        w = P.MoeLayerWeights.random(h, E, seed=0, dtype=torch.bfloat16, device=dev,
                                     experts=range(rank * el, (rank + 1) * el))
        ebr = [w.bank if r == rank else None for r in range(ws)] if distributed else [w.bank]
        params = w.leaf_parameters()
        g_aux = torch.ones((), device=dev)
        for n in a.tokens:
            x = torch.randn(n, h, device=dev, generator=torch.Generator(device=dev).manual_seed(1)).bfloat16()
            x.requires_grad_()
            g_out = torch.ones(n, h, device=dev, dtype=torch.bfloat16)

            def pp_step():
                for p in params:
                    p.grad = None
                x.grad = None
                out, l_aux = P.ppmoe_forward(world, group, x, w.gate, ebr, top_k=k)
                torch.autograd.backward([out, l_aux], [g_out, g_aux])
                P.sync_gate_gradients(world, group, w.gate)

            nr = n // ws
            x_dp = x.detach()[rank * nr:(rank + 1) * nr].clone().requires_grad_()
            g_dp = torch.ones(nr, h, device=dev, dtype=torch.bfloat16)

            def dp_step():
                for p in params:
                    p.grad = None
                x_dp.grad = None
                out, l_aux = P.dpmoe_forward(world, group, x_dp, w.gate, experts_by_rank=ebr, top_k=k)
                torch.autograd.backward([out, l_aux], [g_dp, g_aux])
                P.dpmoe_sync_gradients(world, group, w.gate)

            ms_pp = timed(pp_step, a.steps, a.warmup, dev, distributed)
            ms_dp = timed(dp_step, a.steps, a.warmup, dev, distributed)
            if rank == 0:
                print(json.dumps({"n_gpus": ws, "tokens": n, "experts": E, "hidden": h, "top_k": k,
                                  "ppmoe_tok_s": n / ms_pp * 1e3, "a2a_tok_s": n / ms_dp * 1e3,
                                  "ppmoe_ms": ms_pp, "a2a_ms": ms_dp, "ppmoe_over_a2a": ms_dp / ms_pp}), flush=True)
            del x, x_dp, g_out, g_dp
        del w, ebr, params
        torch.cuda.empty_cache()
    if distributed:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
