"""BASELINE.json configs[3]: GPT-style PPMoE block stack (h 4096, E 8, top-2, bf16) over
pipeline stages x tensor ranks, 1F1B over micro-batches.  Prints one JSON line on rank 0:
tokens/s of whole training iterations (all micro-batches fwd+bwd + gate-gradient sync),
device time, max over ranks.

usage: python -m torch.distributed.run --nproc-per-node P*T tools/pp_bench.py --stages P --tp T
       [--layers 24] [--micro 8] [--mb-tokens 4096] [--steps 3] [--warmup 1]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import paper_2304_11414_b200 as P
from paper_2304_11414_b200.pipeline import PipelineStack


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stages", type=int, default=2)
    ap.add_argument("--tp", type=int, default=2)
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--top-k", type=int, default=2)
    ap.add_argument("--micro", type=int, default=8)
    ap.add_argument("--mb-tokens", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    a = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    world = P.World(1, ws, distributed=ws > 1)
    stack = PipelineStack(world, a.layers, a.stages, a.tp, a.hidden, a.experts, top_k=a.top_k)

    def step():
        for p in stack.parameters():
            p.grad = None
        stack.train_step(a.micro, mb_tokens=a.mb_tokens)
        stack.sync_gate_gradients()

    for _ in range(a.warmup):
        step()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / a.steps], device=dev, dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t)
    tokens = a.micro * a.mb_tokens
    flop = 12 * tokens * a.top_k * a.hidden * 4 * a.hidden * a.layers + 12 * tokens * a.hidden * 4 * a.hidden * a.layers
    if rank == 0:
        print(json.dumps({
            "metric": "PPMoE block stack training tokens/s (1F1B, fwd+bwd)", "value": tokens / ms * 1e3,
            "unit": "tokens/s", "ms_per_iteration": ms, "n_gpus": ws, "stages": a.stages, "tp": a.tp,
            "layers": a.layers, "hidden": a.hidden, "experts": a.experts, "top_k": a.top_k,
            "micro_batches": a.micro, "mb_tokens": a.mb_tokens, "dtype": "bf16", "data": "synthetic",
            "model_tflops_per_gpu": flop / (ms / 1e3) / 1e12 / ws,
            "block": "x + DenseTPFFN(x), then x + PPMoE(x) (no attention: absent from the reference)",
            "bubble_closed_form": (a.stages - 1) / (a.micro + a.stages - 1)}), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
