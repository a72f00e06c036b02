"""Dev tool: per-call times of the forward NVLink exchange (owner gather, barriers, pull)
on the C2 layer over a TP group, forward only.  Env knobs are read once per process, so
compare variants with separate launches.
usage: torchrun --nproc-per-node T tools/nvl_micro.py [experts] [iters]"""
import os
import sys

sys.path.insert(0, ".")
import torch
import torch.distributed as dist

import paper_2304_11414_b200 as P
from paper_2304_11414_b200 import _ops

rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
E = int(sys.argv[1]) if len(sys.argv) > 1 else 8
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h, k, n = 4096, 2, 16384
el = E // ws
w = P.MoeLayerWeights.random(h, E, seed=0, device=dev, experts=range(rank * el, (rank + 1) * el))
x = torch.randn(n, h, device=dev, generator=torch.Generator(device=dev).manual_seed(1)).bfloat16()
world, group = P.World(1, ws), P.ProcessGroup(P.EP, tuple(range(ws)))
ebr = [w.bank if r == rank else None for r in range(ws)]

with torch.no_grad():
    for _ in range(5):
        P.ppmoe_forward(world, group, x, w.gate, ebr, top_k=k)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with _ops.KernelProfile() as prof:
        e0.record()
        for _ in range(iters):
            P.ppmoe_forward(world, group, x, w.gate, ebr, top_k=k)
        e1.record()
    summ = prof.summary()
tot = e0.elapsed_time(e1) / iters
t = torch.tensor([tot], device=dev)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
keys = ("ppmoe_nvl_owner_gather", "ppmoe_nvl_barrier", "ppmoe_nvl_pull_blocks_ce", "ppmoe_nvl_pull_blocks",
        "ppmoe_expert_fc2_fwd", "ppmoe_expert_fc1_fwd")
parts = " ".join(f"{kk.replace('ppmoe_', '')}={summ[kk]['ms'] / iters * 1e3:.0f}us/{summ[kk]['launches'] // iters}"
                 for kk in keys if kk in summ)
env = " ".join(f"{k_}={v}" for k_, v in sorted(os.environ.items()) if k_.startswith("PPMOE_"))
print(f"[T={ws} E={E} rank {rank}] {env or 'default'}: fwd {tot:.3f} ms (max over ranks {float(t):.3f}) {parts}",
      flush=True)
dist.destroy_process_group()
