"""Dev tool: host enqueue time of one C2 PPMoE step at T = WORLD_SIZE (torchrun), cProfile on rank 0.
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/host_cprofile_dist.py"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch
import torch.distributed as dist

import paper_2304_11414_b200 as P

rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
h, E, k, n = 4096, 8, 2, 16384
el = E // ws
w = P.MoeLayerWeights.random(h, E, seed=0, device=dev, experts=range(rank * el, (rank + 1) * el))
x = torch.randn(n, h, device=dev, generator=torch.Generator(device=dev).manual_seed(1)).bfloat16().requires_grad_()
g_out = torch.ones(n, h, device=dev, dtype=torch.bfloat16)
g_aux = torch.ones((), device=dev)
world, group = P.World(1, ws), P.ProcessGroup(P.EP, tuple(range(ws)))
ebr = [w.bank if r == rank else None for r in range(ws)]


def step():
    for p in w.leaf_parameters():
        p.grad = None
    x.grad = None
    out, l_aux = P.ppmoe_forward(world, group, x, w.gate, ebr, top_k=k)
    torch.autograd.backward([out, l_aux], [g_out, g_aux])
    P.sync_gate_gradients(world, group, w.gate)


for _ in range(3):
    step()
torch.cuda.synchronize()
dist.barrier()
ts = []
for i in range(10):
    t0 = time.perf_counter()
    step()
    ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    dist.barrier()
if rank == 0:
    print(f"T={ws} host enqueue per step: median {1e3 * sorted(ts)[5]:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    step()
    torch.cuda.synchronize()
    dist.barrier()
pr.disable()
if rank == 0:
    pstats.Stats(pr).sort_stats("tottime").print_stats(30)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
dist.destroy_process_group()
