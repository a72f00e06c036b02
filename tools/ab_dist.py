"""Dev tool: interleaved A/B of environment-switched code paths on the C2 step over a TP
group (torchrun, one process per GPU).  usage: torchrun ... tools/ab_dist.py VAR=v1,v2"""
import os, statistics, sys
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
var, vals = sys.argv[1].split("=")
vals = vals.split(",")


def step():
    for p in w.leaf_parameters():
        p.grad = None
    x.grad = None
    out, l_aux = P.ppmoe_forward(world, group, x, w.gate, ebr, top_k=k)
    torch.autograd.backward([out, l_aux], [g_out, g_aux])
    P.sync_gate_gradients(world, group, w.gate)


res = {v: [] for v in vals}
for v in vals:
    os.environ[var] = v
    for _ in range(3):
        step()
torch.cuda.synchronize()
for rnd in range(8):
    for v in vals:
        os.environ[var] = v
        step()
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            step()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 5], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[v].append(float(t))
if rank == 0:
    for v in vals:
        ms = statistics.median(res[v])
        print(f"T={ws} {var}={v:8s} median {ms:.3f} ms/step  {n / ms * 1e3:,.0f} tok/s  all={[round(t, 2) for t in res[v]]}")
dist.destroy_process_group()
