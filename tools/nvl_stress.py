"""Dev tool: per-step times of the C2 step over a TP group, per rank, for several env
settings (torchrun).  usage: torchrun ... tools/nvl_stress.py VAR=v1,v2 [steps]"""
import os, sys
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
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 60


def step():
    for p in w.leaf_parameters():
        p.grad = None
    x.grad = None
    out, l_aux = P.ppmoe_forward(world, group, x, w.gate, ebr, top_k=k)
    torch.autograd.backward([out, l_aux], [g_out, g_aux])
    P.sync_gate_gradients(world, group, w.gate)


for v in vals.split(","):
    os.environ[var] = v
    for _ in range(3):
        step()
    dist.barrier()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    evs[0].record()
    for i in range(steps):
        step()
        evs[i + 1].record()
    torch.cuda.synchronize()
    t = torch.tensor([evs[i].elapsed_time(evs[i + 1]) for i in range(steps)], device=dev)
    allt = [torch.empty_like(t) for _ in range(ws)]
    dist.all_gather(allt, t)
    if rank == 0:
        m = torch.stack(allt).max(0).values.cpu()
        q = torch.quantile(m, torch.tensor([0.1, 0.5, 0.9, 1.0]))
        slow = int((m > 1.3 * q[1]).sum())
        print(f"T={ws} {var}={v:6s} p10 {q[0]:.2f} p50 {q[1]:.2f} p90 {q[2]:.2f} max {q[3]:.2f} ms  slow steps {slow}/{steps}",
              flush=True)
dist.destroy_process_group()
