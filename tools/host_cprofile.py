"""Dev tool: where the host enqueue time of one C2 PPMoE step goes (cProfile over 20 steps)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2304_11414_b200 as P

h, E, k, n = 4096, 8, 2, 16384
dev = torch.device("cuda", 0)
w = P.MoeLayerWeights.random(h, E, seed=0, device=dev)
x = torch.randn(n, h, device=dev).bfloat16().requires_grad_()
g_out = torch.ones(n, h, device=dev, dtype=torch.bfloat16)
g_aux = torch.ones((), device=dev)
world, group = P.World(1, 1), P.ProcessGroup(P.EP, (0,))


def step():
    for p in w.leaf_parameters():
        p.grad = None
    x.grad = None
    out, l_aux = P.ppmoe_forward(world, group, x, w.gate, [w.bank], top_k=k)
    torch.autograd.backward([out, l_aux], [g_out, g_aux])


for _ in range(3):
    step()
torch.cuda.synchronize()
ts = []
for i in range(10):
    t0 = time.perf_counter()
    step()
    ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
print(f"host enqueue per step: median {1e3 * sorted(ts)[5]:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    step()
    torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(35)
