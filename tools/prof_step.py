"""Dev tool: two C2 (PROF_C3=1: C3) PPMoE steps (fwd+bwd) for ncu captures (TP = 1, default combine mode)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2304_11414_b200 as P

import os

h, E, k, n = (8192, 16, 2, 16384) if os.environ.get("PROF_C3") else (4096, 8, 2, 16384)
cf = 1.25 if os.environ.get("PROF_C3") else float("inf")
if len(sys.argv) > 1:
    n = int(sys.argv[1])
dev = torch.device("cuda", 0)
w = P.MoeLayerWeights.random(h, E, seed=0, device=dev)
x = torch.randn(n, h, device=dev).bfloat16().requires_grad_()
g_out = torch.ones(n, h, device=dev, dtype=torch.bfloat16)
g_aux = torch.ones((), device=dev)
world, group = P.World(1, 1), P.ProcessGroup(P.EP, (0,))
for _ in range(2):
    for p in w.leaf_parameters():
        p.grad = None
    out, l_aux = P.ppmoe_forward(world, group, x, w.gate, [w.bank], top_k=k, capacity_factor=cf)
    torch.autograd.backward([out, l_aux], [g_out, g_aux])
torch.cuda.synchronize()
print("ok")
