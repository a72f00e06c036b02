"""Dev tool: one launch of each of the C2 step's six products through cuBLAS (torch.bmm)
and through our kernels (one step), for an ncu metrics pass comparing the two.
usage: ncu ... python tools/cublas_probe.py"""
import sys

sys.path.insert(0, ".")
import torch

import paper_2304_11414_b200 as P

h, E, k, n = 4096, 8, 2, 16384
f = 4 * h
dev = torch.device("cuda", 0)
pe = n * k // E
w = P.MoeLayerWeights.random(h, E, seed=0, device=dev)
up, down = w.bank.up.detach(), w.bank.down.detach()
xs = torch.randn(E, pe, h, device=dev).bfloat16()
act = torch.randn(E, pe, f, device=dev).bfloat16()
dy = torch.randn(E, pe, h, device=dev).bfloat16()
dh = torch.randn(E, pe, f, device=dev).bfloat16()
prods = [lambda: torch.bmm(xs, up), lambda: torch.bmm(act, down), lambda: torch.bmm(dy, down.transpose(1, 2)),
         lambda: torch.bmm(dh, up.transpose(1, 2)), lambda: torch.bmm(act.transpose(1, 2), dy),
         lambda: torch.bmm(xs.transpose(1, 2), dh)]
for p in prods:
    p()
torch.cuda.synchronize()
for p in prods:
    p()
torch.cuda.synchronize()
x = torch.randn(n, h, device=dev).bfloat16().requires_grad_()
out, l_aux = P.ppmoe_forward(P.World(1, 1), P.ProcessGroup(P.EP, (0,)), x, w.gate, [w.bank], top_k=k)
torch.autograd.backward([out, l_aux], [torch.ones_like(out), torch.ones_like(l_aux)])
torch.cuda.synchronize()
