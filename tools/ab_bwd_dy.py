"""Dev tool: A/B of the two bwd_dy forms (PPMOE_BWD_DY=block vs the default column-slab
kernel).  `python tools/ab_bwd_dy.py save OUT.pt` runs one C2-like TP=1 step and saves the
gradients; `python tools/ab_bwd_dy.py cmp A.pt B.pt` compares them."""
import sys
sys.path.insert(0, ".")
import torch

if sys.argv[1] == "cmp":
    a, b = torch.load(sys.argv[2]), torch.load(sys.argv[3])
    for k in a:
        same = torch.equal(a[k], b[k])
        d = (a[k].float() - b[k].float()).abs().max().item()
        s = a[k].float().abs().max().item()
        print(f"{k:28s} bit-identical={same} max|diff|={d:.3e} max|a|={s:.3e}")
    sys.exit(0)

import paper_2304_11414_b200 as P
h, E, k, n = 4096, 8, 2, 8192
dev = torch.device("cuda", 0)
torch.manual_seed(0)
w = P.MoeLayerWeights.random(h, E, seed=0, device=dev)
x = torch.randn(n, h, device=dev).bfloat16().requires_grad_()
g_out = torch.randn(n, h, device=dev).bfloat16()
g_aux = torch.ones((), device=dev)
world, group = P.World(1, 1), P.ProcessGroup(P.EP, (0,))
out, l_aux = P.ppmoe_forward(world, group, x, w.gate, [w.bank], top_k=k)
torch.autograd.backward([out, l_aux], [g_out, g_aux])
res = {"dx": x.grad}
for name, gr in w.named_grads().items():
    if gr is not None:
        res[name] = gr
torch.save({kk: v.detach().cpu() for kk, v in res.items()}, sys.argv[2])
print("saved", sys.argv[2], len(res))
