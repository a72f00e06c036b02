"""Dev tool: interleaved A/B timing of GEMM kernel modes on the C2 step (median of rounds)."""
import statistics, sys
sys.path.insert(0, ".")
import torch
import paper_2304_11414_b200 as P
from paper_2304_11414_b200 import _lib

h, E, k, n = 4096, 8, 2, 16384
dev = torch.device("cuda", 0)
w = P.MoeLayerWeights.random(h, E, seed=0, device=dev)
x = torch.randn(n, h, device=dev).bfloat16().requires_grad_()
g_out = torch.ones(n, h, device=dev, dtype=torch.bfloat16)
g_aux = torch.ones((), device=dev)
world, group = P.World(1, 1), P.ProcessGroup(P.EP, (0,))
modes = {"auto": 0, "single": 1, "pair": 2}
sel = sys.argv[1:] or ["auto", "single", "pair"]

def step():
    for p in w.leaf_parameters():
        p.grad = None
    x.grad = None
    out, l_aux = P.ppmoe_forward(world, group, x, w.gate, [w.bank], top_k=k)
    torch.autograd.backward([out, l_aux], [g_out, g_aux])

res = {m: [] for m in sel}
for _ in range(3):
    step()
for rnd in range(6):
    for m in sel:
        _lib.call("ppmoe_set_gemm_mode", modes[m])
        step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            step()
        e1.record()
        torch.cuda.synchronize()
        res[m].append(e0.elapsed_time(e1) / 5)
for m in sel:
    ms = statistics.median(res[m])
    print(f"{m:7s} median {ms:.3f} ms/step  {n / ms * 1e3:,.0f} tok/s   all={[round(v, 2) for v in res[m]]}")
