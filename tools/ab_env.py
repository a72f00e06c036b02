"""Dev tool: interleaved A/B of environment-switched code paths on the C2 step, one process.
usage: python tools/ab_env.py VAR=val1,val2          (one variable, one arm per value)
       python tools/ab_env.py A=x+B=y C=z+D=w ...    (one arm per argument, '+'-joined settings)"""
import os, statistics, sys
sys.path.insert(0, ".")
import torch
import paper_2304_11414_b200 as P

h, E, k, n = 4096, 8, 2, 16384
dev = torch.device("cuda", 0)
w = P.MoeLayerWeights.random(h, E, seed=0, device=dev)
x = torch.randn(n, h, device=dev).bfloat16().requires_grad_()
g_ones = torch.ones(n, h, device=dev, dtype=torch.bfloat16)
g_normal = torch.randn(n, h, device=dev).bfloat16()  # AB_UPSTREAM=normal (arm setting)
g_aux = torch.ones((), device=dev)
world, group = P.World(1, 1), P.ProcessGroup(P.EP, (0,))
if len(sys.argv) > 2 or "+" in sys.argv[1]:
    var, vals = "arm", sys.argv[1:]
else:
    var, vals = sys.argv[1].split("=")
    vals = vals.split(",")


def set_arm(v):
    if var != "arm":
        os.environ[var] = v
        return
    for kv in v.split("+"):
        k_, v_ = kv.split("=")
        os.environ[k_] = v_


def step():
    for p in w.leaf_parameters():
        p.grad = None
    x.grad = None
    out, l_aux = P.ppmoe_forward(world, group, x, w.gate, [w.bank], top_k=k)
    g_out = g_normal if os.environ.get("AB_UPSTREAM") == "normal" else g_ones
    torch.autograd.backward([out, l_aux], [g_out, g_aux])


res = {v: [] for v in vals}
for v in vals:
    set_arm(v)
    for _ in range(2):
        step()
torch.cuda.synchronize()
for rnd in range(int(os.environ.get("AB_ROUNDS", "6"))):
    for v in vals:
        set_arm(v)
        step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            step()
        e1.record()
        torch.cuda.synchronize()
        res[v].append(e0.elapsed_time(e1) / 5)
for v in vals:
    ms = statistics.median(res[v])
    print(f"{var}={v} median {ms:.3f} ms/step  {n / ms * 1e3:,.0f} tok/s   all={[round(t, 2) for t in res[v]]}")
