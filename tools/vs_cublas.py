"""Dev tool: the six expert GEMMs of the C2 step (our tcgen05 kernels, timed per C-ABI call
inside the real fwd+bwd step) against cuBLAS doing the same six products as batched
matmuls with no epilogue work (torch.bmm, bf16 out), in the same sustained, power-capped
regime: rounds alternate between the two, 10 steps each.
usage: python tools/vs_cublas.py [rounds]"""
import statistics
import sys

sys.path.insert(0, ".")
import torch

import paper_2304_11414_b200 as P
from paper_2304_11414_b200 import _ops

h, E, k, n = 4096, 8, 2, 16384
f = 4 * h
dev = torch.device("cuda", 0)
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 4
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


pe = n * k // E  # rows per expert (balanced: the step's routing gives 3967-4201)
xs = torch.randn(E, pe, h, device=dev).bfloat16()
up, down = w.bank.up.detach(), w.bank.down.detach()
act = torch.randn(E, pe, f, device=dev).bfloat16()
dy = torch.randn(E, pe, h, device=dev).bfloat16()
dh = torch.randn(E, pe, f, device=dev).bfloat16()
cub = {
    "fc1_fwd": lambda: torch.bmm(xs, up),
    "fc2_fwd": lambda: torch.bmm(act, down),
    "fc2_dgrad": lambda: torch.bmm(dy, down.transpose(1, 2)),
    "fc1_dgrad": lambda: torch.bmm(dh, up.transpose(1, 2)),
    "fc2_wgrad": lambda: torch.bmm(act.transpose(1, 2), dy),
    "fc1_wgrad": lambda: torch.bmm(xs.transpose(1, 2), dh),
}
ours = {nm: [] for nm in cub}
theirs = {nm: [] for nm in cub}
for _ in range(3):
    step()
    for fn in cub.values():
        fn()
torch.cuda.synchronize()
for _ in range(rounds):
    with _ops.KernelProfile() as prof:
        for _ in range(10):
            step()
    s = prof.summary()
    for nm in cub:
        ours[nm].append(s[f"ppmoe_expert_{nm}"]["ms"] / 10)
    for nm, fn in cub.items():
        evs = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            evs.append((a, b))
        # the other five products run between repeats, as in a step
        for other, g in cub.items():
            if other != nm:
                g()
        torch.cuda.synchronize()
        theirs[nm].append(sum(a.elapsed_time(b) for a, b in evs) / 10)
flop = 2.0 * E * pe * h * f
print(f"{'GEMM':10s} {'ours ms':>8s} {'TFLOP/s':>8s}   {'cuBLAS ms':>9s} {'TFLOP/s':>8s}   ours/cuBLAS time")
to = tc = 0.0
for nm in cub:
    mo, mc = statistics.median(ours[nm]), statistics.median(theirs[nm])
    to += mo
    tc += mc
    print(f"{nm:10s} {mo:8.3f} {flop / mo / 1e9:8.0f}   {mc:9.3f} {flop / mc / 1e9:8.0f}   {mo / mc:.3f}")
print(f"{'sum':10s} {to:8.3f} {6 * flop / to / 1e9:8.0f}   {tc:9.3f} {6 * flop / tc / 1e9:8.0f}   {to / tc:.3f}")
print("(ours: in the step, with the fused epilogues and the real routing, 3967-4201 rows per expert; "
      "cuBLAS: 4096 rows per expert, no bias/GeLU/GeLU'/partials)")
