"""Dev tool: the six expert GEMMs of the C2 step (8 experts x 4096 rows) through cuBLAS
(torch.matmul, bf16 out) vs our grouped GEMM kernels, interleaved, same process."""
import statistics, sys
sys.path.insert(0, ".")
import torch
import paper_2304_11414_b200 as P
from paper_2304_11414_b200 import _ops

h, E, k, n = 4096, 8, 2, 16384
f = 4 * h
dev = torch.device("cuda", 0)
w = P.MoeLayerWeights.random(h, E, seed=0, device=dev)
x = torch.randn(n, h, device=dev).bfloat16().requires_grad_()
g_out = torch.ones(n, h, device=dev, dtype=torch.bfloat16)
g_aux = torch.ones((), device=dev)
world, group = P.World(1, 1), P.ProcessGroup(P.EP, (0,))
rows = 4096
Xs = torch.randn(E, rows, h, device=dev).bfloat16()
A = torch.randn(E, rows, f, device=dev).bfloat16()
dY = torch.randn(E, rows, h, device=dev).bfloat16()
up, down = w.bank.up.detach(), w.bank.down.detach()


def cublas_step():
    for e in range(E):
        torch.matmul(Xs[e], up[e])            # fc1 fwd
        torch.matmul(A[e], down[e])           # fc2 fwd
        torch.matmul(dY[e], down[e].T)        # fc2 dgrad
        torch.matmul(A[e].T, dY[e])           # fc2 wgrad
        torch.matmul(A[e], up[e].T)           # fc1 dgrad
        torch.matmul(Xs[e].T, A[e])           # fc1 wgrad


def ours_step():
    for p in w.leaf_parameters():
        p.grad = None
    x.grad = None
    out, l_aux = P.ppmoe_forward(world, group, x, w.gate, [w.bank], top_k=k)
    torch.autograd.backward([out, l_aux], [g_out, g_aux])


gemm_names = ["ppmoe_expert_fc1_fwd", "ppmoe_expert_fc2_fwd", "ppmoe_expert_fc2_dgrad", "ppmoe_expert_fc2_wgrad",
              "ppmoe_expert_fc1_dgrad", "ppmoe_expert_fc1_wgrad"]
res = {"cublas": [], "ours_gemm": [], "ours_step": []}
for _ in range(3):
    cublas_step(); ours_step()
torch.cuda.synchronize()
for rnd in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        cublas_step()
    e1.record(); torch.cuda.synchronize()
    res["cublas"].append(e0.elapsed_time(e1) / 5)
    with _ops.KernelProfile() as prof:
        e0.record()
        for _ in range(5):
            ours_step()
        e1.record(); torch.cuda.synchronize()
    s = prof.summary()
    res["ours_gemm"].append(sum(s[nm]["ms"] for nm in gemm_names if nm in s) / 5)
    res["ours_step"].append(e0.elapsed_time(e1) / 5)
flops = 12 * 32768 * h * f
for kk, v in res.items():
    ms = statistics.median(v)
    print(f"{kk:10s} {ms:7.3f} ms  {flops / ms / 1e9:6.0f} TFLOP/s  {[round(t, 2) for t in v]}")
