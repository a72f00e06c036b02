"""Dev tool: warm CUDA-event timing of the non-GEMM kernels at the C2 shape (TP=1)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2304_11414_b200 as P
from paper_2304_11414_b200 import _ops, _lib

h, E, k, n = 4096, 8, 2, 16384
dev = torch.device("cuda", 0)
w = P.MoeLayerWeights.random(h, E, seed=0, device=dev)
x = torch.randn(n, h, device=dev).bfloat16()
wg = w.gate.wg.detach()


def timeit(name, fn, nbytes=None, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    bw = f"  {nbytes / us / 1e3:7.0f} GB/s" if nbytes else ""
    print(f"{name:28s} {us:8.1f} us{bw}", flush=True)


rt = _ops.route(x, wg, k)
pl = _ops.plan(rt.idx, rt.w, E)
timeit("route (router+finalize)", lambda: _ops.route(x, wg, k), n * h * 2)
timeit("dispatch_plan", lambda: _ops.plan(rt.idx, rt.w, E))
out_acc = torch.zeros(n, h, device=dev)
st = _ops.experts_forward(x, pl, 0, E, w.bank.up.detach(), w.bank.down.detach(), w.bank.bias_up.detach(),
                          w.bank.bias_down.detach(), k, True, out_acc)
rows = n * k
timeit("gather", lambda: _lib.call("ppmoe_gather", _ops.ptr(x), 0, n, h, _ops.ptr(st.seg), E, _ops.ptr(pl.tok_sorted),
                                   _ops.ptr(pl.w_sorted), st.rows_cap, _ops.ptr(st.xs), _ops.ptr(st.tok_l),
                                   _ops.ptr(st.w_l), _ops._stream()), rows * h * 4)
timeit("cast_out", lambda: _ops.cast_out(out_acc, torch.bfloat16), n * h * 6)
timeit("zeros fp32 NxH", lambda: torch.zeros(n, h, device=dev), n * h * 4)
g_out = torch.ones(n, h, device=dev, dtype=torch.bfloat16)
dx_acc = torch.zeros(n, h, device=dev)
dy = torch.empty(st.rows_cap, h, device=dev, dtype=torch.bfloat16)
dw = torch.empty(st.rows_cap, device=dev)
timeit("bwd_dy", lambda: _lib.call("ppmoe_bwd_dy", 0, _ops.ptr(g_out), _ops.ptr(st.y), _ops.ptr(st.seg), E, h,
                                   st.rows_cap, _ops.ptr(st.tok_l), _ops.ptr(st.w_l), 1, 0.0, 0, _ops.ptr(dy),
                                   _ops.ptr(dw), None, _ops._stream()), rows * h * 6)
part = torch.empty(st.rows_cap // 32, h, device=dev)
timeit("bwd_dy (+dY colsum parts)", lambda: _lib.call("ppmoe_bwd_dy", 0, _ops.ptr(g_out), _ops.ptr(st.y),
                                   _ops.ptr(st.seg), E, h, st.rows_cap, _ops.ptr(st.tok_l), _ops.ptr(st.w_l), 1, 0.0,
                                   0, _ops.ptr(dy), _ops.ptr(dw), _ops.ptr(part), _ops._stream()), rows * h * 6)
aux = torch.ones(1, device=dev)
dl = _ops.gate_backward(rt, pl, st, dw, aux)
timeit("gate_bwd", lambda: _ops.gate_backward(rt, pl, st, dw, aux))
timeit("gate_grads (dX + dWg)", lambda: _ops.gate_grads(dx_acc, x, dl, wg, True, True), n * h * 8)
outb = torch.empty_like(x)
timeit("combine fwd (Y gather, w)", lambda: _ops.combine(st.y, st, pl, rt.w, outb), n * h * 6)
timeit("input_grads (dX + dWg)", lambda: _ops.input_grads(st.y, st, pl, x, dl, wg, True, True), n * h * 8)
timeit("input_grads (dX only)", lambda: _ops.input_grads(st.y, st, pl, x, dl, wg, True, False), n * h * 6)
timeit("owner gather fwd (T=1)", lambda: _ops.local_combine(st.y, st, pl, rt.idx, rt.w, outb), n * h * 6)
timeit("owner gather bwd (T=1, +gate)", lambda: _ops.local_combine(st.y, st, pl, rt.idx, None, outb, dl, wg), n * h * 6)
timeit("gate_weight_grad (dWg)", lambda: _ops.gate_weight_grad(x, dl, wg), n * h * 2)
