"""Dev tool: does the B-operand layout set the grouped GEMM's speed?  Times the pair kernel
(EpiStore<float>) on the fc1-fwd shape (8 x 4096 rows, K 4096, N 16384) and the fc1-dgrad
shape (K 16384, N 4096) with B MN-major (mode 0) and K-major (mode 2), interleaved."""
import statistics, sys
sys.path.insert(0, ".")
import torch
from paper_2304_11414_b200 import _lib

G, per = 8, 4096
rows = G * per
seg = torch.tensor([g * per for g in range(G + 1)], dtype=torch.int32, device="cuda")
res = {}
for K, N in ((4096, 16384), (16384, 4096)):
    A = torch.randn(rows, K, device="cuda").bfloat16()
    Bmn = torch.randn(G * K, N, device="cuda").bfloat16()
    Bk = torch.randn(G * N, K, device="cuda").bfloat16()
    D = torch.empty(rows, N, device="cuda")
    arms = {f"K{K} N{N} B MN-major": (0, Bmn), f"K{K} N{N} B K-major": (2, Bk)}
    for _ in range(2):
        for nm, (mode, B) in arms.items():
            _lib.call("ppmoe_gemm_selftest", mode, 3, 0, _lib.ptr(A), _lib.ptr(B), _lib.ptr(seg), G, 0, N, K, rows,
                      _lib.ptr(D), _lib.stream_ptr())
    for rnd in range(6):
        for nm, (mode, B) in arms.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                _lib.call("ppmoe_gemm_selftest", mode, 3, 0, _lib.ptr(A), _lib.ptr(B), _lib.ptr(seg), G, 0, N, K, rows,
                          _lib.ptr(D), _lib.stream_ptr())
            e1.record()
            torch.cuda.synchronize()
            res.setdefault(nm, []).append(e0.elapsed_time(e1) / 3)
    del A, Bmn, Bk, D
for nm, v in res.items():
    ms = statistics.median(v)
    print(f"{nm:28s} median {ms:.3f} ms  {2 * rows * 4096 * 16384 / ms / 1e9:.0f} TFLOP/s  all={[round(t, 3) for t in v]}")
