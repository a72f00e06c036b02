"""Dev tool: time the grouped GEMM self-test in 1-CTA (use_tc=2) vs CTA-pair (use_tc=3) mode."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2304_11414_b200 import _lib

G, K, N = 8, 4096, 16384
counts = [4096] * G
seg = [0]
for c in counts:
    seg.append(seg[-1] + (c + 127) // 128 * 128)
rows = seg[-1]
segt = torch.tensor(seg, dtype=torch.int32, device="cuda")
A = torch.randn(rows, K, device="cuda").bfloat16()
B = torch.randn(G * K, N, device="cuda").bfloat16()
D = torch.empty(rows, N, device="cuda")
modes = [int(m) for m in sys.argv[1:]] or [2, 3]
for use_tc in modes:
    def run():
        _lib.call("ppmoe_gemm_selftest", 0, use_tc, 0, _lib.ptr(A), _lib.ptr(B), _lib.ptr(segt), G, 0, N, K, rows,
                  _lib.ptr(D), _lib.stream_ptr())
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"use_tc={use_tc}: {ms:.3f} ms  {2 * rows * N * K / ms / 1e9:.0f} TFLOP/s", flush=True)
