"""Dev tool: DRAM traffic / time of the fc2-shaped grouped GEMM (K=16384) in 1-CTA vs pair mode."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2304_11414_b200 import _lib

G, K, N, rows_e = 8, 16384, 4096, 4096
seg = [g * rows_e for g in range(G + 1)]
rows = seg[-1]
segt = torch.tensor(seg, dtype=torch.int32, device="cuda")
A = torch.randn(rows, K, device="cuda").bfloat16()
B = torch.randn(G * K, N, device="cuda").bfloat16()
D = torch.empty(rows, N, device="cuda")
for use_tc in [int(m) for m in sys.argv[1:]] or [2, 3]:
    for _ in range(2):
        _lib.call("ppmoe_gemm_selftest", 0, use_tc, 0, _lib.ptr(A), _lib.ptr(B), _lib.ptr(segt), G, 0, N, K, rows,
                  _lib.ptr(D), _lib.stream_ptr())
    torch.cuda.synchronize()
    print("ok", use_tc)
