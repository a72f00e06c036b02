"""Dev tool: where the rows / columns of an M = 128 pair-MMA tail tile land (selftest, one
group of 128 rows, A = I): D[r][n] should be B[r][n]; with B[k][n] = k the printed matrix
shows which source row each output row holds, with B[k][n] = n which column."""
import sys

sys.path.insert(0, ".")
import torch

from paper_2304_11414_b200 import _lib

rows, K, N = 128, 128, 256
A = torch.eye(rows, K, device="cuda").bfloat16()
segt = torch.tensor([0, rows], dtype=torch.int32, device="cuda")
for name, B in (("row", torch.arange(K, device="cuda")[:, None].expand(K, N).float()),
                ("col", torch.arange(N, device="cuda")[None, :].expand(K, N).float())):
    B = B.contiguous().bfloat16()
    D = torch.full((rows, N), float("nan"), device="cuda")
    _lib.call("ppmoe_gemm_selftest", 0, 3, 0, _lib.ptr(A), _lib.ptr(B), _lib.ptr(segt), 1, 0, N, K, rows,
              _lib.ptr(D), _lib.stream_ptr())
    torch.cuda.synchronize()
    print(name, "D[:, 0]:", D[:, 0].int().tolist())
    print(name, "D[0, :]:", D[0, :].int().tolist())
    print(name, "D[70, :]:", D[70, :].int().tolist())
