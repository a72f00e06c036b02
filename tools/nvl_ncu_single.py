"""Dev tool: NVLink evidence for the owner gather without a multi-process job.  One process
drives 2 GPUs: rank 0's owner-gather kernel (C2 layout at T = 2, E 8, top-2, N 16384) runs on
GPU 0 and reads the pairs whose expert lives on "rank 1" straight out of GPU 1's memory
(P2P loads over NVLink), exactly as in the distributed exchange.  Prints the event-timed
bandwidth; run under ncu with nvlrx__bytes / nvltx__bytes for the link counters:
    ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum \\
        -k regex:nvl_owner_gather -c 2 python tools/nvl_ncu_single.py"""
import ctypes
import sys

sys.path.insert(0, ".")
import torch
from cuda.bindings import runtime as cudart

import paper_2304_11414_b200 as P  # noqa: F401
from paper_2304_11414_b200 import _lib, _ops

h, E, k, n, T = 4096, 8, 2, 16384, 2
el = E // T
d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
for a, b in ((0, 1), (1, 0)):
    cudart.cudaSetDevice(a)
    err = cudart.cudaDeviceEnablePeerAccess(b, 0)[0]
    assert err in (cudart.cudaError_t.cudaSuccess, cudart.cudaError_t.cudaErrorPeerAccessAlreadyEnabled), err
torch.cuda.set_device(0)
x = P.Rng(1, 99).normal_tensor((n, h), dtype=torch.bfloat16, device=d0)
wg = P.GateParams.init(h, E, P.Rng(0).spawn(1), device=d0).wg.detach()
rt = _ops.route(x, wg, k)
pl = _ops.plan(rt.idx, rt.w, E)
rows_cap = _ops.local_rows_cap(n, k, el, pl.capacity)
r0 = torch.randn(rows_cap, h, device=d0).bfloat16()
with torch.cuda.device(1):
    r1 = torch.randn(rows_cap, h, device=d1).bfloat16()
    torch.cuda.synchronize()
rows = (ctypes.c_void_p * 2)(r0.data_ptr(), r1.data_ptr())
out = torch.empty(n, h, device=d0, dtype=torch.bfloat16)


def gather():
    _lib.call("ppmoe_nvl_owner_gather", rows, _lib.ptr(pl.seg), el, _lib.ptr(rt.idx), _lib.ptr(pl.pair_pos),
              _lib.ptr(rt.w), n, k, h, T, 0, None, None, 0, _lib.ptr(out), None, None, 0, _lib.stream_ptr())


for _ in range(3):
    gather()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    gather()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
idx = rt.idx[: n // T].long()
remote_pairs = int((idx >= el).sum())
local_pairs = int((idx < el).sum())
rb, lb, wb = remote_pairs * h * 2, local_pairs * h * 2, (n // T) * h * 2
print(f"owner gather rank 0 of T=2: {ms * 1e3:.1f} us; NVLink reads {rb / 1e6:.1f} MB ({rb / ms / 1e6:.0f} GB/s), "
      f"local reads {lb / 1e6:.1f} MB, writes {wb / 1e6:.1f} MB; total {(rb + lb + wb) / ms / 1e6:.0f} GB/s")
