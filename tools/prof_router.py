"""Dev tool: C2 (or C3 with argv[1] == 'c3') router calls for ncu (-k regex:route); prints the
host enqueue time of one route() call so a host-bound loop is visible."""
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2304_11414_b200 as P
from paper_2304_11414_b200 import _ops

c3 = len(sys.argv) > 1 and sys.argv[1] == "c3"
h, e, k, n = (8192, 16, 2, 16384) if c3 else (4096, 8, 2, 16384)
if len(sys.argv) > 2:
    n = int(sys.argv[2])  # a TP rank's routing slice: N / T tokens
dev = torch.device("cuda", 0)
x = P.Rng(1, 99).normal_tensor((n, h), dtype=torch.bfloat16, device=dev)
wg = P.GateParams.init(h, e, P.Rng(0).spawn(1), device=dev).wg.detach()
for _ in range(3):
    _ops.route(x, wg, k)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    _ops.route(x, wg, k)
t1 = time.perf_counter()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    _ops.route(x, wg, k)
b.record()
torch.cuda.synchronize()
print(f"route() host enqueue {(t1 - t0) / 20 * 1e6:.1f} us/call, device {a.elapsed_time(b) / 20 * 1e3:.1f} us/call")
