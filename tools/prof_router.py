"""Dev tool: one C2 (or C3 with argv[1] == 'c3') router call for ncu (-k regex:router)."""
import sys

sys.path.insert(0, ".")
import torch

import paper_2304_11414_b200 as P
from paper_2304_11414_b200 import _ops

c3 = len(sys.argv) > 1 and sys.argv[1] == "c3"
h, e, k, n = (8192, 16, 2, 16384) if c3 else (4096, 8, 2, 16384)
dev = torch.device("cuda", 0)
x = P.Rng(1, 99).normal_tensor((n, h), dtype=torch.bfloat16, device=dev)
wg = P.GateParams.init(h, e, P.Rng(0).spawn(1), device=dev).wg.detach()
for _ in range(3):
    _ops.route(x, wg, k)
torch.cuda.synchronize()
