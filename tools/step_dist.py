"""Dev tool: a few fwd+bwd steps of a small PPMoE layer over the NVLink exchange (T = WORLD_SIZE),
for compute-sanitizer runs (tools/sanitize_rank.sh).  Shape: h 1024, E 8, top-2, N 2048,
capacity 1.25 (drops exercised), dropout 0.1 (Philox masks exercised), check_replicas on."""
import os
import sys

sys.path.insert(0, ".")
import torch
import torch.distributed as dist

import paper_2304_11414_b200 as P

rank, ws = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
if ws > 1:
    dist.init_process_group("nccl", device_id=dev)
h, E, k, n = 1024, 8, 2, 2048
el = E // ws
w = P.MoeLayerWeights.init(h, E, P.Rng(0), device=dev, experts=range(rank * el, (rank + 1) * el))
x = P.Rng(1, 99).normal_tensor((n, h), dtype=torch.bfloat16, device=dev).requires_grad_()
world, group = P.World(1, ws), P.ProcessGroup(P.EP, tuple(range(ws)))
ebr = [w.bank if r == rank else None for r in range(ws)]
rng = P.Rng(5, 5)
for step in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    for p in w.leaf_parameters():
        p.grad = None
    x.grad = None
    out, l_aux = P.ppmoe_forward(world, group, x, w.gate, ebr, top_k=k, capacity_factor=1.25, dropout_p=0.1, rng=rng,
                                 check_replicas=ws > 1)
    (out.float().sum() + l_aux).backward()
    P.sync_gate_gradients(world, group, w.gate)
torch.cuda.synchronize()
print(f"rank {rank}: step_dist ok, out sum {float(out.float().sum()):.4f}", flush=True)
if ws > 1:
    dist.barrier()
    dist.destroy_process_group()
