"""Dev tool: GPU kernel timeline of the C2 step on rank 0 of a TP group (torch.profiler /
CUPTI), summarised as the step's critical path: which kernels run while no expert GEMM is
running, and the idle gaps.  usage: torchrun --nproc-per-node T tools/tp_timeline.py [experts]"""
import json
import os
import sys

sys.path.insert(0, ".")
import torch
import torch.distributed as dist

import paper_2304_11414_b200 as P

rank, ws = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
if ws > 1:
    dist.init_process_group("nccl", device_id=dev)
E = int(sys.argv[1]) if len(sys.argv) > 1 else 8
h, k, n = 4096, 2, 16384
el = E // ws
w = P.MoeLayerWeights.random(h, E, seed=0, device=dev, experts=range(rank * el, (rank + 1) * el))
x = torch.randn(n, h, device=dev, generator=torch.Generator(device=dev).manual_seed(1)).bfloat16().requires_grad_()
g_out = torch.ones(n, h, device=dev, dtype=torch.bfloat16)
g_aux = torch.ones((), device=dev)
world = P.World(1, ws, distributed=ws > 1)
group = P.ProcessGroup(P.EP, tuple(range(ws)))
ebr = [w.bank if r == rank else None for r in range(ws)] if ws > 1 else [w.bank]


def step():
    for p in w.leaf_parameters():
        p.grad = None
    x.grad = None
    out, l_aux = P.ppmoe_forward(world, group, x, w.gate, ebr, top_k=k)
    torch.autograd.backward([out, l_aux], [g_out, g_aux])
    P.sync_gate_gradients(world, group, w.gate)


for _ in range(5):
    step()
torch.cuda.synchronize()
if ws > 1:
    dist.barrier()
steps, skip = 3, 4  # the first steps after the sync wait on the host: summarise the last 3
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA], acc_events=True) as prof:
    for _ in range(skip + steps):
        step()
    torch.cuda.synchronize()
if rank == 0:
    os.makedirs("gpurun_out", exist_ok=True)
    path = f"gpurun_out/timeline_T{ws}_E{E}.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    starts = [i for i, e in enumerate(ev) if "router_tc_prep" in e["name"] or "router_dmma" in e["name"]]
    ev = ev[starts[skip]:] if len(starts) > skip else ev
    gaps = []
    end, prev = ev[0]["ts"], ev[0]
    for e in ev:
        if e["ts"] - end > 5:
            gaps.append((e["ts"] - end, prev["name"].split("(")[0][-40:], e["name"].split("(")[0][-40:]))
        if e["ts"] + e["dur"] > end:
            end, prev = e["ts"] + e["dur"], e
    for g in sorted(gaps, reverse=True)[:12]:
        print(f"  gap {g[0]:8.1f} us  {g[1]} -> {g[2]}")
    t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
    # intervals covered by GEMMs; everything else is exposed
    gem = [(e["ts"], e["ts"] + e["dur"]) for e in ev if "grouped_gemm" in e["name"]]
    gem.sort()
    merged = []
    for a, b in gem:
        if merged and a <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], b)
        else:
            merged.append([a, b])
    gemm_us = sum(b - a for a, b in merged)
    exposed = {}
    idle = 0.0
    cur = t0
    # walk the non-GEMM windows and attribute them to the kernels running there
    windows = []
    for a, b in merged:
        if a > cur:
            windows.append((cur, a))
        cur = max(cur, b)
    if t1 > cur:
        windows.append((cur, t1))
    for a, b in windows:
        covered = []
        for e in ev:
            s, f = max(a, e["ts"]), min(b, e["ts"] + e["dur"])
            if f > s and "grouped_gemm" not in e["name"]:
                nm = e["name"].split("<")[0].split("(")[0][:48]
                exposed[nm] = exposed.get(nm, 0.0) + (f - s)
                covered.append((s, f))
        covered.sort()
        c = a
        for s, f in covered:
            if s > c:
                idle += s - c
            c = max(c, f)
        if b > c:
            idle += b - c
    total = t1 - t0
    print(f"[T={ws} E={E}] {steps} steps: span {total / steps / 1e3:.3f} ms/step, GEMM-covered "
          f"{gemm_us / steps / 1e3:.3f} ms/step, idle (no kernel) {idle / steps / 1e3:.3f} ms/step")
    for nm, us in sorted(exposed.items(), key=lambda kv: -kv[1]):
        print(f"  exposed {nm:50s} {us / steps:8.1f} us/step")
if ws > 1:
    dist.destroy_process_group()
