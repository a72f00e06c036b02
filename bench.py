#!/usr/bin/env python3
"""Benchmark of the B200 PPMoE MoE layer: tokens/s of one layer forward + backward.

Workload (BASELINE.json configs[1], "C2"): hidden 4096, ffn 16384, 8 experts, top-2,
16384 tokens, bf16 activations/expert weights, fp32 gate, BASELINE.md's Philox inputs.
With --gpus N (one process per GPU; without a launcher the command re-runs itself under
torch.distributed.run) the N GPUs form one tensor-parallel group (TP=N): every rank holds
the replicated tokens, runs its E/N experts, and the group combines the output (forward)
and the input gradient (backward) with the NVLink owner-gather exchange; the gate-weight
gradient is all-reduced once per step (= one global batch).  Total work is fixed as N
grows ("scaling": "strong").

One step = route + dispatch plan + gather + expert fc1/fc2 (+combine) + all-reduce,
then the full backward (all parameter and input gradients) + the dX all-reduce +
the gate-gradient all-reduce.

    python bench.py [--gpus N --steps K --warmup W]             # our CUDA path
    python bench.py --impl reference [--steps K --warmup W]     # CPU reference path (oracle port)
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MoE-layer tokens/sec (fwd+bwd) at 1/2/4/8 B200; % of HBM/tensor roofline"
UNIT = "tokens/s"
C2 = {"hidden": 4096, "ffn": 16384, "experts": 8, "top_k": 2, "tokens": 16384}
# BASELINE.json configs[2] ("C3"): the token count is not given there; 16384 assumed
C3 = {"hidden": 8192, "ffn": 32768, "experts": 16, "top_k": 2, "tokens": 16384, "capacity_factor": 1.25}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--config", choices=["c2", "c3"], default="c2", help="BASELINE.json configs[1] or configs[2]")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--tokens", type=int, default=None)
    ap.add_argument("--hidden", type=int, default=None)
    ap.add_argument("--experts", type=int, default=None)
    ap.add_argument("--top-k", type=int, default=None)
    ap.add_argument("--capacity-factor", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-a2a", action="store_true", help="skip the all-to-all (DPMoE) comparator")
    ap.add_argument("--upstream", choices=["ones", "normal"], default="ones",
                    help="upstream gradient dOut: ones (loss = sum(out) + l_aux, test_moe.py:400; SURVEY 8(d)) "
                         "or N(0,1) bf16; the other one is timed as well and reported under upstream_alt")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time of the cpu_baseline sample")
    a = ap.parse_args()
    base = C3 if a.config == "c3" else C2
    a.tokens = a.tokens if a.tokens is not None else base["tokens"]
    a.hidden = a.hidden if a.hidden is not None else base["hidden"]
    a.experts = a.experts if a.experts is not None else base["experts"]
    a.top_k = a.top_k if a.top_k is not None else base["top_k"]
    if a.capacity_factor is None:
        a.capacity_factor = base.get("capacity_factor", math.inf)
    return a


def config_of(a, n_gpus):
    return {
        "workload": f"{a.config.upper()} PPMoE layer h={a.hidden} ffn={4 * a.hidden} E={a.experts} top-{a.top_k} "
                    f"N={a.tokens} cf={a.capacity_factor} bf16, TP={n_gpus}",
        "hidden": a.hidden, "ffn": 4 * a.hidden, "experts": a.experts, "top_k": a.top_k, "tokens": a.tokens,
        "capacity_factor": "inf" if math.isinf(a.capacity_factor) else a.capacity_factor,
        "tp": n_gpus, "parallelism": f"tp{n_gpus} (experts {a.experts // n_gpus}/GPU)",
        "l2": "per-step working set (weights 2.1 GB + activations) >> 126 MB L2; no flush needed",
        "upstream_grad": getattr(a, "upstream", "ones"),
    }


# ----------------------------------------------------------------------------- clocks


class ClockSampler:
    """SM clock / throttle-reason sampling during the timed region (B200_PROFILING.md clocks
    line).  One `nvidia-smi -lms` process started by rank 0 samples every GPU of the job:
    in-process NVML polling on every rank stalled the CUDA launch path often enough to
    skew the barrier-coupled ranks."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, indices, period_ms: int = 20, active: bool = True):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:  # local ordinals -> the ids nvidia-smi knows (ints or UUIDs)
            ids = [v.strip() for v in vis.split(",") if v.strip()]
            indices = [ids[i] if i < len(ids) else str(i) for i in indices]
        self.indices = list(indices)
        self.period = period_ms
        self.active = active and os.environ.get("PPMOE_CLOCKS", "smi") != "off"
        self.sm, self.smax, self.reasons = [], [], set()
        self.proc = None
        self.thread = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            try:
                rec = (time.perf_counter(), float(parts[1]), float(parts[2]),
                       {nm for nm, v in zip(self.NAMES, parts[3:7]) if v.lower().startswith("active")})
            except (ValueError, IndexError):
                continue
            self.samples.append(rec)

    def __enter__(self):
        """Start sampling (before the warm-up: nvidia-smi needs ~0.5 s to its first line);
        only samples inside mark_start()/mark_end() count."""
        self.samples, self.t0, self.t1 = [], None, None
        if not self.active:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", ",".join(str(i) for i in self.indices), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_end(self):
        self.t1 = time.perf_counter()
        # a timed region shorter than the sampling period still gets the next sample
        deadline = self.t1 + 4 * self.period / 1e3
        while self.proc is not None and time.perf_counter() < deadline and not any(
                r[0] >= self.t1 for r in self.samples):
            time.sleep(self.period / 4e3)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=5)
        return False

    def summary(self):
        recs = list(self.samples)
        whole = set().union(*(r[3] for r in recs)) if recs else set()
        if self.t0 is not None and self.t1 is not None:
            inside = [r for r in recs if self.t0 <= r[0] <= self.t1]
            if not inside:  # region shorter than the period: the samples bracketing it
                before = [r for r in recs if r[0] < self.t0][-1:]
                after = [r for r in recs if r[0] > self.t1][:1]
                inside = before + after
            recs = inside
        if not recs:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [r[1] for r in recs]
        reasons = set().union(*(r[3] for r in recs))
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[2] for r in recs), "reasons": sorted(reasons),
                "samples": len(sm), "sm_mhz_min": min(sm), "gpus": len(self.indices),
                # throttle reasons seen anywhere from the warm-up to the end of the timed region
                # (the power-cap bit toggles; a short region can miss it in its few samples)
                "reasons_around": sorted(whole)}


# ----------------------------------------------------------------------------- CPU baseline


def cpu_baseline(hidden, experts, top_k, ffn, weights_np=None, target_s=12.0, max_tokens=4096):
    """Time the CPU oracle port (numpy fp64, all host BLAS threads) on a bounded token
    sample of the same layer shape.  Test infrastructure; never on the product path."""
    import numpy as np

    from oracle import ppmoe_oracle as O

    try:
        from threadpoolctl import threadpool_info
        threads = max((i.get("num_threads", 1) for i in threadpool_info()), default=os.cpu_count())
    except Exception:  # pragma: no cover
        threads = os.cpu_count()
    if weights_np is None:
        import torch
        g = torch.Generator().manual_seed(0)
        sc = hidden ** -0.5

        def rnd(*s):
            return (torch.randn(*s, generator=g) * sc).to(torch.bfloat16).double().numpy()

        weights_np = O.OracleLayer(rnd(hidden, experts), [rnd(hidden, ffn) for _ in range(experts)],
                                   [rnd(ffn, hidden) for _ in range(experts)], [rnd(ffn) for _ in range(experts)],
                                   [rnd(hidden) for _ in range(experts)])
    rng = np.random.default_rng(1)

    def run(n):
        x = rng.standard_normal((n, hidden))
        t0 = time.perf_counter()
        O.ppmoe_layer(x, weights_np, k=top_k)
        return time.perf_counter() - t0

    n = 128
    t = run(n)
    n2 = int(min(max_tokens, max(n, n * target_s / max(t, 1e-3))))
    n2 = max(64, n2 // 64 * 64)
    t2 = run(n2)
    return {"value": n2 / t2, "unit": UNIT, "cores": int(threads), "kind": "port",
            "sample": f"{n2} tokens of the same layer (h={hidden}, ffn={ffn}, E={experts}, top-{top_k}), "
                      f"one fwd+bwd of oracle/ppmoe_oracle.py (numpy fp64 closed form of moesim ppmoe_forward + "
                      f"tensor.backward), {t2:.1f} s; host os.cpu_count()={os.cpu_count()}"}, weights_np


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # torch.distributed.run sets OMP_NUM_THREADS=1 for its ranks; the reference arm runs on rank 0
    # alone and gets every host core back (the BLAS pools are resized at run time)
    try:
        import numpy  # noqa: F401 -- load the BLAS first: threadpoolctl only sees loaded pools
        from threadpoolctl import threadpool_limits
        limits = threadpool_limits(limits=os.cpu_count() or 1)
    except Exception:  # pragma: no cover
        limits = None
    try:
        return _run_reference(a)
    finally:
        if limits is not None:
            limits.restore_original_limits()


def _run_reference(a):
    hidden, experts, top_k = a.hidden, a.experts, a.top_k
    ffn = 4 * hidden
    steps, warmup = a.steps, a.warmup
    cb, weights = cpu_baseline(hidden, experts, top_k, ffn, target_s=min(a.cpu_seconds, 8.0), max_tokens=2048)
    n = int(cb["sample"].split()[0])
    import numpy as np

    from oracle import ppmoe_oracle as O
    rng = np.random.default_rng(2)
    times = []
    for i in range(warmup + steps):
        x = rng.standard_normal((n, hidden))
        t0 = time.perf_counter()
        O.ppmoe_layer(x, weights, k=top_k)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    t = sum(times)
    value = n * steps / t
    cb = dict(cb)
    cb["value"] = value
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": steps, "warmup": warmup,
            "ms_per_step": 1e3 * t / steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference", "config": config_of(a, a.gpus),
            "cpu_baseline": cb, "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU path


def relaunch_under_torchrun(a) -> int | None:
    """`python bench.py --gpus N` without a launcher: re-run this command under
    torch.distributed.run with N local ranks (one process per GPU, 127.0.0.1 rendezvous);
    rank 0 prints the JSON line.  Returns the launcher's exit code, or None when this
    process is already a rank (or N == 1)."""
    if a.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    a = parse()
    rc = relaunch_under_torchrun(a)
    if rc is not None:
        return rc
    if a.impl == "reference":
        return run_reference(a)

    import torch
    import torch.distributed as dist

    import paper_2304_11414_b200 as P
    from paper_2304_11414_b200 import _lib, _ops

    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world_size != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world_size}")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    distributed = world_size > 1
    if distributed:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    tp = world_size
    h, E, k, n = a.hidden, a.experts, a.top_k, a.tokens
    f = 4 * h
    if E % tp:
        raise SystemExit(f"experts {E} must divide over {tp} GPUs")
    world = P.World(1, tp, distributed=distributed)
    group = P.ProcessGroup(P.EP, tuple(range(tp)))
    el = E // tp
    block = range(rank * el, (rank + 1) * el)
    # BASELINE.md §3 inputs: MoeLayerWeights.init(h, E, Rng(0)) rounded to bf16 (this rank's
    # expert block only; Philox streams per expert, so every block matches the full layer),
    # hidden Rng(1, 99).normal((N, h)) rounded to bf16, identical on every rank
    t_init = time.perf_counter()
    w = P.MoeLayerWeights.init(h, E, P.Rng(0), dtype=torch.bfloat16, device=dev, experts=block,
                               threads=max(1, (os.cpu_count() or 1) // world_size))
    x = P.Rng(1, 99).normal_tensor((n, h), dtype=torch.bfloat16, device=dev).requires_grad_()
    init_s = time.perf_counter() - t_init
    experts_by_rank = [w.bank if r == rank else None for r in range(tp)] if distributed else [w.bank]
    if not distributed:
        group = P.ProcessGroup(P.EP, (0,))
    # dOut: all ones gives constant-per-row dY (low tensor-core switching power, so ~3 % more
    # clock under the power cap than a random gradient); both are timed (upstream_alt)
    g_ones = torch.ones(n, h, device=dev, dtype=torch.bfloat16)
    g_normal = torch.randn(n, h, device=dev, generator=torch.Generator(device=dev).manual_seed(99)).bfloat16()
    g_out = g_ones if a.upstream == "ones" else g_normal
    g_aux = torch.ones((), device=dev, dtype=torch.float32)
    params = w.leaf_parameters()

    def step(xin):
        for p in params:
            p.grad = None
        xin.grad = None
        out, l_aux = P.ppmoe_forward(world, group, xin, w.gate, experts_by_rank, top_k=k,
                                     capacity_factor=a.capacity_factor)
        torch.autograd.backward([out, l_aux], [g_out, g_aux])
        P.sync_gate_gradients(world, group, w.gate)
        return out, l_aux

    def barrier():
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()

    clk = ClockSampler(range(world_size), active=(rank == 0))
    clk.__enter__()  # sampling starts before the warm-up; only the timed window counts
    for _ in range(a.warmup):
        step(x)
    barrier()

    lib = _lib.load()
    launches0 = lib.ppmoe_kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    clk.mark_start()
    ev0.record()
    h0 = time.perf_counter()
    for _ in range(a.steps):
        step(x)
    host_ms = (time.perf_counter() - h0) * 1e3 / a.steps  # host enqueue time (the step never syncs)
    ev1.record()
    barrier()
    clk.mark_end()
    clk.__exit__(None, None, None)
    launches = lib.ppmoe_kernel_launches() - launches0
    ms = ev0.elapsed_time(ev1) / a.steps
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t)
    value = n / (ms / 1e3)
    # per-entry-point CUDA-event times (roofline inputs) from a separate pass of the same
    # steps, so the headline timed region carries no profiling events
    with _ops.KernelProfile() as prof:
        barrier()
        for _ in range(a.steps):
            step(x)
        barrier()
    ksum = prof.summary()

    # ---- the same step with the other upstream gradient (untimed warm-up step first)
    alt_name = "normal" if a.upstream == "ones" else "ones"
    g_out = g_normal if a.upstream == "ones" else g_ones
    step(x)
    barrier()
    ev0.record()
    for _ in range(a.steps):
        step(x)
    ev1.record()
    barrier()
    t = torch.tensor([ev0.elapsed_time(ev1) / a.steps], device=dev, dtype=torch.float64)
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    upstream_alt = {"upstream_grad": alt_name, "value": n / (float(t) / 1e3), "ms_per_step": float(t)}
    g_out = g_ones if a.upstream == "ones" else g_normal

    # ---- roofline of the dominant kernel: the grouped expert GEMM (six launches per step)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("bf16_tflops_sustained", 1400.0)
    peak_src = "MEASURED_PEAKS.json bf16_tflops_sustained" if "bf16_tflops_sustained" in peaks else "fallback 1.4 PF/s"
    gemm_names = ["ppmoe_expert_fc1_fwd", "ppmoe_expert_fc2_fwd", "ppmoe_expert_fc2_dgrad", "ppmoe_expert_fc2_wgrad",
                  "ppmoe_expert_fc1_dgrad", "ppmoe_expert_fc1_wgrad"]
    # algorithmic work: kept (token, expert) pairs of this rank's experts (capacity may drop some)
    rt_ = _ops.route(x.detach(), w.gate.wg.detach(), k)
    pl_ = _ops.plan(rt_.idx, rt_.w, E, _ops.capacity_for(a.capacity_factor, n, k, E))
    router_fixups = int(rt_.fixups[0]) if (rt_.fixups is not None and E <= 16) else 0
    kept_all = pl_.kept.cpu()
    pairs = int(kept_all.sum())
    local_pairs = int(kept_all[rank * el:(rank + 1) * el].sum())
    flop_per_gemm = 2.0 * local_pairs * h * f
    gemm_ms = sum(ksum.get(nm, {}).get("ms", 0.0) for nm in gemm_names) / a.steps
    gemm_launches = sum(ksum.get(nm, {}).get("launches", 0) for nm in gemm_names) / a.steps
    achieved = 6 * flop_per_gemm / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists() and a.config == "c2" and tp == 1:
        try:
            traffic = json.loads(tfile.read_text()).get("grouped_gemm_sm100_bytes_per_launch")
        except Exception:
            traffic = None
    per_kernel = {nm: {"ms_per_step": round(v["ms"] / a.steps, 4), "launches_per_step": v["launches"] / a.steps}
                  for nm, v in sorted(ksum.items())}
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "kernel": "grouped_gemm_sm100 (6 launches/step: fc1/fc2 fwd, dgrad, wgrad)",
                "algorithmic": f"12*P_r*h*f flop per step on this rank, P_r={local_pairs} of P={pairs} kept pairs; "
                               f"{gemm_ms:.3f} ms of GEMM per step",
                "peak_source": peak_src, "gemm_share_of_step": gemm_ms / ms if ms else None,
                "timing": "kernel times from a profiled pass of the same K steps after the timed region",
                "frac_of_burst_peak": (achieved / peaks["bf16_tflops"]) if (achieved and "bf16_tflops" in peaks) else None,
                "peak_note": "peak = cuBLAS bf16 8192^3 back-to-back for 4 s on this pool (power-capped, the regime a "
                             "long step runs in); frac_of_burst_peak uses the short-burst figure. The power-capped "
                             "clock differs from box to box (see clocks), so frac can exceed 1 on a box that holds "
                             "a higher clock than the one the sustained figure was measured on"}

    # ---- end to end: host (pinned) input -> device -> fwd+bwd -> loss back to host
    e2e = None
    if not a.no_e2e:
        x_host = x.detach().cpu().pin_memory()  # the same BASELINE batch, from pinned host memory
        loss_host = [torch.empty(1, dtype=torch.float32).pin_memory() for _ in range(2)]
        loss_ev = [torch.cuda.Event() for _ in range(2)]
        # each rank copies its 1/T row slice over PCIe, NCCL all_gather replicates it; the next
        # batch's copy overlaps this batch's compute (P.ReplicatedFeed).  Step i's loss is read
        # on the host while step i+1 is already queued, so the device never idles on the host.
        feed = P.ReplicatedFeed(world, group, (n, h), torch.bfloat16, dev)

        def e2e_run(steps):
            losses = []
            feed.submit(x_host)
            for i in range(steps):
                xin = feed.take().detach().requires_grad_()
                if i + 1 < steps:
                    feed.submit(x_host)
                out, l_aux = step(xin)
                loss = out.sum(dtype=torch.float32) + l_aux
                loss_host[i % 2].copy_(loss.detach().reshape(1), non_blocking=True)
                loss_ev[i % 2].record()
                if i > 0:
                    loss_ev[(i - 1) % 2].synchronize()
                    losses.append(float(loss_host[(i - 1) % 2][0]))
            loss_ev[(steps - 1) % 2].synchronize()
            losses.append(float(loss_host[(steps - 1) % 2][0]))
            return losses

        e2e_run(2)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        e2e_run(a.steps)
        e1.record()
        barrier()
        ems = e0.elapsed_time(e1) / a.steps
        te = torch.tensor([ems], device=dev, dtype=torch.float64)
        if distributed:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": n / (float(te) / 1e3), "unit": UNIT, "h2d_bytes_per_step": feed.h2d_bytes,
               "d2h_bytes_per_step": 4, "ms_per_step": float(te),
               "h2d_scope": ("per rank: its 1/T row slice of the pinned [N,H] bf16 batch, replicated over "
                             + ("NVLink peer memory (copy-engine pulls)" if feed.arena is not None else
                                "an NCCL all_gather") if world_size > 1 else
                             "the whole pinned [N,H] bf16 batch (one rank)")
                            + "; the next batch's copy overlaps this batch's compute",
               "path": "paper_2304_11414_b200.ReplicatedFeed + ppmoe_forward + backward (C-ABI) from pinned host"}

    # ---- conventional all-to-all expert-parallel layer (DPMoE) at the same global N:
    # each rank routes its own N/T tokens and exchanges rows with two all-to-alls per pass
    a2a = None
    if not a.no_a2a:
        nr = n // tp
        x_dp = x.detach()[rank * nr:(rank + 1) * nr].clone().requires_grad_()
        g_dp = torch.ones(nr, h, device=dev, dtype=torch.bfloat16)

        def dp_step():
            for p in params:
                p.grad = None
            x_dp.grad = None
            out, l_aux = P.dpmoe_forward(world, group, x_dp, w.gate, experts_by_rank=experts_by_rank, top_k=k,
                                         capacity_factor=a.capacity_factor)
            torch.autograd.backward([out, l_aux], [g_dp, g_aux])
            P.dpmoe_sync_gradients(world, group, w.gate)

        for _ in range(a.warmup):
            dp_step()
        barrier()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record()
        for _ in range(a.steps):
            dp_step()
        d1.record()
        barrier()
        dms = torch.tensor([d0.elapsed_time(d1) / a.steps], device=dev, dtype=torch.float64)
        if distributed:
            dist.all_reduce(dms, op=dist.ReduceOp.MAX)
        a2a_value = n / (float(dms) / 1e3)
        a2a = {"value": a2a_value, "unit": UNIT, "ms_per_step": float(dms), "ppmoe_over_a2a": value / a2a_value,
               "layer": "dpmoe_forward (all-to-all dispatch/return, same grouped GEMM kernels), N/T tokens per rank"}

    cb = None
    if rank == 0 and world_size == 1 and not a.no_cpu_baseline:
        cb, _ = cpu_baseline(h, E, k, f, target_s=a.cpu_seconds)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world_size, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "bf16", "data": f"synthetic: BASELINE.md inputs of the {a.config.upper()} layer, weights "
                                f"MoeLayerWeights.init(h, E, Rng(0)) and hidden Rng(1, 99).normal((N, h)), both "
                                f"rounded to bf16 (Philox, bit-identical to the reference init; {init_s:.1f} s)",
                "config": config_of(a, world_size), "roofline": roofline, "cpu_baseline": cb, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clk.summary(), "a2a_comparator": a2a, "kernels": per_kernel,
                "host_enqueue_ms_per_step": round(host_ms, 3), "upstream_alt": upstream_alt,
                "router": {"kernel": "tensor-core logits + guard band + fp64 fix-up" if E <= 16 else
                           "FP64 tensor-core (DMMA) logits",
                           "fixup_tokens": router_fixups if E <= 16 else None,
                           "fixup_scope": "tokens of the full N-token batch re-routed in fp64 by one routing call "
                                          "(adjacent top-(k+1) logit gap within the error bound)"},
                "gemm_launches_per_step": gemm_launches}
        print(json.dumps(line), flush=True)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
