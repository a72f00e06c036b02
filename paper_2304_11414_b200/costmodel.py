"""Cost model of the MoE layer recalibrated with measured B200 numbers.

Restates the reference's analytical layer model (costmodel.py:171-310: FFN FLOPs, ring
all-reduce / all-to-all latencies, `layer_forward_latency` for "moe_ppmoe" and
"moe_dpmoe", `breakdown_report`'s percentage view) and feeds it B200 parameters measured
by this repo: the grouped-GEMM throughput inside the step, the NVLink bandwidth of the
exchange, the barrier latency.  `measured_breakdown` turns a bench.py JSON line (its
per-entry-point CUDA-event timings) into the same component rows, so model and
measurement can be put side by side (tools/costmodel_report.py).

Two deliberate differences from the reference formulas, both noted in SURVEY §8(f):
the all-reduce term uses NCCL's bus-bandwidth convention 2(T-1)/T·m/B (the reference's
2(T-1)·m/B omits the ring's 1/T, costmodel.py:188-192), and the expert FLOPs use the
top-k pair count 2·N·k·h·f per GEMM (the reference's 16·b·s·h² is the k = 1, f = 4h case).
"""

from __future__ import annotations

from dataclasses import dataclass

ELEM_BYTES = 2.0


@dataclass(frozen=True)
class B200Profile:
    flops: float        # grouped expert GEMM, FLOP/s, measured inside the step
    nvlink_bw: float    # bytes/s per GPU, measured exchange pull bandwidth
    startup: float      # s per collective step (barrier / hop latency)
    hbm_bw: float       # bytes/s, measured copy bandwidth
    fp64_flops: float = 37e12  # router logits are fp64 (bit-exact routing)


def lat_all_reduce(n: int, payload: float, bw: float, startup: float = 0.0, ring_factor: bool = True) -> float:
    """Ring all-reduce: 2(n-1)(t_s + m/(n B)) (bus-bandwidth convention) or the reference's
    2(n-1)(t_s + m/B) with ring_factor=False (costmodel.py:188-192)."""
    if n <= 1:
        return 0.0
    per = payload / n if ring_factor else payload
    return 2.0 * (n - 1) * (startup + per / bw)


def lat_all_to_all(n: int, chunk: float, bw: float, startup: float = 0.0) -> float:
    """(n-1)(t_s + m n/(2B)) for a per-peer chunk of m bytes (costmodel.py:181-185)."""
    if n <= 1:
        return 0.0
    return (n - 1) * (startup + chunk * n / (2.0 * bw))


def expert_flops(tokens: int, hidden: int, top_k: int, ffn: int | None = None, backward: bool = False) -> float:
    """Expert GEMM FLOPs of one layer: 4·N·k·h·f forward, 12·N·k·h·f forward+backward."""
    f = ffn or 4 * hidden
    return (12.0 if backward else 4.0) * tokens * top_k * hidden * f


def layer_latency(kind: str, tokens: int, hidden: int, experts: int, top_k: int, tp: int, prof: B200Profile,
                  backward: bool = True) -> dict:
    """Model of one MoE layer (fwd, or fwd+bwd) on a group of tp GPUs
    (layer_forward_latency, costmodel.py:259-309), in seconds per component."""
    act = ELEM_BYTES * tokens * hidden
    passes = 2 if backward else 1
    # router: X·Wg in fp64 (FP64 pipe) or the X read, whichever is slower; the backward
    # re-reads X for dWg and writes the gate term into dX
    gating = max(ELEM_BYTES * tokens * hidden / prof.hbm_bw, 2.0 * tokens * hidden * experts / prof.fp64_flops)
    if backward:
        gating += 2.0 * ELEM_BYTES * tokens * hidden / prof.hbm_bw
    compute = expert_flops(tokens, hidden, top_k, backward=backward) / (tp * prof.flops)
    if kind == "moe_ppmoe":
        comm = passes * lat_all_reduce(tp, act, prof.nvlink_bw, prof.startup)
        return {"gating": gating, "expert_compute": compute, "moe_all_reduce": comm,
                "total": gating + compute + comm}
    if kind == "moe_dpmoe":
        a2a = lat_all_to_all(tp, act / tp * top_k / tp, prof.nvlink_bw, prof.startup)
        comm = 2 * passes * a2a
        return {"gating": gating / tp, "expert_compute": compute, "a2a": comm, "total": gating / tp + compute + comm}
    raise ValueError(f"unknown layer kind {kind!r}")


GEMM_CALLS = ("ppmoe_expert_fc1_fwd", "ppmoe_expert_fc2_fwd", "ppmoe_expert_fc2_dgrad", "ppmoe_expert_fc2_wgrad",
              "ppmoe_expert_fc1_dgrad", "ppmoe_expert_fc1_wgrad")
GATING_CALLS = ("ppmoe_route", "ppmoe_dispatch_plan", "ppmoe_gate_bwd")
EXCHANGE_CALLS = ("ppmoe_nvl_barrier", "ppmoe_nvl_owner_gather", "ppmoe_nvl_pull_blocks", "ppmoe_nvl_pull_blocks_ce",
                  "ppmoe_nvl_sum_rows")


def measured_breakdown(bench: dict) -> dict:
    """Component rows (seconds per step) from a bench.py JSON line: gating (router, plan,
    gate backward), expert compute (the six grouped GEMMs), exchange (the NVLink exchange
    calls; on one GPU the owner-gather combines), others (gather, bwd_dy, dWg, ...), and the
    remainder of the measured step (overlap gaps, NCCL, launch latency)."""
    k = bench.get("kernels", {})

    def s(names):
        return sum(k.get(n, {}).get("ms_per_step", 0.0) for n in names) / 1e3

    total = bench["ms_per_step"] / 1e3
    gating, compute, exchange = s(GATING_CALLS), s(GEMM_CALLS), s(EXCHANGE_CALLS)
    listed = sum(v.get("ms_per_step", 0.0) for v in k.values()) / 1e3
    others = listed - gating - compute - exchange
    return {"gating": gating, "expert_compute": compute, "exchange": exchange, "others": others,
            "unaccounted": total - listed, "total": total}


def breakdown_rows(parts: dict) -> list[tuple[str, float, float]]:
    """(name, value, % of total) rows in the reference's Table-1 style (breakdown_report,
    costmodel.py:483-509)."""
    total = parts["total"]
    if total <= 0:
        raise ValueError("breakdown total must be positive")
    return [(name, v, 100.0 * v / total) for name, v in parts.items() if name != "total"]
