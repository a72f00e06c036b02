"""Orchestration of the sm_100a kernels for one PPMoE layer step (forward + backward).

Every device computation below goes through the C-ABI library (``_lib``); torch
only allocates buffers, provides the stream and runs NCCL collectives.  There is
no host synchronisation between routing and the expert GEMMs: the dispatch plan
stays on the device (padded segments) and the GEMM tile schedulers read it.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import ptr

INT32_MAX = 2**31 - 1
_DTYPE_CODE = {torch.bfloat16: 0, torch.float32: 1}


def dtype_code(dt: torch.dtype) -> int:
    try:
        return _DTYPE_CODE[dt]
    except KeyError:
        raise ValueError(f"PPMoE kernels support bf16 and fp32 activations, got {dt}") from None


_GUARDS: list = []  # (guard view, expected bytes) of PPMOE_GUARD=1 buffers
_GUARD_ROWS = 64


def _act(shape, dtype, device) -> torch.Tensor:
    """Activation/scratch buffer.  PPMOE_POISON=1 fills it with NaN (ints: -7) so that any
    read of a row a kernel should have written shows up in the parity tests.
    PPMOE_GUARD=1 (test mode; compute-sanitizer is not available on the pool) allocates 64
    extra rows after the buffer, filled with a random byte pattern that ``check_guards``
    verifies: a kernel writing past the rows it was given corrupts them."""
    poison = os.environ.get("PPMOE_POISON") == "1"
    if os.environ.get("PPMOE_GUARD") == "1":
        shape = tuple(shape) if isinstance(shape, (tuple, list)) else (int(shape),)
        full = torch.empty((shape[0] + _GUARD_ROWS,) + shape[1:], dtype=dtype, device=device)
        main, guard = full[: shape[0]], full[shape[0]:]
        pattern = torch.randint(0, 256, (guard.numel() * guard.element_size(),), dtype=torch.uint8, device=device)
        guard.view(torch.uint8).view(-1).copy_(pattern)
        _GUARDS.append((guard, pattern))
        if poison:
            main.fill_(float("nan") if dtype.is_floating_point else -7)
        return main
    if poison:
        shape = tuple(shape) if isinstance(shape, (tuple, list)) else (int(shape),)
        return torch.full(shape, float("nan") if dtype.is_floating_point else -7, dtype=dtype, device=device)
    return torch.empty(shape, dtype=dtype, device=device)


def check_guards(clear: bool = True) -> int:
    """Verify every PPMOE_GUARD guard region (synchronises); raises on a corrupted one.
    Returns the number of guards checked."""
    torch.cuda.synchronize()
    n = len(_GUARDS)
    bad = [i for i, (g, pat) in enumerate(_GUARDS) if not torch.equal(g.view(torch.uint8).reshape(-1), pat)]
    if clear:
        _GUARDS.clear()
    if bad:
        raise RuntimeError(f"out-of-bounds write: {len(bad)} of {n} guard regions past PPMoE buffers were modified")
    return n


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def _stream():
    return _lib.stream_ptr()


class sm_budget:
    """Context manager: persistent GEMMs use at most `sms` SMs (0 = all) so that an NCCL
    collective running concurrently on its own stream gets SMs (overlap instead of queueing)."""

    def __init__(self, sms: int):
        self.sms = int(sms)

    active = 0  # the budget in force (0 = none)

    def __enter__(self):
        if self.sms:
            _lib.call("ppmoe_set_gemm_sm_budget", self.sms)
            sm_budget.active = self.sms
        return self

    def __exit__(self, *exc):
        if self.sms:
            _lib.call("ppmoe_set_gemm_sm_budget", 0)
            sm_budget.active = 0
        return False

    @staticmethod
    def release():
        """Drop the budget early (the rest of the block runs on every SM)."""
        if sm_budget.active:
            _lib.call("ppmoe_set_gemm_sm_budget", 0)
            sm_budget.active = 0


def overlap_sm_budget() -> int:
    """GEMM SM budget while a collective is in flight: PPMOE_OVERLAP_SMS (default: all but 16)."""
    v = os.environ.get("PPMOE_OVERLAP_SMS")
    if v is not None:
        return int(v)
    n = _lib.query("ppmoe_num_sms")
    return max(2, n - 16)


class KernelProfile:
    """Per-entry-point CUDA-event timing of the C-ABI calls made inside the block
    (events on the launching stream; used by bench.py for the roofline numbers)."""

    def __init__(self):
        self.records = []

    def __enter__(self):
        global _PROFILE
        _PROFILE = self
        return self

    def __exit__(self, *exc):
        global _PROFILE
        _PROFILE = None
        return False

    def summary(self) -> dict:
        torch.cuda.synchronize()
        out: dict = {}
        for name, a, b in self.records:
            cell = out.setdefault(name, {"launches": 0, "ms": 0.0})
            cell["launches"] += 1
            cell["ms"] += a.elapsed_time(b)
        return out


_PROFILE: KernelProfile | None = None


def call(name: str, *args):
    """C-ABI call; timed with CUDA events when a KernelProfile is active."""
    prof = _PROFILE
    if prof is None:
        return _lib.call(name, *args)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    rc = _lib.call(name, *args)
    b.record()
    prof.records.append((name, a, b))
    return rc


# --------------------------------------------------------------------- routing


@dataclass
class Route:
    idx: torch.Tensor  # [N, k] int32
    w: torch.Tensor  # [N, k] fp32
    scores: torch.Tensor  # [N, E] fp32
    l_aux: torch.Tensor  # [2] fp64 (value, sum of fractions)
    top1_counts: torch.Tensor  # [E] int32
    fixups: torch.Tensor | None = None  # [1] int32: tokens the tensor-core router re-routed in fp64


@dataclass
class Plan:
    counts: torch.Tensor  # [E] routed pairs per expert (pre-capacity)
    kept: torch.Tensor  # [E]
    seg: torch.Tensor  # [E+1] padded segment starts
    tok_sorted: torch.Tensor  # [rows_cap_global]
    w_sorted: torch.Tensor
    pair_pos: torch.Tensor  # [N, k]
    capacity: int


def route(hidden: torch.Tensor, wg: torch.Tensor, k: int, override: torch.Tensor | None = None,
          score_sums: torch.Tensor | None = None) -> Route:
    """Gate GEMV + softmax + top-k + aux loss (moe.py:196-223) on the device."""
    n, h = hidden.shape
    e = wg.shape[1]
    dev = hidden.device
    idx = torch.empty((n, k), dtype=torch.int32, device=dev)
    w = torch.empty((n, k), dtype=torch.float32, device=dev)
    scores = torch.empty((n, e), dtype=torch.float32, device=dev)
    l_aux = torch.empty(2, dtype=torch.float64, device=dev)
    cnt1 = torch.empty(e, dtype=torch.int32, device=dev)
    ws = _ws(_lib.query("ppmoe_route_workspace_bytes_h", n, h, e, k), dev)
    call("ppmoe_route", ptr(hidden), dtype_code(hidden.dtype), ptr(wg), n, h, e, k, ptr(override), ptr(idx), ptr(w),
         ptr(scores), ptr(l_aux), ptr(cnt1), ptr(score_sums), ptr(ws), ws.numel(), _stream())
    # workspace layout (route.cu): score-sum records (one per 16 tokens) | top-1 counts, fix-up count | queue
    off = ((n + 15) // 16 * e * 8 + 255) // 256 * 256 + e * 4
    return Route(idx, w, scores, l_aux, cnt1, ws[off:off + 4].view(torch.int32))


def route_sliced(world, group, hidden: torch.Tensor, wg: torch.Tensor, k: int,
                 override: torch.Tensor | None = None) -> Route:
    """Routing of a replicated activation split across the TP group: each rank routes its
    N/T-token slice, and the slices are gathered identically on every rank -- over NVLink
    peer memory (one barrier + ppmoe_nvl_route_gather), or in-place NCCL all-gathers without
    the arena (the reference gates every replica identically, moe.py:288-291; the logits are
    computed once instead of T times).  l_aux is
    recombined on the device from the per-slice score sums and top-1 counts in rank order
    (ppmoe_route_combine_stats: deterministic, identical on all ranks)."""
    n, h = hidden.shape
    e = wg.shape[1]
    t = group.size
    me = world.rank_in(group)
    nr = n // t
    dev = hidden.device
    sl = slice(me * nr, (me + 1) * nr)
    idx = torch.empty((n, k), dtype=torch.int32, device=dev)
    w = torch.empty((n, k), dtype=torch.float32, device=dev)
    scores = torch.empty((n, e), dtype=torch.float32, device=dev)
    stats = torch.zeros((t, 4 * e), dtype=torch.int32, device=dev)  # per rank: E fp64 sums | E counts | pad
    mine = stats[me]
    l_aux_slice = torch.empty(2, dtype=torch.float64, device=dev)
    ws = _ws(_lib.query("ppmoe_route_workspace_bytes_h", nr, h, e, k), dev)
    ov = None if override is None else override[sl].contiguous()
    from . import nvlink

    if nvlink.enabled(world, group, torch.bfloat16, 8):
        # peer memory instead of four NCCL all-gathers: route into this rank's record of a
        # peer-visible buffer, one barrier, every rank copies the T records (one kernel).
        # Two records alternate, so a rank that runs ahead cannot overwrite one a peer still
        # reads (it would have to pass the next call's barrier first).
        ar = nvlink.arena(world, group)
        ar.route_parity = getattr(ar, "route_parity", 0) ^ 1
        name = f"route{ar.route_parity}"
        rec = ar.tensor(name, (4 * e + nr * (2 * k + e),), torch.int32)
        r_idx = rec[4 * e:4 * e + nr * k]
        r_w = rec[4 * e + nr * k:4 * e + 2 * nr * k].view(torch.float32)
        r_sc = rec[4 * e + 2 * nr * k:].view(torch.float32)
        call("ppmoe_route", ptr(hidden[sl]), dtype_code(hidden.dtype), ptr(wg), nr, h, e, k, ptr(ov), ptr(r_idx),
             ptr(r_w), ptr(r_sc), ptr(l_aux_slice), ptr(rec[2 * e:3 * e]), ptr(rec[:2 * e]), ptr(ws), ws.numel(),
             _stream())
        ar.barrier(nvlink.CH_ROUTE)
        call("ppmoe_nvl_route_gather", ar.table(name), t, nr, k, e, ptr(idx), ptr(w), ptr(scores), ptr(stats),
             _stream())
    else:
        _route_slice_nccl(world, group, hidden, wg, k, sl, ov, idx, w, scores, stats, mine, l_aux_slice, ws)
    l_aux = torch.empty(2, dtype=torch.float64, device=dev)
    cnt = torch.empty(e, dtype=torch.int32, device=dev)
    call("ppmoe_route_combine_stats", ptr(stats), t, n, e, ptr(l_aux), ptr(cnt), _stream())
    return Route(idx, w, scores, l_aux, cnt)


def _route_slice_nccl(world, group, hidden, wg, k, sl, ov, idx, w, scores, stats, mine, l_aux_slice, ws):
    """route_sliced without the NVLink arena: route the slice in place, then in-place NCCL
    all-gathers of the four routing tensors."""
    import torch.distributed as dist

    n, h = hidden.shape
    e = wg.shape[1]
    t = group.size
    me = world.rank_in(group)
    nr = n // t
    call("ppmoe_route", ptr(hidden[sl]), dtype_code(hidden.dtype), ptr(wg), nr, h, e, k, ptr(ov), ptr(idx[sl]),
         ptr(w[sl]), ptr(scores[sl]), ptr(l_aux_slice), ptr(mine[2 * e:3 * e]), ptr(mine[:2 * e]), ptr(ws), ws.numel(),
         _stream())
    pg = world.torch_group(group)
    for full in (idx, w, scores, stats):
        dist.all_gather_into_tensor(full, full[me * full.shape[0] // t:(me + 1) * full.shape[0] // t], group=pg)


def capacity_for(capacity_factor: float, tokens: int, k: int, num_experts: int) -> int:
    """C = ceil(cf * k * tokens / E), the k-slot generalisation of moe.py:352."""
    if math.isinf(capacity_factor):
        return INT32_MAX
    return min(INT32_MAX, math.ceil(capacity_factor * k * tokens / num_experts))


def plan(idx: torch.Tensor, w: torch.Tensor | None, num_experts: int, capacity: int = INT32_MAX,
         rank_offset: torch.Tensor | None = None) -> Plan:
    """Stable per-expert dispatch plan with capacity (moe.py:226-235, 345-360)."""
    n, k = idx.shape
    dev = idx.device
    e = num_experts
    rows_cap = n * k + 128 * e
    counts = torch.empty(e, dtype=torch.int32, device=dev)
    kept = torch.empty(e, dtype=torch.int32, device=dev)
    seg = torch.empty(e + 1, dtype=torch.int32, device=dev)
    tok_sorted = torch.empty(rows_cap, dtype=torch.int32, device=dev)
    w_sorted = torch.empty(rows_cap, dtype=torch.float32, device=dev)
    pair_pos = torch.empty((n, k), dtype=torch.int32, device=dev)
    ws = _ws(_lib.query("ppmoe_dispatch_workspace_bytes", n, e, k), dev)
    call("ppmoe_dispatch_plan", ptr(idx), ptr(w), n, e, k, int(capacity), ptr(rank_offset), ptr(counts), ptr(kept),
         ptr(seg),
         ptr(tok_sorted), ptr(w_sorted), ptr(pair_pos), rows_cap, ptr(ws), ws.numel(), _stream())
    return Plan(counts, kept, seg, tok_sorted, w_sorted, pair_pos, capacity)


def dropout_descriptor(kept: torch.Tensor, num_experts: int, e0: int, el: int, h: int, key0: int, key1: int,
                       threshold: int, first_draw: int) -> torch.Tensor:
    """Device descriptor of the reference's dropout stream for local experts [e0, e0+el)
    (ppmoe_dropout_stream): [key0, key1, threshold, first draw of each local expert]."""
    desc = torch.empty(3 + el, dtype=torch.int64, device=kept.device)
    call("ppmoe_dropout_stream", ptr(kept), num_experts, e0, el, h, ctypes.c_ulonglong(key0), ctypes.c_ulonglong(key1),
         ctypes.c_ulonglong(threshold), ctypes.c_ulonglong(first_draw), ptr(desc), _stream())
    return desc


def local_rows_cap(n: int, k: int, el: int, capacity: int) -> int:
    """Upper bound of the padded rows of `el` experts (no host sync on the true count)."""
    pairs = min(n * k, n * el)
    if capacity < INT32_MAX:
        pairs = min(pairs, capacity * el)
    return pairs + 128 * el


# --------------------------------------------------------------------- experts


@dataclass
class ExpertFwdState:
    e0: int
    el: int
    rows_cap: int
    seg: torch.Tensor  # view of plan.seg starting at e0 (el+1 entries)
    xs: torch.Tensor
    tok_l: torch.Tensor
    w_l: torch.Tensor
    gelu_grad: torch.Tensor
    act: torch.Tensor
    y: torch.Tensor
    drop_p: float = 0.0
    drop: torch.Tensor | None = None  # dropout stream descriptor (moe.DropoutStream.descriptor)


def experts_forward(hidden, pl: Plan, e0: int, el: int, up, down, bias_up, bias_down, k: int, weight_scaling: bool,
                    out_acc: torch.Tensor, chunks: int = 1, on_chunk=None, drop_p: float = 0.0,
                    drop: torch.Tensor | None = None, y_mirror: torch.Tensor | None = None, owner_table: torch.Tensor | None = None,
                    owner_rows: int = 0, owner_slots: torch.Tensor | None = None) -> ExpertFwdState:
    """index-slice gather -> fc1 (+bias, GeLU) -> fc2 (+bias, gate-scaled scatter-add combine)
    for experts [e0, e0+el) (moe.py:294-305).  out_acc None: fc2 only stores Y and the
    combine is done by ``combine`` (gather, no atomics).  With chunks > 1 the two GEMMs run per token
    chunk (each expert segment is ascending in token id, so a chunk is a row range) and
    ``on_chunk(c)`` is called once chunk c's rows of out_acc are final on this rank."""
    n, h = hidden.shape
    f = up.shape[2]
    dt = dtype_code(hidden.dtype)
    dev = hidden.device
    rows_cap = local_rows_cap(n, k, el, pl.capacity)
    seg = pl.seg[e0:e0 + el + 1]
    xs = _act((rows_cap, h), hidden.dtype, dev)
    tok_l = _act(rows_cap, torch.int32, dev)
    w_l = _act(rows_cap, torch.float32, dev)
    s = _stream()
    call("ppmoe_gather", ptr(hidden), dt, n, h, ptr(seg), el, ptr(pl.tok_sorted), ptr(pl.w_sorted), rows_cap, ptr(xs),
         ptr(tok_l), ptr(w_l), s)
    gelu_grad = _act((rows_cap, f), hidden.dtype, dev)
    act = _act((rows_cap, f), hidden.dtype, dev)
    y = _act((rows_cap, h), hidden.dtype, dev)

    def gemms(rlo, rhi):
        call("ppmoe_expert_fc1_fwd", dt, ptr(xs), ptr(up), ptr(bias_up), ptr(seg), el, h, f, rows_cap, ptr(rlo),
             ptr(rhi), ptr(gelu_grad), ptr(act), s)
        if owner_table is not None or owner_slots is not None:
            # combine fused into the epilogue: rows go to their owners (fp32 accumulators or bf16 slots)
            call("ppmoe_expert_fc2_fwd_owner", dt, ptr(act), ptr(down), ptr(bias_down), ptr(seg), el, h, f, rows_cap,
                 ptr(tok_l), ptr(w_l), int(bool(weight_scaling)), float(drop_p), ptr(drop), ptr(y), ptr(owner_table),
                 ptr(owner_slots), ptr(pl.pair_pos), k, int(owner_rows), s)
            return
        call("ppmoe_expert_fc2_fwd", dt, ptr(act), ptr(down), ptr(bias_down), ptr(seg), el, h, f, rows_cap, ptr(rlo),
             ptr(rhi), ptr(tok_l), ptr(w_l), int(bool(weight_scaling)), float(drop_p), ptr(drop), ptr(y), ptr(y_mirror),
             ptr(out_acc), s)

    if chunks <= 1:
        gemms(None, None)
    else:
        rlo = torch.empty((chunks + 1) * el, dtype=torch.int32, device=dev)
        rhi = torch.empty((chunks + 1) * el, dtype=torch.int32, device=dev)
        call("ppmoe_chunk_rows", ptr(tok_l), ptr(seg), ptr(pl.kept[e0:e0 + el]), el, n, chunks, ptr(rlo), ptr(rhi), s)
        budget = overlap_sm_budget()
        for c in range(chunks):
            # from chunk 1 on, the previous chunk's all-reduce runs concurrently
            with sm_budget(budget if c > 0 else 0):
                gemms(rlo[c * el:(c + 1) * el], rhi[c * el:(c + 1) * el])
            if on_chunk is not None:
                on_chunk(c)
        # padding rows still need fc1 (their GeLU'/Act rows meet zero dY in the backward)
        pad_lo, pad_hi = rlo[chunks * el:], rhi[chunks * el:]
        call("ppmoe_expert_fc1_fwd", dt, ptr(xs), ptr(up), ptr(bias_up), ptr(seg), el, h, f, rows_cap, ptr(pad_lo),
             ptr(pad_hi), ptr(gelu_grad), ptr(act), s)
    return ExpertFwdState(e0, el, rows_cap, seg, xs, tok_l, w_l, gelu_grad, act, y, drop_p, drop)


def expert_pipeline(xsrc: torch.Tensor, seg: torch.Tensor, el: int, tok_sorted: torch.Tensor,
                    w_sorted: torch.Tensor | None, rows_cap: int, up, down, bias_up, bias_down, weight_scaling: bool,
                    out_acc: torch.Tensor, drop_p: float = 0.0, drop: torch.Tensor | None = None) -> ExpertFwdState:
    """gather(xsrc rows by tok_sorted) -> fc1 -> fc2 with the scatter-add into out_acc[tok],
    for an arbitrary padded-segment layout (used by the all-to-all comparator's owner side,
    where tok_sorted maps owner rows to receive-buffer rows)."""
    n, h = xsrc.shape
    f = up.shape[2]
    dt = dtype_code(xsrc.dtype)
    dev = xsrc.device
    xs = _act((rows_cap, h), xsrc.dtype, dev)
    tok_l = _act(rows_cap, torch.int32, dev)
    w_l = _act(rows_cap, torch.float32, dev)
    s = _stream()
    call("ppmoe_gather", ptr(xsrc), dt, n, h, ptr(seg), el, ptr(tok_sorted), ptr(w_sorted), rows_cap, ptr(xs),
         ptr(tok_l), ptr(w_l), s)
    gelu_grad = _act((rows_cap, f), xsrc.dtype, dev)
    act = _act((rows_cap, f), xsrc.dtype, dev)
    y = _act((rows_cap, h), xsrc.dtype, dev)
    call("ppmoe_expert_fc1_fwd", dt, ptr(xs), ptr(up), ptr(bias_up), ptr(seg), el, h, f, rows_cap, None, None,
         ptr(gelu_grad), ptr(act), s)
    call("ppmoe_expert_fc2_fwd", dt, ptr(act), ptr(down), ptr(bias_down), ptr(seg), el, h, f, rows_cap, None, None,
         ptr(tok_l), ptr(w_l), int(bool(weight_scaling)), float(drop_p), ptr(drop), ptr(y), None, ptr(out_acc), s)
    return ExpertFwdState(0, el, rows_cap, seg, xs, tok_l, w_l, gelu_grad, act, y, drop_p, drop)


def combine_mode(dtype: torch.dtype, hidden: int) -> str:
    """How one rank sums its tokens' expert rows: "owner" (the owner-gather kernel of the
    NVLink exchange with a group of one, bf16), "gather" (ppmoe_combine / ppmoe_input_grads)
    or "scatter" (fp32 scatter-add in the GEMM epilogues).  PPMOE_COMBINE overrides."""
    mode = os.environ.get("PPMOE_COMBINE")
    if mode is None:
        mode = "owner"
    if mode == "owner" and not (dtype == torch.bfloat16 and hidden % 8 == 0):
        mode = "gather"
    return mode


def local_combine(rows: torch.Tensor, st: ExpertFwdState, pl: Plan, idx: torch.Tensor, w: torch.Tensor | None,
                  out: torch.Tensor, dl: torch.Tensor | None = None, wg: torch.Tensor | None = None) -> torch.Tensor:
    """out[t] = sum over t's pairs (slot order) of w·rows[row] (+ dl[t]·wgᵀ): the owner-gather
    kernel of csrc/nvlink.cu for a group of one (all experts local, e0 = 0)."""
    n, h = out.shape
    k = pl.pair_pos.shape[1]
    e = wg.shape[1] if wg is not None else 0
    rows_set = (ctypes.c_void_p * 1)(rows.data_ptr())
    call("ppmoe_nvl_owner_gather", rows_set, ptr(pl.seg), st.el, ptr(idx), ptr(pl.pair_pos), ptr(w), n, k, h, 1, 0,
         ptr(dl), ptr(wg), e, ptr(out), None, None, 0, _stream())
    return out


def combine(rows: torch.Tensor, st: ExpertFwdState, pl: Plan, w: torch.Tensor | None, out: torch.Tensor,
            dl: torch.Tensor | None = None, wg: torch.Tensor | None = None) -> torch.Tensor:
    """out[t] = sum over t's local pairs (slot order) of w·rows[row] (+ dl[t]·wgᵀ): the top-k
    combine of Y (scale_rows + index_assign, tensor.py:184-272), or with the per-row dX and
    the gate term the input gradient, as a deterministic gather."""
    n, h = out.shape
    k = pl.pair_pos.shape[1]
    e = wg.shape[1] if wg is not None else 0
    call("ppmoe_combine", dtype_code(out.dtype), ptr(rows), ptr(st.seg), st.el, ptr(pl.pair_pos), ptr(w), n, k, h,
         ptr(dl), ptr(wg), e, ptr(out), _stream())
    return out


def a2a_compact(pl: Plan, idx: torch.Tensor, num_experts: int):
    """Compact expert-major layout of the kept pairs: (cstart [E+1], tok_c, w_c, pair_pos_c)."""
    dev = idx.device
    n, k = idx.shape
    rows = n * k
    cstart = torch.empty(num_experts + 1, dtype=torch.int32, device=dev)
    tok_c = _act(max(rows, 1), torch.int32, dev)
    w_c = _act(max(rows, 1), torch.float32, dev)
    pos_c = torch.empty((n, k), dtype=torch.int32, device=dev)
    call("ppmoe_a2a_compact", ptr(pl.tok_sorted), ptr(pl.w_sorted), ptr(pl.seg), ptr(pl.kept), num_experts, ptr(idx),
         ptr(pl.pair_pos), n * k, ptr(cstart), ptr(tok_c), ptr(w_c), ptr(pos_c), _stream())
    return cstart, tok_c, w_c, pos_c


def owner_layout(recv_counts: torch.Tensor, t: int, el: int, rows_cap: int):
    dev = recv_counts.device
    seg = torch.empty(el + 1, dtype=torch.int32, device=dev)
    rmap = torch.empty(max(rows_cap, 1), dtype=torch.int32, device=dev)
    call("ppmoe_a2a_owner_layout", ptr(recv_counts), t, el, rows_cap, ptr(seg), ptr(rmap), _stream())
    return seg, rmap


def permute_rows(src: torch.Tensor, rows: int, rmap: torch.Tensor, dst: torch.Tensor) -> None:
    """dst[rmap[o]] = src[o] for the first `rows` owner rows (rmap < 0: padding)."""
    call("ppmoe_a2a_permute_rows", ptr(src), dtype_code(src.dtype), src.shape[1], int(rows), ptr(rmap), ptr(dst),
         _stream())


def compact_combine(rows: torch.Tensor, cstart: torch.Tensor, idx: torch.Tensor, pos_c: torch.Tensor,
                    w: torch.Tensor | None, out: torch.Tensor, dl: torch.Tensor | None = None,
                    wg: torch.Tensor | None = None) -> torch.Tensor:
    """out[t] = sum over t's kept pairs (slot order) of w·rows[pos_c[t, s]] (+ dl[t]·wgᵀ), for
    rows in the compact expert-major layout of the all-to-all comparator: the owner-gather
    kernel with a group of one and every expert "local" (row = pos_c - cstart[0] = pos_c)."""
    n, h = out.shape
    k = pos_c.shape[1]
    e_cols = wg.shape[1] if wg is not None else 0
    num_experts = cstart.numel() - 1
    if out.dtype != torch.bfloat16 or h % 8:  # fp32 reference-precision mode: the generic gather
        call("ppmoe_combine", dtype_code(out.dtype), ptr(rows), ptr(cstart), num_experts, ptr(pos_c), ptr(w), n, k, h,
             ptr(dl), ptr(wg), e_cols, ptr(out), _stream())
        return out
    rows_set = (ctypes.c_void_p * 1)(rows.data_ptr())
    call("ppmoe_nvl_owner_gather", rows_set, ptr(cstart), num_experts, ptr(idx), ptr(pos_c), ptr(w), n, k, h, 1, 0,
         ptr(dl), ptr(wg), e_cols, ptr(out), None, None, 0, _stream())
    return out


def scatter_rows(src: torch.Tensor, nrows: torch.Tensor, tok: torch.Tensor, w: torch.Tensor | None,
                 dst: torch.Tensor) -> None:
    call("ppmoe_scatter_rows", ptr(src), dtype_code(src.dtype), src.shape[1], ptr(nrows), ptr(tok), ptr(w), ptr(dst),
         _stream())


def _fused_colsums(dt: int, h: int) -> bool:
    """Bias-gradient column sums produced by bwd_dy / the fc2 dgrad epilogue (bf16 path)."""
    return dt == 0 and h % 256 == 0 and os.environ.get("PPMOE_FUSED_COLSUM", "1") != "0"


def experts_backward_data(grad_out, st: ExpertFwdState, up, down, weight_scaling: bool, dx_acc: torch.Tensor | None,
                          has_bias: bool = True, dxs: torch.Tensor | None = None):
    """Data-gradient half of the experts' backward: dY/dw (scale_rows + index_assign backward),
    dH = dY·downᵀ ⊙ GeLU', and dX_acc[tok] += dH·upᵀ (or, with ``dxs``, the per-row dH·upᵀ
    stored for the gather in ``gate_grads``).  Returns (dy, dh, dw, parts) where parts
    are the per-32-row column-sum partials of dY and dH (bias gradients) or None."""
    h = grad_out.shape[1]
    f = up.shape[2]
    el, rows_cap = st.el, st.rows_cap
    dt = dtype_code(grad_out.dtype)
    dev = grad_out.device
    s = _stream()
    fused = has_bias and _fused_colsums(dt, h)
    dy_part = torch.empty((max(rows_cap // 32, 1), h), dtype=torch.float32, device=dev) if fused else None
    dh_part = torch.empty((max(rows_cap // 32, 1), f), dtype=torch.float32, device=dev) if fused else None
    dy = _act((rows_cap, h), grad_out.dtype, dev)
    dw = _act(rows_cap, torch.float32, dev)
    call("ppmoe_bwd_dy", dt, ptr(grad_out), ptr(st.y), ptr(st.seg), el, h, rows_cap, ptr(st.tok_l), ptr(st.w_l),
         int(bool(weight_scaling)), float(st.drop_p), ptr(st.drop), ptr(dy), ptr(dw), ptr(dy_part), s)
    dh = _act((rows_cap, f), grad_out.dtype, dev)
    call("ppmoe_expert_fc2_dgrad", dt, ptr(dy), ptr(down), ptr(st.gelu_grad), ptr(st.seg), el, h, f, rows_cap, ptr(dh),
         ptr(dh_part), s)
    call("ppmoe_expert_fc1_dgrad", dt, ptr(dh), ptr(up), ptr(st.seg), el, h, f, rows_cap, ptr(st.tok_l), ptr(dx_acc),
         ptr(dxs), s)
    return dy, dh, dw, (dy_part, dh_part)


def experts_backward_weights(st: ExpertFwdState, dy, dh, up, down, has_bias: bool, parts=(None, None)):
    """Weight-gradient half: d down = Actᵀ·dY, d up = Xsᵀ·dH (variable-K grouped GEMMs) and
    the bias gradients.  Independent of dX, so it overlaps the dX all-reduce: under an
    `sm_budget` only the first GEMM leaves SMs free for it (PPMOE_BUDGET_SPLIT=0: both)."""
    h = dy.shape[1]
    f = up.shape[2]
    el, rows_cap = st.el, st.rows_cap
    dt = dtype_code(dy.dtype)
    dev = dy.device
    s = _stream()
    dy_part, dh_part = parts
    d_down = torch.empty_like(down)
    d_bd = torch.empty((el, h), dtype=dy.dtype, device=dev) if has_bias else None
    call("ppmoe_expert_fc2_wgrad", dt, ptr(st.act), ptr(dy), ptr(st.seg), el, h, f, rows_cap, ptr(d_down), ptr(d_bd),
         ptr(dy_part), s)
    if os.environ.get("PPMOE_BUDGET_SPLIT", "1") == "1":
        # the collective beside us finishes within the first GEMM: the second takes every SM
        # (T = 4: 5.82 vs 5.93 ms per step, T = 2: 10.79 vs 11.05; profiles/r01_sm_budget.md)
        sm_budget.release()
    d_up = torch.empty_like(up)
    d_bu = torch.empty((el, f), dtype=dy.dtype, device=dev) if has_bias else None
    call("ppmoe_expert_fc1_wgrad", dt, ptr(st.xs), ptr(dh), ptr(st.seg), el, h, f, rows_cap, ptr(d_up), ptr(d_bu),
         ptr(dh_part), s)
    return d_up, d_down, d_bu, d_bd


def gate_backward(rt: Route, pl: Plan, st: ExpertFwdState, dw: torch.Tensor, aux_grad: torch.Tensor | None,
                  out: torch.Tensor | None = None) -> torch.Tensor:
    """dL = d(loss)/d(logits) from the local pairs' dw and (on one rank) the aux loss."""
    n, e = rt.scores.shape
    k = rt.idx.shape[1]
    dl = out if out is not None else torch.empty((n, e), dtype=torch.float32, device=rt.scores.device)
    call("ppmoe_gate_bwd", ptr(rt.scores), ptr(rt.idx), ptr(pl.pair_pos), ptr(dw), ptr(st.seg), st.el,
         ptr(rt.top1_counts), n, e, k, ptr(aux_grad), ptr(dl), _stream())
    return dl


def input_grads(dxs, st: ExpertFwdState, pl: Plan, hidden, dl, wg, want_dx: bool, want_dwg: bool):
    """dX = gather of the token's per-row dX (slot order) + dL Wgᵀ and dWg = Xᵀ dL, one pass."""
    n, h = hidden.shape
    e = wg.shape[1]
    k = pl.pair_pos.shape[1]
    dt = dtype_code(hidden.dtype)
    dev = hidden.device
    dx = torch.empty_like(hidden) if want_dx else None
    dwg = torch.empty((h, e), dtype=torch.float32, device=dev) if want_dwg else None
    ws = _ws(_lib.query("ppmoe_input_grads_workspace_bytes", dt, n, h, e) if want_dwg else 0, dev)
    call("ppmoe_input_grads", dt, ptr(dxs), ptr(st.seg), st.el, ptr(pl.pair_pos), n, k, h, ptr(hidden), ptr(dl),
         ptr(wg), e, ptr(dx), ptr(dwg), ptr(ws), ws.numel(), _stream())
    return dx, dwg


def gate_weight_grad(hidden_rows: torch.Tensor, dl_rows: torch.Tensor, wg: torch.Tensor,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    """dWg = Xᵀ dL over the given token rows (fp32 [H x E]; deterministic partials)."""
    n, h = hidden_rows.shape
    e = wg.shape[1]
    dt = dtype_code(hidden_rows.dtype)
    dwg = out if out is not None else torch.empty((h, e), dtype=torch.float32, device=hidden_rows.device)
    if n == 0:
        return dwg.zero_()
    ws = _ws(_lib.query("ppmoe_input_grads_workspace_bytes", dt, n, h, e), hidden_rows.device)
    call("ppmoe_input_grads", dt, None, None, 1, None, n, 1, h, ptr(hidden_rows), ptr(dl_rows), ptr(wg), e, None,
         ptr(dwg), ptr(ws), ws.numel(), _stream())
    return dwg


def gate_grads(dx_acc, hidden, dl, wg, want_dx: bool, want_dwg: bool):
    """dX = dx_acc + dL Wg^T (activation dtype) and dWg = X^T dL (fp32)."""
    n, h = hidden.shape
    e = wg.shape[1]
    dev = hidden.device
    dx = torch.empty_like(hidden) if want_dx else None
    dwg = torch.empty((h, e), dtype=torch.float32, device=dev) if want_dwg else None
    ws = _ws(_lib.query("ppmoe_gate_grad_workspace_bytes", n, h, e) if want_dwg else 0, dev)
    call("ppmoe_gate_grads", ptr(dx_acc), ptr(hidden), dtype_code(hidden.dtype), ptr(dl), ptr(wg), n, h, e, ptr(dx),
         ptr(dwg), ptr(ws), ws.numel(), _stream())
    return dx, dwg


def cast_out(acc: torch.Tensor, dtype: torch.dtype, out: torch.Tensor | None = None) -> torch.Tensor:
    if out is None:
        out = torch.empty(acc.shape, dtype=dtype, device=acc.device)
    call("ppmoe_cast_out", ptr(acc), acc.numel(), ptr(out), dtype_code(dtype), _stream())
    return out
