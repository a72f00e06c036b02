"""PPMoE MoE layer on B200: the reference's MoE-layer API (moesim/moe.py) over sm_100a kernels.

Drop-in surface (same names, argument meaning and error messages as
/root/reference/pkg/src/moesim/moe.py): ``GateParams``, ``GateOutput``,
``DispatchPlan``, ``ExpertFfn``, ``MoeLayerWeights``, ``LayerConfig``,
``gate_top1``, ``aux_loss``, ``build_dispatch_plan``, ``ppmoe_forward``,
``sync_gate_gradients``.  Extensions: ``top_k`` (>= 1; k = 1 is the reference),
``capacity_factor`` on the PPMoE path, bf16 compute, real NCCL tensor parallelism.

Tensors are torch CUDA tensors: hidden [N, h] in bf16 (or fp32 for the
reference-precision mode), gate weight fp32 [h, E], expert weights in the
hidden dtype.  Experts of a rank are stored stacked (``ExpertBank``) so one
grouped GEMM serves all of them; ``ExpertFfn`` objects are views into a bank.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _ops, nvlink
from .collectives import EP, ProcessGroup, World
from .rng import Rng

# ---------------------------------------------------------------------- parameters


def _draw_into(rng: Rng, dst: torch.Tensor, scale: float, chunk_elems: int = 1 << 24) -> None:
    """dst <- rng.normal(dst.shape, scale) rounded to dst.dtype, drawn in row chunks."""
    shape = tuple(dst.shape)
    if len(shape) == 1:
        dst.copy_(torch.from_numpy(rng.normal(shape, scale)))
        return
    cols = int(np.prod(shape[1:]))
    step = max(1, chunk_elems // max(cols, 1))
    for r0 in range(0, shape[0], step):
        r1 = min(shape[0], r0 + step)
        dst[r0:r1].copy_(torch.from_numpy(rng.normal((r1 - r0,) + shape[1:], scale)))


def _as_param(a, dtype, device, requires_grad=True) -> torch.Tensor:
    t = torch.as_tensor(np.asarray(a), dtype=torch.float64).to(device=device, dtype=dtype).contiguous()
    return t.requires_grad_(requires_grad)


@dataclass
class GateParams:
    """Routing linear map of shape hidden x experts, replicated on every rank (moe.py:30-53)."""

    wg: torch.Tensor

    def __post_init__(self):
        if self.wg.dim() != 2:
            raise ValueError(f"gate weight must be 2-D, got {tuple(self.wg.shape)}")
        if not bool(torch.isfinite(self.wg.detach()).all()):
            raise ValueError("gate weight has non-finite entries")

    @property
    def hidden(self) -> int:
        return self.wg.shape[0]

    @property
    def num_experts(self) -> int:
        return self.wg.shape[1]

    @classmethod
    def init(cls, hidden: int, num_experts: int, rng: Rng, scale: float | None = None,
             device="cuda") -> "GateParams":
        scale = scale if scale is not None else hidden ** -0.5
        return cls(_as_param(rng.normal((hidden, num_experts), scale), torch.float32, device))


@dataclass
class ExpertFfn:
    """One expert: Dropout(GeLU(x @ up + bias_up) @ down + bias_down) (moe.py:80-110)."""

    up: torch.Tensor
    down: torch.Tensor
    bias_up: torch.Tensor | None = None
    bias_down: torch.Tensor | None = None
    _bank: "ExpertBank | None" = field(default=None, repr=False, compare=False)
    _local: int = field(default=-1, repr=False, compare=False)

    @classmethod
    def init(cls, hidden: int, rng: Rng, ffn_mult: int = 4, bias: bool = True, scale: float | None = None,
             dtype=torch.bfloat16, device="cuda") -> "ExpertFfn":
        scale = scale if scale is not None else hidden ** -0.5
        inner = ffn_mult * hidden
        up = rng.normal((hidden, inner), scale)
        down = rng.normal((inner, hidden), scale)
        bu = rng.normal((inner,), scale) if bias else None
        bd = rng.normal((hidden,), scale) if bias else None
        return cls(_as_param(up, dtype, device), _as_param(down, dtype, device),
                   None if bu is None else _as_param(bu, dtype, device),
                   None if bd is None else _as_param(bd, dtype, device))

    def parameters(self) -> list:
        return [p for p in (self.up, self.down, self.bias_up, self.bias_down) if p is not None]

    def forward(self, x: torch.Tensor, dropout_p: float = 0.0, rng=None) -> torch.Tensor:
        """Dense FFN of every row through the expert kernels (single-expert route)."""
        bank = ExpertBank.stack([self])
        n = x.shape[0]
        gate = GateParams(torch.zeros((x.shape[1], 1), dtype=torch.float32, device=x.device))
        world = World(1, 1, distributed=False)  # a private one-rank world, also inside a multi-GPU job
        out, _ = ppmoe_forward(world, ProcessGroup(EP, (0,)), x, gate, [bank], weight_scaling=False,
                               dropout_p=dropout_p, rng=rng,
                               route_override=torch.zeros(n, dtype=torch.int64, device=x.device))
        return out


class ExpertBank:
    """Stacked weights of a contiguous block of experts [first, first + count).

    up [El, h, f], down [El, f, h], bias_up [El, f] | None, bias_down [El, h] | None.
    """

    def __init__(self, up, down, bias_up=None, bias_down=None, first: int = 0, _root=None, _offset: int = 0):
        if up.dim() != 3 or down.dim() != 3 or up.shape[0] != down.shape[0]:
            raise ValueError(f"expert bank needs stacked [El,h,f]/[El,f,h] weights, got {tuple(up.shape)}, {tuple(down.shape)}")
        if up.shape[1] != down.shape[2] or up.shape[2] != down.shape[1]:
            raise ValueError(f"expert shapes disagree: up {tuple(up.shape)} vs down {tuple(down.shape)}")
        if (bias_up is None) != (bias_down is None):
            raise ValueError("bias_up and bias_down must both be given or both be None")
        self.up, self.down, self.bias_up, self.bias_down = up, down, bias_up, bias_down
        self.first = first
        self._root = _root  # bank this one is a zero-copy slice of (None: it is a root)
        self._offset = _offset

    @property
    def count(self) -> int:
        return self.up.shape[0]

    @property
    def has_bias(self) -> bool:
        return self.bias_up is not None

    def __len__(self) -> int:
        return self.count

    @property
    def experts(self) -> list:
        return [ExpertFfn(self.up[i], self.down[i], None if self.bias_up is None else self.bias_up[i],
                          None if self.bias_down is None else self.bias_down[i], self, i) for i in range(self.count)]

    def slice(self, lo: int, hi: int) -> "ExpertBank":
        root = self._root or self
        off = self._offset + lo
        return ExpertBank(self.up[lo:hi], self.down[lo:hi], None if self.bias_up is None else self.bias_up[lo:hi],
                          None if self.bias_down is None else self.bias_down[lo:hi], self.first + lo, root, off)

    @staticmethod
    def stack(experts) -> "ExpertBank":
        """Bank for a list of experts: zero-copy when they are consecutive views of one
        bank, else a differentiable torch.stack."""
        experts = list(experts)
        if not experts:
            raise ValueError("need at least one expert")
        b0 = experts[0]._bank
        if b0 is not None and all(ex._bank is b0 for ex in experts):
            locs = [ex._local for ex in experts]
            if locs == list(range(locs[0], locs[0] + len(locs))):
                return b0.slice(locs[0], locs[-1] + 1)
        has_bias = experts[0].bias_up is not None
        return ExpertBank(torch.stack([ex.up for ex in experts]), torch.stack([ex.down for ex in experts]),
                          torch.stack([ex.bias_up for ex in experts]) if has_bias else None,
                          torch.stack([ex.bias_down for ex in experts]) if has_bias else None)

    @staticmethod
    def concat(banks) -> "ExpertBank":
        """One bank of all experts: a zero-copy slice when the banks are consecutive slices
        of one root (the output of MoeLayerWeights.shard), else a differentiable cat."""
        banks = list(banks)
        if len(banks) == 1:
            return banks[0]
        roots = {id(b._root or b) for b in banks}
        if len(roots) == 1 and all(b._root is not None for b in banks):
            if all(banks[i]._offset + banks[i].count == banks[i + 1]._offset for i in range(len(banks) - 1)):
                root = banks[0]._root
                return root.slice(banks[0]._offset, banks[-1]._offset + banks[-1].count)
        b0 = banks[0]
        return ExpertBank(torch.cat([b.up for b in banks]), torch.cat([b.down for b in banks]),
                          torch.cat([b.bias_up for b in banks]) if b0.has_bias else None,
                          torch.cat([b.bias_down for b in banks]) if b0.has_bias else None, b0.first)


@dataclass
class MoeLayerWeights:
    """Gate plus the ascending-id experts, stored as one bank (moe.py:113-147)."""

    gate: GateParams
    bank: ExpertBank

    @property
    def experts(self) -> list:
        return self.bank.experts

    @classmethod
    def init(cls, hidden: int, num_experts: int, rng: Rng, bias: bool = True, dtype=torch.bfloat16, device="cuda",
             ffn_mult: int = 4, experts: range | None = None, threads: int | None = None) -> "MoeLayerWeights":
        """Bit-identical draws to the reference init (gate stream 1, expert e stream 10+e,
        moe.py:120-124), rounded to ``dtype``.  ``experts`` restricts the bank to a
        block of expert ids (the local block of a tensor-parallel rank).

        Each expert's Philox stream is drawn in row chunks straight into the device bank
        (a stream drawn in pieces equals the one-shot draw), one host thread per expert
        (numpy releases the GIL), so BASELINE-size banks (C3: 17 GB of bf16) initialise in
        seconds without a 69 GB fp64 host copy."""
        from concurrent.futures import ThreadPoolExecutor

        gate = GateParams.init(hidden, num_experts, rng.spawn(1), device=device)
        ids = range(num_experts) if experts is None else experts
        scale = hidden ** -0.5
        inner = ffn_mult * hidden
        el = len(ids)
        up = torch.empty((el, hidden, inner), dtype=dtype, device=device)
        down = torch.empty((el, inner, hidden), dtype=dtype, device=device)
        bu = torch.empty((el, inner), dtype=dtype, device=device) if bias else None
        bd = torch.empty((el, hidden), dtype=dtype, device=device) if bias else None

        def fill(i):
            r = rng.spawn(10 + ids[i])
            _draw_into(r, up[i], scale)
            _draw_into(r, down[i], scale)
            if bias:
                _draw_into(r, bu[i], scale)
                _draw_into(r, bd[i], scale)

        workers = max(1, min(el, threads or (os.cpu_count() or 1)))
        if workers == 1:
            for i in range(el):
                fill(i)
        else:
            with ThreadPoolExecutor(workers) as ex:
                list(ex.map(fill, range(el)))
        if torch.device(device).type == "cuda":
            torch.cuda.synchronize(device)
        bank = ExpertBank(*(None if t is None else t.requires_grad_() for t in (up, down, bu, bd)), first=ids[0])
        return cls(gate, bank)

    @classmethod
    def random(cls, hidden: int, num_experts: int, seed: int = 0, bias: bool = True, dtype=torch.bfloat16,
               device="cuda", ffn_mult: int = 4, experts: range | None = None) -> "MoeLayerWeights":
        """Same distribution as ``init`` drawn with torch's device generator (fast; for
        benchmark-scale layers where host Philox draws would dominate set-up time)."""
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        scale = hidden ** -0.5
        inner = ffn_mult * hidden
        ids = range(num_experts) if experts is None else experts
        el = len(ids)

        def draw(*shape, dt):
            return (torch.randn(*shape, generator=g, device=device, dtype=torch.float32) * scale).to(dt).requires_grad_()

        wg = draw(hidden, num_experts, dt=torch.float32)
        bank = ExpertBank(draw(el, hidden, inner, dt=dtype), draw(el, inner, hidden, dt=dtype),
                          draw(el, inner, dt=dtype) if bias else None, draw(el, hidden, dt=dtype) if bias else None,
                          first=ids[0])
        return cls(GateParams(wg), bank)

    def named_parameters(self) -> dict:
        out = {"gate.wg": self.gate.wg}
        for i, ex in enumerate(self.experts):
            e = self.bank.first + i
            out[f"expert{e}.up"] = ex.up
            out[f"expert{e}.down"] = ex.down
            if ex.bias_up is not None:
                out[f"expert{e}.bias_up"] = ex.bias_up
                out[f"expert{e}.bias_down"] = ex.bias_down
        return out

    def leaf_parameters(self) -> list:
        b = self.bank
        return [p for p in (self.gate.wg, b.up, b.down, b.bias_up, b.bias_down) if p is not None]

    def named_grads(self) -> dict:
        """Gradients under the reference's parameter names (None where not computed)."""
        b = self.bank
        out = {"gate.wg": self.gate.wg.grad}
        for i in range(b.count):
            e = b.first + i
            out[f"expert{e}.up"] = None if b.up.grad is None else b.up.grad[i]
            out[f"expert{e}.down"] = None if b.down.grad is None else b.down.grad[i]
            if b.has_bias:
                out[f"expert{e}.bias_up"] = None if b.bias_up.grad is None else b.bias_up.grad[i]
                out[f"expert{e}.bias_down"] = None if b.bias_down.grad is None else b.bias_down.grad[i]
        return out

    def zero_grad(self) -> None:
        for p in self.leaf_parameters():
            p.grad = None

    def shard(self, ranks: int) -> list:
        """Contiguous expert blocks, ascending ids, one block per rank (moe.py:141-147)."""
        e = self.bank.count
        if e % ranks != 0:
            raise ValueError(f"{e} experts do not divide over {ranks} ranks")
        n = e // ranks
        return [self.bank.slice(r * n, (r + 1) * n) for r in range(ranks)]


@dataclass
class LayerConfig:
    """MoE layer settings as ingested from planner JSON (moe.py:150-190), plus ``top_k``."""

    hidden: int
    experts: int
    tp: int
    capacity_factor: float = math.inf
    weight_scaling: bool = True
    dropout_p: float = 0.0
    seed: int = 0
    top_k: int = 1

    _FIELDS = ("hidden", "experts", "tp", "capacity_factor", "weight_scaling", "dropout_p", "seed", "top_k")

    @classmethod
    def from_dict(cls, raw: dict) -> "LayerConfig":
        unknown = set(raw) - set(cls._FIELDS)
        if unknown:
            raise ValueError(f"unknown layer config fields: {sorted(unknown)}")
        if raw.get("capacity_factor") == "inf":
            raw = {**raw, "capacity_factor": math.inf}
        cfg = cls(**raw)
        if cfg.hidden < 1 or cfg.experts < 1 or cfg.tp < 1:
            raise ValueError("hidden, experts and tp must be positive")
        if cfg.experts % cfg.tp != 0:
            raise ValueError(f"experts must divide over tp ranks: {cfg.experts} % {cfg.tp} != 0")
        if not (cfg.capacity_factor > 0):
            raise ValueError("capacity_factor must be positive (may be inf)")
        if not 1 <= cfg.top_k <= cfg.experts:
            raise ValueError(f"top_k must be in [1, experts], got {cfg.top_k}")
        return cfg

    def to_dict(self) -> dict:
        cf = self.capacity_factor
        return {"hidden": self.hidden, "experts": self.experts, "tp": self.tp,
                "capacity_factor": cf if math.isfinite(cf) else "inf", "weight_scaling": self.weight_scaling,
                "dropout_p": self.dropout_p, "seed": self.seed, "top_k": self.top_k}


# ---------------------------------------------------------------------- gating


@dataclass
class GateOutput:
    """Routing decision for one batch of token rows (moe.py:56-63).

    indices / weights are [N] for top-1 (the reference shape) and [N, k] otherwise.
    """

    indices: torch.Tensor
    weights: torch.Tensor
    l_aux: torch.Tensor
    scores: torch.Tensor


@dataclass
class DispatchPlan:
    """Ascending token row ids per expert (moe.py:66-77), plus the device-side plan."""

    per_expert: list
    kept_mask: torch.Tensor | None = None
    device_plan: object = None

    @property
    def num_experts(self) -> int:
        return len(self.per_expert)

    def tokens(self) -> int:
        return sum(len(rows) for rows in self.per_expert)


def _override_tensor(route_override, n: int, k: int, num_experts: int, device) -> torch.Tensor | None:
    if route_override is None:
        return None
    ov = torch.as_tensor(route_override, device=device)
    if ov.dim() == 1 and k == 1:
        ov = ov[:, None]
    if tuple(ov.shape) != (n, k):
        if k == 1:
            raise ValueError(f"route override needs one expert id per token, got {tuple(ov.shape)}")
        raise ValueError(f"route override needs {k} expert ids per token, got {tuple(ov.shape)}")
    if ov.numel() and (int(ov.min()) < 0 or int(ov.max()) >= num_experts):
        raise ValueError("route override contains expert ids out of range")
    if k > 1 and ov.numel():
        srt = ov.sort(dim=1).values
        if bool((srt[:, 1:] == srt[:, :-1]).any()):
            # the router never picks an expert twice for a token, and the per-rank row bounds
            # (_ops.local_rows_cap) rely on it
            raise ValueError("route override repeats an expert id within a token's top-k")
    return ov.to(torch.int32).contiguous()


def gate_topk(hidden: torch.Tensor, gate: GateParams, k: int = 1, route_override=None) -> GateOutput:
    """Softmax scores, top-k routing (lowest expert id wins ties), balance loss (moe.py:196-208)."""
    n = hidden.shape[0]
    if n == 0:
        raise ValueError("aux_loss of zero tokens is undefined")
    ov = _override_tensor(route_override, n, k, gate.num_experts, hidden.device)
    rt = _ops.route(hidden.contiguous(), gate.wg.detach().contiguous(), k, ov)
    idx, w = rt.idx.long(), rt.w
    if k == 1:
        idx, w = idx[:, 0], w[:, 0]
    return GateOutput(idx, w, rt.l_aux[0].float(), rt.scores)


def gate_top1(hidden: torch.Tensor, gate: GateParams, route_override=None) -> GateOutput:
    return gate_topk(hidden, gate, 1, route_override)


def aux_loss(indices: torch.Tensor, scores: torch.Tensor, num_experts: int) -> torch.Tensor:
    """Balance regularizer E * sum_e frac_e * mean_t s[t,e] (moe.py:211-223); frac from slot 0."""
    n = indices.shape[0]
    if n == 0:
        raise ValueError("aux_loss of zero tokens is undefined")
    ids = indices if indices.dim() == 1 else indices[:, 0]
    frac = torch.bincount(ids.long(), minlength=num_experts).to(scores.dtype) / n
    return (scores @ frac).sum() * (num_experts / n)


def build_dispatch_plan(indices, num_experts: int, capacity: int | None = None) -> DispatchPlan:
    """Ascending token positions per expert from per-token expert ids (moe.py:226-235),
    computed by the device counting sort; ``capacity`` applies the keep-first rule."""
    idx = torch.as_tensor(indices)
    if idx.dim() == 1:
        idx = idx[:, None]
    if idx.numel() and (int(idx.min()) < 0 or int(idx.max()) >= num_experts):
        bad = idx[(idx < 0) | (idx >= num_experts)][0]
        raise ValueError(f"expert id {int(bad)} out of range for {num_experts} experts")
    dev = idx.device if idx.is_cuda else torch.device("cuda")
    idx_d = idx.to(device=dev, dtype=torch.int32).contiguous()
    cap = _ops.INT32_MAX if capacity is None else int(capacity)
    pl = _ops.plan(idx_d, None, num_experts, cap)
    seg = pl.seg.cpu().tolist()
    kept = pl.kept.cpu().tolist()
    tok = pl.tok_sorted.cpu()
    per = [tok[seg[e]:seg[e] + kept[e]].tolist() for e in range(num_experts)]
    return DispatchPlan(per, (pl.pair_pos >= 0), pl)


# ---------------------------------------------------------------------- ppmoe


@dataclass
class _Spec:
    world: World
    group: ProcessGroup
    k: int
    capacity_factor: float
    weight_scaling: bool
    override: torch.Tensor | None
    e0: int
    el: int
    aux_here: bool
    fwd_chunks: int = 1
    dropout_p: float = 0.0
    drop: "DropoutStream | None" = None
    sliced_router: bool = False
    route: object = None  # the forward's routing (for check_replicas)


class _PPMoEFunction(torch.autograd.Function):
    """Forward: route -> plan -> gather -> fc1 -> fc2+combine -> TP all-reduce.
    Backward: closed form of tensor.backward through that graph (tensor.py:368-374) ->
    TP all-reduce of dX (tp_region, collectives.py:205-228)."""

    @staticmethod
    def forward(ctx, hidden, wg, up, down, bias_up, bias_down, spec: _Spec):
        nvlink.check_all()  # a barrier of an earlier exchange timed out: fail loudly
        n, h = hidden.shape
        e = wg.shape[1]
        if spec.sliced_router:
            rt = _ops.route_sliced(spec.world, spec.group, hidden, wg, spec.k, spec.override)
        else:
            rt = _ops.route(hidden, wg, spec.k, spec.override)
        spec.route = (rt, None)
        cap = _ops.capacity_for(spec.capacity_factor, n, spec.k, e)
        pl = _ops.plan(rt.idx, rt.w, e, cap)
        spec.route = (rt, pl)
        desc = None
        if spec.drop is not None:  # the reference's per-expert dropout draws (moe.py:301, tensor.py:315-330)
            desc = spec.drop.descriptor(pl.kept, e, spec.e0, spec.el, h)
            spec.drop.advance(h * int(pl.kept.sum()))
        if spec.fwd_chunks > 1:
            out_acc = torch.zeros((n, h), dtype=torch.float32, device=hidden.device)
            # combine all-reduce pipelined by token chunk: chunk c goes on the wire while the
            # expert GEMMs of chunk c+1 run (reduce_from_tensor_parallel_region, moe.py:307)
            out = torch.empty((n, h), dtype=hidden.dtype, device=hidden.device)
            works = []
            bounds = [c * n // spec.fwd_chunks for c in range(spec.fwd_chunks + 1)]

            def on_chunk(c):
                lo, hi = bounds[c], bounds[c + 1]
                if hi > lo:
                    _ops.cast_out(out_acc[lo:hi], hidden.dtype, out[lo:hi])
                    works.append(spec.world.all_reduce_async(spec.group, out[lo:hi], charge=False))

            st = _ops.experts_forward(hidden, pl, spec.e0, spec.el, up, down, bias_up, bias_down, spec.k,
                                      spec.weight_scaling, out_acc, spec.fwd_chunks, on_chunk, spec.dropout_p,
                                      desc)
            spec.world.charge_all_reduce(spec.group, out.numel())
            for wk in works:
                if wk is not None:
                    wk.wait()
            del out_acc
        elif nvlink.enabled(spec.world, spec.group, hidden.dtype, h):
            # fc2 also mirrors Y into peer-visible memory; every rank sums its owned tokens'
            # expert rows straight from the peers and the owners' blocks are all-gathered
            # (replaces reduce_from_tensor_parallel_region's all-reduce, moe.py:307)
            ar = nvlink.arena(spec.world, spec.group)
            mode = nvlink.fused_forward_mode(ar, n, spec.k)
            if mode == "slots":
                # the fc2 epilogue stores w*Y into the owning rank's slot rows over NVLink
                # (plain P2P stores, tile by tile during the GEMM); owners sum, then all-gather
                table, rows = nvlink.owner_slots(ar, n, spec.k, h)
                st = _ops.experts_forward(hidden, pl, spec.e0, spec.el, up, down, bias_up, bias_down, spec.k,
                                          spec.weight_scaling, None, drop_p=spec.dropout_p, drop=desc,
                                          owner_slots=table, owner_rows=rows)
                out = nvlink.finish_slots_forward(ar, n, spec.k, h, pl.pair_pos, torch.empty_like(hidden))
            elif mode == "fused":
                # the fc2 epilogue adds w*Y straight into the owning rank's fp32 accumulator
                # over NVLink, tile by tile during the GEMM; owners cast, then all-gather
                table, rows = nvlink.owner_accumulator(ar, n, h)
                st = _ops.experts_forward(hidden, pl, spec.e0, spec.el, up, down, bias_up, bias_down, spec.k,
                                          spec.weight_scaling, None, drop_p=spec.dropout_p, drop=desc,
                                          owner_table=table, owner_rows=rows)
                out = nvlink.finish_fused_forward(ar, n, h, torch.empty_like(hidden))
            elif nvlink.forward_chunks(ar, n) > 1:
                # pipelined: the exchange of token chunk c (its owners' blocks) runs on the side
                # stream while the expert GEMMs of chunk c+1 compute (SM budget leaves room)
                chunks = nvlink.forward_chunks(ar, n)
                ym = ar.tensor("y", (_ops.local_rows_cap(n, spec.k, spec.el, cap), h), hidden.dtype)
                out = torch.empty_like(hidden)
                ar.tensor("xch", (n, h), torch.bfloat16)  # allocated before the side stream uses it
                main, side = torch.cuda.current_stream(), ar.stream
                wts = rt.w if spec.weight_scaling else None

                def on_chunk(c):
                    side.wait_stream(main)
                    with torch.cuda.stream(side):
                        nvlink.exchange_chunk(ar, c, chunks, "y", pl.seg, spec.el, rt.idx, pl.pair_pos, wts, n, h,
                                              out)

                st = _ops.experts_forward(hidden, pl, spec.e0, spec.el, up, down, bias_up, bias_down, spec.k,
                                          spec.weight_scaling, None, chunks, on_chunk, spec.dropout_p, desc,
                                          y_mirror=ym)
                main.wait_stream(side)
            else:
                ym = ar.tensor("y", (_ops.local_rows_cap(n, spec.k, spec.el, cap), h), hidden.dtype)
                st = _ops.experts_forward(hidden, pl, spec.e0, spec.el, up, down, bias_up, bias_down, spec.k,
                                          spec.weight_scaling, None, drop_p=spec.dropout_p, drop=desc,
                                          y_mirror=ym)
                out = nvlink.exchange(ar, "y", pl.seg, spec.el, rt.idx, pl.pair_pos,
                                      rt.w if spec.weight_scaling else None, n, h, torch.empty_like(hidden))
            spec.world.charge_all_reduce(spec.group, out.numel())
        elif spec.el == e and _ops.combine_mode(hidden.dtype, h) == "owner":
            # all experts local: fc2 stores Y, the owner-gather kernel sums every token's rows
            st = _ops.experts_forward(hidden, pl, spec.e0, spec.el, up, down, bias_up, bias_down, spec.k,
                                      spec.weight_scaling, None, drop_p=spec.dropout_p, drop=desc)
            out = _ops.local_combine(st.y, st, pl, rt.idx, rt.w if spec.weight_scaling else None,
                                     torch.empty_like(hidden))
            spec.world.all_reduce_(spec.group, out)  # a group of one: ledger only (moe.py:307)
        elif _ops.combine_mode(hidden.dtype, h) != "scatter":
            # fc2 stores Y; the combine gathers each token's local pairs (no fp32 accumulator)
            st = _ops.experts_forward(hidden, pl, spec.e0, spec.el, up, down, bias_up, bias_down, spec.k,
                                      spec.weight_scaling, None, drop_p=spec.dropout_p, drop=desc)
            out = _ops.combine(st.y, st, pl, rt.w if spec.weight_scaling else None, torch.empty_like(hidden))
            spec.world.all_reduce_(spec.group, out)  # reduce_from_tensor_parallel_region (moe.py:307)
        else:
            out_acc = torch.zeros((n, h), dtype=torch.float32, device=hidden.device)
            st = _ops.experts_forward(hidden, pl, spec.e0, spec.el, up, down, bias_up, bias_down, spec.k,
                                      spec.weight_scaling, out_acc, drop_p=spec.dropout_p, drop=desc)
            out = _ops.cast_out(out_acc, hidden.dtype)
            del out_acc
            spec.world.all_reduce_(spec.group, out)  # reduce_from_tensor_parallel_region (moe.py:307)
        ctx.save_for_backward(hidden, wg, up, down)
        ctx.state = (rt, pl, st, bias_up is not None, spec)
        l_aux = rt.l_aux[0].to(torch.float32)
        return out, l_aux

    @staticmethod
    def backward(ctx, g_out, g_aux):
        nvlink.check_all()
        hidden, wg, up, down = ctx.saved_tensors
        rt, pl, st, has_bias, spec = ctx.state
        n, h = hidden.shape
        if g_out is None:
            g_out = torch.zeros_like(hidden)
        g_out = g_out.to(hidden.dtype).contiguous()
        aux = None
        if spec.aux_here and g_aux is not None:
            aux = g_aux.detach().to(torch.float32).reshape(1).contiguous()
        # data gradients first: dX can go on the wire while the weight gradients compute.
        need_dx = ctx.needs_input_grad[0]
        need_dwg = ctx.needs_input_grad[1]
        if nvlink.enabled(spec.world, spec.group, hidden.dtype, h) and need_dx:
            # per-row dX and dL into peer-visible memory; owners gather them (+ the gate term)
            # and the blocks are all-gathered (replaces tp_region's dX all-reduce)
            ar = nvlink.arena(spec.world, spec.group)
            dxs = ar.tensor("dxs", (st.rows_cap, h), hidden.dtype)
            dy, dh, dw, parts = _ops.experts_backward_data(g_out, st, up, down, spec.weight_scaling, None, has_bias,
                                                           dxs)
            e = wg.shape[1]
            _ops.gate_backward(rt, pl, st, dw, aux, out=ar.tensor("dl", (n, e), torch.float32))
            t0, t1 = nvlink.owned_range(ar, n)
            dx = torch.empty_like(hidden)
            dwg = torch.empty((h, e), dtype=torch.float32, device=hidden.device) if need_dwg else None
            main = torch.cuda.current_stream()
            side = ar.stream if os.environ.get("PPMOE_NVL_OVERLAP", "1") == "1" else main
            side.wait_stream(main)
            # no record_stream: every tensor the side stream touches outlives the
            # main.wait_stream(side) below (inputs are saved tensors, outputs are returned)
            with torch.cuda.stream(side):
                # the exchange runs beside the weight-gradient GEMMs (their SM budget leaves room)
                ar.barrier(0)  # every rank's dX rows and dL partials are published
                dl_own = nvlink.sum_owned_rows(ar, "dl", n, e)
                if need_dwg:  # dWg over the owned tokens; sync_gate_gradients sums the ranks' shares
                    _ops.gate_weight_grad(hidden[t0:t1], dl_own, wg, out=dwg)
                nvlink.exchange(ar, "dxs", pl.seg, spec.el, rt.idx, pl.pair_pos, None, n, h, dx, dl_own, wg,
                                barrier_first=False)
            spec.world.charge_all_reduce(spec.group, dx.numel())
            with _ops.sm_budget(_ops.overlap_sm_budget()):
                d_up, d_down, d_bu, d_bd = _ops.experts_backward_weights(st, dy, dh, up, down, has_bias, parts)
            main.wait_stream(side)
            ctx.state = None
            return dx, dwg, d_up, d_down, d_bu, d_bd, None
        if spec.el == wg.shape[1] and _ops.combine_mode(hidden.dtype, h) == "owner":
            # all experts local: per-row dX gathered per token with the gate term (owner gather)
            dxs = _ops._act((st.rows_cap, h), hidden.dtype, hidden.device)
            dy, dh, dw, parts = _ops.experts_backward_data(g_out, st, up, down, spec.weight_scaling, None, has_bias,
                                                           dxs)
            dl = _ops.gate_backward(rt, pl, st, dw, aux)
            dx = None
            if need_dx:
                dx = _ops.local_combine(dxs, st, pl, rt.idx, None, torch.empty_like(hidden), dl, wg)
                spec.world.all_reduce_(spec.group, dx)  # a group of one: ledger only
            dwg = _ops.gate_weight_grad(hidden, dl, wg) if need_dwg else None
            del dxs
            d_up, d_down, d_bu, d_bd = _ops.experts_backward_weights(st, dy, dh, up, down, has_bias, parts)
            ctx.state = None
            return dx, dwg, d_up, d_down, d_bu, d_bd, None
        # fc1 dgrad stores per-row dX; gate_grads gathers them per token (no fp32 scatter)
        if _ops.combine_mode(hidden.dtype, h) != "scatter":
            dx_acc, dxs = None, _ops._act((st.rows_cap, h), hidden.dtype, hidden.device)
        else:
            dx_acc, dxs = torch.zeros((n, h), dtype=torch.float32, device=hidden.device), None
        dy, dh, dw, parts = _ops.experts_backward_data(g_out, st, up, down, spec.weight_scaling, dx_acc, has_bias, dxs)
        dl = _ops.gate_backward(rt, pl, st, dw, aux)
        if dxs is not None:
            dx, dwg = _ops.input_grads(dxs, st, pl, hidden, dl, wg, need_dx, need_dwg)
        else:
            dx, dwg = _ops.gate_grads(dx_acc, hidden, dl, wg, need_dx, need_dwg)
        del dx_acc, dxs
        work = None
        if need_dx:  # copy_to_tensor_parallel_region backward (collectives.py:215-221)
            work = spec.world.all_reduce_async(spec.group, dx)
        with _ops.sm_budget(_ops.overlap_sm_budget() if work is not None else 0):
            d_up, d_down, d_bu, d_bd = _ops.experts_backward_weights(st, dy, dh, up, down, has_bias, parts)
        if work is not None:
            work.wait()  # stream-ordered: the compute stream waits for the NCCL stream
        ctx.state = None
        return dx, dwg, d_up, d_down, d_bu, d_bd, None


class DropoutStream:
    """The reference's expert dropout draws (tensor.dropout, tensor.py:315-330, called in
    ExpertFfn.forward for every expert with rows, ascending id, moe.py:294-301): expert e
    consumes one uniform [rows_e, h] block of the caller's Rng (numpy Philox4x64-10), and an
    element survives iff its uniform >= p.  The device regenerates exactly those draws
    (csrc/common.cuh) from the stream's key and position, so masks equal the reference's
    and the caller's Rng ends where the reference leaves it.  Every rank of a TP group holds
    the same Rng state and routing, so its experts' draws are the simulated reference's."""

    def __init__(self, p: float, rng):
        from .rng import stream_position

        gen = getattr(rng, "_gen", None)
        if not isinstance(gen, np.random.Generator):
            raise ValueError("dropout with p > 0 needs a Philox-backed Rng (moesim's Rng)")
        self.p, self.gen = float(p), gen
        self.key0, self.key1, self.first = stream_position(gen)
        self.threshold = int(math.ceil(self.p * 2.0 ** 53))  # (word >> 11) >= ceil(p 2^53) <=> uniform >= p

    @classmethod
    def of(cls, dropout_p: float, rng) -> "DropoutStream | None":
        """Validate like tensor.dropout (tensor.py:315-322); None when p == 0."""
        if not 0.0 <= dropout_p < 1.0:
            raise ValueError(f"dropout probability must be in [0, 1), got {dropout_p}")
        if dropout_p == 0.0:
            return None
        if rng is None:
            raise ValueError("dropout with p > 0 requires an rng")
        return cls(dropout_p, rng)

    def descriptor(self, kept: torch.Tensor, num_experts: int, e0: int, el: int, h: int) -> torch.Tensor:
        return _ops.dropout_descriptor(kept, num_experts, e0, el, h, self.key0, self.key1, self.threshold, self.first)

    def advance(self, draws: int) -> None:
        """The caller's Rng moves past the layer's draws (host-visible kept counts: one sync)."""
        from .rng import set_stream_position

        set_stream_position(self.gen, self.first + draws)


def _as_single(value, what: str):
    """Collapse a replica list to its logical value, checking exact agreement (moe.py:238-248)."""
    if isinstance(value, (list, tuple)):
        first = value[0]
        ref = first.wg if isinstance(first, GateParams) else first
        for r, other in enumerate(value[1:], start=1):
            data = other.wg if isinstance(other, GateParams) else other
            if data.shape != ref.shape or not torch.equal(ref.detach(), data.detach()):
                raise ValueError(f"TP replica divergence: {what} differs on rank {r}")
        return first
    return value


def _bank_of(entry) -> ExpertBank:
    if isinstance(entry, ExpertBank):
        return entry
    return ExpertBank.stack(entry)


def ppmoe_forward(world: World, group: ProcessGroup, hidden, gate, experts_by_rank, *, weight_scaling: bool = True,
                  dropout_p: float = 0.0, rng=None, route_override=None, top_k: int = 1,
                  capacity_factor: float = math.inf, check_replicas: bool = False):
    """Index-slice dispatch with all-reduce combine over a tensor-parallel group (moe.py:254-308).

    ``experts_by_rank`` has one entry per group member (an ``ExpertBank`` or a list of
    ``ExpertFfn``).  In a simulated world all entries are used on this GPU; in a
    distributed world only this process's entry is needed (others may be None).
    Returns (out [N, h] replicated on every rank, l_aux scalar).
    """
    hidden = _as_single(hidden, "hidden activation")
    gate = _as_single(gate, "gate weight")
    tp = group.size
    if len(experts_by_rank) != tp:
        raise ValueError(f"need one expert list per rank: {len(experts_by_rank)} for group of {tp}")
    drop = DropoutStream.of(dropout_p, rng)
    num_experts = gate.num_experts
    if not 1 <= top_k <= num_experts:
        raise ValueError(f"top_k must be in [1, {num_experts}], got {top_k}")
    if hidden.dim() != 2 or hidden.shape[1] != gate.hidden:
        raise ValueError(f"hidden must be [tokens, {gate.hidden}], got {tuple(hidden.shape)}")
    if hidden.shape[0] == 0:
        raise ValueError("aux_loss of zero tokens is undefined")
    if world.distributed:
        me = world.rank_in(group)
        local = _bank_of(experts_by_rank[me])
        num_local = local.count
        if num_local * tp != num_experts:
            raise ValueError(f"{num_experts} experts must spread evenly over {tp} ranks")
        e0, el, aux_here = me * num_local, num_local, me == 0
    else:
        banks = [_bank_of(x) for x in experts_by_rank]
        num_local = banks[0].count
        if any(b.count != num_local for b in banks) or num_local * tp != num_experts:
            raise ValueError(f"{num_experts} experts must spread evenly over {tp} ranks")
        local = ExpertBank.concat(banks)
        e0, el, aux_here = 0, num_experts, True
    n = hidden.shape[0]
    ov = _override_tensor(route_override, n, top_k, num_experts, hidden.device)
    wdt = hidden.dtype
    for p in (local.up, local.down, local.bias_up, local.bias_down):
        if p is not None and p.dtype != wdt:
            raise ValueError(f"expert weights must match the hidden dtype {wdt}, got {p.dtype}")
    env_chunks = os.environ.get("PPMOE_FWD_CHUNKS")
    if env_chunks is not None:
        chunks = max(1, int(env_chunks))
    else:
        chunks = 1  # token-chunked combine measured slower than one all-reduce
    sliced = (world.distributed and tp > 1 and hidden.shape[0] % tp == 0
              and os.environ.get("PPMOE_SLICED_ROUTER", "1") != "0")
    spec = _Spec(world, group, top_k, float(capacity_factor), bool(weight_scaling), ov, e0, el, aux_here, chunks,
                 float(dropout_p), drop, sliced)
    wg = gate.wg if gate.wg.dtype == torch.float32 else gate.wg.float()
    out, l_aux = _PPMoEFunction.apply(hidden.contiguous(), wg, local.up.contiguous(), local.down.contiguous(),
                                      None if local.bias_up is None else local.bias_up.contiguous(),
                                      None if local.bias_down is None else local.bias_down.contiguous(), spec)
    if check_replicas and world.distributed and tp > 1:
        _check_dispatch_agreement(world, group, hidden, *spec.route)
    return out, l_aux


def _check_dispatch_agreement(world: World, group: ProcessGroup, hidden: torch.Tensor, route=None,
                              plan=None) -> None:
    """Debug-mode replacement of the reference's replica checks (moe.py:289-291): every rank
    of the group must hold the same hidden activation AND the same dispatch (routing indices,
    per-expert kept counts): an int64 position-weighted hash of the indices plus the counts
    are compared across ranks with MIN/MAX all-reduces."""
    import torch.distributed as dist

    pg = world.torch_group(group)
    sig = torch.stack([hidden.float().sum(), (hidden.float() * torch.arange(1, hidden.shape[1] + 1,
                                                                             device=hidden.device)).sum()])
    lo, hi = sig.clone(), sig.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=pg)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=pg)
    if not torch.equal(lo, hi):
        raise ValueError("TP replica divergence: hidden activation differs across ranks")
    if route is None:
        return
    idx = route.idx.long().reshape(-1)
    pos = torch.arange(1, idx.numel() + 1, device=idx.device, dtype=torch.int64)
    parts = [(idx * pos).sum().reshape(1), (idx * idx * (pos % 1009)).sum().reshape(1)]
    if plan is not None:
        parts.append(plan.kept.long())
    dig = torch.cat(parts)
    lo, hi = dig.clone(), dig.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=pg)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=pg)
    if not torch.equal(lo, hi):
        raise ValueError("TP replica divergence: dispatch order differs across ranks")


def sync_gate_gradients(world: World, group: ProcessGroup, gate: GateParams) -> None:
    """Once-per-global-batch all-reduce of the gate weight gradient (moe.py:311-313)."""
    world.account_gradient_sync(group, gate.wg.numel())
    if world.distributed and group.size > 1 and gate.wg.grad is not None:
        import torch.distributed as dist

        nvlink.check_all()
        g = gate.wg.grad
        if (g.is_cuda and g.dtype == torch.float32 and g.is_contiguous()
                and nvlink.enabled(world, group, torch.bfloat16, 8)):
            nvlink.all_reduce_grad(nvlink.arena(world, group), g)  # peer memory, one barrier
        else:
            dist.all_reduce(g, op=dist.ReduceOp.SUM, group=world.torch_group(group))


class PPMoELayer(torch.nn.Module):
    """nn.Module wrapper: one PPMoE layer of a tensor-parallel group, built from a LayerConfig."""

    def __init__(self, cfg: LayerConfig, world: World | None = None, group: ProcessGroup | None = None,
                 dtype=torch.bfloat16, device="cuda", weights: MoeLayerWeights | None = None, fast_init: bool = False):
        super().__init__()
        self.cfg = cfg
        self.world = world or World(1, cfg.tp)
        self.group = group or ProcessGroup(EP, tuple(range(cfg.tp)))
        el = cfg.experts // cfg.tp
        block = None
        if self.world.distributed:
            me = self.world.rank_in(self.group)
            block = range(me * el, (me + 1) * el)
        if weights is None:
            if fast_init:
                weights = MoeLayerWeights.random(cfg.hidden, cfg.experts, cfg.seed, dtype=dtype, device=device,
                                                 experts=block)
            else:
                weights = MoeLayerWeights.init(cfg.hidden, cfg.experts, Rng(cfg.seed), dtype=dtype, device=device,
                                               experts=block)
        self.weights = weights
        self.rng = Rng(cfg.seed, 5)  # the dropout stream the reference's CLI uses (cli.py:137)
        for name, p in zip(("wg", "up", "down", "bias_up", "bias_down"),
                           (weights.gate.wg, weights.bank.up, weights.bank.down, weights.bank.bias_up,
                            weights.bank.bias_down)):
            if p is not None:
                self.register_parameter(name, torch.nn.Parameter(p.detach(), requires_grad=True))
        # keep the weight containers pointing at the registered parameters
        weights.gate.wg = self.wg
        weights.bank.up, weights.bank.down = self.up, self.down
        if weights.bank.has_bias:
            weights.bank.bias_up, weights.bank.bias_down = self.bias_up, self.bias_down

    def experts_by_rank(self):
        if self.world.distributed:
            me = self.world.rank_in(self.group)
            return [self.weights.bank if r == me else None for r in range(self.group.size)]
        return self.weights.shard(self.cfg.tp)

    def forward(self, hidden: torch.Tensor, route_override=None):
        return ppmoe_forward(self.world, self.group, hidden, self.weights.gate, self.experts_by_rank(),
                             weight_scaling=self.cfg.weight_scaling, dropout_p=self.cfg.dropout_p,
                             rng=self.rng if self.cfg.dropout_p > 0 else None,
                             route_override=route_override, top_k=self.cfg.top_k,
                             capacity_factor=self.cfg.capacity_factor)

    def sync_gate_gradients(self):
        sync_gate_gradients(self.world, self.group, self.weights.gate)


def global_batch_equivalence(weights: MoeLayerWeights, global_batch, dp: int, *, tp: int = 1, include_aux: bool = True,
                             weight_scaling: bool = True, top_k: int = 1):
    """Gradients of one global batch spanned spatially vs temporally (moe.py:475-533).

    Spatial: the micro-batches as `dp` expert-parallel ranks of the all-to-all layer with the
    gradient sum of the data-parallel all-reduce (single process: one rank after another on
    this GPU; the ranks share no state when capacity is unlimited).  Temporal: the same
    micro-batches one after another through the PPMoE layer on a `tp` group, gradients
    accumulated, then the gate-gradient sync.  Loss per micro-batch: sum(out) (+ l_aux).
    Returns (spatial, temporal) dicts of fp64 numpy arrays under the reference's names.
    """
    from .dpmoe import dpmoe_forward

    if len(global_batch) != dp:
        raise ValueError(f"global batch of {len(global_batch)} micro-batches does not span dp={dp}")
    dev = weights.gate.wg.device
    dtype = weights.bank.up.dtype

    def snapshot():
        return {k: v.detach().double().cpu().numpy().copy() for k, v in weights.named_grads().items() if v is not None}

    def as_input(x):
        return torch.as_tensor(np.asarray(x), dtype=torch.float64).to(device=dev, dtype=dtype).contiguous()

    def loss_of(out, l_aux):
        term = out.float().sum()
        return term + l_aux if include_aux else term

    weights.zero_grad()
    world_s = World(1, 1, distributed=False)  # single-process helper worlds, also under torchrun
    for x in global_batch:
        out, l_aux = dpmoe_forward(world_s, ProcessGroup(EP, (0,)), as_input(x), weights.gate,
                                   experts_by_rank=weights.shard(1), capacity_factor=math.inf,
                                   weight_scaling=weight_scaling, top_k=top_k)
        loss_of(out, l_aux).backward()
    spatial = snapshot()

    weights.zero_grad()
    world_t = World(1, tp, distributed=False)
    group = ProcessGroup(EP, tuple(range(tp)))
    shards = weights.shard(tp)
    for x in global_batch:
        out, l_aux = ppmoe_forward(world_t, group, as_input(x), weights.gate, shards, weight_scaling=weight_scaling,
                                   top_k=top_k)
        loss_of(out, l_aux).backward()
    sync_gate_gradients(world_t, group, weights.gate)
    temporal = snapshot()
    return spatial, temporal
