"""Conventional all-to-all expert-parallel MoE layer (the reference's DPMoE, moe.py:363-469).

The comparator the PPMoE layer is measured against, built on the same kernels so only the
dispatch differs.  Every expert-parallel rank holds its own micro-batch and a contiguous
block of experts; per layer step:

  route + plan (local tokens, capacity by ascending GLOBAL token id: rank 0's tokens first)
  -> counts exchange (host-visible split sizes)
  -> dispatch all-to-all of the kept rows, expert-major then token order (moe.py:405-423)
  -> owner regroups rows per local expert in source order, runs the expert FFNs (moe.py:426-457)
  -> return all-to-all of the (pre-scale) expert outputs (moe.py:459)
  -> source scatters w * y back to token order (index_assign, moe.py:461-467).

The backward mirrors it (two more all-to-alls).  Gate-weight gradients are local to each
rank's micro-batch; `dpmoe_sync_gradients` sums them over the group (the spatial gradient
all-reduce of global_batch_equivalence, moe.py:496-518).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _ops
from .collectives import ProcessGroup, World


@dataclass
class _A2ASpec:
    world: World
    group: ProcessGroup
    me: int
    tp: int
    el: int
    k: int
    capacity_factor: float
    weight_scaling: bool
    override: torch.Tensor | None
    dropout_p: float = 0.0
    drop: object = None  # moe.DropoutStream


def _a2a(world: World, group: ProcessGroup, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits,
         async_op: bool = False):
    """Variable-size row all-to-all (the simulated world.all_to_all, collectives.py:155-182),
    ledger-charged with the off-diagonal bytes like the reference."""
    row = inp.shape[1] * world.ledger.elem_bytes if inp.dim() > 1 else world.ledger.elem_bytes
    me = world.rank_in(group) if world.distributed else 0
    moved = sum(n for i, n in enumerate(in_splits) if i != me) * row
    world.ledger.charge(group.kind, "all_to_all", moved)
    if not world.distributed or group.size == 1:
        if out.data_ptr() != inp.data_ptr():
            out.copy_(inp)
        return None
    return dist.all_to_all_single(out, inp, output_split_sizes=list(out_splits), input_split_sizes=list(in_splits),
                                  group=world.torch_group(group), async_op=async_op)


class _DPMoEFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, hidden, wg, up, down, bias_up, bias_down, spec: _A2ASpec):
        n, h = hidden.shape
        e = wg.shape[1]
        t, el, k = spec.tp, spec.el, spec.k
        dev = hidden.device
        rt = _ops.route(hidden, wg, k, spec.override)
        cap = _ops.INT32_MAX
        offset = None
        if not math.isinf(spec.capacity_factor):
            # C = ceil(cf * tokens_per_rank * dp / E) (moe.py:352), k-slot generalised
            cap = min(_ops.INT32_MAX, math.ceil(spec.capacity_factor * k * n * t / e))
            if t > 1:
                # pairs of higher priority on lower ranks: all slot-s pairs of ranks < me,
                # plus all lower-slot pairs everywhere (global ascending token id per slot)
                cnt = torch.stack([torch.bincount(rt.idx[:, s].long(), minlength=e) for s in range(k)]).to(torch.int32)
                allc = torch.empty((t, k, e), dtype=torch.int32, device=dev)
                dist.all_gather_into_tensor(allc, cnt.contiguous(), group=spec.world.torch_group(spec.group))
                tot = allc.sum(0)
                off = allc[: spec.me].sum(0) + torch.cumsum(tot, 0) - tot
                offset = off.to(torch.int32).contiguous()
        pl = _ops.plan(rt.idx, rt.w, e, cap, offset)
        if t == 1 and _ops.combine_mode(hidden.dtype, h) == "owner":
            return _DPMoEFunction._forward_solo(ctx, hidden, wg, up, down, bias_up, bias_down, spec, rt, pl)
        cstart, tok_c, w_c, pos_c = _ops.a2a_compact(pl, rt.idx, e)
        # counts exchange: kept rows per destination (owner, local expert)
        recv_counts = torch.empty(t * el, dtype=torch.int32, device=dev)
        _a2a(spec.world, spec.group, recv_counts, pl.kept, [el] * t, [el] * t)
        kept_h = pl.kept.cpu().tolist()  # host-visible split sizes: the conventional a2a sync point
        recv_h = recv_counts.cpu().tolist()
        send_rows = [sum(kept_h[o * el:(o + 1) * el]) for o in range(t)]
        recv_rows = [sum(recv_h[s * el:(s + 1) * el]) for s in range(t)]
        n_send, n_recv = sum(send_rows), sum(recv_rows)
        # dispatch: compact expert-major send buffer
        xsend = _ops._act((max(n_send, 1), h), hidden.dtype, dev)
        tmp_tok = torch.empty(max(n_send, 1), dtype=torch.int32, device=dev)
        tmp_w = torch.empty(max(n_send, 1), dtype=torch.float32, device=dev)
        _ops.call("ppmoe_gather", _ops.ptr(hidden), _ops.dtype_code(hidden.dtype), n, h, _ops.ptr(cstart), e,
                  _ops.ptr(tok_c), _ops.ptr(w_c), n_send, _ops.ptr(xsend), _ops.ptr(tmp_tok), _ops.ptr(tmp_w),
                  _ops._stream())
        # a group of one exchanges nothing: the receive buffers alias the send buffers
        solo = t == 1
        xrecv = xsend if solo else torch.empty((max(n_recv, 1), h), dtype=hidden.dtype, device=dev)
        _a2a(spec.world, spec.group, xrecv[:n_recv], xsend[:n_send], recv_rows, send_rows)
        # owner: regroup per local expert (source order), expert FFNs; fc2 stores the unscaled
        # bf16 outputs in the owner layout and a row permutation puts them in receive order
        rows_cap_o = n_recv + 128 * el
        seg_o, rmap = _ops.owner_layout(recv_counts, t, el, rows_cap_o)
        desc = None
        if spec.drop is not None:
            # the reference draws each expert's [rows received from all sources, h] block in
            # ascending expert id (moe.py:443-448): offsets from the global per-expert counts
            kept_all = pl.kept.clone()
            if t > 1:
                dist.all_reduce(kept_all, group=spec.world.torch_group(spec.group))
            desc = spec.drop.descriptor(kept_all, e, spec.me * el, el, h)
            spec.drop.advance(h * int(kept_all.sum()))
        st = _ops.expert_pipeline(xrecv, seg_o, el, rmap, None, rows_cap_o, up, down, bias_up, bias_down, False, None,
                                  spec.dropout_p, desc)
        yret = _ops._act((max(n_recv, 1), h), hidden.dtype, dev)
        _ops.permute_rows(st.y, rows_cap_o, rmap, yret)
        yback = yret if solo else torch.empty((max(n_send, 1), h), dtype=hidden.dtype, device=dev)
        _a2a(spec.world, spec.group, yback[:n_send], yret[:n_recv], send_rows, recv_rows)
        # source: out[t] = sum_s w * y (index_assign, moe.py:461-467) as a gather in slot order
        out = _ops.compact_combine(yback, cstart, rt.idx, pos_c, rt.w if spec.weight_scaling else None,
                                   torch.empty_like(hidden))
        ctx.save_for_backward(hidden, wg, up, down)
        ctx.state = (rt, pl, cstart, tok_c, w_c, pos_c, send_rows, recv_rows, st, rmap, yback, bias_up is not None,
                     spec)
        return out, rt.l_aux[0].to(torch.float32)

    @staticmethod
    def _forward_solo(ctx, hidden, wg, up, down, bias_up, bias_down, spec, rt, pl):
        """A group of one exchanges nothing: the conventional layer is then local dispatch
        (gather into expert-major padded segments), the expert FFNs and the local combine --
        the same kernels as the PPMoE layer at T = 1, so the comparator measures only what
        the all-to-all adds at T > 1.  The ledger still records the reference's five
        (empty) all-to-alls per step (moe.py:363-469)."""
        n, h = hidden.shape
        e = wg.shape[1]
        desc = None
        if spec.drop is not None:
            desc = spec.drop.descriptor(pl.kept, e, 0, e, h)
            spec.drop.advance(h * int(pl.kept.sum()))
        st = _ops.experts_forward(hidden, pl, 0, e, up, down, bias_up, bias_down, spec.k, spec.weight_scaling, None,
                                  drop_p=spec.dropout_p, drop=desc)
        out = _ops.local_combine(st.y, st, pl, rt.idx, rt.w if spec.weight_scaling else None, torch.empty_like(hidden))
        for _ in range(3):  # counts exchange, dispatch, return
            spec.world.ledger.charge(spec.group.kind, "all_to_all", 0.0)
        ctx.save_for_backward(hidden, wg, up, down)
        ctx.state = ("solo", rt, pl, st, bias_up is not None, spec)
        return out, rt.l_aux[0].to(torch.float32)

    @staticmethod
    def _backward_solo(ctx, g_out, g_aux):
        hidden, wg, up, down = ctx.saved_tensors
        _, rt, pl, st, has_bias, spec = ctx.state
        n, h = hidden.shape
        if g_out is None:
            g_out = torch.zeros_like(hidden)
        g_out = g_out.to(hidden.dtype).contiguous()
        aux = None if g_aux is None else g_aux.detach().to(torch.float32).reshape(1).contiguous()
        dxs = _ops._act((st.rows_cap, h), hidden.dtype, hidden.device)
        dy, dh, dw, parts = _ops.experts_backward_data(g_out, st, up, down, spec.weight_scaling, None, has_bias, dxs)
        dl = _ops.gate_backward(rt, pl, st, dw, aux)
        dx = _ops.local_combine(dxs, st, pl, rt.idx, None, torch.empty_like(hidden), dl, wg) \
            if ctx.needs_input_grad[0] else None
        dwg = _ops.gate_weight_grad(hidden, dl, wg) if ctx.needs_input_grad[1] else None
        del dxs
        d_up, d_down, d_bu, d_bd = _ops.experts_backward_weights(st, dy, dh, up, down, has_bias, parts)
        for _ in range(2):  # dY dispatch and dX return
            spec.world.ledger.charge(spec.group.kind, "all_to_all", 0.0)
        ctx.state = None
        return dx, dwg, d_up, d_down, d_bu, d_bd, None

    @staticmethod
    def backward(ctx, g_out, g_aux):
        if ctx.state[0] == "solo":
            return _DPMoEFunction._backward_solo(ctx, g_out, g_aux)
        hidden, wg, up, down = ctx.saved_tensors
        rt, pl, cstart, tok_c, w_c, pos_c, send_rows, recv_rows, st, rmap, yback, has_bias, spec = ctx.state
        n, h = hidden.shape
        e = wg.shape[1]
        dev = hidden.device
        n_send, n_recv = sum(send_rows), sum(recv_rows)
        if g_out is None:
            g_out = torch.zeros_like(hidden)
        g_out = g_out.to(hidden.dtype).contiguous()
        # source: dY = w * dOut[tok], dw = <dOut[tok], y> per compact row
        dy_c = _ops._act((max(n_send, 1), h), hidden.dtype, dev)
        dw_c = _ops._act(max(n_send, 1), torch.float32, dev)
        _ops.call("ppmoe_bwd_dy", _ops.dtype_code(hidden.dtype), _ops.ptr(g_out), _ops.ptr(yback), _ops.ptr(cstart), e,
                  h, max(n_send, 1), _ops.ptr(tok_c), _ops.ptr(w_c), int(spec.weight_scaling), 0.0, 0, _ops.ptr(dy_c),
                  _ops.ptr(dw_c), None, _ops._stream())
        solo = spec.tp == 1
        dy_recv = dy_c if solo else torch.empty((max(n_recv, 1), h), dtype=hidden.dtype, device=dev)
        _a2a(spec.world, spec.group, dy_recv[:n_recv], dy_c[:n_send], recv_rows, send_rows)
        # owner: data gradients (dY gathered to owner rows by the receive map), per-row dX in the
        # owner layout, permuted back to receive order (bf16, no fp32 scatter)
        dxs = _ops._act((st.rows_cap, h), hidden.dtype, dev)
        dy, dh, _, parts = _ops.experts_backward_data(dy_recv, st, up, down, False, None, has_bias, dxs)
        dx_recv = _ops._act((max(n_recv, 1), h), hidden.dtype, dev)
        _ops.permute_rows(dxs, st.rows_cap, rmap, dx_recv)
        del dxs
        dx_back = dx_recv if solo else torch.empty((max(n_send, 1), h), dtype=hidden.dtype, device=dev)
        work = _a2a(spec.world, spec.group, dx_back[:n_send], dx_recv[:n_recv], send_rows, recv_rows, async_op=True)
        with _ops.sm_budget(_ops.overlap_sm_budget() if work is not None else 0):
            d_up, d_down, d_bu, d_bd = _ops.experts_backward_weights(st, dy, dh, up, down, has_bias, parts)
        if work is not None:
            work.wait()
        # source: dX[t] = sum_s dX rows (slot order) + dL Wg^T in one gather; dWg = X^T dL
        aux = None if g_aux is None else g_aux.detach().to(torch.float32).reshape(1).contiguous()
        dl = torch.empty((n, e), dtype=torch.float32, device=dev)
        _ops.call("ppmoe_gate_bwd", _ops.ptr(rt.scores), _ops.ptr(rt.idx), _ops.ptr(pos_c), _ops.ptr(dw_c),
                  _ops.ptr(cstart), e, _ops.ptr(rt.top1_counts), n, e, spec.k, _ops.ptr(aux), _ops.ptr(dl),
                  _ops._stream())
        dx = None
        if ctx.needs_input_grad[0]:
            dx = _ops.compact_combine(dx_back, cstart, rt.idx, pos_c, None, torch.empty_like(hidden), dl, wg)
        dwg = _ops.gate_weight_grad(hidden, dl, wg) if ctx.needs_input_grad[1] else None
        ctx.state = None
        return dx, dwg, d_up, d_down, d_bu, d_bd, None


def dpmoe_forward(world: World, ep_group: ProcessGroup, hidden_per_rank, gate, *, experts_by_rank,
                  capacity_factor: float = math.inf, weight_scaling: bool = True, dropout_p: float = 0.0, rng=None,
                  route_overrides=None, top_k: int = 1):
    """All-to-all dispatch MoE layer (moe.py:363-469) on this rank's micro-batch.

    Distributed world: ``hidden_per_rank`` is this rank's [tokens, h] tensor (or a per-rank
    list whose own entry is used); returns (out, l_aux) of this rank.  A single-rank world
    runs the same path without communication.
    """
    from .moe import ExpertBank, _bank_of, DropoutStream, _override_tensor

    dp = ep_group.size
    if world.distributed:
        me = world.rank_in(ep_group)
    else:
        if dp != 1:
            raise NotImplementedError("the all-to-all comparator runs one process per rank (torch.distributed) "
                                      "or on a single-rank world")
        me = 0
    if isinstance(hidden_per_rank, (list, tuple)):
        if len(hidden_per_rank) != dp:
            raise ValueError(f"need hidden and experts for each of {dp} ranks")
        hidden = hidden_per_rank[me]
    else:
        hidden = hidden_per_rank
    if len(experts_by_rank) != dp:
        raise ValueError(f"need hidden and experts for each of {dp} ranks")
    drop = DropoutStream.of(dropout_p, rng)
    local: ExpertBank = _bank_of(experts_by_rank[me])
    num_experts = gate.num_experts
    if local.count * dp != num_experts:
        raise ValueError(f"{num_experts} experts must spread evenly over {dp} ranks")
    ov = None
    if route_overrides is not None:
        ov = _override_tensor(route_overrides[me] if isinstance(route_overrides, (list, tuple)) and
                              len(route_overrides) == dp else route_overrides,
                              hidden.shape[0], top_k, num_experts, hidden.device)
    spec = _A2ASpec(world, ep_group, me, dp, local.count, top_k, float(capacity_factor), bool(weight_scaling), ov,
                    float(dropout_p), drop)
    wg = gate.wg if gate.wg.dtype == torch.float32 else gate.wg.float()
    return _DPMoEFunction.apply(hidden.contiguous(), wg, local.up.contiguous(), local.down.contiguous(),
                                None if local.bias_up is None else local.bias_up.contiguous(),
                                None if local.bias_down is None else local.bias_down.contiguous(), spec)


def dpmoe_sync_gradients(world: World, group: ProcessGroup, gate) -> None:
    """Sum the replicated gate weight's gradient over the data-parallel ranks."""
    world.account_gradient_sync(group, gate.wg.numel())
    if world.distributed and group.size > 1 and gate.wg.grad is not None:
        dist.all_reduce(gate.wg.grad, op=dist.ReduceOp.SUM, group=world.torch_group(group))
