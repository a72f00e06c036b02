"""PPMoE block stack over pipeline stages (BASELINE.json configs[3]).

A stack of L residual blocks, each a tensor-parallel dense FFN followed by a PPMoE layer
(the GPT-style alternation of dense and MoE feed-forward layers; the reference has no
attention or LayerNorm, so the block is FFN-only), cut into P pipeline
stages of L/P blocks.  Rank (s, t) = global rank s*T + t holds tensor slot t of stage s;
each stage is one PPMoE tensor-parallel group (the NVLink exchange of nvlink.py), and
activations / their gradients travel between (s, t) and (s+1, t) with NCCL p2p.

The micro-batch order is the reference's 1F1B schedule (`schedule_1f1b`,
pipeline.py:64-82): per stage `p - s` warm-up forwards, then strict backward/forward
alternation, then the drain.  Sends that would cross in opposite directions are issued as
one batched p2p operation (send-forward + receive-backward, and the converse), so the
schedule cannot deadlock on NCCL's per-pair ordering.

The dense FFN is `dense_tp_ffn_forward` (moe.py:316-335): column-sharded up projection,
exact GeLU, row-sharded down projection, one all-reduce; its GEMMs are plain cuBLAS
(a library GEMM outside the MoE hot path).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.distributed as dist

from .collectives import EP, PP, ProcessGroup, World
from .moe import ExpertBank, GateParams, MoeLayerWeights, ppmoe_forward

F, B = "F", "B"


def schedule_1f1b(p: int, m: int) -> list[list[tuple[str, int]]]:
    """Per-stage op order of the reference's 1F1B schedule (pipeline.py:64-82):
    warm-up forwards, strict 1F1B alternation, drain.  Micro-batches are 1-based."""
    if p < 1 or m < 1:
        raise ValueError(f"need at least one stage and one micro-batch, got p={p}, m={m}")
    out = []
    for i in range(p):
        warm = min(p - i, m)
        ops = [(F, mb) for mb in range(1, warm + 1)]
        nb = 1
        for nf in range(warm + 1, m + 1):
            ops += [(B, nb), (F, nf)]
            nb += 1
        ops += [(B, mb) for mb in range(nb, m + 1)]
        out.append(ops)
    return out


class _CopyToTP(torch.autograd.Function):
    """Identity forward; all-reduce of the gradient over the tensor group (tp_region)."""

    @staticmethod
    def forward(ctx, x, pg):
        ctx.pg = pg
        return x.view_as(x)

    @staticmethod
    def backward(ctx, g):
        g = g.contiguous()
        if ctx.pg is not None:
            dist.all_reduce(g, group=ctx.pg)
        return g, None


class _ReduceFromTP(torch.autograd.Function):
    """All-reduce forward over the tensor group; identity backward."""

    @staticmethod
    def forward(ctx, x, pg):
        x = x.contiguous()
        if pg is not None:
            dist.all_reduce(x, group=pg)
        return x

    @staticmethod
    def backward(ctx, g):
        return g, None


@dataclass
class DenseShard:
    """This rank's column/row shard of a dense FFN (dense_tp_ffn_forward, moe.py:316-335)."""

    up: torch.Tensor      # [h, f/T]
    down: torch.Tensor    # [f/T, h]
    bias_down: torch.Tensor  # [h] (added once, after the reduction)

    def parameters(self):
        return [self.up, self.down, self.bias_down]


def dense_tp_ffn(x: torch.Tensor, shard: DenseShard, pg) -> torch.Tensor:
    x = _CopyToTP.apply(x, pg)
    y = torch.nn.functional.gelu(x @ shard.up) @ shard.down
    return _ReduceFromTP.apply(y, pg) + shard.bias_down


class PipelineStack:
    """L blocks (dense TP FFN + PPMoE, residual) over P stages x T tensor ranks.

    Every rank of a distributed world of P*T processes builds the stack with the same
    arguments; it keeps only its stage's blocks and its tensor slot's shards.  In a
    non-distributed world (P = T = 1) it runs every block on the local GPU.
    """

    def __init__(self, world: World, layers: int, stages: int, tp: int, hidden: int, experts: int, *, top_k: int = 2,
                 capacity_factor: float = math.inf, seed: int = 0, dtype=torch.bfloat16, device="cuda"):
        if layers % stages:
            raise ValueError(f"{layers} layers do not split over {stages} pipeline stages")
        if world.world_size != stages * tp:
            raise ValueError(f"world of {world.world_size} ranks is not {stages} stages x {tp} tensor ranks")
        if experts % tp or (4 * hidden) % tp:
            raise ValueError(f"experts ({experts}) and ffn ({4 * hidden}) must divide over tp={tp}")
        self.world, self.P, self.T, self.L = world, stages, tp, layers
        self.h, self.E, self.k, self.cf = hidden, experts, top_k, capacity_factor
        self.dtype, self.device = dtype, torch.device(device)
        rank = dist.get_rank() if world.distributed else 0
        self.stage, self.slot = divmod(rank, tp)
        # every rank creates every torch group in the same order (torch_group is collective)
        self.tp_groups = [ProcessGroup(EP, tuple(s * tp + t for t in range(tp))) for s in range(stages)]
        self.pp_groups = [ProcessGroup(PP, tuple(s * tp + t for s in range(stages))) for t in range(tp)]
        if world.distributed:
            world.register_groups(self.tp_groups + self.pp_groups)
        self.group = self.tp_groups[self.stage]
        self.pg = world.torch_group(self.group) if world.distributed and tp > 1 else None
        per = layers // stages
        self.first_layer = self.stage * per
        el = experts // tp
        fs = 4 * hidden // tp
        self.blocks = []
        for i in range(self.first_layer, self.first_layer + per):
            g = torch.Generator(device=self.device).manual_seed(seed * 1000 + i)
            up = (torch.randn(hidden, 4 * hidden, device=self.device, generator=g) * hidden ** -0.5)
            down = (torch.randn(4 * hidden, hidden, device=self.device, generator=g) * (4 * hidden) ** -0.5)
            dense = DenseShard(up[:, self.slot * fs:(self.slot + 1) * fs].to(dtype).contiguous().requires_grad_(),
                               down[self.slot * fs:(self.slot + 1) * fs].to(dtype).contiguous().requires_grad_(),
                               torch.zeros(hidden, device=self.device, dtype=dtype, requires_grad=True))
            del up, down
            full = MoeLayerWeights.random(hidden, experts, seed=seed * 1000 + i, dtype=dtype, device=self.device)
            part = full.bank.slice(self.slot * el, (self.slot + 1) * el)
            bank = ExpertBank(*(None if t is None else t.detach().clone().requires_grad_()
                                for t in (part.up, part.down, part.bias_up, part.bias_down)), first=self.slot * el)
            moe = MoeLayerWeights(GateParams(full.gate.wg.detach().clone().requires_grad_()), bank)
            del full, part
            self.blocks.append((dense, moe))

    def parameters(self):
        out = []
        for dense, moe in self.blocks:
            out += dense.parameters() + moe.leaf_parameters()
        return out

    def stage_forward(self, x: torch.Tensor):
        """This stage's blocks on one micro-batch; returns (y, summed aux loss)."""
        aux = torch.zeros((), device=self.device, dtype=torch.float32)
        for dense, moe in self.blocks:
            x = x + dense_tp_ffn(x, dense, self.pg)
            ebr = [moe.bank if r == self.slot else None for r in range(self.T)] if self.world.distributed \
                else [moe.bank]
            y, l_aux = ppmoe_forward(self.world, self.group if self.world.distributed else ProcessGroup(EP, (0,)),
                                     x, moe.gate, ebr, top_k=self.k, capacity_factor=self.cf)
            x = x + y
            aux = aux + l_aux
        return x, aux

    # ------------------------------------------------------------------ p2p

    def _peer(self, ds: int) -> int:
        return (self.stage + ds) * self.T + self.slot

    def _p2p(self, send=None, send_to=0, recv_from=0, shape=None):
        """Batched p2p: optionally send `send` to stage+send_to and receive a tensor of
        `shape` from stage+recv_from (one NCCL group, so crossing pairs cannot deadlock)."""
        ops, got = [], None
        if send is not None:
            ops.append(dist.P2POp(dist.isend, send.contiguous(), self._peer(send_to)))
        if shape is not None:
            got = torch.empty(shape, device=self.device, dtype=self.dtype)
            ops.append(dist.P2POp(dist.irecv, got, self._peer(recv_from)))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return got

    # ------------------------------------------------------------------ 1F1B

    def train_step(self, micro_batches: list[torch.Tensor] | int, mb_tokens: int | None = None) -> list[str]:
        """One global batch through the 1F1B schedule: forward + backward of every
        micro-batch (loss = sum of the last stage's outputs + the aux losses), parameter
        gradients accumulated over the micro-batches.  Stage 0 takes `micro_batches`
        (list of [n, h] tensors, or their count with `mb_tokens` for synthetic inputs).
        Returns this stage's executed op order (for the schedule check)."""
        m = micro_batches if isinstance(micro_batches, int) else len(micro_batches)
        n = mb_tokens if isinstance(micro_batches, int) else micro_batches[0].shape[0]
        shape = (n, self.h)
        p, s = self.P, self.stage
        first, last = s == 0, s == p - 1
        ops = schedule_1f1b(p, m)[s]
        saved: dict = {}
        done = []
        gen = torch.Generator(device=self.device).manual_seed(1234)
        for i, (kind, mb) in enumerate(ops):
            nxt = ops[i + 1] if i + 1 < len(ops) else None
            if kind == F:
                if first:
                    x = (micro_batches[mb - 1] if not isinstance(micro_batches, int)
                         else torch.randn(shape, device=self.device, generator=gen).to(self.dtype))
                    x = x.detach()
                else:
                    x = saved.pop(("X", mb), None)  # received together with the last backward send
                    if x is None:
                        x = self._p2p(shape=shape, recv_from=-1)
                x.requires_grad_(not first)
                y, aux = self.stage_forward(x)
                saved[mb] = (x, y, aux)
                if not last:
                    if nxt is not None and nxt[0] == B:  # steady state: send F, receive B together
                        g = self._p2p(send=y.detach(), send_to=+1, shape=shape, recv_from=+1)
                        saved[(B, nxt[1])] = g
                    else:
                        self._p2p(send=y.detach(), send_to=+1)
            else:
                x, y, aux = saved.pop(mb)
                if last:
                    torch.autograd.backward([y, aux], [torch.ones_like(y), torch.ones_like(aux)])
                else:
                    g = saved.pop((B, mb), None)
                    if g is None:
                        g = self._p2p(shape=shape, recv_from=+1)
                    torch.autograd.backward([y, aux], [g, torch.ones_like(aux)])
                if not first:
                    dx = x.grad
                    if nxt is not None and nxt[0] == F:  # steady state: send B, receive next F together
                        saved[("X", nxt[1])] = self._p2p(send=dx, send_to=-1, shape=shape, recv_from=-1)
                    else:
                        self._p2p(send=dx, send_to=-1)
            done.append((kind, mb))
        return done

    def sync_gate_gradients(self):
        from .moe import sync_gate_gradients
        for _, moe in self.blocks:
            sync_gate_gradients(self.world, self.group, moe.gate)
