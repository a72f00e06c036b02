"""Process groups, traffic ledger and the tensor-parallel collectives of the PPMoE path.

Mirrors moesim.collectives (collectives.py:20-228) on real hardware:

* ``World`` runs in one of two modes.  *Simulated* (no torch.distributed
  process group): every rank of a group lives in this process and is executed
  on the local GPU — the reference's own execution model (collectives.py:1-8).
  *Distributed*: one process per GPU, collectives over NCCL (NVLink 5 /
  NVSwitch) through torch.distributed; ``ProcessGroup`` members are global ranks.
* ``TrafficLedger`` charges the same ring-model bytes as the reference
  (2(N-1)*m per all-reduce, collectives.py:112-121) so its byte-parity
  properties (test_moe.py:372-407) carry over.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

DP, TP, PP, EP = "DP", "TP", "PP", "EP"
P2P = "P2P"


class ConfigurationError(ValueError):
    """A parallel layout violates a divisibility or placement constraint."""


@dataclass(frozen=True)
class ProcessGroup:
    """Ordered set of ranks participating in one flavor of parallelism (collectives.py:28-43)."""

    kind: str
    members: tuple[int, ...]

    def __post_init__(self):
        if len(set(self.members)) != len(self.members):
            raise ConfigurationError(f"{self.kind} group has repeated ranks: {self.members}")
        if list(self.members) != sorted(self.members):
            raise ConfigurationError(f"{self.kind} group members must be sorted: {self.members}")

    @property
    def size(self) -> int:
        return len(self.members)


@dataclass
class TrafficLedger:
    """Cumulative bytes and op counts per (group kind, op kind) (collectives.py:46-77)."""

    elem_bytes: float = 2.0
    entries: dict = field(default_factory=dict)

    def charge(self, group_kind: str, op_kind: str, bytes_moved: float, inter_node_bytes: float = 0.0) -> None:
        if bytes_moved < 0 or inter_node_bytes < 0:
            raise ValueError("ledger bytes must be non-negative")
        cell = self.entries.setdefault((group_kind, op_kind), {"bytes": 0.0, "count": 0, "inter_node_bytes": 0.0})
        cell["bytes"] += bytes_moved
        cell["count"] += 1
        cell["inter_node_bytes"] += inter_node_bytes

    def bytes_for(self, group_kind: str, op_kind: str) -> float:
        return self.entries.get((group_kind, op_kind), {}).get("bytes", 0.0)

    def count_for(self, group_kind: str, op_kind: str) -> int:
        return int(self.entries.get((group_kind, op_kind), {}).get("count", 0))

    def inter_node_bytes_for(self, group_kind: str, op_kind: str) -> float:
        return self.entries.get((group_kind, op_kind), {}).get("inter_node_bytes", 0.0)

    def as_dict(self) -> dict:
        out: dict = {}
        for (gk, ok), cell in sorted(self.entries.items()):
            out.setdefault(gk, {})[ok] = dict(cell)
        return out

    def to_json(self, indent: int | None = 2) -> str:
        return json.dumps(self.as_dict(), indent=indent, sort_keys=True)


class World:
    """Rank universe of nodes x devices-per-node plus the traffic ledger (collectives.py:80-228).

    ``distributed`` is decided at construction: True when torch.distributed is
    initialised (one process per GPU), else every rank is simulated locally.
    """

    def __init__(self, nodes: int, devices_per_node: int, elem_bytes: float = 2.0, distributed: bool | None = None):
        if nodes < 1 or devices_per_node < 1:
            raise ConfigurationError(f"need at least one node and one device, got {nodes}x{devices_per_node}")
        self.nodes = nodes
        self.devices_per_node = devices_per_node
        self.world_size = nodes * devices_per_node
        self.ledger = TrafficLedger(elem_bytes)
        if distributed is None:
            distributed = dist.is_available() and dist.is_initialized()
        self.distributed = bool(distributed)
        if self.distributed and dist.get_world_size() != self.world_size:
            raise ConfigurationError(
                f"world of {self.world_size} ranks does not match torch.distributed world size {dist.get_world_size()}"
            )
        self._torch_groups: dict = {}

    def node_of(self, rank: int) -> int:
        self._check_rank(rank)
        return rank // self.devices_per_node

    def _check_rank(self, rank: int) -> None:
        if not 0 <= rank < self.world_size:
            raise ValueError(f"rank {rank} outside world of size {self.world_size}")

    # ------------------------------------------------------------- ledger math

    def _ring_crossings(self, members) -> int:
        n = len(members)
        if n < 2:
            return 0
        return sum(1 for i in range(n) if self.node_of(members[i]) != self.node_of(members[(i + 1) % n]))

    def _ring_bytes(self, group: ProcessGroup, numel: int) -> tuple[float, float]:
        n = group.size
        m = numel * self.ledger.elem_bytes
        total = 2 * (n - 1) * m
        per_edge = total / n if n > 1 else 0.0
        return total, per_edge * self._ring_crossings(group.members)

    def charge_all_reduce(self, group: ProcessGroup, numel: int, op_kind: str = "all_reduce") -> None:
        total, inter = self._ring_bytes(group, numel)
        self.ledger.charge(group.kind, op_kind, total, inter)

    def account_gradient_sync(self, group: ProcessGroup, numel: int) -> None:
        """Ledger record of the deferred parameter-gradient all-reduce (collectives.py:123-131)."""
        self.charge_all_reduce(group, numel, "gradient_sync")

    # ------------------------------------------------------------- real collectives

    def rank_in(self, group: ProcessGroup) -> int:
        """Index of this process inside ``group`` (distributed mode)."""
        if not self.distributed:
            raise RuntimeError("rank_in() is only defined for a distributed world")
        r = dist.get_rank()
        if r not in group.members:
            raise ValueError(f"rank {r} is not a member of {group.kind} group {group.members}")
        return group.members.index(r)

    def register_groups(self, groups) -> None:
        """Create the torch.distributed groups of ``groups`` collectively: every rank of the
        job must call this with the same groups in the same order (dist.new_group is a
        collective over the whole job), including ranks that are not members."""
        if not self.distributed:
            return
        for group in groups:
            if group.members == tuple(range(self.world_size)) or group.members in self._torch_groups:
                continue
            self._torch_groups[group.members] = dist.new_group(list(group.members))

    def torch_group(self, group: ProcessGroup):
        """The torch.distributed (NCCL) group for ``group``: WORLD for the whole job, else a
        group created by ``register_groups`` / ``tp_groups`` (creating one lazily here would
        call dist.new_group on the member ranks only, which hangs or mismatches groups when
        the job has several tensor groups)."""
        if not self.distributed:
            return None
        if group.members == tuple(range(self.world_size)):
            return dist.group.WORLD
        g = self._torch_groups.get(group.members)
        if g is None:
            raise ConfigurationError(
                f"{group.kind} group {group.members} has no torch.distributed group: create the job's groups "
                f"collectively first (tp_groups(world, ...) or World.register_groups)"
            )
        return g

    def all_reduce_(self, group: ProcessGroup, t: torch.Tensor, charge: bool = True, op_kind: str = "all_reduce"):
        """In-place sum over the group (NCCL); in simulated mode partials were already summed."""
        if charge:
            self.charge_all_reduce(group, t.numel(), op_kind)
        if self.distributed and group.size > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.torch_group(group))
        return t

    def all_reduce_async(self, group: ProcessGroup, t: torch.Tensor, op_kind: str = "all_reduce",
                         charge: bool = True):
        """Start an in-place NCCL sum on the process group's stream (after the work already
        queued on the current stream); returns a handle whose ``wait()`` makes the current
        stream wait for it, or None when there is nothing to communicate."""
        if charge:
            self.charge_all_reduce(group, t.numel(), op_kind)
        if self.distributed and group.size > 1:
            return dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.torch_group(group), async_op=True)
        return None

    def all_reduce_sum(self, group: ProcessGroup, per_rank: list) -> list:
        """Simulated-mode reference semantics: ascending-rank sum, every member receives it
        (collectives.py:135-153)."""
        if len(per_rank) != group.size:
            raise ValueError(f"all_reduce_sum needs one tensor per member, got {len(per_rank)} for {group.size}")
        shape = per_rank[0].shape
        for rank, t in zip(group.members, per_rank):
            if t.shape != shape:
                raise ValueError(
                    f"all_reduce_sum shape mismatch: rank {group.members[0]} has {tuple(shape)}, rank {rank} has {tuple(t.shape)}"
                )
        acc = per_rank[0]
        for t in per_rank[1:]:
            acc = acc + t
        self.charge_all_reduce(group, acc.numel())
        return [acc for _ in group.members]


@dataclass(frozen=True)
class GroupSet:
    dp: tuple
    tp: tuple
    pp: tuple
    ep: tuple

    def group_of(self, kind: str, rank: int) -> ProcessGroup:
        for g in getattr(self, kind.lower()):
            if rank in g.members:
                return g
        raise ValueError(f"rank {rank} not in any {kind} group")


def tp_groups(world: World, tp: int, num_experts: int) -> GroupSet:
    """PPMoE layout on one node: contiguous tensor groups, expert groups alias them
    (build_groups ppmoe branch, collectives.py:247-299, without pipeline stages)."""
    if world.devices_per_node % tp != 0:
        raise ConfigurationError(
            f"ppmoe tensor groups must sit inside one node: {world.devices_per_node} devices/node not divisible by tp={tp}"
        )
    if num_experts % tp != 0:
        raise ConfigurationError(f"ppmoe needs experts divisible by tp: {num_experts} % {tp} != 0")
    dp = world.world_size // tp
    tpg = tuple(ProcessGroup(TP, tuple(d * tp + t for t in range(tp))) for d in range(dp))
    dpg = tuple(ProcessGroup(DP, tuple(d * tp + t for d in range(dp))) for t in range(tp))
    epg = tuple(ProcessGroup(EP, g.members) for g in tpg)
    world.register_groups(tpg + dpg)  # eagerly, in one fixed order on every rank
    return GroupSet(dp=dpg, tp=tpg, pp=(), ep=epg)
