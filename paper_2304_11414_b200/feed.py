"""Host -> device feed of the replicated PPMoE activations.

Every rank of a PPMoE tensor-parallel group holds the same [N, H] hidden states (the
input of copy_to_tensor_parallel_region, collectives.py:205-228).  Copying the whole
batch over PCIe on every rank moves T times the bytes the group needs, so
``ReplicatedFeed`` splits it: each rank copies its 1/T row slice of the pinned host
batch (host -> device on a side stream) and the slices are exchanged over NVLink.  With
a distributed bf16 group the exchange uses the group's peer-memory arena (nvlink.py):
each rank's slice lands in its peer-visible buffer, a barrier, then copy-engine pulls of
the other slices -- no SMs are taken from the layer running on the main stream.
Otherwise one NCCL all_gather.  Batches are double-buffered: ``submit`` of batch i+1
overlaps the layer's compute on batch i, and ``take`` orders the current stream after
the copies.  With T = 1 it is a prefetching pinned copy.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist

from . import _lib
from ._lib import ptr
from .collectives import ProcessGroup, World

# barrier channels of the arena reserved for the feed (the layer's exchange uses 0 and 1)
_CH_FREE, _CH_LANDED = 2, 3


class ReplicatedFeed:
    def __init__(self, world: World, group: ProcessGroup, shape, dtype, device, depth: int = 2):
        n = shape[0]
        self.world, self.group = world, group
        self.tp = group.size if world.distributed else 1
        if n % self.tp:
            raise ValueError(f"{n} rows do not split over a tensor group of {self.tp}")
        self.rank = world.rank_in(group) if world.distributed else 0
        self.rows = n // self.tp
        self.shape, self.dtype, self.depth = tuple(shape), dtype, depth
        self.stream = torch.cuda.Stream(device=device)
        self.pending: list = []
        self.next = 0
        self.arena = None
        from . import nvlink
        if (self.tp > 1 and os.environ.get("PPMOE_FEED", "nvl") == "nvl"
                and nvlink.enabled(world, group, dtype, shape[1])):
            self.arena = nvlink.arena(world, group)
            self.bufs = [self.arena.tensor(f"feed{i}", self.shape, dtype) for i in range(depth)]
        else:
            self.bufs = [torch.empty(self.shape, dtype=dtype, device=device) for _ in range(depth)]

    @property
    def h2d_bytes(self) -> int:
        """Host -> device bytes one batch costs this rank."""
        b = self.bufs[0]
        return self.rows * b[0].numel() * b.element_size()

    def submit(self, host: torch.Tensor) -> None:
        """Start moving `host` (pinned, the full [N, H] batch) to the device."""
        slot = self.next
        buf = self.bufs[slot]
        self.next = (self.next + 1) % len(self.bufs)
        lo = self.rank * self.rows
        mine = buf[lo:lo + self.rows]
        # the buffer was last read by work queued on the current stream
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            work = None
            if self.arena is not None:
                ar = self.arena
                ar.barrier(_CH_FREE)  # every rank is done pulling from this buffer's last batch
                mine.copy_(host[lo:lo + self.rows], non_blocking=True)
                ar.barrier(_CH_LANDED)  # every slice has landed in its owner's buffer
                n, h = self.shape
                _lib.call("ppmoe_nvl_pull_blocks_ce", ar.table(f"feed{slot}"), ar.tp, ar.rank, n, h, ptr(buf),
                          _lib.stream_ptr())
            else:
                mine.copy_(host[lo:lo + self.rows], non_blocking=True)
                if self.tp > 1:
                    work = dist.all_gather_into_tensor(buf, mine, group=self.world.torch_group(self.group),
                                                       async_op=True)
            done = torch.cuda.Event()
            done.record(self.stream)
        self.pending.append((buf, work, done))

    def take(self) -> torch.Tensor:
        """The oldest submitted batch, replicated on this rank; the current stream waits for it."""
        buf, work, done = self.pending.pop(0)
        torch.cuda.current_stream().wait_event(done)
        if work is not None:
            work.wait()
        return buf
