"""Peer-memory arena of a tensor-parallel group: the NVLink exchange of the PPMoE layer.

``NvlArena`` owns, per (World, ProcessGroup), a set of device buffers that every rank
of the group can address directly (CUDA IPC handles exchanged once through
torch.distributed), a signal pad per rank for the cross-GPU barriers, and the epoch
counters of those barriers.  The kernels that use it live in csrc/nvlink.cu
(ppmoe_nvl_barrier / ppmoe_nvl_owner_gather / ppmoe_nvl_pull_blocks[_ce] /
ppmoe_nvl_sum_rows); moe.py calls ``exchange`` (forward: the experts' Y rows; backward:
their per-row dX plus the gate term) in place of the two [N x H] all-reduces of the
reference (moe.py:307, collectives.py:205-228).  Barrier channels 0/1 belong to the
layer's exchange, 2/3 to the host feed (feed.py).  ``enabled`` probes the group once and
falls back to NCCL everywhere if any rank cannot map its peers.

Buffers are allocated collectively: every rank requests the same names and sizes in the
same order (the sizes are functions of the layer shape only), so the arenas stay in
lock-step.  A buffer grows by re-allocation when a larger shape arrives.
"""

from __future__ import annotations

import ctypes
import os

import torch
import torch.distributed as dist

from . import _lib
from ._lib import ptr
from ._ops import call  # event-timed under _ops.KernelProfile

_ARENAS: dict = {}
# ~2 minutes at 2 GHz: long enough for host-side skew between ranks (logging, checkpoints,
# eval, first-step allocation), short enough that a dead peer ends in an error, not a hang.
# A timed-out barrier sets the arena's host-mapped error flag; every layer call checks it
# (check_all) and raises, and PPMOE_NVL_STRICT=1 synchronises and checks after each exchange.
_TIMEOUT_CYCLES = int(os.environ.get("PPMOE_NVL_TIMEOUT_CYCLES", str(240_000_000_000)))
_STRICT = os.environ.get("PPMOE_NVL_STRICT", "0") == "1"


def ptr_set(ptrs):
    """ctypes host array of device pointers (the C-ABI pointer-set arguments)."""
    return (ctypes.c_void_p * len(ptrs))(*ptrs)


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (wrapped by torch.as_tensor)."""

    def __init__(self, p: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (p, False),
                                         "version": 3, "strides": None, "stream": None}


def _wrap(p: int, shape, dtype: torch.dtype, device) -> torch.Tensor:
    if dtype == torch.bfloat16:
        t = torch.as_tensor(_CudaArray(p, shape, "<i2"), device=device)
        return t.view(torch.bfloat16)
    typestr = {torch.float32: "<f4", torch.int32: "<i4", torch.uint8: "|u1"}[dtype]
    return torch.as_tensor(_CudaArray(p, shape, typestr), device=device)


class _PeerBuffer:
    def __init__(self, arena: "NvlArena", nbytes: int):
        lib = _lib.load()
        hsize = lib.ppmoe_ipc_handle_bytes()
        local = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(hsize)
        _lib.call("ppmoe_ipc_alloc", nbytes, ctypes.byref(local), handle)
        handles = [None] * arena.tp
        dist.all_gather_object(handles, handle.raw, group=arena.torch_group)
        self.local = local.value
        self.nbytes = nbytes
        self.opened = []
        ptrs = []
        for q, hb in enumerate(handles):
            if q == arena.rank:
                ptrs.append(self.local)
                continue
            peer = ctypes.c_void_p()
            _lib.call("ppmoe_ipc_open", ctypes.create_string_buffer(hb, hsize), ctypes.byref(peer))
            self.opened.append(peer.value)
            ptrs.append(peer.value)
        self.ptrs = ptrs
        self.table = ptr_set(ptrs)  # host array of the T ranks' pointers (kernel parameters)

    def release(self):
        for p in self.opened:
            _lib.call("ppmoe_ipc_close", ctypes.c_void_p(p))
        _lib.call("ppmoe_ipc_free", ctypes.c_void_p(self.local))
        self.opened = []


class NvlArena:
    """Peer buffers, signal pads and barrier epochs of one tensor-parallel group."""

    def __init__(self, world, group):
        if not world.distributed:
            raise RuntimeError("the NVLink arena needs a distributed world (one process per GPU)")
        self.world, self.group = world, group
        self.tp = group.size
        self.rank = world.rank_in(group)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.torch_group = world.torch_group(group)
        lib = _lib.load()
        self.pads = _PeerBuffer(self, lib.ppmoe_nvl_pad_bytes())
        # barrier error flag in pinned host memory, mapped into the device address space
        # (UVA): the barrier kernel stores 1 on a timeout and the host reads it without a sync
        self.err = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self._err_view = self.err.numpy()  # host view of the same pinned word (cheap reads)
        self._views: dict = {}  # (name, shape, dtype) -> tensor view of a peer buffer
        self.epoch = [0] * 16  # kNvlChannels
        self.bufs: dict = {}
        self.mc_bufs: dict = {}
        self.mc_disabled = False
        self.stream = torch.cuda.Stream(device=self.device)  # exchange beside the weight-gradient GEMMs

    # ------------------------------------------------------------------ buffers

    def buffer(self, name: str, nbytes: int) -> _PeerBuffer:
        b = self.bufs.get(name)
        if b is None or b.nbytes < nbytes:
            if b is not None:
                torch.cuda.synchronize()
                dist.barrier(group=self.torch_group)  # no peer still reads the old buffer
                b.release()
                self._views = {k: v for k, v in self._views.items() if k[0] != name}
            b = _PeerBuffer(self, nbytes)
            self.bufs[name] = b
        return b

    def tensor(self, name: str, shape, dtype: torch.dtype) -> torch.Tensor:
        key = (name, tuple(shape), dtype)
        t = self._views.get(key)
        if t is not None:
            return t
        n = 1
        for s in shape:
            n *= s
        nbytes = max(n * torch.empty((), dtype=dtype).element_size(), 16)
        t = _wrap(self.buffer(name, nbytes).local, shape, dtype, self.device)
        self._views[key] = t
        return t

    def table(self, name: str):
        return self.bufs[name].table

    def device_table(self, name: str) -> torch.Tensor:
        """Device array of the T ranks' pointers to `name` (built once per allocation)."""
        b = self.bufs[name]
        if getattr(b, "dtab", None) is None:
            b.dtab = torch.tensor(b.ptrs, dtype=torch.int64, device=self.device)
        return b.dtab

    def multicast(self, name: str, shape):
        """(local bf16 tensor, NVLS multicast address) of a symmetric buffer of the group
        (torch symmetric memory), or None when the box has no multicast; grown collectively."""
        if self.mc_disabled:
            return None
        n = shape[0] * shape[1]
        cur = self.mc_bufs.get(name)
        if cur is None or cur[0].numel() < n:
            ok, entry = 1, None
            try:
                import torch.distributed._symmetric_memory as symm_mem
                t = symm_mem.empty(n, dtype=torch.bfloat16, device=self.device)
                hdl = symm_mem.rendezvous(t, self.torch_group)
                mc = int(getattr(hdl, "multicast_ptr", 0) or 0)
                ok = 1 if mc else 0
                entry = (t, mc, hdl)
            except Exception:
                ok = 0
            flag = torch.tensor([ok], dtype=torch.int32, device=self.device)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.torch_group)
            if int(flag.item()) == 0:
                self.mc_disabled = True
                return None
            self.mc_bufs[name] = entry
            cur = entry
        t, mc, _ = cur
        return t[:n].view(shape), mc

    def local_table(self, name: str):
        """A T-entry pointer set that names this rank's own copy of `name` T times."""
        b = self.bufs[name]
        if getattr(b, "local_tab", None) is None:
            b.local_tab = ptr_set([b.local] * self.tp)
        return b.local_tab

    # ------------------------------------------------------------------ sync

    def barrier(self, ch: int) -> None:
        self.epoch[ch] = (self.epoch[ch] + 1) & 0xFFFFFFFF
        call("ppmoe_nvl_barrier", self.pads.table, self.tp, self.rank, ch, self.epoch[ch], ptr(self.err),
             _TIMEOUT_CYCLES, _lib.stream_ptr())

    def check_nonblocking(self) -> None:
        """Raise if a barrier of this arena that already ran timed out (no device sync)."""
        if self._err_view[0] != 0:
            raise RuntimeError(f"NVLink barrier timed out on rank {self.rank} of tensor group {self.group.members}: "
                               "a peer stopped responding; the exchanges since then read unfinished peer rows")

    def check(self) -> None:
        """Raise if any barrier of this arena timed out (synchronises the device first)."""
        torch.cuda.synchronize(self.device)
        self.check_nonblocking()


def check_all(sync: bool = False) -> None:
    """Raise if a barrier of any arena of this process timed out (ppmoe_forward and its
    backward call this on entry; sync=True waits for the queued work first)."""
    for a in _ARENAS.values():
        a.check() if sync else a.check_nonblocking()


_UNAVAILABLE: set = set()


def arena(world, group) -> NvlArena:
    key = (id(world), group.members)
    a = _ARENAS.get(key)
    if a is None:
        a = NvlArena(world, group)
        _ARENAS[key] = a
    return a


def _probe(world, group) -> bool:
    """Create the group's arena once; every rank learns whether all of them could map
    their peers (a MIN all-reduce), so the group takes the same path everywhere."""
    key = (id(world), group.members)
    if key in _ARENAS:
        return True
    if key in _UNAVAILABLE:
        return False
    ok = 1
    try:
        arena(world, group)
    except Exception as exc:  # no P2P / IPC on this box: fall back to NCCL, loudly
        if os.environ.get("PPMOE_NVL_REQUIRE") == "1":  # tests: the exchange must come up
            raise
        import warnings
        warnings.warn(f"NVLink exchange unavailable, using NCCL all-reduces: {exc}")
        ok = 0
    flag = torch.tensor([ok], dtype=torch.int32, device=torch.device("cuda", torch.cuda.current_device()))
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=world.torch_group(group))
    if int(flag.item()) == 0:
        _UNAVAILABLE.add(key)
        _ARENAS.pop(key, None)
        return False
    return True


def enabled(world, group, dtype: torch.dtype, hidden: int) -> bool:
    """NVLink exchange for distributed bf16 groups of 2..8 ranks (PPMOE_TP_COMM=nccl opts out)."""
    if os.environ.get("PPMOE_TP_COMM", "nvl") != "nvl":
        return False
    if not (world.distributed and 1 < group.size <= 8 and dtype == torch.bfloat16 and hidden % 8 == 0):
        return False
    return _probe(world, group)


def owned_range(ar: NvlArena, n: int) -> tuple[int, int]:
    """Tokens [t0, t1) this rank owns in the exchange (contiguous blocks in rank order)."""
    return ar.rank * n // ar.tp, (ar.rank + 1) * n // ar.tp


def sum_owned_rows(ar: NvlArena, name: str, n: int, c: int) -> torch.Tensor:
    """Sum over the group (rank order) of this rank's owned rows of the fp32 [n x c] peer
    buffer `name`; call after a barrier that published it."""
    t0, t1 = owned_range(ar, n)
    out = torch.empty((t1 - t0, c), dtype=torch.float32, device=ar.device)
    call("ppmoe_nvl_sum_rows", ar.table(name), ar.tp, ar.rank, n, c, ptr(out), _lib.stream_ptr())
    return out


_CH_GSYNC = 8  # barrier channel of the gate-gradient sync (0-7: exchange, feed, chunks)
CH_ROUTE = 9  # barrier channel of the sliced routing (_ops.route_sliced)


def all_reduce_grad(ar: NvlArena, grad: torch.Tensor) -> None:
    """In-place sum over the group (rank order, identical on every rank) of an fp32 tensor
    through the arena: publish into a peer-visible buffer, one barrier, every rank sums the
    T copies.  Two buffers alternate, so a rank that runs ahead cannot overwrite a buffer a
    peer still reads (it would have to pass the next sync's barrier first)."""
    ar.gsync = getattr(ar, "gsync", 0) ^ 1
    name = f"gsync{ar.gsync}"
    buf = ar.tensor(name, (grad.numel(),), torch.float32)
    buf.copy_(grad.reshape(-1))
    ar.barrier(_CH_GSYNC)
    call("ppmoe_nvl_sum_all", ar.table(name), ar.tp, grad.numel(), ptr(grad), _lib.stream_ptr())


def fused_forward_mode(ar: NvlArena, n: int, k: int) -> str:
    """Forward combine over NVLink: "gather" (owner gather after fc2, default), "slots"
    (fc2 epilogue stores w*Y into the owner's bf16 slot rows with P2P stores) or "fused"
    (fc2 epilogue red.adds into the owner's fp32 accumulator).  PPMOE_NVL_FWD selects."""
    mode = os.environ.get("PPMOE_NVL_FWD", "gather")
    if mode in ("fused", "slots") and (k > 2 or n % ar.tp):
        mode = "gather"
    return mode


def owner_slots(ar: NvlArena, n: int, k: int, h: int):
    """(device pointer table, rows per owner) of the bf16 owner slot buffers [rows x k x h]."""
    rows = n // ar.tp
    ar.tensor("slots", (rows, k, h), torch.bfloat16)
    return ar.device_table("slots"), rows


def finish_slots_forward(ar: NvlArena, n: int, k: int, h: int, pair_pos, out: torch.Tensor) -> torch.Tensor:
    """After the owner-slot fc2: barrier -> sum the owned tokens' valid slots -> barrier ->
    pull the other owners' blocks."""
    rows = n // ar.tp
    slots = ar.tensor("slots", (rows, k, h), torch.bfloat16)
    xch = ar.tensor("xch", (n, h), torch.bfloat16)
    s = _lib.stream_ptr()
    ar.barrier(0)
    t0 = ar.rank * rows
    call("ppmoe_nvl_sum_slots", ptr(slots), rows, k, h, t0, ptr(pair_pos), ptr(out[t0:t0 + rows]),
         ptr(xch[t0:t0 + rows]), s)
    ar.barrier(1)
    pull = "ppmoe_nvl_pull_blocks" if os.environ.get("PPMOE_NVL_PULL", "ce") == "sm" else "ppmoe_nvl_pull_blocks_ce"
    call(pull, ar.table("xch"), ar.tp, ar.rank, n, h, ptr(out), s)
    return out


def owner_accumulator(ar: NvlArena, n: int, h: int):
    """(device pointer table, rows per owner) of the fp32 owner accumulators."""
    rows = n // ar.tp
    ar.tensor("acc", (rows, h), torch.float32)
    return ar.device_table("acc"), rows


def finish_fused_forward(ar: NvlArena, n: int, h: int, out: torch.Tensor) -> torch.Tensor:
    """After the owner-mode fc2: barrier -> owned accumulator rows to bf16 (zeroing them) ->
    barrier -> pull the other owners' blocks."""
    rows = n // ar.tp
    acc = ar.tensor("acc", (rows, h), torch.float32)
    xch = ar.tensor("xch", (n, h), torch.bfloat16)
    s = _lib.stream_ptr()
    ar.barrier(0)
    t0 = ar.rank * rows
    call("ppmoe_nvl_cast_owned", ptr(acc), rows, h, ptr(out[t0:t0 + rows]), ptr(xch[t0:t0 + rows]), s)
    ar.barrier(1)
    pull = "ppmoe_nvl_pull_blocks" if os.environ.get("PPMOE_NVL_PULL", "ce") == "sm" else "ppmoe_nvl_pull_blocks_ce"
    call(pull, ar.table("xch"), ar.tp, ar.rank, n, h, ptr(out), s)
    return out


def exchange(ar: NvlArena, rows_name: str, seg, el: int, idx, pair_pos, w, n: int, h: int, out: torch.Tensor,
             dl_own: torch.Tensor | None = None, wg: torch.Tensor | None = None,
             barrier_first: bool = True) -> torch.Tensor:
    """out = the replicated sum over the group of every token's expert rows (+ the gate term
    dl_own . Wg^T of the owned rows), see nvlink.cu: barrier -> owner gather (P2P reads) ->
    barrier -> all-gather of the owners' blocks: copy-engine pulls of the peers' blocks, or
    (PPMOE_NVL_MC=1, NVSwitch multicast) an NVLS multimem store from the owner gather that
    reaches every rank's buffer, then a local copy.  The multicast form is correct but
    measured slower at T = 4 (the multimem stores make the owner gather 2x slower than the
    pull they save)."""
    k = pair_pos.shape[1]
    s = _lib.stream_ptr()
    if barrier_first:
        ar.barrier(0)
    e = wg.shape[1] if wg is not None else 0
    mc = ar.multicast("xchmc", (n, h)) if os.environ.get("PPMOE_NVL_MC", "0") == "1" else None
    if mc is not None:
        local, mc_ptr = mc
        call("ppmoe_nvl_owner_gather", ar.table(rows_name), ptr(seg), el, ptr(idx), ptr(pair_pos), ptr(w), n, k, h,
             ar.tp, ar.rank, ptr(dl_own), ptr(wg), e, ptr(out), ctypes.c_void_p(mc_ptr), None, 1, s)
        ar.barrier(1)  # every owner's multicast rows have landed everywhere
        call("ppmoe_nvl_pull_blocks", ptr_set([local.data_ptr()] * ar.tp), ar.tp, ar.rank, n, h, ptr(out), s)
        return out
    xch = ar.tensor("xch", (n, h), torch.bfloat16)
    push = os.environ.get("PPMOE_NVL_PUSH", "0") == "1"
    call("ppmoe_nvl_owner_gather", ar.table(rows_name), ptr(seg), el, ptr(idx), ptr(pair_pos), ptr(w), n, k, h,
         ar.tp, ar.rank, ptr(dl_own), ptr(wg), e, ptr(out), ptr(xch), ar.table("xch") if push else None, 0, s)
    ar.barrier(1)
    # push: every block already sits in the local exchange buffer; pull: read the owners'
    src = ar.local_table("xch") if push else ar.table("xch")
    # copy engines by default: the all-gather then takes no SMs from the overlapped GEMMs
    # (backward); PPMOE_NVL_PULL_FWD picks the forward's separately (nothing to overlap there)
    mode = os.environ.get("PPMOE_NVL_PULL", "ce")
    if rows_name == "y":
        mode = os.environ.get("PPMOE_NVL_PULL_FWD", mode)
    pull = "ppmoe_nvl_pull_blocks" if mode == "sm" else "ppmoe_nvl_pull_blocks_ce"
    call(pull, src, ar.tp, ar.rank, n, h, ptr(out), s)
    if _STRICT:
        ar.check()
    return out


def forward_chunks(ar: NvlArena, n: int) -> int:
    """Token chunks of the pipelined forward exchange (PPMOE_NVL_CHUNKS): chunk c is the
    token range of owners [c T/C, (c+1) T/C), so C must divide T."""
    c = int(os.environ.get("PPMOE_NVL_CHUNKS", "1"))
    if c <= 1 or ar.tp % c or n % ar.tp:
        return 1
    return c


def exchange_chunk(ar: NvlArena, c: int, chunks: int, rows_name: str, seg, el: int, idx, pair_pos, w, n: int, h: int,
                   out: torch.Tensor) -> None:
    """Exchange of token chunk c (its owners' blocks): barrier (every rank's rows of the
    chunk are final) -> owner gather on the chunk's owners -> barrier -> every rank pulls
    the chunk's blocks.  Runs on the arena's side stream while the next chunk computes."""
    k = pair_pos.shape[1]
    q_lo, q_hi = c * ar.tp // chunks, (c + 1) * ar.tp // chunks
    ch = 4 + 2 * (c % 2)
    xch = ar.tensor("xch", (n, h), torch.bfloat16)
    s = _lib.stream_ptr()
    ar.barrier(ch)
    if q_lo <= ar.rank < q_hi:
        call("ppmoe_nvl_owner_gather", ar.table(rows_name), ptr(seg), el, ptr(idx), ptr(pair_pos), ptr(w), n, k, h,
             ar.tp, ar.rank, None, None, 0, ptr(out), ptr(xch), None, 0, s)
    ar.barrier(ch + 1)
    call("ppmoe_nvl_pull_range_ce", ar.table("xch"), ar.tp, ar.rank, n, h, q_lo, q_hi, ptr(out), s)
