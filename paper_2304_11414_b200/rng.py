"""Deterministic counter-based random streams (the reference's ``Rng``, tensor.py:23-49).

Identical (seed, stream, draw index) give identical values on every platform, so
weights initialised here are bit-identical to ``moesim.MoeLayerWeights.init`` with
the same seed.  Draws happen on the host (numpy Philox) — this is input
generation, not the measured layer path.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np


class Rng:
    def __init__(self, seed: int, stream: int = 0):
        if seed < 0 or stream < 0:
            raise ValueError(f"seed and stream must be non-negative, got ({seed}, {stream})")
        self.seed = seed
        self.stream = stream
        self._gen = np.random.Generator(np.random.Philox(key=np.array([seed, stream], dtype=np.uint64)))

    def normal(self, shape: Sequence[int], scale: float = 1.0) -> np.ndarray:
        return self._gen.normal(0.0, scale, size=tuple(shape))

    def uniform(self, shape: Sequence[int]) -> np.ndarray:
        return self._gen.uniform(0.0, 1.0, size=tuple(shape))

    def integers(self, low: int, high: int, count: int) -> np.ndarray:
        return self._gen.integers(low, high, size=count)

    def normal_tensor(self, shape: Sequence[int], scale: float = 1.0, dtype=None, device="cuda"):
        """``normal(shape, scale)`` rounded to ``dtype`` in a torch tensor on ``device``, drawn
        in row chunks (the same values as one ``normal`` call, without the fp64 host copy):
        BASELINE's hidden batch is ``Rng(1, 99).normal_tensor((N, h), dtype=torch.bfloat16)``."""
        import torch

        from .moe import _draw_into

        out = torch.empty(tuple(shape), dtype=dtype or torch.float32, device=device)
        _draw_into(self, out, scale)
        return out

    def spawn(self, stream: int) -> "Rng":
        """Fresh generator on a sibling sub-stream of the same seed."""
        return Rng(self.seed, stream)


_M64 = (1 << 64) - 1


def philox4x64_block(counter: int, key0: int, key1: int) -> list:
    """One block of numpy's Philox4x64-10 (the bit generator behind Rng): the four 64-bit
    words at `counter` (< 2^64) under key (key0, key1).  Used to rebuild a generator's buffer
    after the device consumed draws (DropoutStream.advance); the device twin is
    csrc/common.cuh philox4x64_10."""
    c = [counter & _M64, 0, 0, 0]
    k0, k1 = key0 & _M64, key1 & _M64
    for r in range(10):
        if r:
            k0 = (k0 + 0x9E3779B97F4A7C15) & _M64
            k1 = (k1 + 0xBB67AE8584CAA73B) & _M64
        p0 = 0xD2E7470EE14C6C93 * c[0]
        p1 = 0xCA5A826395121157 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k0, p1 & _M64, (p0 >> 64) ^ c[3] ^ k1, p0 & _M64]
    return c


def stream_position(gen: np.random.Generator) -> tuple:
    """(key0, key1, draws consumed) of a Philox generator: draw m of the stream is word m % 4
    of the block at counter m // 4 + 1."""
    st = gen.bit_generator.state
    if st.get("bit_generator") != "Philox":
        raise ValueError("dropout needs a Philox-backed Rng (moesim's Rng)")
    ctr = [int(v) for v in st["state"]["counter"]]
    if any(ctr[1:]):
        raise ValueError("Philox counter beyond 2^64 blocks is not supported")
    key = [int(v) for v in st["state"]["key"]]
    return key[0], key[1], 4 * ctr[0] + int(st["buffer_pos"]) - 4


def set_stream_position(gen: np.random.Generator, draws: int) -> None:
    """Move a Philox generator to `draws` consumed draws of its stream (as if drawn)."""
    st = gen.bit_generator.state
    key0, key1 = (int(v) for v in st["state"]["key"])
    if draws == 0:
        ctr, pos, buf = 0, 4, [0, 0, 0, 0]
    else:
        ctr = (draws + 3) // 4
        pos = draws - 4 * (ctr - 1)
        buf = philox4x64_block(ctr, key0, key1)
    st["state"]["counter"] = np.array([ctr, 0, 0, 0], dtype=np.uint64)
    st["buffer"] = np.array(buf, dtype=np.uint64)
    st["buffer_pos"] = pos
    st["has_uint32"] = 0
    st["uinteger"] = 0
    gen.bit_generator.state = st
