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
