"""Loading helpers for the reference-generated golden vectors (tests/golden)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import torch

from oracle import ppmoe_oracle as O

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str):
    z = np.load(GOLDEN / f"{name}.npz")
    meta = json.loads(str(z["meta"]))
    arrays = {k: z[k] for k in z.files if k != "meta"}
    return meta, arrays


def bf16(a):
    return torch.from_numpy(np.array(a, dtype=np.float64)).to(torch.bfloat16).to(torch.float64).numpy()


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def golden_inputs(case):
    """Rebuild (hidden, layer) exactly as make_golden.py fed them to the reference."""
    h, e, n, seed = case["hidden"], case["experts"], case["tokens"], case["seed"]
    layer = O.init_layer(h, e, seed, bias=case.get("bias", True))
    layer = O.OracleLayer(f32(layer.wg), [bf16(u) for u in layer.up], [bf16(d) for d in layer.down],
                          [bf16(b) for b in layer.bias_up], [bf16(b) for b in layer.bias_down])
    hidden = bf16(O.philox(seed, 99).normal(0.0, 1.0, size=(n, h)))
    return hidden, layer


def unpack_lists(flat, offs):
    return [flat[offs[i]:offs[i + 1]].tolist() for i in range(len(offs) - 1)]


def stack_inputs(case):
    """Rebuild (hidden, blocks) of make_golden.stack_case: dense FFN i from Philox (seed,
    200+i) in ExpertFfn.init's draw order (up, down, bias_up, bias_down), MoE layer i from
    init_layer(seed+1+i), all rounded as the reference saw them."""
    h, e, n, seed = case["hidden"], case["experts"], case["tokens"], case["seed"]
    hidden = bf16(O.philox(seed, 99).normal(0.0, 1.0, size=(n, h)))
    blocks = []
    for i in range(case["blocks"]):
        g = O.philox(seed, 200 + i)
        scale = h ** -0.5
        up = g.normal(0.0, scale, size=(h, 4 * h))
        down = g.normal(0.0, scale, size=(4 * h, h))
        g.normal(0.0, scale, size=(4 * h,))  # bias_up: drawn, unused by dense_tp_ffn_forward
        bd = g.normal(0.0, scale, size=(h,))
        lay = O.init_layer(h, e, seed + 1 + i)
        lay = O.OracleLayer(f32(lay.wg), [bf16(u) for u in lay.up], [bf16(d) for d in lay.down],
                            [bf16(b) for b in lay.bias_up], [bf16(b) for b in lay.bias_down])
        blocks.append(O.StackBlock(bf16(up), bf16(down), bf16(bd), lay))
    return hidden, blocks
