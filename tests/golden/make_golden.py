"""Generate golden vectors for the PPMoE hot path from the REFERENCE itself.

Run in the build container (where the read-only reference lives):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``moesim`` from /root/reference/pkg/src, evaluates gate_top1,
build_dispatch_plan, ppmoe_forward (+ tensor.backward) and single-rank
dpmoe_forward with capacity on seeded inputs, and writes small .npz files next to
this script.  Inputs are rounded before they reach the reference — hidden rows
and expert weights to bf16, the gate weight to fp32 — so the same vectors pin
both the bf16 and the fp32 modes of the CUDA path.  Only seeds and outputs are
stored; tests rebuild the inputs with oracle.init_layer (bit-identical Philox
streams, checked through the stored weight checksums).
"""

from __future__ import annotations

import json
import math
import os
import sys
from pathlib import Path

import numpy as np
import torch

REF = Path(os.environ.get("PPMOE_REFERENCE", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))
sys.dont_write_bytecode = True

from moesim import moe  # noqa: E402
from moesim import tensor as T  # noqa: E402
from moesim.collectives import EP, ProcessGroup, World  # noqa: E402

OUT = Path(__file__).resolve().parent


def bf16(a):
    return torch.from_numpy(np.array(a, dtype=np.float64)).to(torch.bfloat16).to(torch.float64).numpy()


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def hidden_of(seed, n, h):
    return bf16(T.Rng(seed, 99).normal((n, h)))


def rounded_layer(h, e, seed, bias=True):
    layer = moe.MoeLayerWeights.init(h, e, T.Rng(seed), bias=bias)
    layer.gate.wg = T.tensor(f32(layer.gate.wg.data), requires_grad=True)
    for ex in layer.experts:
        ex.up = T.tensor(bf16(ex.up.data), requires_grad=True)
        ex.down = T.tensor(bf16(ex.down.data), requires_grad=True)
        if ex.bias_up is not None:
            ex.bias_up = T.tensor(bf16(ex.bias_up.data), requires_grad=True)
            ex.bias_down = T.tensor(bf16(ex.bias_down.data), requires_grad=True)
    return layer


def weight_checksums(layer):
    out = {}
    for name, p in layer.named_parameters().items():
        out[name] = [float(p.data.sum()), float(np.abs(p.data).sum())]
    return out


def ep(n):
    return ProcessGroup(EP, tuple(range(n)))


def run_ppmoe(case):
    h, e, n, tp, seed = case["hidden"], case["experts"], case["tokens"], case["tp"], case["seed"]
    layer = rounded_layer(h, e, seed, case.get("bias", True))
    x0 = hidden_of(seed, n, h)
    x = T.tensor(x0, requires_grad=True)
    override = case.get("override")
    drop = case.get("dropout_p", 0.0)
    rng = T.Rng(seed, 77) if drop > 0 else None
    out, l_aux = moe.ppmoe_forward(World(1, tp), ep(tp), x, layer.gate, layer.shard(tp),
                                   weight_scaling=case.get("weight_scaling", True), route_override=override,
                                   dropout_p=drop, rng=rng)
    T.backward(T.add(T.tsum(out), l_aux))
    gate = moe.gate_top1(T.tensor(x0), layer.gate, route_override=override)
    plan = moe.build_dispatch_plan(gate.indices, e)
    return layer, x, out, l_aux, gate, plan


def run_dpmoe_capacity(case):
    h, e, n, seed = case["hidden"], case["experts"], case["tokens"], case["seed"]
    layer = rounded_layer(h, e, seed, case.get("bias", True))
    x0 = hidden_of(seed, n, h)
    x = T.tensor(x0, requires_grad=True)
    override = case.get("override")
    [(out, l_aux)] = moe.dpmoe_forward(World(1, 1), ep(1), [x], layer.gate, experts_by_rank=layer.shard(1),
                                       capacity_factor=case["capacity_factor"],
                                       route_overrides=None if override is None else [override])
    T.backward(T.add(T.tsum(out), l_aux))
    gate = moe.gate_top1(T.tensor(x0), layer.gate, route_override=override)
    return layer, x, out, l_aux, gate


def pack_lists(lists):
    flat = np.array([i for rows in lists for i in rows], dtype=np.int64)
    offs = np.cumsum([0] + [len(r) for r in lists]).astype(np.int64)
    return flat, offs


def save(name, case, arrays, meta=None):
    meta = dict(meta or {})
    meta["case"] = case
    np.savez_compressed(OUT / f"{name}.npz", meta=np.array(json.dumps(meta)), **arrays)
    print(f"wrote {name}.npz ({(OUT / f'{name}.npz').stat().st_size} bytes)")


def layer_case(name, case, sample_every=1):
    layer, x, out, l_aux, gate, plan = run_ppmoe(case)
    grads = {k: p.grad for k, p in layer.named_parameters().items() if p.grad is not None}
    arrays = {
        "indices": gate.indices.astype(np.int64),
        "weights": gate.weights.data,
        "l_aux": np.array(l_aux.item()),
    }
    flat, offs = pack_lists(plan.per_expert)
    arrays["plan_flat"], arrays["plan_offs"] = flat, offs
    rows = np.arange(0, out.shape[0], sample_every)
    arrays["rows"] = rows
    arrays["out"] = out.data[rows]
    arrays["grad_hidden"] = x.grad[rows]
    arrays["grad_gate.wg"] = grads["gate.wg"]
    checks = {}
    for k, g in grads.items():
        checks[k] = [float(g.sum()), float(np.abs(g).sum()), float((g * g).sum())]
        if k != "gate.wg" and sample_every == 1 and case["hidden"] <= 64:
            arrays[f"grad_{k}"] = g
    meta = {"weights": weight_checksums(layer), "grad_checksums": checks,
            "out_checksum": [float(out.data.sum()), float(np.abs(out.data).sum())],
            "grad_hidden_checksum": [float(x.grad.sum()), float(np.abs(x.grad).sum())]}
    save(name, case, arrays, meta)


def stack_case(name, case):
    """A residual stack of (dense_tp_ffn_forward, ppmoe_forward) blocks (moe.py:316-335,
    254-308) on one TP group: loss = sum(out) + sum of l_aux, tensor.backward.  Dense FFN of
    block i: ExpertFfn.init(h, Rng(seed, 200 + i)) rounded to bf16; MoE of block i:
    MoeLayerWeights.init(h, E, Rng(seed + 1 + i)) rounded like the layer goldens."""
    h, e, n, tp, seed, nb = case["hidden"], case["experts"], case["tokens"], case["tp"], case["seed"], case["blocks"]
    x0 = hidden_of(seed, n, h)
    x = T.tensor(x0, requires_grad=True)
    cur, aux, params = x, None, {}
    for i in range(nb):
        ffn = moe.ExpertFfn.init(h, T.Rng(seed, 200 + i))
        ffn.up = T.tensor(bf16(ffn.up.data), requires_grad=True)
        ffn.down = T.tensor(bf16(ffn.down.data), requires_grad=True)
        ffn.bias_down = T.tensor(bf16(ffn.bias_down.data), requires_grad=True)
        layer = rounded_layer(h, e, seed + 1 + i)
        d = moe.dense_tp_ffn_forward(World(1, tp), ep(tp), cur, ffn)
        x1 = T.add(cur, d)
        out, l_aux = moe.ppmoe_forward(World(1, tp), ep(tp), x1, layer.gate, layer.shard(tp))
        cur = T.add(x1, out)
        aux = l_aux if aux is None else T.add(aux, l_aux)
        params.update({f"{i}.dense.up": ffn.up, f"{i}.dense.down": ffn.down, f"{i}.dense.bias_down": ffn.bias_down})
        params.update({f"{i}.moe.{k}": p for k, p in layer.named_parameters().items()})
    T.backward(T.add(T.tsum(cur), aux))
    arrays = {"out": cur.data, "grad_hidden": x.grad, "aux": np.array(aux.item())}
    for k, p in params.items():
        if p.grad is not None:
            arrays[f"grad_{k}"] = p.grad
    save(name, case, arrays)


def main():
    if sys.argv[1:] == ["dropout"]:
        layer_case("ppmoe_dropout", {"hidden": 32, "experts": 4, "tokens": 64, "tp": 2, "seed": 15,
                                     "dropout_p": 0.25})
        return
    if sys.argv[1:] == ["stack"]:
        stack_case("stack_2blocks_tp2", {"hidden": 32, "experts": 4, "tokens": 40, "tp": 2, "seed": 31, "blocks": 2})
        return
    torch.set_num_threads(1)
    # gate_top1 on a random instance (test_moe.py:44-55 style) and the identity-gate goldens
    rng = T.Rng(50)
    gate = moe.GateParams.init(8, 4, rng)
    hid = rng.normal((64, 8))
    g = moe.gate_top1(T.tensor(hid), gate)
    save("gate_small", {"seed": 50}, {"hidden": hid, "wg": gate.wg.data, "indices": g.indices.astype(np.int64),
                                      "weights": g.weights.data, "scores": g.scores.data,
                                      "l_aux": np.array(g.l_aux.item())})
    # dispatch worked example (test_moe.py:95-97)
    order = [2, 3, 1, 2, 0, 3, 2, 0]
    plan = moe.build_dispatch_plan(order, 4)
    flat, offs = pack_lists(plan.per_expert)
    save("dispatch_example", {"order": order}, {"order": np.array(order), "plan_flat": flat, "plan_offs": offs})
    # random dispatch plan, 6 experts x 40 tokens (test_moe.py:105-112 style)
    ids = T.Rng(52).integers(0, 6, 40)
    plan = moe.build_dispatch_plan(ids, 6)
    flat, offs = pack_lists(plan.per_expert)
    save("dispatch_random", {"seed": 52}, {"order": ids.astype(np.int64), "plan_flat": flat, "plan_offs": offs})

    layer_case("ppmoe_h64_e4_tp2", {"hidden": 64, "experts": 4, "tokens": 96, "tp": 2, "seed": 11})
    layer_case("ppmoe_h128_e8_tp4", {"hidden": 128, "experts": 8, "tokens": 256, "tp": 4, "seed": 12})
    layer_case("ppmoe_nobias_noscale", {"hidden": 64, "experts": 4, "tokens": 64, "tp": 1, "seed": 13,
                                        "bias": False, "weight_scaling": False})
    ov = T.Rng(14, 5).integers(0, 4, 48).tolist()
    layer_case("ppmoe_override", {"hidden": 64, "experts": 4, "tokens": 48, "tp": 2, "seed": 14, "override": ov})
    layer_case("ppmoe_dropout", {"hidden": 32, "experts": 4, "tokens": 64, "tp": 2, "seed": 15, "dropout_p": 0.25})
    # C1 shape (BASELINE configs[0]): h=512, ffn=2048, E=8, top-1, 2048 tokens; rows sampled
    layer_case("ppmoe_c1", {"hidden": 512, "experts": 8, "tokens": 2048, "tp": 1, "seed": 0}, sample_every=16)

    # capacity: single-rank dpmoe_forward is the oracle for top-1 + capacity (moe.py:345-469)
    for name, cf, skew in (("capacity_cf050", 0.5, False), ("capacity_cf100_skew", 1.0, True)):
        case = {"hidden": 64, "experts": 4, "tokens": 64, "seed": 21, "capacity_factor": cf}
        if skew:
            case["override"] = [0 if t % 3 else int(T.Rng(22).integers(0, 4, 1)[0]) for t in range(64)]
        layer, x, out, l_aux, gate = run_dpmoe_capacity(case)
        grads = {k: p.grad for k, p in layer.named_parameters().items() if p.grad is not None}
        arrays = {"indices": gate.indices.astype(np.int64), "out": out.data, "grad_hidden": x.grad,
                  "l_aux": np.array(l_aux.item()), "grad_gate.wg": grads["gate.wg"]}
        for k, gr in grads.items():
            arrays[f"grad_{k}"] = gr
        save(name, case, arrays, {"weights": weight_checksums(layer),
                                  "capacity": math.ceil(cf * 64 / 4)})
    stack_case("stack_2blocks_tp2", {"hidden": 32, "experts": 4, "tokens": 40, "tp": 2, "seed": 31, "blocks": 2})


if __name__ == "__main__":
    main()
