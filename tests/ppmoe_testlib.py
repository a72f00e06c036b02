"""Shared helpers for the parity tests: move oracle layers to the device and run the
CUDA path through the package's public API (which calls the C-ABI library)."""

from __future__ import annotations

import math

import numpy as np
import torch

import paper_2304_11414_b200 as P
from oracle import ppmoe_oracle as O

TOL = {torch.bfloat16: 2e-2, torch.float32: 1e-4}  # north_star tolerances (rtol, scaled by max|ref|)


def scaled_err(got, ref) -> float:
    """max|got - ref| / max|ref|: allclose(rtol, atol = rtol * max|ref|) as one number."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    denom = max(float(np.abs(ref).max(initial=0.0)), 1e-30)
    return float(np.abs(got - ref).max(initial=0.0)) / denom


def device_weights(layer: O.OracleLayer, dtype=torch.bfloat16, device="cuda") -> P.MoeLayerWeights:
    def t(a, dt):
        return torch.as_tensor(np.asarray(a), dtype=torch.float64).to(device=device, dtype=dt).contiguous().requires_grad_()

    gate = P.GateParams(t(layer.wg, torch.float32))
    bank = P.ExpertBank(t(np.stack(layer.up), dtype), t(np.stack(layer.down), dtype),
                        t(np.stack(layer.bias_up), dtype) if layer.bias_up else None,
                        t(np.stack(layer.bias_down), dtype) if layer.bias_down else None)
    return P.MoeLayerWeights(gate, bank)


def run_cuda_layer(hidden: np.ndarray, w: P.MoeLayerWeights, *, tp=1, k=1, capacity_factor=math.inf,
                   weight_scaling=True, route_override=None, dtype=torch.bfloat16, grad_out=None, dropout_p=0.0,
                   rng=None):
    x = torch.as_tensor(hidden, dtype=torch.float64).to("cuda", dtype).requires_grad_()
    world = P.World(1, tp)
    group = P.ProcessGroup(P.EP, tuple(range(tp)))
    out, l_aux = P.ppmoe_forward(world, group, x, w.gate, w.shard(tp), weight_scaling=weight_scaling,
                                 route_override=route_override, top_k=k, capacity_factor=capacity_factor,
                                 dropout_p=dropout_p, rng=rng)
    if grad_out is None:
        loss = out.float().sum() + l_aux
    else:
        loss = (out.float() * torch.as_tensor(grad_out, device="cuda", dtype=torch.float32)).sum() + l_aux
    loss.backward()
    torch.cuda.synchronize()
    grads = {k2: (None if v is None else v.detach().double().cpu().numpy()) for k2, v in w.named_grads().items()}
    return {
        "out": out.detach().double().cpu().numpy(),
        "l_aux": float(l_aux.detach()),
        "grad_hidden": x.grad.detach().double().cpu().numpy(),
        "grads": grads,
        "world": world,
    }


def oracle_rounded(layer: O.OracleLayer, dtype) -> O.OracleLayer:
    """The oracle sees exactly the values the device holds."""
    def r(a):
        return torch.as_tensor(np.asarray(a)).to(dtype).double().numpy()

    return O.OracleLayer(np.asarray(layer.wg, dtype=np.float32).astype(np.float64), [r(u) for u in layer.up],
                         [r(d) for d in layer.down], [r(b) for b in layer.bias_up], [r(b) for b in layer.bias_down])


def per_token_oracle(x64, wg64, bank, tokens, k, n_all, route, kept=None):
    """out[t] and dX[t] of the C2 layer for the sampled tokens t, in fp64, from the closed
    form of oracle.ppmoe_layer (dOut = ones, aux gradient 1) restricted to one token:
    out[t] = sum_e w_te FFN_e(x_t); dX[t] = sum_e (w_te (1 down_e^T) * GeLU'(a)) up_e^T
    + dL_t Wg^T, with dS[t,e] = sum_j Y_e(x_t)_j + (E/N) frac_e.  `kept` [N, k] drops the
    pairs capacity removed (they contribute neither output nor expert gradient)."""
    e_count = wg64.shape[1]
    h = x64.shape[1]
    out = np.zeros((len(tokens), h))
    dx = np.zeros((len(tokens), h))
    ds = np.zeros((len(tokens), e_count))
    for e in range(e_count):
        sel = [(i, s) for i, t in enumerate(tokens) for s in range(k)
               if route.indices[t, s] == e and (kept is None or kept[t, s])]
        if not sel:
            continue
        up = bank.up[e].detach().double().cpu().numpy()
        down = bank.down[e].detach().double().cpu().numpy()
        bu = bank.bias_up[e].detach().double().cpu().numpy()
        bd = bank.bias_down[e].detach().double().cpu().numpy()
        rows = np.array([i for i, _ in sel])
        wt = np.array([route.weights[tokens[i], s] for i, s in sel])
        a = x64[tokens[rows]] @ up + bu
        y = O.gelu(a) @ down + bd
        out[rows] += wt[:, None] * y
        ds[rows, e] += y.sum(axis=1)
        da = wt[:, None] * down.sum(axis=1)[None, :] * O.gelu_grad(a)
        dx[rows] += da @ up.T
    frac = route.top1_counts / n_all
    ds += (e_count / n_all) * frac[None, :]
    s = route.scores[tokens]
    dl = s * (ds - (ds * s).sum(axis=1, keepdims=True))
    dx += dl @ wg64.T
    return out, dx


# ------------------------------------------------------------------ full-size fp64 restatement on the device
#
# oracle.ppmoe_layer restated in torch fp64 so that it runs at BASELINE sizes (C2: 26 TFLOP,
# C3: 106 TFLOP of fp64 GEMMs on the GPU's FP64 pipe instead of hours of host BLAS).  The
# routing (indices, weights, scores, top-1 counts) and the capacity mask come from the host
# oracle (O.gate_topk / O.dispatch_plan), so the only arithmetic restated here is the
# per-expert FFN, its backward and the softmax/gate backward, line for line with
# O.ppmoe_layer (moe.py:100-107, tensor.py:134-138, 190-221).  Checked against the oracle
# on the CPU in tests/test_oracle.py::test_fp64_restatement_matches_oracle.


def _gelu64(a):
    return 0.5 * a * (1.0 + torch.special.erf(a * (2.0 ** -0.5)))


def _gelu_grad64(a):
    return 0.5 * (1.0 + torch.special.erf(a * (2.0 ** -0.5))) + a * torch.exp(-0.5 * a * a) * (2.0 * math.pi) ** -0.5


def fp64_expert_pass(x, bank, expert_ids, indices, weights, kept, num_experts, grad_out=None, weight_scaling=True,
                     on_expert=None):
    """Experts `expert_ids` (global ids; bank index = position in the list) of the layer in
    fp64.  Returns (out_part, dx_part, ds_part): their contribution to out, to dX through
    the experts, and to dS = d loss / d scores.  ``on_expert(e, grads)`` receives each
    expert's parameter gradients (dicts of fp64 device tensors) as soon as they exist.
    `indices`/`weights`/`kept` are [N, k] device tensors (int64 / fp64 / bool)."""
    n, h = x.shape
    dev = x.device
    x64 = x.detach().double()
    out = torch.zeros((n, h), dtype=torch.float64, device=dev)
    dx = torch.zeros((n, h), dtype=torch.float64, device=dev)
    ds = torch.zeros((n, num_experts), dtype=torch.float64, device=dev)
    has_bias = bank.bias_up is not None
    for i, e in enumerate(expert_ids):
        m = (indices == e) & kept
        rows = torch.nonzero(m.any(dim=1)).flatten()
        up = bank.up[i].detach().double()
        down = bank.down[i].detach().double()
        grads = {}
        if rows.numel() == 0:
            grads["up"] = torch.zeros_like(up)
            grads["down"] = torch.zeros_like(down)
            if has_bias:
                grads["bias_up"] = torch.zeros(up.shape[1], dtype=torch.float64, device=dev)
                grads["bias_down"] = torch.zeros(h, dtype=torch.float64, device=dev)
        else:
            wr = (weights * m).sum(dim=1)[rows]
            xe = x64[rows]
            a = xe @ up
            if has_bias:
                a += bank.bias_up[i].detach().double()
            hh = _gelu64(a)
            y = hh @ down
            if has_bias:
                y += bank.bias_down[i].detach().double()
            out.index_add_(0, rows, y * wr[:, None] if weight_scaling else y)
            g = torch.ones_like(y) if grad_out is None else grad_out[rows].double()
            if weight_scaling:
                dy = g * wr[:, None]
                ds[rows, e] += (g * y).sum(dim=1)
            else:
                dy = g
            del y
            grads["down"] = hh.T @ dy
            del hh
            da = (dy @ down.T) * _gelu_grad64(a)
            del a
            grads["up"] = xe.T @ da
            if has_bias:
                grads["bias_down"] = dy.sum(dim=0)
                grads["bias_up"] = da.sum(dim=0)
            dx.index_add_(0, rows, da @ up.T)
            del da, dy
        if on_expert is not None:
            on_expert(e, grads)
        del grads
    return out, dx, ds


def fp64_gate_pass(x, wg, scores, top1_counts, ds, aux_grad=1.0):
    """Aux-loss term + softmax backward + gate GEMMs of O.ppmoe_layer (moe.py:211-223,
    tensor.py:218-221): returns (dWg, dX through the gate) in fp64."""
    n = x.shape[0]
    e_count = scores.shape[1]
    frac = top1_counts.double() / n
    ds = ds + aux_grad * (e_count / n) * frac[None, :]
    s = scores
    dl = s * (ds - (ds * s).sum(dim=1, keepdim=True))
    x64 = x.detach().double()
    return x64.T @ dl, dl @ wg.detach().double().T


def dev_scaled_err(got, ref) -> float:
    """scaled_err on the device: max|got - ref| / max|ref|."""
    got = got.detach().double()
    ref = ref.detach().double()
    denom = max(float(ref.abs().max()), 1e-30) if ref.numel() else 1.0
    return float((got - ref).abs().max()) / denom if ref.numel() else 0.0


def routing_on_device(route, kept, device="cuda"):
    """(indices int64, weights fp64, kept bool, scores fp64, top-1 counts) of an oracle Routing."""
    return (torch.as_tensor(route.indices, dtype=torch.int64, device=device),
            torch.as_tensor(route.weights, dtype=torch.float64, device=device),
            torch.as_tensor(kept, dtype=torch.bool, device=device),
            torch.as_tensor(route.scores, dtype=torch.float64, device=device),
            torch.as_tensor(route.top1_counts, dtype=torch.int64, device=device))


def min_topk_gap(scores: np.ndarray, k: int) -> float:
    """Smallest gap between consecutive scores among a token's top k+1 (how close the
    selection and the slot order are to a tie)."""
    m = min(k + 1, scores.shape[1])
    if m < 2:
        return float("inf")
    top = -np.sort(-scores, axis=1)[:, :m]
    return float((top[:, :-1] - top[:, 1:]).min())
