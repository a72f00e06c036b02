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
                   weight_scaling=True, route_override=None, dtype=torch.bfloat16, grad_out=None):
    x = torch.as_tensor(hidden, dtype=torch.float64).to("cuda", dtype).requires_grad_()
    world = P.World(1, tp)
    group = P.ProcessGroup(P.EP, tuple(range(tp)))
    out, l_aux = P.ppmoe_forward(world, group, x, w.gate, w.shard(tp), weight_scaling=weight_scaling,
                                 route_override=route_override, top_k=k, capacity_factor=capacity_factor)
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
