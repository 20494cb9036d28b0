"""Standalone decoder-MLP passes on the GPU: the reference's mlp_forward /
mlp_backward (mlp.py:55-85) for callers that compose the MLP with their own
upstream gradient (the C3 harness composes encode_forward,
mlp_forward, mlp_backward and encode_backward).

`params` is either the reference's MlpParams-like object (numpy
``weights`` / ``biases`` / ``weight_grads`` / ``bias_grads`` lists, (fan_in,
fan_out) weights) or a device Model's ``mlp`` view; x and upstream follow
the parameters (numpy in -> numpy out, CUDA tensors in -> tensors out).
Gradients ACCUMULATE into params.weight_grads / bias_grads, as the
reference's do.  Arithmetic: the batched numpy / OpenBLAS operation order
(pg_mlp_forward / pg_mlp_backward), so outputs and dx match the reference
to rounding of the summation order only.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ShapeMismatch
from .hyper import mlp_struct


@dataclass
class MlpCache:
    """What mlp_backward needs: the input rows, the output shape, and the
    device copies the forward used (the backward re-runs the forward
    layers from x inside the kernel sequence, pg_mlp_backward)."""
    x: torch.Tensor
    out_shape: tuple
    flat: torch.Tensor
    widths: list


def _widths(params):
    return [params.weights[0].shape[0]] + [w.shape[1] for w in params.weights]


def _flat(params, dev, dt) -> torch.Tensor:
    parts = []
    for w, b in zip(params.weights, params.biases):
        parts += [torch.as_tensor(w).reshape(-1), torch.as_tensor(b).reshape(-1)]
    return torch.cat([p.to(device=dev, dtype=dt) for p in parts])


def _device(x):
    return x.device if isinstance(x, torch.Tensor) and x.is_cuda else torch.device("cuda")


def mlp_forward(params, x):
    """Batched forward: returns (output, cache) (mlp.py:55-70)."""
    as_numpy = not isinstance(x, torch.Tensor)
    n_in = params.weights[0].shape[0]
    if x.ndim != 2 or x.shape[1] != n_in:
        raise ShapeMismatch(f"input shape {tuple(x.shape)} does not match first layer ({n_in} inputs)")
    dev = _device(x)
    dt = torch.float64 if (x.dtype == np.float64 or x.dtype == torch.float64) else torch.float32
    xt = (torch.from_numpy(np.ascontiguousarray(x)) if as_numpy else x).to(device=dev, dtype=dt).contiguous()
    widths = _widths(params)
    flat = _flat(params, dev, dt)
    B = xt.shape[0]
    out = torch.empty((B, widths[-1]), dtype=dt, device=dev)
    desc = mlp_struct(widths)
    ws = torch.empty(max(1, int(_lib.lib().pg_mlp_train_workspace_floats(B, desc))), dtype=dt, device=dev)
    sfx = "f64" if dt == torch.float64 else "f32"
    with torch.cuda.device(dev):
        _lib.call(f"pg_mlp_forward_{sfx}", desc, _lib.ptr(xt), B, _lib.ptr(flat), _lib.ptr(ws), _lib.ptr(out),
                  _lib.stream_ptr())
    cache = MlpCache(xt, tuple(out.shape), flat, widths)
    return (out.cpu().numpy() if as_numpy else out), cache


def mlp_backward(params, cache: MlpCache, upstream):
    """Accumulate parameter gradients; returns dL/dx (mlp.py:73-85)."""
    as_numpy = not isinstance(upstream, torch.Tensor)
    if tuple(upstream.shape) != cache.out_shape:
        raise ShapeMismatch(f"upstream shape {tuple(upstream.shape)} != output shape {cache.out_shape}")
    xt, flat, widths = cache.x, cache.flat, cache.widths
    dev, dt = xt.device, xt.dtype
    up = (torch.from_numpy(np.ascontiguousarray(upstream)) if as_numpy else upstream).to(
        device=dev, dtype=dt).contiguous()
    B = xt.shape[0]
    desc = mlp_struct(widths)
    ws = torch.empty(max(1, int(_lib.lib().pg_mlp_train_workspace_floats(B, desc))), dtype=dt, device=dev)
    g = torch.zeros_like(flat)
    dx = torch.empty((B, widths[0]), dtype=dt, device=dev)
    sfx = "f64" if dt == torch.float64 else "f32"
    with torch.cuda.device(dev):
        _lib.call(f"pg_mlp_backward_{sfx}", desc, _lib.ptr(xt), B, _lib.ptr(flat), _lib.ptr(up), _lib.ptr(g),
                  _lib.ptr(dx), _lib.ptr(ws), _lib.stream_ptr())
    off = 0
    for wg, bg, (fi, fo) in zip(params.weight_grads, params.bias_grads, zip(widths[:-1], widths[1:])):
        gw = g[off:off + fi * fo].view(fi, fo)
        off += fi * fo
        gb = g[off:off + fo]
        off += fo
        if isinstance(wg, torch.Tensor):
            wg += gw.to(wg.dtype)
            bg += gb.to(bg.dtype)
        else:
            wg += gw.cpu().numpy().astype(wg.dtype)
            bg += gb.cpu().numpy().astype(bg.dtype)
    return dx.cpu().numpy() if as_numpy else dx
