"""Fused multiresolution encoding entry points (encoding.py:42-133 of the
reference) on the device-resident model: ONE kernel encodes every level.

``encode_forward(model, xs)`` accepts numpy (returns numpy, like the
reference) or a CUDA tensor (returns a CUDA tensor, no host round trip).
The returned trace keeps the device copy of xs; ``encode_backward``
recomputes corner geometry from it instead of storing per-level index and
weight arrays (12-48 B per point-level the reference keeps in LevelTrace).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import on_device
from .errors import DomainViolation, StaleTrace
from .grid_model import Model
from .hyper import AUX_PRIMES, PRIMARY_PRIMES, LevelMode


@dataclass
class LevelTrace:
    """The reference's per-level trace (encoding.py:22-30)."""
    kind: str                 # "dense" | "hashed" | "probed"
    weights: np.ndarray       # (B, 2^d)
    idx: np.ndarray = None    # dense/hashed: final feature rows (B, 2^d)
    base: np.ndarray = None   # probed: (n_p * hash) mod n_f
    row: np.ndarray = None    # probed: hash2 mod n_c
    feat_shape: tuple = None
    conf_shape: tuple = None


@dataclass
class EncodeTrace:
    """Everything the fused backward needs: the batch's coordinates (the
    backward recomputes corners, hashes and weights on the fly instead of
    storing 2^d x L index/weight arrays).  It still reads like the
    reference's list[LevelTrace]: len() is the level count and indexing or
    iterating materialises a level's LevelTrace (weights, idx / base, row)
    through the per-level protocol kernels, for callers that inspect traces
    (e.g. model_io.py:302-307 counting lookups)."""

    xs: torch.Tensor
    model_id: int
    layout_version: int
    n_levels: int
    feat_shape: tuple
    conf_shape: tuple
    surrogate: bool
    model: object = field(default=None, repr=False, compare=False)

    def __len__(self):  # reference callers check len(traces) == len(levels)
        return self.n_levels

    def __getitem__(self, i) -> LevelTrace:
        from . import backend
        m = self.model
        if m is None:
            raise StaleTrace("trace holds no model to materialise level traces from")
        i = range(self.n_levels)[i]
        spec, lv = m.specs[i], m.levels[i]
        h = m.hyper
        xs = self.xs.cpu().numpy()
        feats = lv.features.values.cpu().numpy()
        fshape = (h.n_f, h.feature_dim) if spec.mode is not LevelMode.DENSE else \
            ((spec.resolution + 1) ** h.d, h.feature_dim)
        if spec.mode is LevelMode.DENSE:
            _, idx, w = backend.dense_fwd(xs, spec.resolution, feats[:fshape[0]])
            return LevelTrace("dense", w, idx=idx, feat_shape=fshape)
        if lv.conf is None:
            _, idx, w = backend.hashed_fwd(xs, spec.resolution, h.n_f, feats, PRIMARY_PRIMES)
            return LevelTrace("hashed", w, idx=idx, feat_shape=fshape)
        _, base, row, w = backend.probed_fwd(xs, spec.resolution, h.n_f, h.n_c, h.n_p.bit_length() - 1, feats,
                                             lv.baked.entries.cpu().numpy(), PRIMARY_PRIMES, AUX_PRIMES)
        return LevelTrace("probed", w, base=base, row=row, feat_shape=fshape,
                          conf_shape=(h.n_c, h.n_p))

    def __iter__(self):
        return (self[i] for i in range(self.n_levels))


def _sfx(model):
    return "f64" if model.tdtype == torch.float64 else "f32"


def _prepare_xs(model: Model, xs, check_domain: bool):
    d = model.hyper.d
    if isinstance(xs, torch.Tensor):
        t = xs.to(device=model.device, dtype=model.tdtype).contiguous()
        if t.ndim != 2 or t.shape[1] != d:
            raise DomainViolation(f"expected (batch, {d}) coordinates, got {tuple(t.shape)}")
        return t, False
    a = np.ascontiguousarray(np.asarray(xs).astype(model.dtype, copy=False))
    if a.ndim != 2 or a.shape[1] != d:
        raise DomainViolation(f"expected (batch, {d}) coordinates, got {a.shape}")
    if check_domain and (np.any(a < 0.0) or np.any(a > 1.0)):
        raise DomainViolation("coordinates outside the unit hypercube")
    return torch.from_numpy(a).to(model.device), True


@on_device
def encode_forward_device(model: Model, xs: torch.Tensor, y: torch.Tensor = None,
                          surrogate: bool = False, bad: torch.Tensor = None, stream=None):
    """Launch the fused forward on device tensors; returns y (B, L*F)."""
    h = model.hyper
    B = xs.shape[0]
    if y is None:
        y = torch.empty((B, h.encoded_width), dtype=model.tdtype, device=model.device)
    flags = _lib.PG_SURROGATE if surrogate else 0
    _lib.call(f"pg_encode_fwd_{_sfx(model)}", model.grid, _lib.ptr(xs), B, _lib.ptr(model.feats),
              _lib.ptr(model.baked), _lib.ptr(model.conf), flags, _lib.ptr(y), _lib.ptr(bad),
              _lib.stream_ptr(stream))
    return y


@on_device
def encode_backward_device(model: Model, xs: torch.Tensor, dy: torch.Tensor, stream=None,
                           deterministic: bool = False, flush: bool = True):
    """Launch the fused backward: accumulate into model.grads / touched.
    deterministic=True accumulates in fixed point (run-to-run identical);
    flush=False leaves the sums in model.grads_fx for the caller to flush."""
    if deterministic:
        if model.tdtype != torch.float32:
            raise ValueError("deterministic mode is float32-only")
        gf, _, gc = model.fx_ptrs()
        _lib.call("pg_encode_bwd_det_f32", model.grid, _lib.ptr(xs), xs.shape[0], _lib.ptr(dy),
                  _lib.ptr(model.feats), _lib.ptr(model.conf), gf, gc, _lib.ptr(model.touched),
                  _lib.stream_ptr(stream))
        if flush:
            model.fx_flush(stream=stream)
        return
    _lib.call(f"pg_encode_bwd_{_sfx(model)}", model.grid, _lib.ptr(xs), xs.shape[0], _lib.ptr(dy),
              _lib.ptr(model.feats), _lib.ptr(model.conf), _lib.ptr(model.gfeats),
              _lib.ptr(model.gconf), _lib.ptr(model.touched), _lib.stream_ptr(stream))


@on_device
def encode_forward(model: Model, xs, surrogate: bool = False):
    """Encode a batch; returns (features (B, L*F), trace).

    ``surrogate=True`` blends the softmax mixture over the probing range
    instead of the argmax probe (gradient checks only, encoding.py:45-47)."""
    t, was_numpy = _prepare_xs(model, xs, check_domain=True)
    bad = None
    if not was_numpy:
        bad = torch.zeros(1, dtype=torch.int32, device=model.device)
    y = encode_forward_device(model, t, surrogate=surrogate, bad=bad)
    if bad is not None and int(bad.item()):
        raise DomainViolation("coordinates outside the unit hypercube")
    trace = EncodeTrace(t, id(model), model.layout_version, model.hyper.n_levels,
                        tuple(model.feats.shape), tuple(model.conf.shape), surrogate, model)
    return (y.cpu().numpy() if was_numpy else y), trace


@on_device
def encode_backward(model: Model, trace: EncodeTrace, upstream, deterministic: bool = False) -> None:
    """Accumulate codebook gradients from an encoded batch (encoding.py:119-133).
    deterministic=True: order-independent fixed-point accumulation (float32)."""
    if not isinstance(trace, EncodeTrace) or len(trace) != len(model.levels):
        raise StaleTrace("trace level count does not match the model")
    if trace.model_id != id(model) or trace.layout_version != model.layout_version:
        raise StaleTrace("trace recorded against other tables")
    if trace.feat_shape != tuple(model.feats.shape) or trace.conf_shape != tuple(model.conf.shape):
        raise StaleTrace("codebook shapes changed since the forward pass")
    if isinstance(upstream, torch.Tensor):
        dy = upstream.to(device=model.device, dtype=model.tdtype).contiguous()
    else:
        dy = torch.from_numpy(np.ascontiguousarray(upstream, dtype=model.dtype)).to(model.device)
    if tuple(dy.shape) != (trace.xs.shape[0], model.hyper.encoded_width):
        raise StaleTrace(f"upstream shape {tuple(dy.shape)} does not match the trace")
    encode_backward_device(model, trace.xs, dy, deterministic=deterministic)
