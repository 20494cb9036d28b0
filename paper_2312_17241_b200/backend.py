"""The reference backend protocol on B200 kernels (NAME = "cuda").

Same module-level functions, argument meaning, dtypes and in-place semantics
as ``probegrid.backends.cython_backend`` (cython_backend.py:24-89) /
``numpy_backend`` (numpy_backend.py:59-216), so it plugs into the reference's
seam ``probegrid.backends`` (backends/__init__.py:12-50) — e.g. by inserting
this module into ``probegrid.backends._BACKENDS["cuda"]`` and calling
``set_backend("cuda")``.  numpy arrays in, numpy arrays out; every call copies
its operands to the device, runs the sm_100a kernel and copies results back.
The device-resident, fused path for throughput lives in encoding.py /
train.py / decode.py.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .hyper import mlp_struct

NAME = "cuda"

_MAX_FEATURE_DIM = _lib.PG_MAX_FEATURE
_MAX_PROBE_RANGE = _lib.PG_MAX_PROBES


def _dev(a, dtype=None):
    a = np.ascontiguousarray(a, dtype=dtype)
    return torch.from_numpy(a).cuda()


def _sfx(dtype):
    return "f64" if np.dtype(dtype) == np.float64 else "f32"


def _tdtype(dtype):
    return torch.float64 if np.dtype(dtype) == np.float64 else torch.float32


def _primes(p, d):
    arr = (_lib.ctypes.c_uint32 * 3)(*[int(x) for x in p[:d]] + [0] * (3 - d))
    return arr


def _check_dims(F, n_p=1):
    if F > _MAX_FEATURE_DIM:
        raise ValueError(f"feature dim {F} beyond compiled limit")
    if n_p > _MAX_PROBE_RANGE:
        raise ValueError(f"probing range {n_p} beyond compiled limit")


def _fwd_common(xs):
    xs = np.ascontiguousarray(xs)
    b, d = xs.shape
    return xs, b, d, 1 << d


def dense_fwd(xs, resolution, feats):
    xs, b, d, c = _fwd_common(xs)
    F = feats.shape[1]
    _check_dims(F)
    tx, tf = _dev(xs), _dev(feats, xs.dtype)
    out = torch.zeros((b, F), dtype=_tdtype(xs.dtype), device="cuda")
    idx = torch.empty((b, c), dtype=torch.int32, device="cuda")
    w = torch.empty((b, c), dtype=_tdtype(xs.dtype), device="cuda")
    _lib.call(f"pg_dense_fwd_{_sfx(xs.dtype)}", _lib.ptr(tx), b, d, int(resolution), _lib.ptr(tf), F,
              _lib.ptr(out), _lib.ptr(idx), _lib.ptr(w), _lib.stream_ptr())
    return out.cpu().numpy(), idx.cpu().numpy(), w.cpu().numpy()


def hashed_fwd(xs, resolution, n_f, feats, primary):
    xs, b, d, c = _fwd_common(xs)
    F = feats.shape[1]
    _check_dims(F)
    tx, tf = _dev(xs), _dev(feats, xs.dtype)
    out = torch.zeros((b, F), dtype=_tdtype(xs.dtype), device="cuda")
    idx = torch.empty((b, c), dtype=torch.int32, device="cuda")
    w = torch.empty((b, c), dtype=_tdtype(xs.dtype), device="cuda")
    _lib.call(f"pg_hashed_fwd_{_sfx(xs.dtype)}", _lib.ptr(tx), b, d, int(resolution), n_f - 1,
              _lib.ptr(tf), F, _primes(primary, d), _lib.ptr(out), _lib.ptr(idx), _lib.ptr(w),
              _lib.stream_ptr())
    return out.cpu().numpy(), idx.cpu().numpy(), w.cpu().numpy()


def probed_fwd(xs, resolution, n_f, n_c, log2_np, feats, baked, primary, aux):
    xs, b, d, c = _fwd_common(xs)
    F = feats.shape[1]
    _check_dims(F, 1 << log2_np)
    tx, tf, tb = _dev(xs), _dev(feats, xs.dtype), _dev(baked, np.uint8)
    out = torch.zeros((b, F), dtype=_tdtype(xs.dtype), device="cuda")
    base = torch.empty((b, c), dtype=torch.int32, device="cuda")
    row = torch.empty((b, c), dtype=torch.int32, device="cuda")
    w = torch.empty((b, c), dtype=_tdtype(xs.dtype), device="cuda")
    _lib.call(f"pg_probed_fwd_{_sfx(xs.dtype)}", _lib.ptr(tx), b, d, int(resolution), n_f - 1,
              n_c - 1, int(log2_np), _lib.ptr(tf), F, _lib.ptr(tb), _primes(primary, d),
              _primes(aux, d), _lib.ptr(out), _lib.ptr(base), _lib.ptr(row), _lib.ptr(w),
              _lib.stream_ptr())
    return out.cpu().numpy(), base.cpu().numpy(), row.cpu().numpy(), w.cpu().numpy()


def indexed_bwd(upstream, idx, weights, gfeat):
    """gfeat[idx] += w * up, in place on the caller's numpy array."""
    _check_dims(gfeat.shape[1])
    dt = gfeat.dtype
    up, ti, tw, tg = _dev(upstream, dt), _dev(idx, np.int32), _dev(weights, dt), _dev(gfeat)
    _lib.call(f"pg_indexed_bwd_{_sfx(dt)}", _lib.ptr(up), up.shape[0], up.shape[1], _lib.ptr(ti),
              _lib.ptr(tw), ti.shape[1], _lib.ptr(tg), _lib.stream_ptr())
    gfeat[...] = tg.cpu().numpy()


def dedup_rows(row, n_c):
    """Unique rows in first-encounter order + inverse (_core.pyx:140-160)."""
    row = np.ascontiguousarray(row, dtype=np.int32)
    n = row.size
    tr = _dev(row)
    ws = torch.empty(int(_lib.lib().pg_dedup_workspace_bytes(n, n_c)), dtype=torch.uint8, device="cuda")
    rows_u = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    inv = torch.empty(row.shape, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("pg_dedup_rows", _lib.ptr(tr), n, n_c, _lib.ptr(ws), _lib.ptr(rows_u), _lib.ptr(inv),
              _lib.ptr(cnt), _lib.stream_ptr())
    u = int(cnt.item())
    return rows_u[:u].cpu().numpy().copy(), inv.cpu().numpy()


def probed_bwd(upstream, base, inv, weights, smu, feats, gfeat, gconf_u):
    """Straight-through scatter into gfeat / gconf_u, in place."""
    dt = gfeat.dtype
    _check_dims(gfeat.shape[1], smu.shape[1])
    up, tb, ti, tw = _dev(upstream, dt), _dev(base, np.int32), _dev(inv, np.int32), _dev(weights, dt)
    ts, tf, tg, tc = _dev(smu, dt), _dev(feats, dt), _dev(gfeat), _dev(gconf_u)
    _lib.call(f"pg_probed_bwd_{_sfx(dt)}", _lib.ptr(up), up.shape[0], up.shape[1], _lib.ptr(tb),
              _lib.ptr(ti), _lib.ptr(tw), tb.shape[1], _lib.ptr(ts), ts.shape[1], _lib.ptr(tf),
              _lib.ptr(tg), _lib.ptr(tc), _lib.stream_ptr())
    gfeat[...] = tg.cpu().numpy()
    gconf_u[...] = tc.cpu().numpy()


def adam_rebake_rows(conf, m, v, baked, rows_u, gconf_u, t, lr, beta1, beta2, eps):
    """Lazy Adam on rows_u then argmax re-bake, in place (bit-exact with _core)."""
    dt = conf.dtype
    tc, tm, tv, tb = _dev(conf), _dev(m), _dev(v), _dev(baked, np.uint8)
    tr, tg = _dev(rows_u, np.int32), _dev(gconf_u, dt)
    _lib.call(f"pg_adam_rebake_rows_{_sfx(dt)}", _lib.ptr(tc), _lib.ptr(tm), _lib.ptr(tv),
              conf.shape[1], _lib.ptr(tb), _lib.ptr(tr), tr.numel(), _lib.ptr(tg),
              1.0 - beta1 ** t, 1.0 - beta2 ** t, lr, beta1, beta2, eps, _lib.stream_ptr())
    conf[...] = tc.cpu().numpy()
    m[...] = tm.cpu().numpy()
    v[...] = tv.cpu().numpy()
    baked[...] = tb.cpu().numpy()


def mlp_infer_rows(xs, weights, biases, out_sigmoid=False):
    """Row-independent MLP inference, reference operation order (bit-exact)."""
    xs = np.ascontiguousarray(xs)
    dt = xs.dtype
    widths = [weights[0].shape[0]] + [w.shape[1] for w in weights]
    flat = np.concatenate([np.concatenate([np.asarray(w, dt).ravel(), np.asarray(b, dt).ravel()])
                           for w, b in zip(weights, biases)])
    tx, tp = _dev(xs), _dev(flat)
    b = xs.shape[0]
    ws = torch.empty(max(1, 2 * b * max(widths)), dtype=_tdtype(dt), device="cuda")
    out = torch.empty((b, widths[-1]), dtype=_tdtype(dt), device="cuda")
    flags = _lib.PG_EXACT_MLP | (_lib.PG_SIGMOID if out_sigmoid else 0)
    _lib.call(f"pg_mlp_infer_rows_{_sfx(dt)}", _lib.ptr(tx), b, mlp_struct(widths), _lib.ptr(tp),
              flags, _lib.ptr(ws), _lib.ptr(out), _lib.stream_ptr())
    return out.cpu().numpy()
