"""TEST INFRASTRUCTURE ONLY — CPU oracle for the learned-hash-probing hot path.

Restates the reference package ``probegrid`` (``/root/reference/pkg``) for the
path named in BASELINE.json: multiresolution probed hash-grid encoding
(forward + straight-through backward), the MLP it feeds, the training step
and random-access decode.  The compiled kernels come from ``pg_oracle.c``
(a C restatement of ``backends/_core.pyx``, built by ``oracle/Makefile``);
everything around them is numpy, in the same operation order as the
reference so results agree bit for bit on the same machine.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline
leg may import this module, and only as the checker.  The product package
(``paper_2312_17241_b200``) never imports it.

Parity is pinned two ways (see tests/test_oracle.py):
  * golden vectors produced by the real reference (tests/golden/make_golden.py);
  * the reference's own Cython core compiled into ``oracle/_ref`` (build_ref.sh),
    used live through :func:`reference_core_backend`.
"""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import math
import os
from dataclasses import dataclass, field, replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

# --------------------------------------------------------------------------
# hash constants and the level ladder — indexing.py:22-23, 66-101
# --------------------------------------------------------------------------
PRIMARY = (1, 2654435761, 805459861)
AUX = (1, 3674653429, 2097192037)
SEED_FEATURES, SEED_CONFIDENCE, SEED_MLP, SEED_BATCH = 0, 1, 2, 3  # model.py:21-24


def level_resolution(level, n_min, n_max, n_levels):
    """indexing.py:66-90: floor(n_min * b^level), endpoints exact, 1e-9 guard."""
    if n_levels == 1 or level == 0:
        return n_min
    if level == n_levels - 1:
        return n_max
    growth = (math.log(n_max) - math.log(n_min)) / (n_levels - 1)
    val = n_min * math.exp(level * growth)
    r = math.floor(val)
    if val - r > 1.0 - 1e-9:
        r += 1
    return r


def level_ladder(h):
    """indexing.py:93-101: (resolution, dense?) per level."""
    out = []
    for lv in range(h.n_levels):
        res = level_resolution(lv, h.n_min, h.n_max, h.n_levels)
        out.append((res, (res + 1) ** h.d <= h.n_f))
    return out


def log2i(n):
    return int(n).bit_length() - 1


# --------------------------------------------------------------------------
# C kernels (pg_oracle.c) under the reference backend protocol
# (backends/cython_backend.py:24-89)
# --------------------------------------------------------------------------
_P = ctypes.c_void_p
_I64, _I32, _U32, _D = ctypes.c_int64, ctypes.c_int, ctypes.c_uint32, ctypes.c_double


def _ptr(a):
    return a.ctypes.data_as(_P)


def _load_orc():
    path = os.path.join(HERE, "liborc.so")
    if not os.path.exists(path):
        import subprocess
        subprocess.run(["make", "-s", "-C", HERE, "liborc.so"], check=True)
    lib = ctypes.CDLL(path)
    for sfx in ("f32", "f64"):
        getattr(lib, f"orc_dense_fwd_{sfx}").argtypes = [_P, _I64, _I32, ctypes.c_long, _P, _I32, _P, _P, _P]
        getattr(lib, f"orc_hashed_fwd_{sfx}").argtypes = [_P, _I64, _I32, ctypes.c_long, _U32, _P, _I32, _P, _P, _P, _P]
        getattr(lib, f"orc_probed_fwd_{sfx}").argtypes = [_P, _I64, _I32, ctypes.c_long, _U32, _U32, _I32, _P, _I32, _P, _P, _P, _P, _P, _P, _P]
        getattr(lib, f"orc_indexed_bwd_{sfx}").argtypes = [_P, _I64, _I32, _P, _P, _I32, _P]
        getattr(lib, f"orc_probed_bwd_{sfx}").argtypes = [_P, _I64, _I32, _P, _P, _P, _I32, _P, _I32, _P, _P, _P]
        getattr(lib, f"orc_adam_rebake_rows_{sfx}").argtypes = [_P, _P, _P, _I32, _P, _P, _I64, _P, _D, _D, _D, _D, _D, _D]
        getattr(lib, f"orc_linear_rows_{sfx}").argtypes = [_P, _I64, _I32, _P, _P, _I32, _P, _I32]
        getattr(lib, f"orc_sigmoid_rows_{sfx}").argtypes = [_P, _I64]
    lib.orc_dedup_rows.argtypes = [_P, _I64, _P, _I64, _P, _P]
    lib.orc_dedup_rows.restype = _I64
    lib.orc_wgrad_blas_f32.argtypes = [_P, _I64, _I32, _P, _I32, _P, _P]
    return lib


_ORC = None


def _orc():
    global _ORC
    if _ORC is None:
        _ORC = _load_orc()
    return _ORC


def _sfx(dtype):
    return "f64" if np.dtype(dtype) == np.float64 else "f32"


def _c(a, dtype=None):
    return np.ascontiguousarray(a, dtype=dtype)


def wgrad_blas(a, delta, gw, gb):
    """gw += a.T @ delta and gb += delta.sum(0) in numpy/OpenBLAS order
    (orc_wgrad_blas_f32; float32 only), in place."""
    a, delta = _c(a, np.float32), _c(delta, np.float32)
    assert gw.flags.c_contiguous and gb.flags.c_contiguous and gw.dtype == np.float32
    _orc().orc_wgrad_blas_f32(_ptr(a), a.shape[0], a.shape[1], _ptr(delta), delta.shape[1],
                              _ptr(gw), _ptr(gb))


class CBackend:
    """The oracle's kernels behind the reference backend protocol."""

    NAME = "oracle-c"

    @staticmethod
    def dense_fwd(xs, resolution, feats):
        xs = _c(xs)
        feats = _c(feats, xs.dtype)
        b, d = xs.shape
        out = np.zeros((b, feats.shape[1]), xs.dtype)
        idx = np.empty((b, 1 << d), np.int32)
        w = np.empty((b, 1 << d), xs.dtype)
        getattr(_orc(), f"orc_dense_fwd_{_sfx(xs.dtype)}")(
            _ptr(xs), b, d, resolution, _ptr(feats), feats.shape[1], _ptr(out), _ptr(idx), _ptr(w))
        return out, idx, w

    @staticmethod
    def hashed_fwd(xs, resolution, n_f, feats, primary):
        xs = _c(xs)
        feats = _c(feats, xs.dtype)
        b, d = xs.shape
        pr = np.asarray(primary[:d], np.uint32)
        out = np.zeros((b, feats.shape[1]), xs.dtype)
        idx = np.empty((b, 1 << d), np.int32)
        w = np.empty((b, 1 << d), xs.dtype)
        getattr(_orc(), f"orc_hashed_fwd_{_sfx(xs.dtype)}")(
            _ptr(xs), b, d, resolution, n_f - 1, _ptr(feats), feats.shape[1], _ptr(pr),
            _ptr(out), _ptr(idx), _ptr(w))
        return out, idx, w

    @staticmethod
    def probed_fwd(xs, resolution, n_f, n_c, log2_np, feats, baked, primary, aux):
        xs = _c(xs)
        feats = _c(feats, xs.dtype)
        baked = _c(baked, np.uint8)
        b, d = xs.shape
        pr = np.asarray(primary[:d], np.uint32)
        ax = np.asarray(aux[:d], np.uint32)
        out = np.zeros((b, feats.shape[1]), xs.dtype)
        base = np.empty((b, 1 << d), np.int32)
        row = np.empty((b, 1 << d), np.int32)
        w = np.empty((b, 1 << d), xs.dtype)
        getattr(_orc(), f"orc_probed_fwd_{_sfx(xs.dtype)}")(
            _ptr(xs), b, d, resolution, n_f - 1, n_c - 1, log2_np, _ptr(feats), feats.shape[1],
            _ptr(baked), _ptr(pr), _ptr(ax), _ptr(out), _ptr(base), _ptr(row), _ptr(w))
        return out, base, row, w

    @staticmethod
    def indexed_bwd(upstream, idx, weights, gfeat):
        up = _c(upstream, gfeat.dtype)
        idx = _c(idx, np.int32)
        w = _c(weights, gfeat.dtype)
        assert gfeat.flags.c_contiguous
        getattr(_orc(), f"orc_indexed_bwd_{_sfx(gfeat.dtype)}")(
            _ptr(up), up.shape[0], up.shape[1], _ptr(idx), _ptr(w), idx.shape[1], _ptr(gfeat))

    @staticmethod
    def dedup_rows(row, n_c):
        row = _c(row, np.int32)
        mark = np.empty(n_c, np.int32)
        rows_u = np.empty(row.size, np.int32)
        inv = np.empty(row.shape, np.int32)
        u = _orc().orc_dedup_rows(_ptr(row), row.size, _ptr(mark), n_c, _ptr(rows_u), _ptr(inv))
        return rows_u[:u].copy(), inv

    @staticmethod
    def probed_bwd(upstream, base, inv, weights, smu, feats, gfeat, gconf_u):
        dt = gfeat.dtype
        up = _c(upstream, dt)
        base = _c(base, np.int32)
        inv = _c(inv, np.int32)
        w = _c(weights, dt)
        smu = _c(smu, dt)
        feats = _c(feats, dt)
        if feats.shape[1] > 16 or smu.shape[1] > 256:  # cython_backend.py:17-21
            raise ValueError("feature dim / probing range beyond compiled limit")
        assert gfeat.flags.c_contiguous and gconf_u.flags.c_contiguous
        getattr(_orc(), f"orc_probed_bwd_{_sfx(dt)}")(
            _ptr(up), up.shape[0], up.shape[1], _ptr(base), _ptr(inv), _ptr(w), base.shape[1],
            _ptr(smu), smu.shape[1], _ptr(feats), _ptr(gfeat), _ptr(gconf_u))

    @staticmethod
    def adam_rebake_rows(conf, m, v, baked, rows_u, gconf_u, t, lr, beta1, beta2, eps):
        rows_u = _c(rows_u, np.int32)
        g = _c(gconf_u, conf.dtype)
        getattr(_orc(), f"orc_adam_rebake_rows_{_sfx(conf.dtype)}")(
            _ptr(conf), _ptr(m), _ptr(v), conf.shape[1], _ptr(baked), _ptr(rows_u), rows_u.size,
            _ptr(g), 1.0 - beta1 ** t, 1.0 - beta2 ** t, lr, beta1, beta2, eps)

    @staticmethod
    def mlp_infer_rows(xs, weights, biases, out_sigmoid=False):
        a = _c(xs)
        n = len(weights)
        for li in range(n):
            w = _c(weights[li], a.dtype)
            bb = _c(biases[li], a.dtype)
            out = np.empty((a.shape[0], w.shape[1]), a.dtype)
            getattr(_orc(), f"orc_linear_rows_{_sfx(a.dtype)}")(
                _ptr(a), a.shape[0], w.shape[0], _ptr(w), _ptr(bb), w.shape[1], _ptr(out),
                1 if li < n - 1 else 0)
            a = out
        if out_sigmoid:
            getattr(_orc(), f"orc_sigmoid_rows_{_sfx(a.dtype)}")(_ptr(a), a.size)
        return a


def reference_core_path():
    hits = sorted(glob.glob(os.path.join(HERE, "_ref", "_core*.so")))
    return hits[0] if hits else None


class _RefCoreBackend:
    """The reference's own compiled Cython kernels (oracle/_ref, built from
    /root/reference by build_ref.sh) wrapped exactly as cython_backend.py:24-89
    wraps them.  Used to pin the C restatement and as the reference CPU arm."""

    NAME = "reference-cython"

    def __init__(self, core):
        self.core = core

    def dense_fwd(self, xs, resolution, feats):
        b, d = xs.shape
        out = np.zeros((b, feats.shape[1]), xs.dtype)
        idx = np.empty((b, 1 << d), np.int32)
        w = np.empty((b, 1 << d), xs.dtype)
        self.core.dense_fwd(xs, resolution, feats, out, idx, w)
        return out, idx, w

    def hashed_fwd(self, xs, resolution, n_f, feats, primary):
        b, d = xs.shape
        out = np.zeros((b, feats.shape[1]), xs.dtype)
        idx = np.empty((b, 1 << d), np.int32)
        w = np.empty((b, 1 << d), xs.dtype)
        self.core.hashed_fwd(xs, resolution, np.uint32(n_f - 1), feats,
                             np.asarray(primary[:d], np.uint32), out, idx, w)
        return out, idx, w

    def probed_fwd(self, xs, resolution, n_f, n_c, log2_np, feats, baked, primary, aux):
        b, d = xs.shape
        out = np.zeros((b, feats.shape[1]), xs.dtype)
        base = np.empty((b, 1 << d), np.int32)
        row = np.empty((b, 1 << d), np.int32)
        w = np.empty((b, 1 << d), xs.dtype)
        self.core.probed_fwd(xs, resolution, np.uint32(n_f - 1), np.uint32(n_c - 1), log2_np,
                             feats, baked, np.asarray(primary[:d], np.uint32),
                             np.asarray(aux[:d], np.uint32), out, base, row, w)
        return out, base, row, w

    def indexed_bwd(self, upstream, idx, weights, gfeat):
        self.core.indexed_bwd(upstream, idx, weights, gfeat)

    def dedup_rows(self, row, n_c):
        return self.core.dedup_rows(np.ascontiguousarray(row), n_c)

    def probed_bwd(self, upstream, base, inv, weights, smu, feats, gfeat, gconf_u):
        self.core.probed_bwd(upstream, base, inv, weights, np.ascontiguousarray(smu),
                             feats, gfeat, gconf_u)

    def adam_rebake_rows(self, conf, m, v, baked, rows_u, gconf_u, t, lr, beta1, beta2, eps):
        self.core.adam_rebake_rows(conf, m, v, baked, rows_u, gconf_u, 1.0 - beta1 ** t,
                                   1.0 - beta2 ** t, lr, beta1, beta2, eps)

    def mlp_infer_rows(self, xs, weights, biases, out_sigmoid=False):
        a = np.ascontiguousarray(xs)
        n = len(weights)
        for li in range(n):
            out = np.empty((a.shape[0], weights[li].shape[1]), a.dtype)
            self.core.linear_rows(a, weights[li], biases[li], out, li < n - 1)
            a = out
        if out_sigmoid:
            self.core.sigmoid_rows(a)
        return a


def reference_core_backend():
    """Backend over oracle/_ref's compiled reference core, or None if absent."""
    path = reference_core_path()
    if path is None:
        return None
    spec = importlib.util.spec_from_file_location("_core", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return _RefCoreBackend(mod)


# --------------------------------------------------------------------------
# numpy-only kernels the reference calls directly (numpy_backend.py)
# --------------------------------------------------------------------------
def softmax_rows(c):
    """numpy_backend.py:115-131: shift by the GLOBAL max, exp, divide by
    row sums computed as a mat-vec with ones (same BLAS call, same bits)."""
    z = c - c.max()
    np.exp(z, out=z)
    if z.ndim == 2:
        z /= (z @ np.ones(z.shape[-1], dtype=z.dtype))[:, None]
    else:
        z /= z.sum(axis=-1, keepdims=True)
    return z


def _geometry(xs, res):
    """numpy_backend.py:22-42 — (corners (B,C,d) int64, weights (B,C))."""
    b, d = xs.shape
    scaled = xs * xs.dtype.type(res)
    cell = np.clip(np.floor(scaled), xs.dtype.type(0), xs.dtype.type(res - 1))
    t = scaled - cell
    cell = cell.astype(np.int64)
    n = 1 << d
    corners = np.empty((b, n, d), np.int64)
    w = np.ones((b, n), xs.dtype)
    for k in range(n):
        for i in range(d):
            bit = (k >> (d - 1 - i)) & 1
            corners[:, k, i] = cell[:, i] + bit
            w[:, k] *= t[:, i] if bit else (xs.dtype.type(1.0) - t[:, i])
    return corners, w


def _hash(corners, primes):
    v = corners.astype(np.uint64) & np.uint64(0xFFFFFFFF)
    h = np.zeros(corners.shape[:2], np.uint64)
    for i in range(corners.shape[2]):
        h ^= (v[:, :, i] * np.uint64(primes[i])) & np.uint64(0xFFFFFFFF)
    return h


def probed_fwd_surrogate(xs, res, n_f, n_c, log2_np, feats, conf, primary, aux):
    """numpy_backend.py:94-112 — softmax-mixture forward, for gradient checks."""
    corners, w = _geometry(xs, res)
    h = _hash(corners, primary)
    h2 = _hash(corners, aux)
    base = ((h << np.uint64(log2_np)) & np.uint64(n_f - 1)).astype(np.int32)
    row = (h2 & np.uint64(n_c - 1)).astype(np.int32)
    sm = softmax_rows(conf[row])
    n_p = conf.shape[1]
    probes = base[:, :, None] + np.arange(n_p, dtype=np.int32)
    mixed = np.einsum("bcj,bcjf->bcf", sm, feats[probes])
    return np.einsum("bc,bcf->bf", w, mixed), base, row, w


# --------------------------------------------------------------------------
# model state — model.py:35-158, codebooks.py:87-98, mlp.py:43-52
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Hyper:
    n_f: int = 2**6
    n_c: int = 2**14
    n_p: int = 2**4
    n_levels: int = 16
    feature_dim: int = 2
    n_min: int = 16
    n_max: int = 512
    n_neurons: int = 64
    n_hidden_layers: int = 2
    d: int = 2
    out_dim: int = 3
    out_sigmoid: bool = False

    @property
    def encoded_width(self):
        return self.n_levels * self.feature_dim

    def widths(self):
        return [self.encoded_width] + [self.n_neurons] * self.n_hidden_layers + [self.out_dim]

    def with_updates(self, **kw):
        return replace(self, **kw)


def seeded_rng(seed, domain, index=0):
    """model.py:24-32."""
    return np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(domain, index)))


@dataclass
class Level:
    level: int
    res: int
    dense: bool
    feats: np.ndarray
    fgrad: np.ndarray
    conf: np.ndarray | None = None
    cgrad: np.ndarray | None = None
    baked: np.ndarray | None = None


@dataclass
class OModel:
    hyper: Hyper
    levels: list
    W: list
    b: list
    dtype: np.dtype
    Wg: list = field(default=None)
    bg: list = field(default=None)

    def __post_init__(self):
        if self.Wg is None:
            self.Wg = [np.zeros_like(w) for w in self.W]
            self.bg = [np.zeros_like(x) for x in self.b]


def init_model(h: Hyper, seed=0, dtype=np.float32, force_probed=False) -> OModel:
    """model.py:133-158 with codebooks.py:87-98 and mlp.py:43-52."""
    dtype = np.dtype(dtype)
    levels = []
    for lv, (res, dense) in enumerate(level_ladder(h)):
        f = seeded_rng(seed, SEED_FEATURES, lv).uniform(-1e-4, 1e-4, (h.n_f, h.feature_dim)).astype(dtype)
        L = Level(lv, res, dense, f, np.zeros_like(f))
        if not dense and (h.n_p > 1 or force_probed):
            c = seeded_rng(seed, SEED_CONFIDENCE, lv).uniform(0.0, 1e-2, (h.n_c, h.n_p)).astype(dtype)
            L.conf, L.cgrad = c, np.zeros_like(c)
            L.baked = np.argmax(c, axis=1).astype(np.uint8)
        levels.append(L)
    rng = seeded_rng(seed, SEED_MLP)
    W, B = [], []
    widths = h.widths()
    for fi, fo in zip(widths[:-1], widths[1:]):
        lim = np.sqrt(6.0 / fi)
        W.append(rng.uniform(-lim, lim, size=(fi, fo)).astype(dtype))
        B.append(np.zeros(fo, dtype))
    return OModel(h, levels, W, B, dtype)


# --------------------------------------------------------------------------
# encoding — encoding.py:22-133
# --------------------------------------------------------------------------
@dataclass
class Trace:
    kind: str
    w: np.ndarray
    idx: np.ndarray = None
    base: np.ndarray = None
    row: np.ndarray = None


class OracleDomainError(ValueError):
    pass


def encode_forward(model: OModel, xs, kern=CBackend, surrogate=False):
    """encoding.py:42-86 — per-level dispatch, concat into (B, L*F)."""
    h = model.hyper
    xs = np.ascontiguousarray(np.asarray(xs).astype(model.dtype, copy=False))
    if xs.ndim != 2 or xs.shape[1] != h.d:
        raise OracleDomainError(f"expected (batch, {h.d}) coordinates")
    if np.any(xs < 0.0) or np.any(xs > 1.0):
        raise OracleDomainError("coordinates outside the unit hypercube")
    F = h.feature_dim
    y = np.empty((xs.shape[0], h.n_levels * F), model.dtype)
    traces = []
    for L in model.levels:
        if L.dense:
            out, idx, w = kern.dense_fwd(xs, L.res, L.feats)
            tr = Trace("dense", w, idx=idx)
        elif L.baked is None:
            out, idx, w = kern.hashed_fwd(xs, L.res, h.n_f, L.feats, PRIMARY)
            tr = Trace("hashed", w, idx=idx)
        elif surrogate:
            out, base, row, w = probed_fwd_surrogate(xs, L.res, h.n_f, h.n_c, log2i(h.n_p),
                                                     L.feats, L.conf, PRIMARY, AUX)
            tr = Trace("probed", w, base=base, row=row)
        else:
            out, base, row, w = kern.probed_fwd(xs, L.res, h.n_f, h.n_c, log2i(h.n_p), L.feats,
                                                L.baked, PRIMARY, AUX)
            tr = Trace("probed", w, base=base, row=row)
        y[:, L.level * F:(L.level + 1) * F] = out
        traces.append(tr)
    return y, traces


def _level_up(model, lv, upstream):
    F = model.hyper.feature_dim
    return np.ascontiguousarray(upstream[:, lv * F:(lv + 1) * F], dtype=model.dtype)


def probed_backward_compact(L: Level, tr: Trace, up, kern=CBackend):
    """encoding.py:95-116: dedup touched rows, softmax, scatter."""
    rows_u, inv = kern.dedup_rows(tr.row, L.conf.shape[0])
    smu = softmax_rows(L.conf[rows_u])
    gconf_u = np.zeros_like(smu)
    kern.probed_bwd(up, tr.base, inv, tr.w, smu, L.feats, L.fgrad, gconf_u)
    return rows_u, gconf_u


def encode_backward(model: OModel, traces, upstream, kern=CBackend):
    """encoding.py:119-133."""
    for L, tr in zip(model.levels, traces):
        up = _level_up(model, L.level, upstream)
        if tr.kind == "probed":
            rows_u, gconf_u = probed_backward_compact(L, tr, up, kern)
            L.cgrad[rows_u] += gconf_u
        else:
            kern.indexed_bwd(up, tr.idx, tr.w, L.fgrad)


# --------------------------------------------------------------------------
# MLP — mlp.py:55-85
# --------------------------------------------------------------------------
def mlp_forward(W, B, x):
    acts, pre = [x], []
    a = x
    for li, (w, b) in enumerate(zip(W, B)):
        z = a @ w + b
        pre.append(z)
        a = np.maximum(z, 0) if li < len(W) - 1 else z
        acts.append(a)
    return a, (acts, pre)


def mlp_backward(W, Wg, Bg, cache, upstream):
    acts, pre = cache
    delta = upstream
    for li in range(len(W) - 1, -1, -1):
        Wg[li] += acts[li].T @ delta
        Bg[li] += delta.sum(axis=0)
        if li > 0:
            delta = (delta @ W[li].T) * (pre[li - 1] > 0)
    return delta @ W[0].T


# --------------------------------------------------------------------------
# training step — trainer.py:34-171
# --------------------------------------------------------------------------
@dataclass
class TrainCfg:
    steps: int = 10_000
    batch_size: int = 8192
    lr: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.99
    eps: float = 1e-15
    seed: int = 0


def adam_update(p, g, m, v, t, lr, b1=0.9, b2=0.99, eps=1e-15):
    """trainer.py:73-84 — numpy in-place ops in the reference's order."""
    dt = p.dtype.type
    m *= dt(b1)
    m += dt(1 - b1) * g
    v *= dt(b2)
    v += dt(1 - b2) * (g * g)
    mhat = m / dt(1 - b1 ** t)
    vhat = v / dt(1 - b2 ** t)
    p -= dt(lr) * mhat / (np.sqrt(vhat) + dt(eps))


def sample_pixels(rng, batch, width, height):
    """trainer.py:109-116 (indices only)."""
    return rng.integers(0, width * height, size=batch)


def pixel_coords(pix, width, height, dtype):
    rows, cols = pix // width, pix % width
    return np.stack([(cols + 0.5) / width, (rows + 0.5) / height], axis=1).astype(dtype)


class TrainState:
    """trainer.py:87-171."""

    def __init__(self, model: OModel, image, cfg: TrainCfg, kern=CBackend):
        self.model, self.cfg, self.kern = model, cfg, kern
        self.image = np.ascontiguousarray(image, dtype=model.dtype)
        self.flat = self.image.reshape(-1, image.shape[2])
        self.height, self.width = image.shape[:2]
        self.rng = seeded_rng(cfg.seed, SEED_BATCH)
        self.t = 0
        z = np.zeros_like
        self.mlp_m = [z(a) for a in model.W + model.b]
        self.mlp_v = [z(a) for a in model.W + model.b]
        self.f_m = [z(L.feats) for L in model.levels]
        self.f_v = [z(L.feats) for L in model.levels]
        self.c_m = [z(L.conf) if L.conf is not None else None for L in model.levels]
        self.c_v = [z(L.conf) if L.conf is not None else None for L in model.levels]
        self.last_pix = None

    def sample_batch(self):
        pix = sample_pixels(self.rng, self.cfg.batch_size, self.width, self.height)
        self.last_pix = pix
        return pixel_coords(pix, self.width, self.height, self.model.dtype), self.flat[pix]

    def step(self):
        model, cfg, kern = self.model, self.cfg, self.kern
        xs, targets = self.sample_batch()
        y, traces = encode_forward(model, xs, kern)
        out, cache = mlp_forward(model.W, model.b, y)
        pred = 1.0 / (1.0 + np.exp(-out)) if model.hyper.out_sigmoid else out
        diff = pred - targets
        loss = float(np.mean(diff.astype(np.float64) ** 2))
        if not math.isfinite(loss):
            raise FloatingPointError(f"non-finite loss at step {self.t}")
        dpred = diff * model.dtype.type(2.0 / diff.size)
        dout = dpred * (pred * (1.0 - pred)) if model.hyper.out_sigmoid else dpred
        dy = mlp_backward(model.W, model.Wg, model.bg, cache, dout)
        compacts = []
        for L, tr in zip(model.levels, traces):
            up = _level_up(model, L.level, dy)
            if tr.kind == "probed":
                compacts.append(probed_backward_compact(L, tr, up, kern))
            else:
                kern.indexed_bwd(up, tr.idx, tr.w, L.fgrad)
                compacts.append(None)
        self.t += 1
        params = model.W + model.b
        grads = model.Wg + model.bg
        for p, g, m, v in zip(params, grads, self.mlp_m, self.mlp_v):
            adam_update(p, g, m, v, self.t, cfg.lr, cfg.beta1, cfg.beta2, cfg.eps)
            g[:] = 0
        for i, L in enumerate(model.levels):
            adam_update(L.feats, L.fgrad, self.f_m[i], self.f_v[i], self.t, cfg.lr,
                        cfg.beta1, cfg.beta2, cfg.eps)
            L.fgrad[:] = 0
            if compacts[i] is not None:
                rows_u, gconf_u = compacts[i]
                kern.adam_rebake_rows(L.conf, self.c_m[i], self.c_v[i], L.baked, rows_u, gconf_u,
                                      self.t, cfg.lr, cfg.beta1, cfg.beta2, cfg.eps)
        return loss


# --------------------------------------------------------------------------
# inference — model_io.py:114-147, 292-349
# --------------------------------------------------------------------------
DECODE_CHUNK = 16384


def to_inference(model: OModel) -> OModel:
    """model_io.py:130-147 + _compute_twin 114-127: fp16 RNE downcast of the
    features and MLP, fp32 compute twin; baked copied; no confidences."""
    levels = []
    for L in model.levels:
        f = L.feats.astype(np.float16).astype(np.float32)
        levels.append(Level(L.level, L.res, L.dense, f, np.zeros_like(f),
                            baked=None if L.baked is None else L.baked.copy()))
    W = [w.astype(np.float16).astype(np.float32) for w in model.W]
    B = [b.astype(np.float16).astype(np.float32) for b in model.b]
    return OModel(model.hyper, levels, W, B, np.dtype(np.float32))


def decode_pixels(inf: OModel, xs, kern=CBackend):
    """model_io.py:292-311: chunked encode + row-wise MLP."""
    xs = np.asarray(xs, dtype=np.float32)
    out = np.empty((xs.shape[0], inf.hyper.out_dim), np.float32)
    for lo in range(0, xs.shape[0], DECODE_CHUNK):
        y, _ = encode_forward(inf, xs[lo:lo + DECODE_CHUNK], kern)
        out[lo:lo + DECODE_CHUNK] = kern.mlp_infer_rows(y, inf.W, inf.b, inf.hyper.out_sigmoid)
    return out


def grid_coords(width, height, x0, y0, x1, y1):
    """model_io.py:321-325 pixel centres."""
    cols, rows = np.meshgrid(np.arange(x0, x1), np.arange(y0, y1))
    return np.stack([(cols.ravel() + 0.5) / width, (rows.ravel() + 0.5) / height],
                    axis=1).astype(np.float32)


# --------------------------------------------------------------------------
# volume compositing head.  NOT in the reference (no
# renderer there): this is the definitional restatement the CUDA kernels
# (pg_composite_fwd_f32 / pg_nerf_train_f32) are checked against, itself
# checked by finite differences (tests/test_nerf_oracle.py).  "parity
# unpinned" for this row: no reference outputs exist to pin it to.
# --------------------------------------------------------------------------
def _softplus(x):
    return np.where(x > 20, x, np.log1p(np.exp(np.minimum(x, 20))))


def _logistic(x):
    return 1.0 / (1.0 + np.exp(-x))


def composite_forward(raw, deltas):
    """raw (R, S, 4) = (sigma_raw, r, g, b) per sample, deltas (R, S) ->
    rgb (R, 3), weights (R, S): sigma = softplus, c = logistic,
    alpha = 1 - exp(-sigma delta), T_i = prod_{j<i}(1 - alpha_j)."""
    raw = np.asarray(raw)
    tr = np.exp(-_softplus(raw[..., 0]) * deltas)
    T = np.cumprod(np.concatenate([np.ones_like(tr[:, :1]), tr[:, :-1]], axis=1), axis=1)
    w = T * (1 - tr)
    c = _logistic(raw[..., 1:])
    return (w[..., None] * c).sum(axis=1), w


def composite_backward(raw, deltas, g_rgb):
    """dL/draw (R, S, 4) for dL/drgb = g_rgb (R, 3): dC/dc_i = w_i,
    dC/dsigma_i = delta_i (T_{i+1} c_i - sum_{k>i} w_k c_k)."""
    raw = np.asarray(raw)
    tr = np.exp(-_softplus(raw[..., 0]) * deltas)
    T = np.cumprod(np.concatenate([np.ones_like(tr[:, :1]), tr[:, :-1]], axis=1), axis=1)
    w = T * (1 - tr)
    c = _logistic(raw[..., 1:])
    cg = (c * g_rgb[:, None, :]).sum(-1)                         # c_i . g
    wcg = w * cg
    after = np.cumsum(wcg[:, ::-1], axis=1)[:, ::-1] - wcg       # sum_{k>i} w_k c_k . g
    dsig = deltas * (T * tr * cg - after)
    out = np.empty_like(raw)
    out[..., 0] = dsig * _logistic(raw[..., 0])
    out[..., 1:] = w[..., None] * g_rgb[:, None, :] * c * (1 - c)
    return out


def nerf_step_grads(model: OModel, pts, deltas, target_rgb, n_samples, scale, kern=CBackend):
    """One NeRF-style gradient pass on the numpy side: encode fwd, MLP fwd,
    compositing, loss sum, dL/draw, MLP bwd, encode bwd (accumulates into
    model.W grads / level grads).  Returns (loss_sum, dy)."""
    y, traces = encode_forward(model, pts, kern)
    raw, cache = mlp_forward(model.W, model.b, y)
    R = target_rgb.shape[0]
    rgb, _ = composite_forward(raw.reshape(R, n_samples, 4), deltas.reshape(R, n_samples))
    diff = rgb - target_rgb
    loss = float((diff.astype(np.float64) ** 2).sum())
    draw = composite_backward(raw.reshape(R, n_samples, 4), deltas.reshape(R, n_samples),
                              diff * np.float32(scale)).reshape(-1, 4).astype(raw.dtype)
    dy = mlp_backward(model.W, model.Wg, model.bg, cache, draw)
    encode_backward(model, traces, dy, kern)
    return loss, dy


def ray_samples(origins, dirs, n_samples):
    """Midpoint samples inside [0,1]^3 (slab entry/exit), float32 like the
    kernel: points (R*S, 3) clamped to [0,1], deltas (R*S)."""
    o = np.asarray(origins, np.float32)
    d = np.asarray(dirs, np.float32)
    dd = np.where(np.abs(d) < np.float32(1e-12), np.float32(1e-12), d)
    inv = np.float32(1) / dd
    t0, t1 = (np.float32(0) - o) * inv, (np.float32(1) - o) * inv
    near = np.maximum(np.minimum(t0, t1).max(axis=1), np.float32(0))
    far = np.maximum(t0, t1).min(axis=1)
    hit = far > near
    near, far = np.where(hit, near, 0).astype(np.float32), np.where(hit, far, 0).astype(np.float32)
    step = (far - near) / np.float32(n_samples)
    t = near[:, None] + (np.arange(n_samples, dtype=np.float32) + np.float32(0.5))[None, :] * step[:, None]
    pts = np.clip(o[:, None, :] + t[..., None] * d[:, None, :], 0, 1).astype(np.float32)
    return pts.reshape(-1, 3), np.repeat(step, n_samples)
