"""Device-resident model state (the reference's Model / LevelState /
codebooks / MlpParams, model.py:90-158, codebooks.py:24-98, mlp.py:16-52).

HBM layout — one allocation per role so each optimizer pass is one launch and
the data-parallel gradient exchange is one buffer:

    dense   [ feats (L, n_f, F) | mlp (W0, b0, W1, b1, ...) ]      float32/64
    grads   [ gfeats | gmlp | pad | gconf (P, n_c, N_p) | pad | touched-as-float (P*n_c) ]
    conf    (P, n_c, N_p)  confidences of the P probed levels, slot order
    baked   (P, n_c)       uint8 argmax probe per row
    touched (P*n_c)        uint8 rows looked up since the last optimizer step

``model.levels[i].features.values`` etc. are torch views into these buffers,
so code written against the reference's attribute paths keeps working (with
device tensors instead of numpy arrays).  ``init_model`` draws every initial
value on the host from the reference's seeded numpy streams
(model.py:24-32, 133-158) and uploads it, so a seed gives the reference's
exact starting point.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import on_device
from .hyper import (SEED_CONFIDENCE, SEED_FEATURES, SEED_MLP, HyperParams, LevelMode, LevelSpec,
                    build_level_specs, grid_struct, mlp_struct, seeded_rng)


class Codebook:
    """A level's table (codebooks.py:24-84 attribute paths) as views into the
    model's device buffers.  Assigning ``values`` / ``grads`` uploads into the
    device table when the shape matches (the reference swaps the array, same
    contents); a different shape cannot live in the fixed device layout, so
    the tables are kept and the model's layout version moves on: traces
    recorded before then raise StaleTrace in encode_backward, as the
    reference's shape check does (encoding.py:122-127)."""

    def __init__(self, values: torch.Tensor, grads: torch.Tensor | None = None, owner=None):
        self._values, self._grads, self._owner = values, grads, owner

    def _assign(self, dst, src):
        src_t = src if isinstance(src, torch.Tensor) else torch.as_tensor(np.asarray(src))
        if tuple(src_t.shape) == tuple(dst.shape):
            with torch.no_grad():
                dst.copy_(src_t.to(device=dst.device, dtype=dst.dtype))
        elif self._owner is not None:
            self._owner.layout_version += 1

    @property
    def values(self) -> torch.Tensor:
        return self._values

    @values.setter
    def values(self, v) -> None:
        self._assign(self._values, v)

    @property
    def grads(self) -> torch.Tensor | None:
        return self._grads

    @grads.setter
    def grads(self, v) -> None:
        self._assign(self._grads, v)


@dataclass
class BakedView:
    entries: torch.Tensor


@dataclass
class LevelState:
    spec: LevelSpec
    features: Codebook
    conf: Codebook | None = None
    baked: BakedView | None = None

    @property
    def probing(self) -> bool:
        return self.conf is not None


@dataclass
class MlpView:
    weights: list
    biases: list
    weight_grads: list
    bias_grads: list

    @property
    def widths(self):
        return [self.weights[0].shape[0]] + [w.shape[1] for w in self.weights]

    def param_count(self) -> int:
        return sum(w.numel() for w in self.weights) + sum(b.numel() for b in self.biases)


def _tdt(dtype):
    return torch.float64 if np.dtype(dtype) == np.float64 else torch.float32


class Model:
    """All trainable state of one probed multiresolution grid + decoder, on one GPU."""

    def __init__(self, hyper: HyperParams, dtype=np.float32, seed: int = 0,
                 force_probed: bool = False, device=None):
        hyper.validate()
        self.hyper = hyper
        self.dtype = np.dtype(dtype)
        self.tdtype = _tdt(dtype)
        self.seed = seed
        self.probing_forced = force_probed
        self.device = torch.device(device or "cuda")
        self.specs = build_level_specs(hyper.n_min, hyper.n_max, hyper.n_levels, hyper.n_f, hyper.d)
        self.probed = [s.level for s in self.specs
                       if s.mode is LevelMode.HASHED and (hyper.n_p > 1 or force_probed)]
        self.grid = grid_struct(hyper, self.specs, self.probed)
        self.widths = hyper.mlp_widths()
        self.mlp_desc = mlp_struct(self.widths)
        h = hyper
        L, F, P = h.n_levels, h.feature_dim, len(self.probed)
        self.n_feat = L * h.n_f * F
        self.n_mlp = sum(a * b + b for a, b in zip(self.widths[:-1], self.widths[1:]))
        self.n_dense = self.n_feat + self.n_mlp
        self.n_conf = P * h.n_c * h.n_p
        self.n_rows = P * h.n_c
        # section starts padded to 64 elements: the scatter kernels issue
        # 16-byte vector reductions into gconf rows (red.global.add.v4.f32)
        self.off_gconf = -(-self.n_dense // 64) * 64
        self.off_touched = -(-(self.off_gconf + self.n_conf) // 64) * 64
        kw = dict(dtype=self.tdtype, device=self.device)
        self.dense = torch.zeros(self.n_dense, **kw)
        # + 1 trailing slot: the step's loss sum rides in the same all-reduce
        self.grads = torch.zeros(self.off_touched + self.n_rows + 1, **kw)
        self.conf = torch.zeros((P, h.n_c, h.n_p), **kw)
        self.baked = torch.zeros((P, h.n_c), dtype=torch.uint8, device=self.device)
        self.touched = torch.zeros(self.n_rows, dtype=torch.uint8, device=self.device)
        self.layout_version = 0
        self._build_views()

    # -- views ---------------------------------------------------------------
    @property
    def feats(self):
        h = self.hyper
        return self.dense[:self.n_feat].view(h.n_levels, h.n_f, h.feature_dim)

    @property
    def mlp_params(self):
        return self.dense[self.n_feat:]

    @property
    def gdense(self):
        return self.grads[:self.n_dense]

    @property
    def gfeats(self):
        h = self.hyper
        return self.grads[:self.n_feat].view(h.n_levels, h.n_f, h.feature_dim)

    @property
    def gmlp(self):
        return self.grads[self.n_feat:self.n_dense]

    @property
    def gconf(self):
        h = self.hyper
        return self.grads[self.off_gconf:self.off_gconf + self.n_conf].view(len(self.probed), h.n_c, h.n_p)

    @property
    def touched_f(self):
        return self.grads[self.off_touched:self.off_touched + self.n_rows]

    @property
    def loss_slot(self):
        return self.grads[self.off_touched + self.n_rows:]

    def _mlp_views(self, flat):
        out_w, out_b, off = [], [], 0
        for a, b in zip(self.widths[:-1], self.widths[1:]):
            out_w.append(flat[off:off + a * b].view(a, b))
            off += a * b
            out_b.append(flat[off:off + b])
            off += b
        return out_w, out_b

    def _build_views(self):
        feats, gfeats = self.feats, self.gfeats
        slot = {lv: i for i, lv in enumerate(self.probed)}
        self.levels = []
        for s in self.specs:
            lv = LevelState(spec=s, features=Codebook(feats[s.level], gfeats[s.level], self))
            if s.level in slot:
                i = slot[s.level]
                lv.conf = Codebook(self.conf[i], self.gconf[i], self)
                lv.baked = BakedView(self.baked[i])
            self.levels.append(lv)
        w, b = self._mlp_views(self.mlp_params)
        gw, gb = self._mlp_views(self.gmlp)
        self.mlp = MlpView(w, b, gw, gb)

    # -- deterministic mode: 64-bit fixed-point accumulators ------------------
    @property
    def grads_fx(self):
        """uint64 accumulators laid out like `grads` (deterministic mode)."""
        if getattr(self, "_grads_fx", None) is None:
            self._grads_fx = torch.zeros(self.off_gconf + self.n_conf, dtype=torch.int64,
                                         device=self.device)
            self._loss_fx = torch.zeros(1, dtype=torch.int64, device=self.device)
        return self._grads_fx

    @property
    def loss_fx(self):
        self.grads_fx  # noqa: B018 (allocates both)
        return self._loss_fx

    def fx_ptrs(self):
        """(gfeat_fx, gmlp_fx, gconf_fx) device pointers into grads_fx."""
        base = self.grads_fx.data_ptr()
        return (_lib.ctypes.c_void_p(base), _lib.ctypes.c_void_p(base + 8 * self.n_feat),
                _lib.ctypes.c_void_p(base + 8 * self.off_gconf))

    @on_device
    def fx_flush(self, loss_sum=None, stream=None) -> None:
        """Add the fixed-point accumulators into the float gradients (and the
        loss into loss_sum), clearing them."""
        s = _lib.stream_ptr(stream)
        _lib.call("pg_fx_accumulate_f32", _lib.ptr(self.grads_fx), self.grads_fx.numel(),
                  _lib.ptr(self.grads), s)
        if loss_sum is not None:
            _lib.call("pg_fx_loss", _lib.ptr(self.loss_fx), _lib.ptr(loss_sum), s)

    # -- reference Model methods (model.py:108-130) -------------------------
    def zero_grads(self) -> None:
        self.grads.zero_()
        self.touched.zero_()

    def parameter_count(self) -> int:
        return self.n_dense + self.n_conf

    def rebake_all(self) -> None:
        """Full argmax bake of every probed level (codebooks.py:147-152; ties
        to the smallest probe like the strict '>' scan)."""
        if self.probed:
            self.bake_into(self.baked)

    @on_device
    def bake_into(self, out: torch.Tensor) -> torch.Tensor:
        """np.argmax of every confidence row (codebooks.py:151-152) into `out`
        (P, n_c) uint8, on the device."""
        sfx = "f64" if self.tdtype == torch.float64 else "f32"
        _lib.call(f"pg_bake_rows_{sfx}", _lib.ptr(self.conf), self.n_rows, self.hyper.n_p,
                  _lib.ptr(out), _lib.stream_ptr())
        return out

    # -- host interchange (parity tests, checkpoints) ------------------------
    @on_device
    def load_host(self, feats, conf=None, weights=None, biases=None, baked=None) -> "Model":
        """Upload per-level numpy tables (lists indexed by level / slot)."""
        with torch.no_grad():
            for lv, f in enumerate(feats):
                self.feats[lv].copy_(torch.as_tensor(np.asarray(f, self.dtype)))
            if conf is not None:
                for i, lv in enumerate(self.probed):
                    self.conf[i].copy_(torch.as_tensor(np.asarray(conf[lv], self.dtype)))
            if weights is not None:
                for dst, src in zip(self.mlp.weights, weights):
                    dst.copy_(torch.as_tensor(np.asarray(src, self.dtype)))
                for dst, src in zip(self.mlp.biases, biases):
                    dst.copy_(torch.as_tensor(np.asarray(src, self.dtype)))
            if baked is not None:
                for i, lv in enumerate(self.probed):
                    self.baked[i].copy_(torch.as_tensor(np.asarray(baked[lv], np.uint8)))
            elif conf is not None:
                self.rebake_all()
        return self

    @on_device
    def to_host(self) -> dict:
        """numpy copies keyed like the reference's attribute paths."""
        feats = self.feats.cpu().numpy()
        conf = self.conf.cpu().numpy()
        baked = self.baked.cpu().numpy()
        out = {"feats": [feats[i] for i in range(self.hyper.n_levels)],
               "conf": {lv: conf[i] for i, lv in enumerate(self.probed)},
               "baked": {lv: baked[i] for i, lv in enumerate(self.probed)},
               "W": [w.cpu().numpy() for w in self.mlp.weights],
               "b": [b.cpu().numpy() for b in self.mlp.biases]}
        return out


def host_init_arrays(hyper: HyperParams, seed: int, dtype, probed):
    """The reference's initial values (codebooks.py:87-98, mlp.py:43-52,
    model.py:133-158), drawn from the same seeded streams."""
    dtype = np.dtype(dtype)
    feats, conf = [], {}
    for lv in range(hyper.n_levels):
        rng = seeded_rng(seed, SEED_FEATURES, lv)
        feats.append(rng.uniform(-1e-4, 1e-4, size=(hyper.n_f, hyper.feature_dim)).astype(dtype))
        if lv in probed:
            rc = seeded_rng(seed, SEED_CONFIDENCE, lv)
            conf[lv] = rc.uniform(0.0, 1e-2, size=(hyper.n_c, hyper.n_p)).astype(dtype)
    rng = seeded_rng(seed, SEED_MLP)
    W, B = [], []
    widths = hyper.mlp_widths()
    for fi, fo in zip(widths[:-1], widths[1:]):
        lim = np.sqrt(6.0 / fi)
        W.append(rng.uniform(-lim, lim, size=(fi, fo)).astype(dtype))
        B.append(np.zeros(fo, dtype))
    return feats, conf, W, B


def init_model(hyper: HyperParams, seed: int = 0, dtype=np.float32, force_probed: bool = False,
               device=None) -> Model:
    """Fresh device model with the reference's initial values (model.py:133-158)."""
    m = Model(hyper, dtype, seed, force_probed, device)
    feats, conf, W, B = host_init_arrays(hyper, seed, dtype, set(m.probed))
    return m.load_host(feats, conf, W, B)
