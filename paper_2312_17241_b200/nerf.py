"""NeRF-style density/colour head with volume compositing (SURVEY 8f row 4,
config C4).  The reference stops at per-point fields (its trainer is
image-only, trainer.py:92-95) and has no renderer, so this row has no
reference to pin against: the tests check it against a numpy restatement of
the compositing equations (test infrastructure, not imported here) and
finite differences.

Rays through the unit cube [0,1]^3 (the grid's domain) are sampled at S
midpoints between the box entry and exit; the 3-D learned-hash-probing
encoding + MLP (out_dim 4) gives per-sample (sigma_raw, r, g, b); the
compositing kernel (pg_composite_fwd_f32 / pg_nerf_train_f32) renders
rgb = sum_i T_i alpha_i c_i with sigma = softplus(sigma_raw),
c = logistic(rgb_raw), alpha_i = 1 - exp(-sigma_i delta_i).

Training step on R rays: sample points (device) -> encode fwd
(pg_encode_fwd_f32) -> MLP fwd + compositing + loss + compositing bwd + MLP
bwd (pg_nerf_train_f32, one call) -> encode bwd (pg_encode_bwd_f32) -> dense
Adam + lazy Adam / re-bake — the same optimizer path as TrainState.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import on_device
from .encoding import encode_backward_device, encode_forward_device
from .errors import InvalidHyperparameter
from .grid_model import Model
from .train import TrainConfig, TrainState


@on_device
def sample_points(origins: torch.Tensor, dirs: torch.Tensor, n_samples: int):
    """Midpoint samples along each ray inside the unit cube (slab entry and
    exit; rays that miss get zero-length segments): points (R*S, 3) clamped
    to [0,1] and segment lengths deltas (R*S) — pg_ray_samples_f32."""
    R = origins.shape[0]
    pts = torch.empty((R * n_samples, 3), dtype=torch.float32, device=origins.device)
    deltas = torch.empty(R * n_samples, dtype=torch.float32, device=origins.device)
    _lib.call("pg_ray_samples_f32", _lib.ptr(origins.contiguous()), _lib.ptr(dirs.contiguous()), R,
              n_samples, _lib.ptr(pts), _lib.ptr(deltas), _lib.stream_ptr())
    return pts, deltas


def orbit_rays(n_rays: int, seed: int = 0, radius: float = 1.5, spread: float = 0.35,
               device="cuda"):
    """Synthetic camera rays: origins on a sphere of `radius` around the cube
    centre, aimed at a point jittered by `spread` around it (unit dirs)."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((n_rays, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    o = 0.5 + radius * v
    aim = 0.5 + spread * (rng.random((n_rays, 3)) - 0.5)
    d = aim - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return (torch.from_numpy(o.astype(np.float32)).to(device),
            torch.from_numpy(d.astype(np.float32)).to(device))


def _check_model(model: Model):
    h = model.hyper
    if h.d != 3 or h.out_dim != 4 or model.tdtype != torch.float32 or h.out_sigmoid:
        raise InvalidHyperparameter("the NeRF head needs a float32 3-D model with out_dim=4 "
                                    "(sigma, r, g, b) and out_sigmoid=False")


@on_device
def mlp_raw(model: Model, y: torch.Tensor) -> torch.Tensor:
    """Per-sample MLP outputs (B, 4) on the device (row-wise kernel)."""
    B = y.shape[0]
    out = torch.empty((B, model.hyper.out_dim), dtype=torch.float32, device=model.device)
    ws = torch.empty(max(1, 2 * B * max(model.widths)), dtype=torch.float32, device=model.device)
    _lib.call("pg_mlp_infer_rows_f32", _lib.ptr(y), B, model.mlp_desc, _lib.ptr(model.mlp_params),
              0, _lib.ptr(ws), _lib.ptr(out), _lib.stream_ptr())
    return out


@on_device
def composite(raw: torch.Tensor, deltas: torch.Tensor, n_samples: int, weights: bool = False):
    """rgb (R, 3) [and per-sample weights (R, S)] from raw (R*S, 4)."""
    R = raw.shape[0] // n_samples
    rgb = torch.empty((R, 3), dtype=torch.float32, device=raw.device)
    w = torch.empty((R, n_samples), dtype=torch.float32, device=raw.device) if weights else None
    _lib.call("pg_composite_fwd_f32", _lib.ptr(raw.contiguous()), _lib.ptr(deltas), R, n_samples,
              _lib.ptr(rgb), _lib.ptr(w), _lib.stream_ptr())
    return (rgb, w) if weights else rgb


@on_device
def render(model: Model, origins, dirs, n_samples: int = 64, chunk: int = 1 << 14) -> torch.Tensor:
    """Render rays (R, 3) -> rgb (R, 3) through the current model."""
    _check_model(model)
    out = []
    for lo in range(0, origins.shape[0], chunk):
        pts, deltas = sample_points(origins[lo:lo + chunk], dirs[lo:lo + chunk], n_samples)
        y = encode_forward_device(model, pts)
        out.append(composite(mlp_raw(model, y), deltas, n_samples))
    return torch.cat(out) if out else torch.empty((0, 3), device=model.device)


class NerfTrainState(TrainState):
    """Fits a radiance field to per-ray target colours.  Batches are
    successive slices of a device-resident ray set (cfg.batch_size rays per
    step, n_samples points each); optimizer path identical to TrainState."""

    def __init__(self, model: Model, origins, dirs, target_rgb, cfg: TrainConfig, n_samples: int = 64,
                 fused: bool | None = None):
        """``fused`` (default: when the shape allows): one fused tensor-core
        kernel per step (pg_train_fused_f32 with PG_COMPOSITE: encode fwd,
        MLP, compositing of one ray per 64-sample tile, backward, encode bwd)
        — needs n_samples == 64 and the [32, 64, 64, 4] MLP over 16 levels of
        F = 2; otherwise generic encode kernels around pg_nerf_train_f32."""
        _check_model(model)
        o = torch.as_tensor(origins, dtype=torch.float32, device=model.device).contiguous()
        d = torch.as_tensor(dirs, dtype=torch.float32, device=model.device).contiguous()
        c = torch.as_tensor(target_rgb, dtype=torch.float32, device=model.device).contiguous()
        if o.ndim != 2 or o.shape[1] != 3 or d.shape != o.shape or c.shape != o.shape:
            raise InvalidHyperparameter("origins, dirs and target_rgb must all be (R, 3)")
        if o.shape[0] < cfg.batch_size:
            raise InvalidHyperparameter("ray set smaller than one batch")
        if n_samples < 1:
            raise InvalidHyperparameter("n_samples must be >= 1")
        super().__init__(model, None, cfg, sampler="points", fused=False)
        h, w = model.hyper, model.widths
        shape_ok = (h.feature_dim == 2 and h.n_levels == 16 and h.n_p <= 16 and list(w) == [32, 64, 64, 4]
                    and n_samples == 64)
        if fused and not shape_ok:
            raise InvalidHyperparameter("the fused NeRF step needs 64 samples per ray and the "
                                        "[32, 64, 64, 4] MLP over 16 levels of F = 2")
        self.nerf_fused = shape_ok if fused is None else bool(fused)
        self.origins, self.dirs, self.rgb = o, d, c
        self.n_samples = n_samples
        R, S = cfg.batch_size, n_samples
        if self.nerf_fused:
            self.tgt4 = torch.empty((R * S, 4), dtype=torch.float32, device=model.device)
        else:
            self.y = torch.empty((R * S, h.encoded_width), dtype=torch.float32, device=model.device)
            self.dy = torch.empty_like(self.y)
            nws = int(_lib.lib().pg_mlp_train_workspace_floats(R * S, model.mlp_desc))
            self.ws = torch.empty(max(nws, 1), dtype=torch.float32, device=model.device)
        self.scale = 2.0 / (R * 3)

    def shard(self, rank: int, world: int) -> "NerfTrainState":
        super().shard(rank, world)
        self.scale = 2.0 / (world * self.cfg.batch_size * 3)
        return self

    def loss_denominator(self) -> int:
        return self.world * self.cfg.batch_size * 3

    @on_device
    def sample_batch(self):
        """Next contiguous ray slice -> (points (R*S, 3), (deltas, target rgb))."""
        n, R = self.origins.shape[0], self.cfg.batch_size
        lo = (self.t * self.world + self.rank) * R % n
        if lo + R > n:
            lo = 0
        if not self.nerf_fused:
            pts, deltas = sample_points(self.origins[lo:lo + R], self.dirs[lo:lo + R], self.n_samples)
            return pts, (deltas, self.rgb[lo:lo + R])
        # fused step: the per-sample targets (delta, rgb) written by the same kernel
        S = self.n_samples
        pts = torch.empty((R * S, 3), dtype=torch.float32, device=self.origins.device)
        deltas = torch.empty(R * S, dtype=torch.float32, device=self.origins.device)
        t4 = self.tgt4[:R * S]
        _lib.call("pg_ray_samples_targets_f32", _lib.ptr(self.origins[lo:lo + R]), _lib.ptr(self.dirs[lo:lo + R]),
                  _lib.ptr(self.rgb[lo:lo + R]), R, S, _lib.ptr(pts), _lib.ptr(deltas), _lib.ptr(t4),
                  _lib.stream_ptr())
        return pts, (deltas, self.rgb[lo:lo + R], t4)

    @on_device
    def compute_grads(self, xs, targets, dy_out=None) -> None:
        m, s = self.model, _lib.stream_ptr()
        deltas, rgb = targets[0], targets[1]
        R = rgb.shape[0]
        if self.nerf_fused:
            S = self.n_samples
            if len(targets) > 2:
                t4 = targets[2]          # written by pg_ray_samples_targets_f32
            else:                        # caller-supplied (deltas, rgb)
                t4 = self.tgt4[:R * S].view(R, S, 4)
                t4[:, :, 0] = deltas.view(R, S)
                t4[:, :, 1:] = rgb[:, None, :]
            self._fused_step(xs, t4, R * S, float(np.float32(self.scale)),
                             _lib.PG_COMPOSITE | (_lib.PG_TOUCH_ALL if self.touch_all else 0), dy_out)
            return
        encode_forward_device(m, xs, self.y)
        _lib.call("pg_nerf_train_f32", m.mlp_desc, _lib.ptr(self.y), _lib.ptr(deltas), _lib.ptr(rgb), R,
                  self.n_samples, _lib.ptr(m.mlp_params), float(np.float32(self.scale)), _lib.ptr(m.gmlp),
                  _lib.ptr(self.dy), _lib.ptr(self.loss_sum), _lib.ptr(self.ws), s)
        if dy_out is not None:
            dy_out.copy_(self.dy)
        encode_backward_device(m, xs, self.dy)
