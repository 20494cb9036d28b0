"""Device-resident training step (trainer.py:34-242 of the reference).

One ``TrainState.step()`` on the GPU:

    pixel batch -> fused encode fwd (all levels) -> MLP fwd + squared error
    + MLP bwd -> fused encode bwd (straight-through scatter, touched rows)
    -> dense Adam over [features | MLP] (one launch) -> lazy Adam + re-bake
    over touched confidence rows (one launch)

Batches come from the reference's own seeded stream on the host
(``sampler="reference"``: identical pixels, hence comparable loss curves) or
from a counter-based generator on the device (``sampler="device"``: no host
work in the step).  The loss is the fp64 mean of squared errors
(trainer.py:129-132); a non-finite loss leaves parameters untouched and raises
TrainingDiverged, as the reference does.
"""

from __future__ import annotations

import json
import os
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import on_device
from .encoding import encode_backward_device, encode_forward_device
from .errors import InvalidHyperparameter, TrainingDiverged
from .grid_model import Model, init_model
from .hyper import SEED_BATCH, HyperParams, seeded_rng


@dataclass
class TrainConfig:
    steps: int = 10_000
    batch_size: int = 8192
    lr: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.99
    eps: float = 1e-15
    seed: int = 0
    precision: str = "f32"      # "f32" | "f64"
    metrics_path: str | None = None
    debug_check_every: int = 0  # assert incremental bake == full bake every N steps

    def validate(self) -> "TrainConfig":
        if self.batch_size < 1:
            raise InvalidHyperparameter("batch size must be at least 1")
        if self.lr < 0:
            raise InvalidHyperparameter("learning rate must be non-negative")
        if self.steps < 0:
            raise InvalidHyperparameter("step count must be non-negative")
        if self.precision not in ("f32", "f64"):
            raise InvalidHyperparameter(f"unknown precision {self.precision!r}")
        return self

    @property
    def dtype(self):
        return np.float64 if self.precision == "f64" else np.float32


@dataclass
class AdamSlot:
    m: torch.Tensor
    v: torch.Tensor

    @classmethod
    def like(cls, t: torch.Tensor) -> "AdamSlot":
        return cls(torch.zeros_like(t), torch.zeros_like(t))


def _sfx(t: torch.Tensor) -> str:
    return "f64" if t.dtype == torch.float64 else "f32"


def adam_update(param: torch.Tensor, grad: torch.Tensor, slot: AdamSlot, t: int, lr: float,
                betas=(0.9, 0.99), eps: float = 1e-15) -> None:
    """Standard Adam with bias correction, in place, the reference's rounding
    order (trainer.py:73-84).  ``grad`` is left unchanged."""
    g = grad.detach().clone().contiguous()
    _lib.call(f"pg_adam_{_sfx(param)}", _lib.ptr(param), _lib.ptr(g), _lib.ptr(slot.m),
              _lib.ptr(slot.v), param.numel(), int(t), float(lr), float(betas[0]), float(betas[1]),
              float(eps), None, _lib.stream_ptr())


def train_cell_budget() -> int:
    """Bytes of the per-step fp32 cell cache the fused training forward
    reads its coarsest levels from (PG_TRAIN_CELL_MB; 0 disables).  Rebuilt
    from the current tables at every step (one launch, ~22 MB at C1, all 16
    levels); C1 step 0.554 -> 0.530 ms, other shapes 1-3%."""
    return int(float(os.environ.get("PG_TRAIN_CELL_MB", "32")) * (1 << 20))


def grad_replicas(hyper: HyperParams, dtype) -> int:
    """Copies of the feature-gradient table the fused fp32 step spreads its
    reductions over (pg_train_fused_rep_f32): small tables see every lookup
    land on a few rows, and same-address reductions from all SMs serialise
    in L2.  PG_TRAIN_REPS overrides."""
    env = os.environ.get("PG_TRAIN_REPS")
    if env:
        return max(1, min(256, int(env)))
    # probing ranges per level: <= 8 are warp-aggregated in the kernel
    # (pg_train_mma.cu, AGG); 9..256 gain from 8 copies (measured, 2^18
    # samples: n_f 2^8 N_p 16 3.66 -> 1.94 ms, n_f 2^10 N_p 16 1.87 -> 1.67,
    # n_f 2^8 N_p 4 0.665 -> 0.619); C1 (1024 ranges) is faster without
    # (0.555 vs 0.563 ms)
    ranges = hyper.n_f // hyper.n_p
    return 8 if 8 < ranges <= 256 and np.dtype(dtype) == np.float32 else 1


class TrainState:
    """Optimizer state bound to one device model; drives individual steps."""

    def __init__(self, model: Model, image, cfg: TrainConfig, sampler: str = "reference",
                 fused: bool | None = None, deterministic: bool = False,
                 reference_order: bool = False, exact_mlp: bool = False):
        """``exact_mlp``: the fused step's MLP on CUDA cores in numpy/OpenBLAS
        operation order (activations and dL/dy bit-identical to the
        reference's) instead of the default 3xTF32 tensor-core MLP (fp32-level,
        ~1e-6).  ``reference_order``: additionally the MLP weight/bias
        gradients in OpenBLAS summation order (pg_mlp_wgrad_blas_f32), making
        every MLP gradient bit-identical to the reference's (parity mode)."""
        cfg.validate()
        if sampler not in ("reference", "device", "points"):
            raise InvalidHyperparameter(f"unknown sampler {sampler!r}")
        self.model, self.cfg, self.sampler = model, cfg, sampler
        if sampler != "points":
            img = image if isinstance(image, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(image, dtype=model.dtype))
            if img.ndim != 3 or img.shape[2] != model.hyper.out_dim:
                raise InvalidHyperparameter(
                    f"image shape {tuple(img.shape)} does not match output dim {model.hyper.out_dim}")
            if model.hyper.d != 2:
                raise InvalidHyperparameter("the image trainer is 2-D (trainer.py:109-116)")
            self.image = img.to(device=model.device, dtype=model.tdtype).contiguous()
            self.height, self.width = int(img.shape[0]), int(img.shape[1])
        self.rng = seeded_rng(cfg.seed, SEED_BATCH)
        self.t = 0
        dev, tdt = model.device, model.tdtype
        self.dm = torch.zeros_like(model.dense)
        self.dv = torch.zeros_like(model.dense)
        self.cm = torch.zeros_like(model.conf)
        self.cv = torch.zeros_like(model.conf)
        B, h = cfg.batch_size, model.hyper
        w = model.widths
        self.fused = (model.tdtype == torch.float32 and h.feature_dim == 2 and h.n_levels == 16
                      and h.n_p <= 16 and len(w) == 4 and w[1] == 64 and w[2] == 64
                      and w[3] <= 4)
        self.pix_host = torch.empty(B, dtype=torch.int64, pin_memory=True)
        self.pix_copied = torch.cuda.Event()
        self.pix = torch.empty(B, dtype=torch.int64, device=dev)
        self.xs = torch.empty((B, h.d), dtype=tdt, device=dev)
        self.targets = torch.empty((B, h.out_dim), dtype=tdt, device=dev)
        if fused is not None:
            self.fused = self.fused and bool(fused)
        if deterministic and model.tdtype != torch.float32:
            raise InvalidHyperparameter("deterministic mode is float32-only")
        self.deterministic = deterministic
        self.reference_order = reference_order
        self.exact_mlp = exact_mlp or reference_order
        if reference_order:
            if not self.fused:
                raise InvalidHyperparameter("reference_order needs the fused float32 shape")
            na = int(_lib.lib().pg_mlp_acts_floats(B, model.mlp_desc))
            self.acts = torch.empty(na, dtype=tdt, device=dev)
        if not self.fused:
            self.y = torch.empty((B, h.encoded_width), dtype=tdt, device=dev)
            self.dy = torch.empty_like(self.y)
            nws = int(_lib.lib().pg_mlp_train_workspace_floats(B, model.mlp_desc))
            self.ws = torch.empty(max(nws, 1), dtype=tdt, device=dev)
        self.loss_sum = torch.zeros(1, dtype=torch.float64, device=dev)
        self.loss_host = torch.zeros(1, dtype=torch.float64, pin_memory=True)
        self.rank, self.world = 0, 1
        self.touch_all = False
        self.grad_replicas = grad_replicas(model.hyper, model.dtype)
        self.scale = 2.0 / (B * h.out_dim)   # trainer.py:134, cast to the model dtype

    def shard(self, rank: int, world: int) -> "TrainState":
        """Make this state one of `world` data-parallel replicas: the batch is
        rank's slice of a global batch of world*batch_size samples, and the
        loss gradient is scaled by 2/(world*B*out_dim) so the summed gradients
        equal the global-batch gradient."""
        self.rank, self.world = rank, world
        self.scale = 2.0 / (world * self.cfg.batch_size * self.model.hyper.out_dim)
        # replicas' gconf sums meet only in the all-reduce, where a row's
        # contributions can cancel to an exact 0.0: flag every lookup so the
        # touched union is the reference's touched set exactly
        self.touch_all = world > 1
        return self

    # ---------------------------------------------------------------- batch
    @on_device
    def sample_batch(self):
        """Draw the next batch; returns device (xs, targets)."""
        m, B, s = self.model, self.cfg.batch_size, _lib.stream_ptr()
        sfx = "f64" if m.tdtype == torch.float64 else "f32"
        if self.sampler == "points":
            # next contiguous slice of a resident point set (cyclic): zero-copy views
            n = self.points.shape[0]
            lo = (self.t * self.world + self.rank) * B % n
            if lo + B > n:
                lo = 0
            return self.points[lo:lo + B], self.values[lo:lo + B]
        if self.sampler == "reference":
            # trainer.py:110-111; replicas draw the global batch and keep their slice
            pix = self.rng.integers(0, self.width * self.height, size=B * self.world)
            pix = pix[self.rank * B:(self.rank + 1) * B]
            self.pix_copied.synchronize()   # previous upload of pix_host has landed
            self.pix_host.numpy()[:] = pix
            self.pix.copy_(self.pix_host, non_blocking=True)
            self.pix_copied.record()
            _lib.call(f"pg_pixel_batch_{sfx}", _lib.ptr(self.pix), B, self.width, self.height,
                      _lib.ptr(self.image), m.hyper.out_dim, 0, 0, None, _lib.ptr(self.xs),
                      _lib.ptr(self.targets), s)
        else:
            _lib.call(f"pg_pixel_batch_{sfx}", None, B, self.width, self.height,
                      _lib.ptr(self.image), m.hyper.out_dim, int(self.cfg.seed) * 1000003 + self.rank,
                      int(self.t), _lib.ptr(self.pix), _lib.ptr(self.xs), _lib.ptr(self.targets), s)
        return self.xs, self.targets

    # ------------------------------------------------------- DP exchange
    def exchange_buffer(self) -> torch.Tensor:
        """The ONE buffer a data-parallel step all-reduces:
        [gfeats | gmlp | pad | gconf | pad | touched-as-float | loss]."""
        return self.model.grads

    @on_device
    def pack_exchange(self) -> None:
        m, s = self.model, _lib.stream_ptr()
        if m.n_rows:
            sfx = "f64" if m.touched_f.dtype == torch.float64 else "f32"
            _lib.call(f"pg_touched_to_{sfx}", _lib.ptr(m.touched), m.n_rows, _lib.ptr(m.touched_f), s)
        m.loss_slot.copy_(self.loss_sum)

    @on_device
    def unpack_exchange(self) -> None:
        """After the all-reduce: touched = union over replicas (every replica
        then updates the same rows, keeping replicas identical), loss = sum."""
        m, s = self.model, _lib.stream_ptr()
        if m.n_rows:
            sfx = "f64" if m.touched_f.dtype == torch.float64 else "f32"
            _lib.call(f"pg_touched_from_{sfx}", _lib.ptr(m.touched_f), m.n_rows, _lib.ptr(m.touched), s)
        self.loss_sum.copy_(m.loss_slot)

    def loss_denominator(self) -> int:
        return self.world * self.cfg.batch_size * self.model.hyper.out_dim

    # ----------------------------------------------------------------- step
    @on_device
    def launch_step(self) -> None:
        """Enqueue one full step on the current stream (no host sync)."""
        m, cfg = self.model, self.cfg
        s = _lib.stream_ptr()
        sfx = "f64" if m.tdtype == torch.float64 else "f32"
        xs, targets = self.sample_batch()
        self.loss_sum.zero_()
        self.compute_grads(xs, targets)
        self.t += 1
        self.apply_updates()

    @on_device
    def compute_grads(self, xs, targets, dy_out=None) -> None:
        """Forward + backward of one batch into model.grads / touched /
        loss_sum: the fused single-kernel path when the shape allows it, else
        fused encode kernels around the generic MLP kernels."""
        m, cfg, s = self.model, self.cfg, _lib.stream_ptr()
        flags = _lib.PG_SIGMOID if m.hyper.out_sigmoid else 0
        if self.exact_mlp and self.fused:
            flags |= _lib.PG_EXACT_MLP
        if self.touch_all:
            flags |= _lib.PG_TOUCH_ALL
        scale = float(np.dtype(m.dtype).type(self.scale))
        if self.reference_order and self.deterministic:
            if dy_out is not None:
                raise InvalidHyperparameter("dy_out is not produced in reference_order mode")
            gf, gm, gc = m.fx_ptrs()
            _lib.call("pg_train_fused_ref_det_f32", m.grid, m.mlp_desc, _lib.ptr(xs), _lib.ptr(targets),
                      xs.shape[0], _lib.ptr(m.feats), _lib.ptr(m.baked), _lib.ptr(m.conf),
                      _lib.ptr(m.mlp_params), scale, flags, gf, gc, _lib.ptr(m.touched),
                      _lib.ptr(m.loss_fx), _lib.ptr(self.acts), s)
            m.fx_flush(loss_sum=self.loss_sum)
            _lib.call("pg_mlp_wgrad_blas_f32", m.mlp_desc, _lib.ptr(self.acts), xs.shape[0],
                      _lib.ptr(m.gmlp), s)
            return
        if self.deterministic:
            gf, gm, gc = m.fx_ptrs()
            if self.fused:
                _lib.call("pg_train_fused_det_f32", m.grid, m.mlp_desc, _lib.ptr(xs),
                          _lib.ptr(targets), xs.shape[0], _lib.ptr(m.feats), _lib.ptr(m.baked),
                          _lib.ptr(m.conf), _lib.ptr(m.mlp_params), scale, flags, gf, gc,
                          _lib.ptr(m.touched), gm, _lib.ptr(m.loss_fx), _lib.ptr(dy_out), s)
            else:
                encode_forward_device(m, xs, self.y)
                _lib.call("pg_mlp_train_det_f32", m.mlp_desc, _lib.ptr(self.y), _lib.ptr(targets),
                          xs.shape[0], _lib.ptr(m.mlp_params), scale, flags, gm,
                          _lib.ptr(self.dy), _lib.ptr(m.loss_fx), _lib.ptr(self.ws), s)
                if dy_out is not None:
                    dy_out.copy_(self.dy)
                encode_backward_device(m, xs, self.dy, deterministic=True, flush=False)
            m.fx_flush(loss_sum=self.loss_sum)
            return
        if self.reference_order:
            if dy_out is not None:
                raise InvalidHyperparameter("dy_out is not produced in reference_order mode")
            _lib.call("pg_train_fused_ref_f32", m.grid, m.mlp_desc, _lib.ptr(xs), _lib.ptr(targets),
                      xs.shape[0], _lib.ptr(m.feats), _lib.ptr(m.baked), _lib.ptr(m.conf),
                      _lib.ptr(m.mlp_params), scale, flags, _lib.ptr(m.gfeats), _lib.ptr(m.gconf),
                      _lib.ptr(m.touched), _lib.ptr(self.loss_sum), _lib.ptr(self.acts), s)
            _lib.call("pg_mlp_wgrad_blas_f32", m.mlp_desc, _lib.ptr(self.acts), xs.shape[0],
                      _lib.ptr(m.gmlp), s)
            return
        if self.fused:
            self._fused_step(xs, targets, xs.shape[0], scale, flags, dy_out)
            return
        sfx = "f64" if m.tdtype == torch.float64 else "f32"
        encode_forward_device(m, xs, self.y)
        _lib.call(f"pg_mlp_train_{sfx}", m.mlp_desc, _lib.ptr(self.y), _lib.ptr(targets),
                  xs.shape[0], _lib.ptr(m.mlp_params), scale, flags, _lib.ptr(m.gmlp),
                  _lib.ptr(self.dy), _lib.ptr(self.loss_sum), _lib.ptr(self.ws), s)
        if dy_out is not None:
            dy_out.copy_(self.dy)
        encode_backward_device(m, xs, self.dy)

    @on_device
    def _fused_step(self, xs, targets, n, scale, flags, dy_out) -> None:
        """One fused fp32 training pass (pg_train_fused_ex_f32): the forward
        reads this step's cell cache (rebuilt here from the current tables),
        feature gradients go through the replica buffer for small tables;
        the OpenBLAS-order MLP (exact_mlp) takes neither."""
        m, s = self.model, _lib.stream_ptr()
        exact = bool(flags & _lib.PG_EXACT_MLP)
        reps = 1 if exact else self.grad_replicas
        cells = None if exact else self._train_cells()
        if reps > 1 and getattr(self, "_gfeat_rep", None) is None:
            self._gfeat_rep = torch.zeros(reps * m.n_feat, dtype=torch.float32, device=m.device)
        if cells is not None:
            _lib.call("pg_cells_build_f32", m.grid, _lib.ptr(m.feats), _lib.ptr(m.baked), cells, s)
        _lib.call("pg_train_fused_ex_f32", m.grid, m.mlp_desc, _lib.ptr(xs), _lib.ptr(targets), n,
                  _lib.ptr(m.feats), _lib.ptr(m.baked), _lib.ptr(m.conf), _lib.ptr(m.mlp_params), scale, flags,
                  _lib.ptr(m.gfeats), _lib.ptr(m.gconf), _lib.ptr(m.touched), _lib.ptr(m.gmlp),
                  _lib.ptr(self.loss_sum), _lib.ptr(dy_out),
                  _lib.ptr(self._gfeat_rep) if reps > 1 else None, reps, cells, s)

    def _train_cells(self):
        """fp32 cell cache plan + buffer for the fused forward (None: off)."""
        if not hasattr(self, "_cells"):
            self._cells = None
            budget = train_cell_budget()
            if budget > 0 and self.model.tdtype == torch.float32 and self.model.hyper.feature_dim == 2:
                plan = _lib.PgCells()
                n = int(_lib.lib().pg_cells_plan_rows(self.model.grid, budget, 8, plan))
                if n > 0:
                    self._cells_buf = torch.empty(n, dtype=torch.uint8, device=self.model.device)
                    plan.data = self._cells_buf.data_ptr()
                    self._cells = plan
        return self._cells

    def apply_updates(self) -> None:
        """Dense Adam over [features | MLP] and lazy Adam + re-bake over the
        touched confidence rows; both skip the update if the loss diverged."""
        m, cfg, s = self.model, self.cfg, _lib.stream_ptr()
        sfx = "f64" if m.tdtype == torch.float64 else "f32"
        _lib.call(f"pg_adam_{sfx}", _lib.ptr(m.dense), _lib.ptr(m.gdense), _lib.ptr(self.dm),
                  _lib.ptr(self.dv), m.n_dense, self.t, cfg.lr, cfg.beta1, cfg.beta2, cfg.eps,
                  _lib.ptr(self.loss_sum), s)
        if m.probed:
            _lib.call(f"pg_lazy_adam_rebake_{sfx}", _lib.ptr(m.conf), _lib.ptr(self.cm),
                      _lib.ptr(self.cv), _lib.ptr(m.baked), _lib.ptr(m.gconf), _lib.ptr(m.touched),
                      m.n_rows, m.hyper.n_p, self.t, cfg.lr, cfg.beta1, cfg.beta2, cfg.eps,
                      _lib.ptr(self.loss_sum), s)

    @on_device
    def loss_value(self) -> float:
        self.loss_host.copy_(self.loss_sum, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return float(self.loss_host[0]) / self.loss_denominator()

    @on_device
    def step(self) -> float:
        self.launch_step()
        return self.finish_step()

    def finish_step(self) -> float:
        """Read the launched step's loss; on a non-finite loss (the optimizer
        kernels skipped the update) undo the step count and raise, as the
        reference raises before counting the step (trainer.py:131-133)."""
        loss = self.loss_value()
        if not math.isfinite(loss):
            self.t -= 1
            raise TrainingDiverged(f"non-finite loss at step {self.t}")
        if self.cfg.debug_check_every and self.t % self.cfg.debug_check_every == 0:
            self.check_bake_consistency()
        return loss

    @on_device
    def check_bake_consistency(self) -> None:
        m = self.model
        if m.probed:
            full = m.bake_into(torch.empty_like(m.baked))     # codebooks.bake
            bad = (full != m.baked).any(dim=-1).nonzero()
            if bad.numel():
                raise TrainingDiverged(
                    f"incremental bake diverged on level {m.probed[int(bad[0])]}")


class FieldTrainState(TrainState):
    """Training on an arbitrary d-dimensional field (2-D or 3-D SDF, density,
    radiance samples): batches are successive slices of a device-resident
    point set with target values.  The reference has no trainer for these
    (trainer.py:92-95 is image-only); the step is the same composition of
    encode / MLP / Adam / lazy-Adam it uses (SURVEY 7.4 hazard 13)."""

    def __init__(self, model: Model, points, values, cfg: TrainConfig, **kw):
        pts = torch.as_tensor(points).to(device=model.device, dtype=model.tdtype).contiguous()
        val = torch.as_tensor(values).to(device=model.device, dtype=model.tdtype).contiguous()
        if pts.ndim != 2 or pts.shape[1] != model.hyper.d:
            raise InvalidHyperparameter(f"points must be (N, {model.hyper.d})")
        if val.shape != (pts.shape[0], model.hyper.out_dim):
            raise InvalidHyperparameter(f"values must be (N, {model.hyper.out_dim})")
        if pts.shape[0] < cfg.batch_size:
            raise InvalidHyperparameter("point set smaller than one batch")
        super().__init__(model, None, cfg, sampler="points", **kw)
        self.points, self.values = pts, val


@dataclass
class FitResult:
    model: Model
    inference: object
    final_psnr: float
    final_loss: float
    steps: int
    wall_time_s: float
    ms_per_step: float
    losses: list = field(default_factory=list, repr=False)

    @property
    def size_report(self):
        """Exact .cngp byte breakdown of this model (trainer.py FitResult)."""
        from .model_io import size_report
        return size_report(self.model.hyper)


def psnr(reference, test) -> float:
    """20*log10(1/RMSE) over [0,1] values in fp64 (metrics.py:12-26)."""
    a = np.asarray(reference, dtype=np.float64)
    b = np.asarray(test, dtype=np.float64)
    mse = float(np.mean((a - b) ** 2))
    return float("inf") if mse == 0.0 else -10.0 * math.log10(mse)


def fit(image, hyper: HyperParams, cfg: TrainConfig, force_probed: bool = False,
        sampler: str = "reference", deterministic: bool = False,
        reference_order: bool = False) -> FitResult:
    """Fit one image on the GPU (trainer.py:196-242)."""
    from .decode import decode_image, to_inference
    model = init_model(hyper, cfg.seed, cfg.dtype, force_probed=force_probed)
    state = TrainState(model, image, cfg, sampler=sampler, deterministic=deterministic,
                       reference_order=reference_order)
    sink = open(cfg.metrics_path, "w") if cfg.metrics_path else None
    losses, step_ms = [], []
    t_start = time.perf_counter()
    try:
        for step in range(cfg.steps):
            t0 = time.perf_counter()
            loss = state.step()
            ms = (time.perf_counter() - t0) * 1e3
            losses.append(loss)
            step_ms.append(ms)
            if sink is not None:
                bp = -10.0 * math.log10(loss) if loss > 0 else float("inf")
                sink.write(json.dumps({"step": step, "loss": loss, "psnr": bp, "ms": ms}) + "\n")
    finally:
        if sink is not None:
            sink.close()
    wall = time.perf_counter() - t_start
    inf = to_inference(model, width=state.width, height=state.height)
    decoded = decode_image(inf)
    img = image.cpu().numpy() if isinstance(image, torch.Tensor) else np.asarray(image)
    final = psnr(img, np.clip(decoded, 0.0, 1.0))
    return FitResult(model, inf, final, losses[-1] if losses else float("nan"), cfg.steps, wall,
                     float(np.median(step_ms)) if step_ms else 0.0, losses)


# size-budgeted hyper-parameters (trainer.py:27-31, 245-281)
RECIPE_NF_MIN, RECIPE_NF_MAX = 2**6, 2**12
RECIPE_NC_MIN, RECIPE_NC_MAX = 2**10, 2**16
RECIPE_NP = 2**1


def select_hyperparams(target_size_bytes: int, base: HyperParams | None = None) -> HyperParams:
    """Largest tables that fit a .cngp byte budget: feature table from the
    plain-hash lower bound (<= a third of the budget), then the index table
    toward its ceiling, then the feature table with what remains — the
    reference's recipe, so both pick the same configuration."""
    from .errors import TargetTooSmall
    from .model_io import size_report
    base = base or HyperParams()
    hyper = base.with_updates(n_f=RECIPE_NF_MIN, n_c=RECIPE_NC_MIN, n_p=RECIPE_NP)
    total = lambda h: size_report(h).total_bytes  # noqa: E731
    minimum = total(hyper)
    if target_size_bytes < minimum:
        raise TargetTooSmall(f"target {target_size_bytes} B below the smallest model ({minimum} B)")
    n_f = RECIPE_NF_MIN
    while n_f * 2 <= RECIPE_NF_MAX and \
            total(hyper.with_updates(n_f=n_f * 2, n_p=1)) <= target_size_bytes // 3:
        n_f *= 2
    n_c = RECIPE_NC_MIN
    while n_c * 2 <= RECIPE_NC_MAX and total(hyper.with_updates(n_f=n_f, n_c=n_c * 2)) <= target_size_bytes:
        n_c *= 2
    while n_f * 2 <= RECIPE_NF_MAX and total(hyper.with_updates(n_f=n_f * 2, n_c=n_c)) <= target_size_bytes:
        n_f *= 2
    return hyper.with_updates(n_f=n_f, n_c=n_c).validate()
