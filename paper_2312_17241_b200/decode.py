"""Random-access decode on the GPU (model_io.py:92-147, 280-349 of the reference).

``to_inference`` performs the reference's fp16 downcast of features and MLP
(model_io.py:130-147).  The device keeps the feature tables IN binary16 (half
the gather bytes of the fp32 twin) and widens them in registers — the widened
values are exactly the reference twin's fp32 values (model_io.py:114-127).
``decode_pixels`` runs ONE fused kernel per call: all-level encode + MLP per
128-query tile.  With ``exact=True`` (the default for the reference-facing
functions) the MLP uses the reference's operation order without FMA, so the
output equals the reference's ``decode_pixels`` bit for bit; ``exact=False``
uses FMA (within ~1e-6 relative).  Every output row depends only on its own
input row either way (model_io.py:294-295), so any batching is bit-identical.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import on_device
from .errors import DomainViolation, UnbakedModel
from .grid_model import Model
from .hyper import HyperParams, build_level_specs, grid_struct, mlp_struct


@dataclass
class TouchCounter:
    """Rows touched by instrumented decode queries (model_io.py:280-289)."""

    feature_rows: int = 0
    index_rows: int = 0

    @property
    def total(self) -> int:
        return self.feature_rows + self.index_rows


class InferenceModel:
    """Half-precision tables + fp16-rounded MLP resident on one GPU."""

    def __init__(self, hyper: HyperParams, width: int, height: int, feats16: torch.Tensor,
                 baked: torch.Tensor, probed: list, params: torch.Tensor, device=None):
        self.hyper, self.width, self.height = hyper, width, height
        self.device = torch.device(device or "cuda")
        self.specs = build_level_specs(hyper.n_min, hyper.n_max, hyper.n_levels, hyper.n_f, hyper.d)
        self.probed = list(probed)
        self.grid = grid_struct(hyper, self.specs, self.probed)
        self.widths = hyper.mlp_widths()
        self.mlp_desc = mlp_struct(self.widths)
        self.feats16 = feats16.to(self.device).contiguous()      # (L, n_f, F) float16
        self.baked = baked.to(self.device).contiguous()          # (P, n_c) uint8
        self.params = params.to(self.device).contiguous()        # fp32 of fp16-rounded MLP
        self.fast = (hyper.feature_dim == 2 and hyper.n_levels == 16 and len(self.widths) == 4
                     and self.widths[1] == 64 and self.widths[2] == 64 and hyper.out_dim <= 4)
        self.cell_budget = CELL_BUDGET
        self._cells = None

    def cells(self):
        """The decode cell cache of this model's tables (built on first use;
        None when no level fits the budget or the tables are not fp16)."""
        if self._cells is None:
            plan = _lib.PgCells()
            nbytes = 0
            if self.feats16.dtype == torch.float16 and self.cell_budget > 0:
                nbytes = int(_lib.lib().pg_cells_plan(self.grid, int(self.cell_budget), plan))
            if nbytes <= 0:
                self._cells = (None, None)
            else:
                buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
                plan.data = buf.data_ptr()
                with torch.cuda.device(self.device):
                    _lib.call("pg_cells_build", self.grid, _lib.ptr(self.feats16), _lib.ptr(self.baked), plan,
                              _lib.stream_ptr())
                self._cells = (plan, buf)
        return self._cells[0]

    def invalidate_cells(self) -> None:
        """Drop the cell cache (call after editing feats16 / baked in place)."""
        self._cells = None

    @property
    def cell_cache_bytes(self) -> int:
        return 0 if self._cells is None or self._cells[1] is None else self._cells[1].numel()

    @property
    def out_dim(self) -> int:
        return self.hyper.out_dim

    @classmethod
    def from_host(cls, hyper, feats16, baked, w16, b16, width=0, height=0, device=None):
        """Build from the reference's InferenceModel payload (per-level fp16
        tables, per-level baked entries or None, fp16 weights/biases)."""
        probed = [i for i, b in enumerate(baked) if b is not None]
        f = torch.from_numpy(np.stack([np.asarray(x, np.float16) for x in feats16]))
        bk = torch.from_numpy(np.stack([np.asarray(baked[i], np.uint8) for i in probed])
                              if probed else np.zeros((0, hyper.n_c), np.uint8))
        flat = np.concatenate([np.concatenate([np.asarray(w, np.float16).astype(np.float32).ravel(),
                                               np.asarray(b, np.float16).astype(np.float32).ravel()])
                               for w, b in zip(w16, b16)])
        return cls(hyper, width, height, f, bk, probed, torch.from_numpy(flat), device)


@on_device
def to_inference(model: Model, width: int = 0, height: int = 0) -> InferenceModel:
    """Downcast a trained device model to its storable half-precision form."""
    if model.probed and model.baked.numel() == 0:
        raise UnbakedModel("probed levels have no baked indices")
    feats16 = model.feats.to(torch.float16)                      # RNE, as numpy astype
    params = model.mlp_params.to(torch.float16).to(torch.float32)
    return InferenceModel(model.hyper, width, height, feats16, model.baked.clone(), model.probed,
                          params, model.device)


# Bytes of device memory the decode cell cache may use per inference model
# (coarsest levels first; pg_cells_plan).  0 disables it.  Measured at C2
# (log2 n_f 16, N_p 4, 2^24 queries): no cache 3.37e9 q/s, 8 MiB 4.01e9,
# 32 MiB (28 used) 4.63e9, 96 MiB (65 used: the 11 coarsest levels) 5.22e9;
# the next level would need 88 MB more and no longer stays L2-resident.
CELL_BUDGET = int(float(os.environ.get("PG_DECODE_CELL_MB", "96")) * (1 << 20))


def _flags(inf: InferenceModel, exact: bool, tensor: bool = True, smem_tables=None) -> int:
    f = _lib.PG_HALF_FEATS
    if exact:
        f |= _lib.PG_EXACT_MLP
    if not tensor:
        f |= _lib.PG_NO_TENSOR
    if smem_tables is not None:
        f |= _lib.PG_SMEM_TABLES if smem_tables else _lib.PG_NO_SMEM_TABLES
    if inf.hyper.out_sigmoid:
        f |= _lib.PG_SIGMOID
    return f


@on_device
def decode_device(inf: InferenceModel, xs: torch.Tensor, out: torch.Tensor = None,
                  exact: bool = True, stream=None, tensor: bool = True,
                  smem_tables=None, cells: bool = True) -> torch.Tensor:
    """Fused encode + MLP on device-resident queries; returns (B, out_dim).

    exact=True: reference operation order on CUDA cores (bit-identical).
    exact=False: the MLP's 64-wide layers on the tcgen05 tensor core (2-term
    tf32, fp32-level accuracy); tensor=False keeps FFMA instead (ablation);
    smem_tables forces (True) or forbids (False) serving the probed levels'
    baked indices from bit-packed shared-memory copies; None = automatic
    (on for N_p = 2 and 4, where it measured faster).  cells: read the
    coarsest levels from the model's decode cell cache (tcgen05 engine;
    bit-identical — the records are copies of the resolved table rows)."""
    B = xs.shape[0]
    if out is None:
        out = torch.empty((B, inf.out_dim), dtype=torch.float32, device=inf.device)
    ws = None
    if not inf.fast:
        n = B * inf.hyper.encoded_width + 2 * B * max(inf.widths)
        ws = torch.empty(max(n, 1), dtype=torch.float32, device=inf.device)
    cells = inf.cells() if (cells and inf.fast) else None
    if cells is not None:
        _lib.call("pg_decode_cells_f32", inf.grid, inf.mlp_desc, _lib.ptr(xs), B, _lib.ptr(inf.feats16),
                  _lib.ptr(inf.baked), _lib.ptr(inf.params), _flags(inf, exact, tensor, smem_tables), cells,
                  _lib.ptr(ws), _lib.ptr(out), _lib.stream_ptr(stream))
    else:
        _lib.call("pg_decode_f32", inf.grid, inf.mlp_desc, _lib.ptr(xs), B, _lib.ptr(inf.feats16),
                  _lib.ptr(inf.baked), _lib.ptr(inf.params), _flags(inf, exact, tensor, smem_tables), _lib.ptr(ws),
                  _lib.ptr(out), _lib.stream_ptr(stream))
    return out


@on_device
def decode_pixels(inf: InferenceModel, xs, counter: TouchCounter | None = None,
                  exact: bool = True):
    """Decode arbitrary coordinates (numpy in -> numpy out, or CUDA tensor in
    -> CUDA tensor out); model_io.py:292-311."""
    d = inf.hyper.d
    as_numpy = not isinstance(xs, torch.Tensor)
    if as_numpy:
        a = np.ascontiguousarray(np.asarray(xs, dtype=np.float32))
        if a.ndim != 2 or a.shape[1] != d:
            raise DomainViolation(f"expected (batch, {d}) coordinates, got {a.shape}")
        if not (a.shape[0] >= HOST_PATH_MIN and inf.fast) and (np.any(a < 0.0) or np.any(a > 1.0)):
            raise DomainViolation("coordinates outside the unit hypercube")
    else:
        t = xs.to(device=inf.device, dtype=torch.float32).contiguous()
        if t.ndim != 2 or t.shape[1] != d:
            raise DomainViolation(f"expected (batch, {d}) coordinates, got {tuple(t.shape)}")
        if t.numel() and bool(((t < 0.0) | (t > 1.0)).any()):   # encoding.py:37-38 (NaN passes, as there)
            raise DomainViolation("coordinates outside the unit hypercube")
    if counter is not None:
        per = (a if as_numpy else t).shape[0] * (1 << d)
        counter.feature_rows += per * inf.hyper.n_levels
        counter.index_rows += per * len(inf.probed)
    if as_numpy:
        if a.shape[0] >= HOST_PATH_MIN and inf.fast:
            return _decode_host_numpy(inf, a, exact)
        t = torch.from_numpy(a).to(inf.device)
    out = decode_device(inf, t, exact=exact)
    return out.cpu().numpy() if as_numpy else out


# numpy batches at least this large take the pipelined host path below
# instead of pageable copies (~10x slower at 2^24 queries, tools/e2e_dropin.py)
HOST_PATH_MIN = 1 << 16
HOST_CHUNK = 1 << 21


class _NumpyPipe:
    """Chunked host pipeline for numpy in / numpy out: two pinned slots per
    direction and two device slots; chunk i's host copy into pinned memory
    (multi-threaded torch copy), H2D, decode kernel and D2H run while the
    host copies chunk i-1's outputs into the result array and stages chunk
    i+1 — host copies, PCIe and the kernels overlap."""

    def __init__(self, inf: InferenceModel, chunk: int):
        d, od, dev = inf.hyper.d, inf.out_dim, inf.device
        self.chunk = chunk
        self.px = [torch.empty((chunk, d), dtype=torch.float32).pin_memory() for _ in range(2)]
        self.po = [torch.empty((chunk, od), dtype=torch.float32).pin_memory() for _ in range(2)]
        self.dx = [torch.empty((chunk, d), dtype=torch.float32, device=dev) for _ in range(2)]
        self.do = [torch.empty((chunk, od), dtype=torch.float32, device=dev) for _ in range(2)]
        self.s_in, self.s_k, self.s_out = (torch.cuda.Stream(device=dev) for _ in range(3))
        self.e_in = [torch.cuda.Event() for _ in range(2)]
        self.e_k = [torch.cuda.Event() for _ in range(2)]
        self.e_out = [torch.cuda.Event() for _ in range(2)]


def _decode_host_numpy(inf: InferenceModel, a: np.ndarray, exact: bool) -> np.ndarray:
    B, od = a.shape[0], inf.out_dim
    pipe = inf.__dict__.get("_numpy_pipe")
    if pipe is None:
        pipe = inf._numpy_pipe = _NumpyPipe(inf, HOST_CHUNK)
    inf.cells()                                   # built (on the current stream) before the pipeline starts
    cur = torch.cuda.current_stream(inf.device)
    for st in (pipe.s_in, pipe.s_k, pipe.s_out):
        st.wait_stream(cur)
    res = np.empty((B, od), np.float32)
    res_t = torch.from_numpy(res)
    src = torch.from_numpy(a)
    C = pipe.chunk
    n_chunks = -(-B // C)
    pending = None                                # (slot, lo, n) of the chunk whose outputs are in flight
    for i in range(n_chunks + 1):
        if i < n_chunks:
            slot, lo = i % 2, i * C
            n = min(C, B - lo)
            if i >= 2:
                pipe.e_in[slot].synchronize()     # the slot's previous H2D has read px[slot]
            hx = pipe.px[slot][:n]
            hx.copy_(src[lo:lo + n])              # multi-threaded host copy into pinned memory
            mn, mx = torch.aminmax(hx)            # encoding.py:37-38 (NaN passes, as there)
            if float(mn) < 0.0 or float(mx) > 1.0:
                torch.cuda.synchronize(inf.device)
                raise DomainViolation("coordinates outside the unit hypercube")
            with torch.cuda.stream(pipe.s_in):
                if i >= 2:
                    pipe.s_in.wait_event(pipe.e_k[slot])      # device slot free
                pipe.dx[slot][:n].copy_(hx, non_blocking=True)
                pipe.e_in[slot].record()
            with torch.cuda.stream(pipe.s_k):
                pipe.s_k.wait_event(pipe.e_in[slot])
                if i >= 2:
                    pipe.s_k.wait_event(pipe.e_out[slot])     # the slot's previous D2H read do[slot]
                decode_device(inf, pipe.dx[slot][:n], pipe.do[slot][:n], exact=exact, stream=pipe.s_k)
                pipe.e_k[slot].record()
            with torch.cuda.stream(pipe.s_out):
                pipe.s_out.wait_event(pipe.e_k[slot])
                pipe.po[slot][:n].copy_(pipe.do[slot][:n], non_blocking=True)
                pipe.e_out[slot].record()
        if pending is not None:                   # previous chunk's outputs to the result array
            ps, plo, pn = pending
            pipe.e_out[ps].synchronize()
            res_t[plo:plo + pn].copy_(pipe.po[ps][:pn])
        pending = (slot, lo, n) if i < n_chunks else None
    return res


def decode_at(inf: InferenceModel, x, counter: TouchCounter | None = None) -> np.ndarray:
    """Random-access decode of one point (model_io.py:314-318)."""
    return decode_pixels(inf, np.asarray(x, dtype=np.float32).reshape(1, -1), counter)[0]


def grid_coords(width: int, height: int, x0: int, y0: int, x1: int, y1: int) -> np.ndarray:
    """Pixel centres of a half-open rectangle (model_io.py:321-325)."""
    cols, rows = np.meshgrid(np.arange(x0, x1), np.arange(y0, y1))
    return np.stack([(cols.ravel() + 0.5) / width, (rows.ravel() + 0.5) / height],
                    axis=1).astype(np.float32)


@on_device
def decode_rect(inf: InferenceModel, rect, width: int | None = None,
                height: int | None = None, exact: bool = True) -> np.ndarray:
    """Decode the half-open pixel rectangle (x0, y0, x1, y1) (model_io.py:327-339)."""
    width = width or inf.width
    height = height or inf.height
    if width < 1 or height < 1:
        raise DomainViolation("model stores no image dimensions; pass them")
    x0, y0, x1, y1 = (int(v) for v in rect)
    if not (0 <= x0 < x1 <= width and 0 <= y0 < y1 <= height):
        raise DomainViolation(f"rect {rect} invalid for {width}x{height} image")
    # pixel centres generated on the device (bit-identical to grid_coords)
    w, h = x1 - x0, y1 - y0
    xs = torch.empty((w * h, 2), dtype=torch.float32, device=inf.device)
    _lib.call("pg_raster_coords_f32", x0, y0, w, h, width, height, _lib.ptr(xs), _lib.stream_ptr())
    out = decode_device(inf, xs, exact=exact)
    return out.cpu().numpy().reshape(h, w, inf.out_dim)


def decode_image(inf: InferenceModel, width: int | None = None,
                 height: int | None = None, exact: bool = True) -> np.ndarray:
    """Decode the full image (model_io.py:342-349)."""
    width = width or inf.width
    height = height or inf.height
    if width < 1 or height < 1:
        raise DomainViolation("model stores no image dimensions; pass them")
    return decode_rect(inf, (0, 0, width, height), width, height, exact=exact)


class HostDecoder:
    """End-to-end decode from pinned host memory through the C ABI.

    Streaming mode (default when the device supports stream memory
    operations and the tensor-core path applies): pg_decode_host_stream_f32
    — ONE decode launch over the whole batch, fed `stream_chunk`-query pieces
    by the copy engine and draining its outputs piece by piece, so H2D, the
    kernel and D2H overlap without per-chunk launch costs.  Needs device
    buffers for the whole batch (20 B/query for 2-D, 3 outputs).
    Chunked mode (stream=False, or the exact / FFMA engines):
    pg_decode_host_f32 — successive chunks on three streams, two buffer
    slots, event-ordered."""

    @on_device
    def __init__(self, inf: InferenceModel, chunk: int = 1 << 21, exact: bool = False,
                 stream: bool | None = None, stream_chunk: int = 1 << 19, cells: bool = True):
        if not inf.fast:
            raise ValueError("host decode needs the fused [32,64,64,<=4] shape")
        if stream_chunk < 128 or stream_chunk & (stream_chunk - 1):
            raise ValueError("stream_chunk must be a power of two >= 128")
        self.inf, self.chunk, self.exact, self.stream_chunk = inf, chunk, exact, stream_chunk
        self.cells = cells
        d, od = inf.hyper.d, inf.out_dim
        ok = bool(_lib.lib().pg_decode_stream_supported(inf.grid, inf.mlp_desc, _flags(inf, exact)))
        if stream and not ok:
            raise ValueError("streaming host decode is not available for this model / device")
        self.streaming = ok if stream is None else bool(stream)
        self.s_in = torch.cuda.Stream(device=inf.device)
        self.s_k = torch.cuda.Stream(device=inf.device)
        self.s_out = torch.cuda.Stream(device=inf.device)
        self._cap = 0
        self.fallbacks = 0
        if not self.streaming:
            self.d_xs = torch.empty(2 * chunk * d, dtype=torch.float32, device=inf.device)
            self.d_out = torch.empty(2 * chunk * od, dtype=torch.float32, device=inf.device)

    def _reserve(self, B: int) -> None:
        if B <= self._cap:
            return
        inf = self.inf
        self.d_xs = torch.empty(B * inf.hyper.d, dtype=torch.float32, device=inf.device)
        self.d_out = torch.empty(B * inf.out_dim, dtype=torch.float32, device=inf.device)
        n = -(-B // self.stream_chunk)
        # [ready per chunk | done per chunk | host-fallback count]
        self.d_flags = torch.empty(2 * n + 1, dtype=torch.int32, device=inf.device)
        self._cap = B

    @on_device
    def __call__(self, h_xs: torch.Tensor, h_out: torch.Tensor) -> torch.Tensor:
        inf = self.inf
        self.fallbacks = 0
        if h_xs.shape[0] == 0:
            return h_out
        assert h_xs.is_pinned() and h_out.is_pinned(), "host buffers must be pinned"
        # the model's tables (to_inference, deserialize) and its cell cache
        # (built on first use) are written on the caller's stream: order this
        # decode's streams after it
        cells = inf.cells() if self.cells else None
        cur = torch.cuda.current_stream(inf.device)
        for s in (self.s_in, self.s_k, self.s_out):
            s.wait_stream(cur)
        streams = (_lib.ctypes.c_void_p(self.s_in.cuda_stream), _lib.ctypes.c_void_p(self.s_k.cuda_stream),
                   _lib.ctypes.c_void_p(self.s_out.cuda_stream))
        if self.streaming:
            B = h_xs.shape[0]
            self._reserve(B)
            if cells is not None:
                _lib.call("pg_decode_host_stream_cells_f32", inf.grid, inf.mlp_desc, _lib.ptr(h_xs), B,
                          _lib.ptr(inf.feats16), _lib.ptr(inf.baked), _lib.ptr(inf.params),
                          _flags(inf, self.exact), cells, self.stream_chunk, _lib.ptr(self.d_xs),
                          _lib.ptr(self.d_out), _lib.ptr(self.d_flags), _lib.ptr(h_out), *streams)
            else:
                _lib.call("pg_decode_host_stream_f32", inf.grid, inf.mlp_desc, _lib.ptr(h_xs), B,
                          _lib.ptr(inf.feats16), _lib.ptr(inf.baked), _lib.ptr(inf.params),
                          _flags(inf, self.exact), self.stream_chunk, _lib.ptr(self.d_xs), _lib.ptr(self.d_out),
                          _lib.ptr(self.d_flags), _lib.ptr(h_out), *streams)
            n = -(-B // self.stream_chunk)
            self.fallbacks = int(self.d_flags[2 * n])   # pipelines that read inputs from host memory
            return h_out
        if cells is not None:
            _lib.call("pg_decode_host_cells_f32", inf.grid, inf.mlp_desc, _lib.ptr(h_xs), h_xs.shape[0],
                      _lib.ptr(inf.feats16), _lib.ptr(inf.baked), _lib.ptr(inf.params),
                      _flags(inf, self.exact), cells, self.chunk, _lib.ptr(self.d_xs), _lib.ptr(self.d_out),
                      _lib.ptr(h_out), *streams)
        else:
            _lib.call("pg_decode_host_f32", inf.grid, inf.mlp_desc, _lib.ptr(h_xs), h_xs.shape[0],
                      _lib.ptr(inf.feats16), _lib.ptr(inf.baked), _lib.ptr(inf.params),
                      _flags(inf, self.exact), self.chunk, _lib.ptr(self.d_xs), _lib.ptr(self.d_out),
                      _lib.ptr(h_out), *streams)
        return h_out
