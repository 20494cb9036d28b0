"""ctypes binding of the C ABI in include/probegrid_b200.h.

The shared library is built in-tree (``paper_2312_17241_b200/libprobegrid_b200.so``,
see csrc/Makefile / __graft_entry__.build()).  There is no fallback: if the
library or a CUDA device is missing, :func:`lib` raises, loudly.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libprobegrid_b200.so")

PG_OK, PG_ERR_ARG, PG_ERR_CUDA, PG_ERR_DOMAIN = 0, 1, 2, 3
PG_MAX_LEVELS, PG_MAX_FEATURE, PG_MAX_PROBES, PG_MAX_LAYERS = 64, 16, 256, 17
PG_LEVEL_DENSE, PG_LEVEL_HASHED, PG_LEVEL_PROBED = 0, 1, 2
PG_EXACT_MLP, PG_SIGMOID, PG_SURROGATE, PG_HALF_FEATS, PG_NO_TENSOR = 1, 2, 4, 8, 16
PG_SMEM_TABLES, PG_NO_SMEM_TABLES = 32, 64
PG_COMPOSITE = 128
PG_TOUCH_ALL = 256


class PgGrid(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32),
        ("n_levels", ctypes.c_int32),
        ("feature_dim", ctypes.c_int32),
        ("n_f", ctypes.c_int32),
        ("n_c", ctypes.c_int32),
        ("log2_np", ctypes.c_int32),
        ("res", ctypes.c_int32 * PG_MAX_LEVELS),
        ("kind", ctypes.c_int32 * PG_MAX_LEVELS),
        ("slot", ctypes.c_int32 * PG_MAX_LEVELS),
        ("primary", ctypes.c_uint32 * 3),
        ("aux", ctypes.c_uint32 * 3),
    ]


class PgMlp(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("widths", ctypes.c_int32 * (PG_MAX_LAYERS + 1))]


class PgCells(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("off", ctypes.c_int64 * PG_MAX_LEVELS)]


class PgError(RuntimeError):
    """A non-zero status from the CUDA library (message from pg_last_error)."""


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_U32 = ctypes.c_uint32
_U64 = ctypes.c_uint64
_D = ctypes.c_double
_F = ctypes.c_float
_G = ctypes.POINTER(PgGrid)
_M = ctypes.POINTER(PgMlp)
_C = ctypes.POINTER(PgCells)

_SIGS = {}
for _t, _s in (("f32", _F), ("f64", _D)):
    _SIGS.update({
        f"pg_dense_fwd_{_t}": [_P, _I64, _I, _I64, _P, _I, _P, _P, _P, _P],
        f"pg_hashed_fwd_{_t}": [_P, _I64, _I, _I64, _U32, _P, _I, _P, _P, _P, _P, _P],
        f"pg_probed_fwd_{_t}": [_P, _I64, _I, _I64, _U32, _U32, _I, _P, _I, _P, _P, _P, _P, _P,
                                _P, _P, _P],
        f"pg_indexed_bwd_{_t}": [_P, _I64, _I, _P, _P, _I, _P, _P],
        f"pg_probed_bwd_{_t}": [_P, _I64, _I, _P, _P, _P, _I, _P, _I, _P, _P, _P, _P],
        f"pg_adam_rebake_rows_{_t}": [_P, _P, _P, _I, _P, _P, _I64, _P, _D, _D, _D, _D, _D, _D, _P],
        f"pg_mlp_infer_rows_{_t}": [_P, _I64, _M, _P, ctypes.c_uint, _P, _P, _P],
        f"pg_encode_fwd_{_t}": [_G, _P, _I64, _P, _P, _P, ctypes.c_uint, _P, _P, _P],
        f"pg_encode_bwd_{_t}": [_G, _P, _I64, _P, _P, _P, _P, _P, _P, _P],
        f"pg_mlp_train_{_t}": [_M, _P, _P, _I64, _P, _s, ctypes.c_uint, _P, _P, _P, _P, _P],
        f"pg_mlp_forward_{_t}": [_M, _P, _I64, _P, _P, _P, _P],
        f"pg_mlp_backward_{_t}": [_M, _P, _I64, _P, _P, _P, _P, _P, _P],
        f"pg_pixel_batch_{_t}": [_P, _I64, _I, _I, _P, _I, _U64, _U64, _P, _P, _P, _P],
        f"pg_adam_{_t}": [_P, _P, _P, _P, _I64, _I64, _D, _D, _D, _D, _P, _P],
        f"pg_lazy_adam_rebake_{_t}": [_P, _P, _P, _P, _P, _P, _I64, _I, _I64, _D, _D, _D, _D, _P, _P],
    })
_SIGS.update({
    "pg_dedup_rows": [_P, _I64, _I64, _P, _P, _P, _P, _P],
    "pg_decode_f32": [_G, _M, _P, _I64, _P, _P, _P, ctypes.c_uint, _P, _P, _P],
    "pg_decode_cells_f32": [_G, _M, _P, _I64, _P, _P, _P, ctypes.c_uint, _C, _P, _P, _P],
    "pg_decode_host_stream_cells_f32": [_G, _M, _P, _I64, _P, _P, _P, ctypes.c_uint, _C, _I64, _P, _P, _P, _P,
                                        _P, _P, _P],
    "pg_cells_build": [_G, _P, _P, _C, _P],
    "pg_cells_build_f32": [_G, _P, _P, _C, _P],
    "pg_decode_host_cells_f32": [_G, _M, _P, _I64, _P, _P, _P, ctypes.c_uint, _C, _I64, _P, _P, _P, _P, _P, _P],
    "pg_decode_host_f32": [_G, _M, _P, _I64, _P, _P, _P, ctypes.c_uint, _I64, _P, _P, _P, _P, _P, _P],
    "pg_touched_to_f32": [_P, _I64, _P, _P],
    "pg_composite_fwd_f32": [_P, _P, _I64, _I, _P, _P, _P],
    "pg_ray_samples_f32": [_P, _P, _I64, _I, _P, _P, _P],
    "pg_ray_samples_targets_f32": [_P, _P, _P, _I64, _I, _P, _P, _P, _P],
    "pg_decode_stream_supported": [_G, _M, ctypes.c_uint],
    "pg_decode_host_zc_f32": [_G, _M, _P, _I64, _P, _P, _P, ctypes.c_uint, _P, _P],
    "pg_decode_host_stream_f32": [_G, _M, _P, _I64, _P, _P, _P, ctypes.c_uint, _I64, _P, _P, _P, _P, _P, _P, _P],
    "pg_nerf_train_f32": [_M, _P, _P, _P, _I64, _I, _P, _F, _P, _P, _P, _P, _P],
    "pg_touched_from_f32": [_P, _I64, _P, _P],
    "pg_touched_to_f64": [_P, _I64, _P, _P],
    "pg_bake_rows_f32": [_P, _I64, _I, _P, _P],
    "pg_quantize_u8_f32": [_P, _I64, _P, _P],
    "pg_bake_rows_f64": [_P, _I64, _I, _P, _P],
    "pg_touched_from_f64": [_P, _I64, _P, _P],
    "pg_train_fused_f32": [_G, _M, _P, _P, _I64, _P, _P, _P, _P, _F, ctypes.c_uint, _P, _P, _P,
                           _P, _P, _P, _P],
    "pg_train_fused_rep_f32": [_G, _M, _P, _P, _I64, _P, _P, _P, _P, _F, ctypes.c_uint, _P, _P, _P,
                               _P, _P, _P, _P, _I, _P],
    "pg_train_fused_ex_f32": [_G, _M, _P, _P, _I64, _P, _P, _P, _P, _F, ctypes.c_uint, _P, _P, _P,
                              _P, _P, _P, _P, _I, _C, _P],
    "pg_train_fused_ref_f32": [_G, _M, _P, _P, _I64, _P, _P, _P, _P, _F, ctypes.c_uint, _P, _P,
                               _P, _P, _P, _P],
    "pg_mlp_wgrad_blas_f32": [_M, _P, _I64, _P, _P],
    "pg_train_fused_ref_det_f32": [_G, _M, _P, _P, _I64, _P, _P, _P, _P, _F, ctypes.c_uint, _P, _P,
                                   _P, _P, _P, _P],
    "pg_unpack_indices": [_P, _I64, _I64, _I, _P, _P],
    "pg_raster_coords_f32": [_I, _I, _I, _I, _I, _I, _P, _P],
    "pg_pack_indices": [_P, _I64, _I64, _I, _P, _P],
    "pg_encode_bwd_det_f32": [_G, _P, _I64, _P, _P, _P, _P, _P, _P, _P],
    "pg_mlp_train_det_f32": [_M, _P, _P, _I64, _P, _F, ctypes.c_uint, _P, _P, _P, _P, _P],
    "pg_train_fused_det_f32": [_G, _M, _P, _P, _I64, _P, _P, _P, _P, _F, ctypes.c_uint, _P, _P,
                               _P, _P, _P, _P, _P],
    "pg_fx_accumulate_f32": [_P, _I64, _P, _P],
    "pg_fx_loss": [_P, _P, _P],
    "pg_selftest_umma_tf32": [_P, _P, _P, _I, _P],
    "pg_probe_stream_read": [_P, _I64, _I, _P, _P],
    "pg_probe_gather": [_P, _I64, _I64, _U32, _P, _P],
})
_RESTYPE_I64 = {"pg_dedup_workspace_bytes": [_I64, _I64],
                "pg_cells_plan": [_G, _I64, _C],
                "pg_cells_plan_rows": [_G, _I64, _I, _C],
                "pg_mlp_train_workspace_floats": [_I64, _M],
                "pg_mlp_acts_floats": [_I64, _M]}

_LIB = None


def exported_symbols():
    """Names the header declares (used by the CPU test that the .so exports them)."""
    return sorted(list(_SIGS) + list(_RESTYPE_I64) +
                  ["pg_last_error", "pg_version", "pg_device_sm_count"])


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """dlopen the library and declare every signature (no device needed)."""
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    for name, args in _RESTYPE_I64.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int64
    lib.pg_last_error.restype = ctypes.c_char_p
    lib.pg_version.restype = ctypes.c_char_p
    lib.pg_device_sm_count.argtypes = [ctypes.c_int]
    return lib


def lib() -> ctypes.CDLL:
    """The loaded library; requires a CUDA device (fails loudly otherwise)."""
    global _LIB
    if _LIB is None:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("probegrid_b200 needs a CUDA device (B200, sm_100a); no CPU fallback")
        torch.cuda.init()
        _LIB = load()
    return _LIB


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point; raise PgError on failure."""
    fn = getattr(lib(), name)
    rc = fn(*args)
    if rc != PG_OK:
        msg = lib().pg_last_error().decode()
        if rc == PG_ERR_ARG:
            raise ValueError(f"{name}: {msg}")
        raise PgError(f"{name} failed ({rc}): {msg}")


def ptr(t) -> ctypes.c_void_p:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(t.data_ptr())


def _device_of(obj):
    for o in (obj, getattr(obj, "model", None), getattr(obj, "inf", None), getattr(obj, "state", None)):
        dev = getattr(o, "device", None)
        if dev is not None:
            return dev
    return None


def on_device(fn):
    """Run a host entry point with its object's CUDA device current.

    The library launches on the current device and on that device's current
    stream (stream_ptr), so a model living on cuda:1 must make cuda:1
    current around every call; the first positional argument (a Model,
    InferenceModel, TrainState, HostDecoder, or a tensor) names the device."""
    import functools

    @functools.wraps(fn)
    def wrapped(*args, **kw):
        import torch
        dev = _device_of(args[0]) if args else None
        if dev is None or torch.device(dev).type != "cuda":
            return fn(*args, **kw)
        with torch.cuda.device(dev):
            return fn(*args, **kw)
    return wrapped


def stream_ptr(stream=None) -> ctypes.c_void_p:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
