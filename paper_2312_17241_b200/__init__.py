"""B200-native learned-hash-probing hot path (arXiv 2312.17241).

Drop-in for the reference package ``probegrid``'s encoder / model / trainer /
decode entry points and its backend plugin protocol (``backend``), running
hand-written sm_100a CUDA through the C ABI in include/probegrid_b200.h.
Importing this package does not touch the GPU; the first kernel call loads
libprobegrid_b200.so and fails loudly if it or a CUDA device is missing.
"""

__version__ = "0.1.0"

from .errors import (BadMagic, DimensionMismatch, DomainViolation, InvalidHyperparameter,
                     InvariantViolation, ModelFileError, ProbeGridError, ShapeMismatch, StaleTrace,
                     TargetTooSmall, TrainingDiverged, TruncatedFile, UnbakedModel, UnsupportedFormat,
                     VersionMismatch)
from .hyper import (AUX_PRIMES, PRIMARY_PRIMES, HyperParams, LevelMode, LevelSpec,
                    build_level_specs, level_resolution)

__all__ = [
    "AUX_PRIMES", "PRIMARY_PRIMES", "HyperParams", "LevelMode", "LevelSpec", "build_level_specs",
    "level_resolution", "ProbeGridError", "InvalidHyperparameter", "DomainViolation",
    "ShapeMismatch", "StaleTrace", "TrainingDiverged", "UnbakedModel", "DimensionMismatch",
    "TargetTooSmall",
    "init_model", "Model", "encode_forward", "encode_backward", "TrainConfig", "TrainState", "fit",
    "to_inference", "decode_pixels", "decode_at", "decode_rect", "decode_image", "InferenceModel",
    "ModelFileError", "BadMagic", "VersionMismatch", "TruncatedFile", "InvariantViolation",
    "serialize", "deserialize", "read_header", "size_report", "SizeReport", "pack_indices",
    "unpack_indices", "HEADER_BYTES", "load", "save", "select_hyperparams",
    "expand_grid", "run_sweep", "write_csv", "SweepPoint", "psnr", "pareto_front",
    "NerfTrainState", "render", "composite", "orbit_rays", "sample_points",
    "UnsupportedFormat", "save_image", "load_image", "mlp_forward", "mlp_backward", "MlpCache",
]


def __getattr__(name):
    # lazy: these import torch-backed modules
    if name in ("init_model", "Model"):
        from . import grid_model
        return getattr(grid_model, name)
    if name in ("encode_forward", "encode_backward"):
        from . import encoding
        return getattr(encoding, name)
    if name in ("TrainConfig", "TrainState", "FieldTrainState", "fit", "adam_update", "select_hyperparams"):
        from . import train
        return getattr(train, name)
    if name in ("to_inference", "decode_pixels", "decode_at", "decode_rect", "decode_image",
                "InferenceModel", "TouchCounter", "HostDecoder"):
        from . import decode
        return getattr(decode, name)
    if name in ("NerfTrainState", "render", "composite", "orbit_rays", "sample_points"):
        from . import nerf
        return getattr(nerf, name)
    if name in ("expand_grid", "run_sweep", "write_csv", "SweepPoint", "psnr", "pareto_front", "CSV_COLUMNS"):
        from . import sweep
        return getattr(sweep, name)
    if name in ("serialize", "deserialize", "read_header", "size_report", "SizeReport", "pack_indices",
                "unpack_indices", "HEADER_BYTES", "parse", "load", "save"):
        from . import model_io
        return getattr(model_io, name)
    if name in ("save_image", "load_image"):
        from . import pngio
        return getattr(pngio, name)
    if name in ("mlp_forward", "mlp_backward", "MlpCache"):
        from . import mlp
        return getattr(mlp, name)
    raise AttributeError(name)
