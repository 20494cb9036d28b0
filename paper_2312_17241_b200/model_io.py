"""The ``.cngp`` model file on the GPU (model_io.py:40-277 of the reference,
FORMAT.md).

Same names and behaviour as the reference module: ``serialize``,
``deserialize``, ``read_header``, ``size_report`` / ``SizeReport``,
``pack_indices`` / ``unpack_indices``, ``HEADER_BYTES``, and the same typed
errors for malformed input (BadMagic, VersionMismatch, TruncatedFile,
InvariantViolation — all ModelFileError).  Validation happens on the host
(``parse``) before anything touches the device, so fuzzed input yields
typed errors, never a crash.

``deserialize`` uploads the payload as it lies in the file — binary16
feature tables, the probed levels' index blocks still bit-packed — and
expands the index blocks on the device (``pg_unpack_indices``); the result
is a device-resident ``InferenceModel`` whose decode is bit-identical to
the reference's decode of the same file.  ``serialize`` packs on the device
(``pg_pack_indices``) and is byte-identical to the reference's writer.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import BadMagic, InvariantViolation, TruncatedFile, UnbakedModel, VersionMismatch
from .hyper import HyperParams, LevelMode, build_level_specs

MAGIC = b"CNGP"
VERSION = 1
_HEADER = struct.Struct("<4sIBBBBIIIIIIIIII")
HEADER_BYTES = _HEADER.size  # 52


@dataclass(frozen=True)
class SizeReport:
    """Exact byte breakdown of a serialized model (model_io.py:47-60)."""

    header_bytes: int
    feature_bytes: int
    index_bytes: int
    mlp_bytes: int

    @property
    def total_bytes(self) -> int:
        return self.header_bytes + self.feature_bytes + self.index_bytes + self.mlp_bytes


def _log2(n: int) -> int:
    return int(n).bit_length() - 1


def _index_block_bytes(hyper: HyperParams) -> int:
    return 0 if hyper.n_p <= 1 else (hyper.n_c * _log2(hyper.n_p) + 7) // 8


def _mlp_param_count(hyper: HyperParams) -> int:
    w = hyper.mlp_widths()
    return sum(a * b + b for a, b in zip(w[:-1], w[1:]))


def size_report(hyper: HyperParams) -> SizeReport:
    """model_io.py:76-88: hashed levels carry an index block when N_p > 1."""
    hyper.validate()
    specs = build_level_specs(hyper.n_min, hyper.n_max, hyper.n_levels, hyper.n_f, hyper.d)
    n_hashed = sum(1 for s in specs if s.mode is LevelMode.HASHED)
    return SizeReport(header_bytes=HEADER_BYTES,
                      feature_bytes=hyper.n_levels * hyper.n_f * hyper.feature_dim * 2,
                      index_bytes=n_hashed * _index_block_bytes(hyper),
                      mlp_bytes=_mlp_param_count(hyper) * 2)


def pack_indices(entries: np.ndarray, n_p: int) -> bytes:
    """Host packing of one level's offsets at log2(n_p) bits, LSB-first
    (model_io.py:150-156)."""
    w = _log2(n_p)
    if w == 0:
        return b""
    bits = np.unpackbits(np.asarray(entries, np.uint8)[:, None], axis=1, bitorder="little")[:, :w]
    return np.packbits(bits.ravel(), bitorder="little").tobytes()


def unpack_indices(raw: bytes, n_c: int, n_p: int) -> np.ndarray:
    """Host inverse of pack_indices (model_io.py:159-165)."""
    w = _log2(n_p)
    if w == 0:
        return np.zeros(n_c, dtype=np.uint8)
    bits = np.unpackbits(np.frombuffer(raw, dtype=np.uint8), bitorder="little", count=n_c * w)
    return (bits.reshape(n_c, w).astype(np.uint16) @ (1 << np.arange(w, dtype=np.uint16))).astype(np.uint8)


def read_header(data: bytes):
    """Parse + validate the 52-byte header; returns (hyper, width, height)
    (model_io.py:190-226, same limits and error types)."""
    if len(data) < HEADER_BYTES:
        raise TruncatedFile(f"need {HEADER_BYTES} header bytes, have {len(data)}")
    (magic, version, d, n_levels, feature_dim, flags, n_min, n_max, n_f, n_c, n_p, n_neurons,
     n_hidden, out_dim, width, height) = _HEADER.unpack_from(data)
    if magic != MAGIC:
        raise BadMagic(f"bad magic {magic!r}")
    if version != VERSION:
        raise VersionMismatch(f"unsupported version {version}")
    if flags > 1:
        raise InvariantViolation(f"unknown flag bits 0x{flags:02x}")
    limits = [(d, 2, 3, "d"), (n_levels, 1, 64, "levels"), (feature_dim, 1, 16, "feature dim"),
              (n_min, 1, 2**24, "n_min"), (n_max, 1, 2**24, "n_max"), (n_f, 1, 2**24, "n_f"),
              (n_c, 1, 2**26, "n_c"), (n_p, 1, 256, "n_p"), (n_neurons, 1, 2**14, "neurons"),
              (n_hidden, 1, 16, "hidden layers"), (out_dim, 1, 64, "out dim"),
              (width, 0, 2**20, "width"), (height, 0, 2**20, "height")]
    for value, lo, hi, name in limits:
        if not lo <= value <= hi:
            raise InvariantViolation(f"{name}={value} outside [{lo}, {hi}]")
    try:
        hyper = HyperParams(n_f=n_f, n_c=n_c, n_p=n_p, n_levels=n_levels, feature_dim=feature_dim,
                            n_min=n_min, n_max=n_max, n_neurons=n_neurons, n_hidden_layers=n_hidden,
                            d=d, out_dim=out_dim, out_sigmoid=bool(flags & 1))
        hyper.validate()
    except Exception as exc:  # InvalidHyperparameter -> the file-format error type
        raise InvariantViolation(str(exc)) from None
    return hyper, width, height


@dataclass
class ParsedFile:
    """Host view of a validated file: payload slices, nothing copied yet."""

    hyper: HyperParams
    width: int
    height: int
    feats16: np.ndarray        # (L, n_f, F) float16
    probed: list               # levels carrying an index block
    packed: np.ndarray         # (len(probed), block_bytes) uint8, as in the file
    mlp16: np.ndarray          # flat fp16 [W0 | b0 | W1 | b1 | ...]


def parse(data: bytes) -> ParsedFile:
    """Validate a whole file on the host (model_io.py:229-277): header,
    exact payload size (TruncatedFile / trailing bytes), then slice it."""
    hyper, width, height = read_header(data)
    report = size_report(hyper)
    if len(data) < report.total_bytes:
        raise TruncatedFile(f"payload needs {report.total_bytes} bytes, file has {len(data)}")
    if len(data) > report.total_bytes:
        raise InvariantViolation(f"{len(data) - report.total_bytes} trailing bytes")
    specs = build_level_specs(hyper.n_min, hyper.n_max, hyper.n_levels, hyper.n_f, hyper.d)
    buf = np.frombuffer(data, dtype=np.uint8)
    pos = HEADER_BYTES
    fbytes = hyper.n_f * hyper.feature_dim * 2
    ibytes = _index_block_bytes(hyper)
    feats, probed, blocks = [], [], []
    for spec in specs:
        feats.append(buf[pos:pos + fbytes])
        pos += fbytes
        if spec.mode is LevelMode.HASHED and hyper.n_p > 1:
            probed.append(spec.level)
            blocks.append(buf[pos:pos + ibytes])
            pos += ibytes
    n_mlp = _mlp_param_count(hyper)
    mlp16 = np.frombuffer(data, dtype="<f2", count=n_mlp, offset=pos)
    pos += 2 * n_mlp
    assert pos == report.total_bytes
    feats16 = np.stack(feats).view("<f2").reshape(hyper.n_levels, hyper.n_f, hyper.feature_dim)
    packed = np.stack(blocks) if blocks else np.zeros((0, ibytes), np.uint8)
    return ParsedFile(hyper, width, height, feats16, probed, packed, mlp16)


def deserialize(data: bytes, device=None):
    """Validate on the host, upload the payload, unpack the index blocks on
    the device; returns a device-resident InferenceModel (model_io.py:229)."""
    from .decode import InferenceModel
    pf = parse(data)
    hyper = pf.hyper
    dev = torch.device(device or "cuda")
    feats16 = torch.from_numpy(np.ascontiguousarray(pf.feats16)).to(dev)
    baked = torch.empty((len(pf.probed), hyper.n_c), dtype=torch.uint8, device=dev)
    if pf.probed:
        packed = torch.from_numpy(np.ascontiguousarray(pf.packed)).to(dev)
        with torch.cuda.device(dev):
            _lib.call("pg_unpack_indices", _lib.ptr(packed), len(pf.probed), hyper.n_c,
                      _log2(hyper.n_p), _lib.ptr(baked), _lib.stream_ptr())
    params = torch.from_numpy(pf.mlp16.astype(np.float32)).to(dev)
    return InferenceModel(hyper, pf.width, pf.height, feats16, baked, pf.probed, params, dev)


def serialize(model) -> bytes:
    """Byte-identical to the reference's writer (model_io.py:168-187) for a
    device Model (downcast first, as the reference) or InferenceModel."""
    from .decode import InferenceModel, to_inference
    from .grid_model import Model
    if isinstance(model, Model):
        model = to_inference(model)
    if not isinstance(model, InferenceModel):
        raise TypeError("serialize expects a Model or an InferenceModel")
    inf, hyper = model, model.hyper
    specs = build_level_specs(hyper.n_min, hyper.n_max, hyper.n_levels, hyper.n_f, hyper.d)
    hashed = [s.level for s in specs if s.mode is LevelMode.HASHED]
    if hyper.n_p > 1 and list(inf.probed) != hashed:
        raise UnbakedModel("every hashed level needs baked indices when N_p > 1")
    w = _log2(hyper.n_p)
    ibytes = _index_block_bytes(hyper)
    packed = np.zeros((len(inf.probed), ibytes), np.uint8)
    if inf.probed and w > 0:
        dpk = torch.empty((len(inf.probed), ibytes), dtype=torch.uint8, device=inf.device)
        with torch.cuda.device(inf.device):
            _lib.call("pg_pack_indices", _lib.ptr(inf.baked), len(inf.probed), hyper.n_c, w,
                      _lib.ptr(dpk), _lib.stream_ptr())
        packed = dpk.cpu().numpy()
    feats = inf.feats16.cpu().numpy().astype("<f2", copy=False)
    mlp16 = inf.params.cpu().numpy().astype("<f2")   # fp16-rounded values: exact
    parts = [_HEADER.pack(MAGIC, VERSION, hyper.d, hyper.n_levels, hyper.feature_dim,
                          1 if hyper.out_sigmoid else 0, hyper.n_min, hyper.n_max, hyper.n_f,
                          hyper.n_c, hyper.n_p, hyper.n_neurons, hyper.n_hidden_layers,
                          hyper.out_dim, inf.width, inf.height)]
    slot = {lv: i for i, lv in enumerate(inf.probed)}
    for lv in range(hyper.n_levels):
        parts.append(feats[lv].tobytes())
        if lv in slot and w > 0:
            parts.append(packed[slot[lv]].tobytes())
    parts.append(mlp16.tobytes())
    out = b"".join(parts)
    assert len(out) == size_report(hyper).total_bytes
    return out


def load(path: str, device=None):
    with open(path, "rb") as f:
        return deserialize(f.read(), device)


def save(model, path: str) -> int:
    raw = serialize(model)
    with open(path, "wb") as f:
        f.write(raw)
    return len(raw)
