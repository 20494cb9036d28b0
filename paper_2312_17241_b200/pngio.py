"""8-bit RGB PNG output of decoded images (the
reference's pngio.py:34-41 ``save_image`` contract: (H, W, 3) values in
[0, 1] are clipped, scaled by 255 and rounded half-to-even to uint8).

The quantisation runs on the GPU when the pixels are a device tensor
(``pg_quantize_u8_f32``: the same float32 arithmetic numpy performs on a
float32 array, so the bytes are identical to the reference's), which also
cuts the device->host copy to one byte per channel; the PNG container is
written on the host with zlib (filter type 0 per row, one IDAT chunk).
``load_image`` reads 8-bit PNGs (any filter type; RGB, RGBA, grayscale).
"""

from __future__ import annotations

import struct
import zlib

import numpy as np

from .errors import UnsupportedFormat

_SIG = b"\x89PNG\r\n\x1a\n"


def _chunk(kind: bytes, data: bytes) -> bytes:
    return struct.pack(">I", len(data)) + kind + data + struct.pack(">I", zlib.crc32(kind + data) & 0xFFFFFFFF)


def quantize(pixels) -> np.ndarray:
    """(H, W, 3) floats -> uint8 as the reference (np.rint(clip(p, 0, 1) * 255)).
    Device tensors are quantised by a CUDA kernel and copied back as bytes."""
    try:
        import torch
        if isinstance(pixels, torch.Tensor):
            if pixels.ndim != 3 or pixels.shape[2] != 3:
                raise UnsupportedFormat(f"expected (H, W, 3) pixels, got {tuple(pixels.shape)}")
            if pixels.is_cuda:
                from . import _lib
                src = pixels.to(torch.float32).contiguous()
                out = torch.empty(src.shape, dtype=torch.uint8, device=src.device)
                with torch.cuda.device(src.device):
                    _lib.call("pg_quantize_u8_f32", _lib.ptr(src), src.numel(), _lib.ptr(out), _lib.stream_ptr())
                return out.cpu().numpy()
            pixels = pixels.numpy()
    except ImportError:
        pass
    pixels = np.asarray(pixels)
    if pixels.ndim != 3 or pixels.shape[2] != 3:
        raise UnsupportedFormat(f"expected (H, W, 3) pixels, got {pixels.shape}")
    return np.rint(np.clip(pixels, 0.0, 1.0) * 255.0).astype(np.uint8)


def encode_png(rgb8: np.ndarray, level: int = 6) -> bytes:
    """PNG bytes of an (H, W, 3) uint8 array."""
    h, w, _ = rgb8.shape
    rows = np.concatenate([np.zeros((h, 1), np.uint8), np.ascontiguousarray(rgb8).reshape(h, w * 3)], axis=1)
    ihdr = struct.pack(">IIBBBBB", w, h, 8, 2, 0, 0, 0)      # 8-bit truecolour, no interlace
    return _SIG + _chunk(b"IHDR", ihdr) + _chunk(b"IDAT", zlib.compress(rows.tobytes(), level)) + \
        _chunk(b"IEND", b"")


def save_image(path, pixels) -> None:
    """Write (H, W, 3) values in [0, 1] (numpy or CUDA tensor) as 8-bit RGB PNG."""
    with open(path, "wb") as f:
        f.write(encode_png(quantize(pixels)))


def _unfilter(raw: bytes, h: int, stride: int, bpp: int) -> np.ndarray:
    out = np.zeros((h, stride), np.uint8)
    prev = np.zeros(stride, np.int32)
    pos = 0
    for y in range(h):
        ft = raw[pos]
        line = np.frombuffer(raw, np.uint8, stride, pos + 1).astype(np.int32)
        pos += stride + 1
        if ft == 0:
            cur = line
        elif ft == 2:
            cur = (line + prev) & 0xFF
        else:   # sub / average / paeth depend on the reconstructed left pixel
            cur = np.zeros(stride, np.int32)
            for x in range(stride):
                a = cur[x - bpp] if x >= bpp else 0
                b = prev[x]
                c = prev[x - bpp] if x >= bpp else 0
                if ft == 1:
                    p = a
                elif ft == 3:
                    p = (a + b) >> 1
                elif ft == 4:
                    pa, pb, pc = abs(b - c), abs(a - c), abs(a + b - 2 * c)
                    p = a if pa <= pb and pa <= pc else (b if pb <= pc else c)
                else:
                    raise UnsupportedFormat(f"bad PNG filter type {ft}")
                cur[x] = (line[x] + p) & 0xFF
        out[y] = cur
        prev = cur
    return out


def load_image(path) -> np.ndarray:
    """Read an 8-bit PNG as (H, W, 3) float32 in [0, 1] (pngio.py:18-31:
    grayscale replicated to three channels, alpha dropped, 16-bit refused)."""
    data = open(path, "rb").read()
    if data[:8] != _SIG:
        raise UnsupportedFormat(f"{path}: not a PNG")
    pos, idat, hdr = 8, [], None
    while pos < len(data):
        n, kind = struct.unpack(">I4s", data[pos:pos + 8])
        body = data[pos + 8:pos + 8 + n]
        pos += 12 + n
        if kind == b"IHDR":
            hdr = struct.unpack(">IIBBBBB", body)
        elif kind == b"IDAT":
            idat.append(body)
        elif kind == b"IEND":
            break
    if hdr is None:
        raise UnsupportedFormat(f"{path}: no IHDR")
    w, h, depth, ctype, _, _, interlace = hdr
    chans = {0: 1, 2: 3, 4: 2, 6: 4}.get(ctype)
    if depth != 8 or chans is None or interlace:
        raise UnsupportedFormat(f"{path}: {depth}-bit colour type {ctype} unsupported (8-bit only)")
    px = _unfilter(zlib.decompress(b"".join(idat)), h, w * chans, chans).reshape(h, w, chans)
    rgb = np.repeat(px[:, :, :1], 3, axis=2) if chans <= 2 else px[:, :, :3]
    return rgb.astype(np.float32) / 255.0
