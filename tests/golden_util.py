"""Helpers shared by the golden-vector generator and the parity tests."""

import hashlib

import numpy as np


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def smooth_image(h=256, w=256):
    """SURVEY 8(d) C1 smooth target, sampled at pixel centres."""
    yy, xx = np.mgrid[0:h, 0:w]
    u = (xx + 0.5) / w
    v = (yy + 0.5) / h
    return np.stack([0.5 + 0.5 * np.sin(6 * np.pi * u) * np.cos(4 * np.pi * v), u,
                     0.5 + 0.25 * np.sin(10 * np.pi * (u + v))], -1).astype(np.float32)
