"""Probe MN-major kind::tf32 descriptor variants with the UMMA self-test."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_17241_b200 import _lib  # noqa: E402

rng = np.random.default_rng(0)
A = rng.standard_normal((128, 32)).astype(np.float16).astype(np.float32)
B = rng.standard_normal((64, 32)).astype(np.float16).astype(np.float32)
ref = A.astype(np.float64) @ B.astype(np.float64).T
for mode in (6, 8):
    pass
for mode, var in ((10, 0),):
    tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    tD = torch.full((128, 64), float("nan"), device="cuda")
    _lib.call("pg_selftest_umma_tf32", _lib.ptr(tA), _lib.ptr(tB), _lib.ptr(tD), mode << 4, _lib.stream_ptr())
    D = tD.cpu().numpy()
    print(f"kind::f16 control, A MN-major: max abs err {np.abs(D - ref).max():.3e}, D[0,:4] {D[0, :4]}", flush=True)
for mode in (6, 8):
    for var in ((0, 1, 2, 3) if mode == 6 else (0, 1, 2)):
        tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        tD = torch.full((128, 64), float("nan"), device="cuda")
        _lib.call("pg_selftest_umma_tf32", _lib.ptr(tA), _lib.ptr(tB), _lib.ptr(tD), (mode << 4) | (var << 1),
                  _lib.stream_ptr())
        D = tD.cpu().numpy()
        err = np.abs(D - ref).max()
        print(f"mode {mode} variant {var}: max abs err {err:.3e}, D[0,:4] {D[0, :4]}, ref {ref[0, :4]}", flush=True)
