"""Dump raw TMEM results of one UMMA self-test mode for layout analysis:
python tools/umma_probe.py MODE"""
import sys

import numpy as np
import torch

from paper_2312_17241_b200 import _lib

mode = int(sys.argv[1])
shapes = {1: ((128, 64), (128, 64)), 3: ((128, 128), (128, 64)), 4: ((64, 64), (64, 64))}
rng = np.random.default_rng(3)
ash, bsh = shapes[mode]
A = rng.standard_normal(ash).astype(np.float16).astype(np.float32)
B = rng.standard_normal(bsh).astype(np.float16).astype(np.float32)
tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
tD = torch.full((128, 64), np.nan, device="cuda")
_lib.call("pg_selftest_umma_tf32", _lib.ptr(tA), _lib.ptr(tB), _lib.ptr(tD), mode << 4, _lib.stream_ptr())
np.savez(f"gpurun_out/umma_probe{mode}.npz", A=A, B=B, D=tD.cpu().numpy())
print("saved", mode)
