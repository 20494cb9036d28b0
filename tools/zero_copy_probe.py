"""Probe: the standard decode kernel reading coordinates from and writing
outputs to pinned host memory directly (zero-copy over PCIe, UVA)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200.decode import decode_device, HostDecoder  # noqa: E402

_, inf = bench.inference_model(pg, pg.HyperParams(**bench.C2), seed=0)
B = bench.B_INFER
hx = torch.rand((B, 2), generator=torch.Generator().manual_seed(1)).pin_memory()
ho = torch.empty((B, 3)).pin_memory()
for _ in range(2):
    decode_device(inf, hx, ho, exact=False)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    decode_device(inf, hx, ho, exact=False)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    print(f"zero-copy decode: {el * 1e3:.3f} ms  {B / el:.4g} q/s")
ref = decode_device(inf, hx.cuda(), exact=False).cpu()
print("equal to device decode:", bool(torch.equal(ref, ho)))
hd = HostDecoder(inf)
for _ in range(3):
    t0 = time.perf_counter()
    hd(hx, ho)
    el = time.perf_counter() - t0
    print(f"streaming HostDecoder: {el * 1e3:.3f} ms  {B / el:.4g} q/s")
from paper_2312_17241_b200 import _lib  # noqa: E402
from paper_2312_17241_b200.decode import _flags  # noqa: E402
ho2 = torch.full((B, 3), float("nan")).pin_memory()
for i in range(4):
    t0 = time.perf_counter()
    _lib.call("pg_decode_host_zc_f32", inf.grid, inf.mlp_desc, _lib.ptr(hx), B, _lib.ptr(inf.feats16),
              _lib.ptr(inf.baked), _lib.ptr(inf.params), _flags(inf, False), _lib.ptr(ho2), _lib.stream_ptr())
    el = time.perf_counter() - t0
    print(f"pg_decode_host_zc_f32 (prefetch): {el * 1e3:.3f} ms  {B / el:.4g} q/s")
print("zc equal to device decode:", bool(torch.equal(ref, ho2)))
