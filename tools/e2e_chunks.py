"""Sweep HostDecoder chunk sizes on the C2 headline workload (end-to-end
from pinned host memory)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200.decode import HostDecoder  # noqa: E402

hyper = pg.HyperParams(**bench.C2)
_, inf = bench.inference_model(pg, hyper, seed=0)
B = bench.B_INFER
hx = torch.rand((B, 2), generator=torch.Generator().manual_seed(1)).pin_memory()
ho = torch.empty((B, 3)).pin_memory()
for lg in (19, 20, 21, 22):
    hd = HostDecoder(inf, chunk=1 << lg, stream=False)
    for _ in range(2):
        hd(hx, ho)
    t0 = time.perf_counter()
    for _ in range(5):
        hd(hx, ho)
    el = (time.perf_counter() - t0) / 5
    print(f"chunk 2^{lg}: {B / el:.4g} q/s ({el * 1e3:.3f} ms)", flush=True)

for lg in (16, 17, 18, 19, 20):
    hd = HostDecoder(inf, stream=True, stream_chunk=1 << lg)
    for _ in range(2):
        hd(hx, ho)
    t0 = time.perf_counter()
    for _ in range(5):
        hd(hx, ho)
    el = (time.perf_counter() - t0) / 5
    print(f"streaming, chunk 2^{lg}: {B / el:.4g} q/s ({el * 1e3:.3f} ms)", flush=True)
