"""Fixed cost of one decode launch (prologue: weights + shared-memory tables,
TMEM alloc; epilogue; tail): time launches over growing batches."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200.decode import decode_device  # noqa: E402

hyper = pg.HyperParams(**bench.C2)
_, inf = bench.inference_model(pg, hyper, seed=0)
x = torch.rand((1 << 22, 2), device="cuda")
o = torch.empty((1 << 22, 3), device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for tables in (None, False):
    for n in (128, 148 * 3 * 128, 148 * 3 * 128 * 4, 1 << 20, 1 << 22):
        for _ in range(3):
            decode_device(inf, x[:n], o[:n], exact=False, smem_tables=tables)
        a.record()
        for _ in range(20):
            decode_device(inf, x[:n], o[:n], exact=False, smem_tables=tables)
        b.record()
        torch.cuda.synchronize()
        print(f"tables={tables} n={n:8d}: {a.elapsed_time(b) / 20 * 1e3:9.1f} us")
