"""Streaming host decode with PG_DEBUG_STREAM=1 (kernel time vs total), then
the same streaming kernel on resident inputs with every chunk flagged ready
(PG_DEBUG_STREAM_NOCOPY): separates the copies' effect from the kernel's."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200.decode import HostDecoder  # noqa: E402

os.environ["PG_DEBUG_STREAM"] = "1"
hyper = pg.HyperParams(**bench.C2)
_, inf = bench.inference_model(pg, hyper, seed=0)
B = bench.B_INFER
hx = torch.rand((B, 2), generator=torch.Generator().manual_seed(1)).pin_memory()
ho = torch.empty((B, 3)).pin_memory()
for lg in (18, 19):
    hd = HostDecoder(inf, stream=True, stream_chunk=1 << lg)
    for _ in range(3):
        t0 = time.perf_counter()
        hd(hx, ho)
        print(f"chunk 2^{lg}: wall {1e3 * (time.perf_counter() - t0):.3f} ms", flush=True)
    os.environ["PG_DEBUG_STREAM_NOCOPY"] = "1"      # inputs now resident in hd.d_xs
    for _ in range(2):
        hd(hx, ho)
    print("  ^ kernel only (resident inputs, all chunks ready)", flush=True)
    del os.environ["PG_DEBUG_STREAM_NOCOPY"]
