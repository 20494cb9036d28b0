"""e2e streaming decode (pinned host in/out) vs stream_chunk (GPU box)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200.decode import HostDecoder  # noqa: E402

B = 1 << 24
_, inf = bench.inference_model(pg, pg.HyperParams(**bench.C2))
hx = torch.rand((B, 2), generator=torch.Generator().manual_seed(0)).pin_memory()
ho = torch.empty((B, 3)).pin_memory()
for sc in (1 << 18, 1 << 19, 1 << 20, 1 << 21):
    hd = HostDecoder(inf, stream_chunk=sc)
    for _ in range(3):
        hd(hx, ho)
    t0 = time.perf_counter()
    for _ in range(10):
        hd(hx, ho)
    el = (time.perf_counter() - t0) / 10
    print(f"stream_chunk {sc:8d}: {el * 1e3:.3f} ms  {B / el:.3e} q/s  fallbacks {hd.fallbacks}", flush=True)
