"""Where the time of decode_pixels(inf, numpy) goes (GPU box)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200 import decode as dec  # noqa: E402

B = 1 << 24
_, inf = bench.inference_model(pg, pg.HyperParams(**bench.C2))
q = np.random.default_rng(1234).random((B, 2), dtype=np.float32)
for exact in (False, True):
    pg.decode_pixels(inf, q, exact=exact)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        pg.decode_pixels(inf, q, exact=exact)
    print(f"exact={exact}: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms", flush=True)
# the same with per-stage host timings
import cProfile  # noqa: E402
import pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
pg.decode_pixels(inf, q, exact=False)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
