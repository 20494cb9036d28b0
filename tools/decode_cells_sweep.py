"""C2 decode q/s against the decode cell-cache budget (GPU box)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200.decode import decode_device  # noqa: E402

B = 1 << 24
xs = torch.rand((B, 2), device="cuda", generator=torch.Generator("cuda").manual_seed(1234))
out = torch.empty((B, 3), device="cuda")
cfgs = [dict(bench.C2)] + [dict(n_f=2 ** lnf, n_c=2 ** 16, n_p=n_p, n_max=8192)
                           for lnf in (14, 18) for n_p in (1, 4, 16)]
for kw in cfgs:
    _, inf = bench.inference_model(pg, pg.HyperParams(**kw))
    for mib in (0, 1, 4, 8, 16, 32, 64, 96):
        inf.cell_budget = mib << 20
        inf.invalidate_cells()
        for _ in range(3):
            decode_device(inf, xs, out, exact=False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            decode_device(inf, xs, out, exact=False)
        e1.record()
        torch.cuda.synchronize()
        print(f"{kw} cells {mib:3d} MiB ({inf.cell_cache_bytes / 2**20:6.1f} used): "
              f"{B * 10 / (e0.elapsed_time(e1) * 1e-3):.3e} q/s", flush=True)
