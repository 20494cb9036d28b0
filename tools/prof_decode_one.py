"""One C2 decode config, a few launches (for ncu): python tools/prof_decode_one.py LOG2NF NP"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200.decode import decode_device  # noqa: E402

log2nf = int(sys.argv[1]) if len(sys.argv) > 1 else 16
npb = int(sys.argv[2]) if len(sys.argv) > 2 else 4
B = 1 << 24
hyper = pg.HyperParams(**dict(bench.C2, n_f=2 ** log2nf, n_p=npb))
_, inf = bench.inference_model(pg, hyper, seed=0)
xs = torch.rand((B, 2), generator=torch.Generator(device="cuda").manual_seed(1234), device="cuda")
out = torch.empty((B, hyper.out_dim), device="cuda")
for _ in range(3):
    decode_device(inf, xs, out, exact=False)
torch.cuda.synchronize()
print("ok")
