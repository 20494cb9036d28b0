"""A/B timing of the fused decode (tcgen05) on C2-family configs; prints one
JSON line per config.  argv: TAG [tables].  With "tables" the PG_SMEM_TABLES
variant runs; its budget / table kinds come from PG_DECODE_TABLE_BYTES and
PG_DECODE_TABLE_KINDS (read once per process)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200.decode import decode_device  # noqa: E402

B = 1 << 24
tag = sys.argv[1] if len(sys.argv) > 1 else "run"
tables = len(sys.argv) > 2 and sys.argv[2] == "tables"
for log2nf, npb in ((16, 4), (14, 4), (18, 4), (16, 1), (16, 2), (16, 8), (16, 16)):
    hyper = pg.HyperParams(**dict(bench.C2, n_f=2 ** log2nf, n_p=npb))
    _, inf = bench.inference_model(pg, hyper, seed=0)
    g = torch.Generator(device="cuda").manual_seed(1234)
    xs = torch.rand((B, 2), generator=g, device="cuda")
    out = torch.empty((B, hyper.out_dim), device="cuda")
    for _ in range(3):
        decode_device(inf, xs, out, exact=False, smem_tables=tables)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        decode_device(inf, xs, out, exact=False, smem_tables=tables)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    o = out[:1 << 16].cpu().numpy()
    key = f"gpurun_out/decode_ab_{log2nf}_{npb}.npy"
    diff = None
    if os.path.exists(key):
        diff = float(np.abs(np.load(key) - o).max())
    else:
        np.save(key, o)
    print(json.dumps({"tag": tag, "log2_nf": log2nf, "n_p": npb, "ms": round(ms, 4),
                      "qps": B / (ms * 1e-3), "maxdiff_vs_first": diff}), flush=True)
