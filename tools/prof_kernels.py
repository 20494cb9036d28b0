#!/usr/bin/env python3
"""Small driver for ncu: a few launches of the hot kernels at bench shapes.

    python tools/prof_kernels.py --what decode|train|all [--n 3]

Same models/shapes as bench.py (C2 decode, C1 train step), fewer
launches so `ncu --set full` replays stay short.  Numbers printed here are
never bench values (they may run under a profiler)."""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200.decode import decode_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="all", choices=["decode", "train", "all"])
    ap.add_argument("--n", type=int, default=3)
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--bq", type=int, default=1 << 24)
    ap.add_argument("--train-cfg", default=None, help="HyperParams kwargs as JSON (default: bench.C1)")
    args = ap.parse_args()
    if args.what in ("decode", "all"):
        _, inf = bench.inference_model(pg, pg.HyperParams(**bench.C2))
        xs = torch.rand((args.bq, 2), device="cuda", generator=torch.Generator("cuda").manual_seed(1))
        out = torch.empty((args.bq, 3), device="cuda")
        for _ in range(args.n):
            decode_device(inf, xs, out, exact=args.exact)
        torch.cuda.synchronize()
        print("decode ok", float(out[:4].sum()))
    if args.what in ("train", "all"):
        from tests.golden_util import smooth_image
        kw = json.loads(args.train_cfg) if args.train_cfg else bench.C1
        st = pg.TrainState(pg.init_model(pg.HyperParams(**kw)), smooth_image(),
                           pg.TrainConfig(batch_size=bench.B_TRAIN, seed=0), sampler="device")
        for _ in range(args.n):
            st.launch_step()
        torch.cuda.synchronize()
        print("train ok", st.loss_value())


if __name__ == "__main__":
    main()
