"""Train-step times (ms) for a list of HyperParams configurations at a given
batch (device sampler, CUDA events, median of 5 blocks), for A/B runs of
kernel variants selected by environment knobs (e.g. PG_TRAIN_NO_PRIV=1)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2312_17241_b200 as pg  # noqa: E402
from tests.golden_util import smooth_image  # noqa: E402

CFGS = [dict(n_f=2**12, n_c=2**14, n_p=4), dict(n_f=2**8, n_c=2**12, n_p=1), dict(n_f=2**8, n_c=2**12, n_p=4),
        dict(n_f=2**8, n_c=2**12, n_p=16), dict(), dict(n_f=2**9, n_c=2**12, n_p=4)]
if os.environ.get("CFGS"):
    CFGS = json.loads(os.environ["CFGS"])
B = int(os.environ.get("B", 1 << 18))
img = smooth_image(256, 256)
res = []
for kw in CFGS:
    st = pg.TrainState(pg.init_model(pg.HyperParams(**kw), seed=0), img, pg.TrainConfig(batch_size=B, seed=0),
                       sampler="device")
    for _ in range(5):
        st.launch_step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        e0.record()
        for _ in range(10):
            st.launch_step()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 10)
    res.append({"cfg": kw or "HyperParams()", "B": B, "ms": float(np.median(ts)), "loss": st.loss_value()})
    print(json.dumps(res[-1]), flush=True)
