"""60-step C1 loss curves with and without the training cell cache, twice
each (float-atomic run-to-run spread vs the cache's effect)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2312_17241_b200 as pg  # noqa: E402
from tests.golden_util import smooth_image  # noqa: E402

curves = {}
for mb in ("0", "32"):
    for run in range(2):
        os.environ["PG_TRAIN_CELL_MB"] = mb
        st = pg.TrainState(pg.init_model(pg.HyperParams(n_f=2**12, n_c=2**14, n_p=4), seed=0), smooth_image(256, 256),
                           pg.TrainConfig(batch_size=1 << 18, seed=0), sampler="device")
        curves[(mb, run)] = np.array([st.step() for _ in range(60)])
ref = curves[("0", 0)]
for k, c in curves.items():
    rel = np.abs(c - ref) / ref
    print(k, "max rel vs (0,0): first 10", rel[:10].max(), "all 60", rel.max(), "final", c[-1])
