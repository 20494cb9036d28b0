"""Forward of the fused training step with and without the per-step fp32 cell
cache: dL/dy must be bit-identical (same y values, same MLP)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200 import train as tr  # noqa: E402
from tests.golden_util import smooth_image  # noqa: E402

for kw in (dict(n_f=2**12, n_c=2**14, n_p=4), dict(), dict(n_f=2**8, n_c=2**12, n_p=16)):
    res = []
    for mb in ("0", "32"):
        os.environ["PG_TRAIN_CELL_MB"] = mb
        m = pg.init_model(pg.HyperParams(**kw), seed=0)
        rng = np.random.default_rng(0)
        with torch.no_grad():
            m.feats.copy_(torch.from_numpy((rng.standard_normal(tuple(m.feats.shape)) * 0.1).astype(np.float32)))
            if m.probed:
                m.conf.copy_(torch.from_numpy(rng.standard_normal(tuple(m.conf.shape)).astype(np.float32)))
                m.rebake_all()
        st = pg.TrainState(m, smooth_image(64, 64), pg.TrainConfig(batch_size=1 << 16, seed=0))
        print(kw, mb, "cells:", st._train_cells() is not None)
        xs, tg = st.sample_batch()
        dy = torch.empty((1 << 16, 32), device="cuda")
        st.loss_sum.zero_()
        st.compute_grads(xs, tg, dy_out=dy)
        res.append((dy.cpu().numpy(), float(st.loss_sum.item())))
    print(kw, "dy identical:", np.array_equal(res[0][0], res[1][0]), "max |diff|", np.abs(res[0][0] - res[1][0]).max(),
          "loss", res[0][1], res[1][1])
