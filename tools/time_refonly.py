"""A few C1 reference_order steps (for an ncu launch list of the parity mode)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_17241_b200 as pg  # noqa: E402
from tests.golden_util import smooth_image  # noqa: E402

st = pg.TrainState(pg.init_model(pg.HyperParams(n_f=2**12, n_c=2**14, n_p=4), seed=0), smooth_image(256, 256),
                   pg.TrainConfig(batch_size=1 << 18, seed=0), sampler="device", reference_order=True)
for _ in range(3):
    st.launch_step()
torch.cuda.synchronize()
print("ok")
