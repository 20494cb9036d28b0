"""C3 (3-D SDF, 2^22 points) training step time with the library at argv[1]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17241_b200 import _lib  # noqa: E402

_lib._LIB = _lib.load(sys.argv[1])
import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402

hk = dict(d=3, n_f=2**8, n_c=2**16, n_p=4, n_max=512, out_dim=1)
B = 1 << 22
x, v = bench.field_points("c3", 2 * B, seed=1)
st = pg.FieldTrainState(pg.init_model(pg.HyperParams(**hk), seed=0), x, v, pg.TrainConfig(batch_size=B, seed=0))
for _ in range(3):
    st.launch_step()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    st.launch_step()
e1.record()
torch.cuda.synchronize()
print(sys.argv[2] if len(sys.argv) > 2 else "", "C3 ms/step", e0.elapsed_time(e1) / 5)
