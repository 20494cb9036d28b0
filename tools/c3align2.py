"""One C3 training-kernel launch with conf/grads placed at a given delta (argv[1] MB)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402

hk = dict(d=3, n_f=2**8, n_c=2**16, n_p=4, n_max=512, out_dim=1)
B = 1 << 22
x, v = bench.field_points("c3", 2 * B, seed=1)
st = pg.FieldTrainState(pg.init_model(pg.HyperParams(**hk), seed=0), x, v, pg.TrainConfig(batch_size=B, seed=0))
m = st.model
conf0, grads0 = m.conf.clone(), m.grads.clone()
MB = 1 << 20
arena = torch.empty(96 * MB, dtype=torch.uint8, device="cuda")
align = (2 * MB - arena.data_ptr() % (2 * MB)) % (2 * MB)
og = int(float(sys.argv[1]) * MB)
m.conf = arena[align:align + conf0.numel() * 4].view(torch.float32).view(conf0.shape)
m.conf.copy_(conf0)
m.grads = arena[align + og:align + og + grads0.numel() * 4].view(torch.float32)
m.grads.copy_(grads0)
xs, tg = st.sample_batch()
for _ in range(3):
    st.compute_grads(xs, tg)
torch.cuda.synchronize()
print("done")
