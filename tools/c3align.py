"""C3 training-kernel time vs the placement of the confidence table and the
gradient buffer (investigating an allocation-dependent slowdown)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "c1":
    from tests.golden_util import smooth_image
    st = pg.TrainState(pg.init_model(pg.HyperParams(n_f=2**12, n_c=2**14, n_p=4), seed=0), smooth_image(256, 256),
                       pg.TrainConfig(batch_size=1 << 18, seed=0), sampler="device")
else:
    hk = dict(d=3, n_f=2**8, n_c=2**16, n_p=4, n_max=512, out_dim=1)
    B = 1 << 22
    x, v = bench.field_points("c3", 2 * B, seed=1)
    st = pg.FieldTrainState(pg.init_model(pg.HyperParams(**hk), seed=0), x, v,
                            pg.TrainConfig(batch_size=B, seed=0))
m = st.model
conf0, grads0 = m.conf.clone(), m.grads.clone()
MB = 1 << 20
arena = torch.empty(96 * MB, dtype=torch.uint8, device="cuda")
base = arena.data_ptr()
print("arena % 2MB", base % (2 * MB))


def place(off_conf, off_grads):
    m.conf = arena[off_conf:off_conf + conf0.numel() * 4].view(torch.float32).view(conf0.shape)
    m.conf.copy_(conf0)
    m.grads = arena[off_grads:off_grads + grads0.numel() * 4].view(torch.float32)
    m.grads.copy_(grads0)


def timed():
    for _ in range(2):
        st.launch_step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    xs, tg = st.sample_batch()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        st.compute_grads(xs, tg)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 3


align = (2 * MB - base % (2 * MB)) % (2 * MB)
for oc, og in [(0, 32 * MB), (0, 34 * MB), (0, 33 * MB), (0, 32 * MB + 65536), (65536, 32 * MB),
               (65536, 32 * MB + 65536), (4096, 32 * MB + 4096), (0, 48 * MB), (0, 40 * MB), (0, 36 * MB),
               (0, 18 * MB), (0, 16 * MB + 65536)]:
    place(align + oc, align + og)
    print(f"conf@+{oc // 1024}K grads@+{og / MB:.3f}MB  delta={(og - oc) / MB:.3f}MB  ->  {timed():.3f} ms")
