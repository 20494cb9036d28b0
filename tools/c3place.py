"""C3 training-step time vs the distance between the confidence table and the
gradient buffer, all placements in ONE process (one arena, 2 MiB aligned).

  python tools/c3place.py [delta_MB ...]

Prints one JSON line per delta: {"delta_mb": d, "ms": median of 5 compute_grads}.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402

deltas = [float(a) for a in sys.argv[1:]] or [16.06, 17, 18, 20, 24, 28, 32, 33, 34, 36, 40, 48, 56, 64, 80, 96]
hk = dict(d=3, n_f=2**8, n_c=2**16, n_p=4, n_max=512, out_dim=1)
B = 1 << 22
x, v = bench.field_points("c3", 2 * B, seed=1)
st = pg.FieldTrainState(pg.init_model(pg.HyperParams(**hk), seed=0), x, v, pg.TrainConfig(batch_size=B, seed=0))
m = st.model
conf0, grads0 = m.conf.clone(), m.grads.clone()
xs, tg = st.sample_batch()


def timed(n=5):
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st.compute_grads(xs, tg)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


for _ in range(3):
    st.compute_grads(xs, tg)
torch.cuda.synchronize()
print(json.dumps({"delta_mb": "separate", "conf_ptr_mod_2mb": m.conf.data_ptr() % (2 << 20),
                  "delta_actual_mb": (m.grads.data_ptr() - m.conf.data_ptr()) / 2**20, "ms": timed()}), flush=True)
MB = 1 << 20
arena = torch.empty(int(max(deltas) * MB) + 40 * MB, dtype=torch.uint8, device="cuda")
align = (2 * MB - arena.data_ptr() % (2 * MB)) % (2 * MB)
for d in deltas:
    og = int(d * MB) // 256 * 256
    m.conf = arena[align:align + conf0.numel() * 4].view(torch.float32).view(conf0.shape)
    m.conf.copy_(conf0)
    m.grads = arena[align + og:align + og + grads0.numel() * 4].view(torch.float32)
    m.grads.copy_(grads0)
    m._build_views()
    st.compute_grads(xs, tg)
    torch.cuda.synchronize()
    print(json.dumps({"delta_mb": d, "ms": timed()}), flush=True)
