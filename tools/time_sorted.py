"""Kernel-side effect of processing the C1 batch in spatial order: time
compute_grads on the same 2^18 samples in sampler order, raster order and
Morton (Z) order of their pixels."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1:   # A/B: the library at argv[1]
    import ctypes
    from paper_2312_17241_b200 import _lib
    _raw = ctypes.CDLL(sys.argv[1])
    _lib._SIGS = {k: v for k, v in _lib._SIGS.items() if hasattr(_raw, k)}
    _lib._LIB = _lib.load(sys.argv[1])
    print("lib", sys.argv[1])
import paper_2312_17241_b200 as pg  # noqa: E402
from tests.golden_util import smooth_image  # noqa: E402


def morton2(x, y):
    def spread(v):
        v = (v | (v << 8)) & 0x00FF00FF
        v = (v | (v << 4)) & 0x0F0F0F0F
        v = (v | (v << 2)) & 0x33333333
        v = (v | (v << 1)) & 0x55555555
        return v
    return spread(x) | (spread(y) << 1)


st = pg.TrainState(pg.init_model(pg.HyperParams(n_f=2**12, n_c=2**14, n_p=4), seed=0),
                   smooth_image(256, 256), pg.TrainConfig(batch_size=1 << 18, seed=0), sampler="device")
xs, tg = st.sample_batch()
xs, tg = xs.clone(), tg.clone()
pix = st.pix.clone().long()
orders = {"sampler": torch.arange(xs.shape[0], device="cuda"),
          "raster": torch.argsort(pix),
          "morton": torch.argsort(morton2(pix % 256, pix // 256))}
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for rep in range(2):
    for name, o in orders.items():
        x, t = xs[o].contiguous(), tg[o].contiguous()
        for _ in range(3):
            st.compute_grads(x, t)
        torch.cuda.synchronize()
        ev[0].record()
        for _ in range(20):
            st.compute_grads(x, t)
        ev[1].record()
        torch.cuda.synchronize()
        print(f"{name:8s} compute_grads {ev[0].elapsed_time(ev[1]) / 20:.4f} ms")
# sort cost for reference
ev[0].record()
for _ in range(20):
    torch.argsort(pix)
ev[1].record()
torch.cuda.synchronize()
print(f"torch.argsort(2^18) {ev[0].elapsed_time(ev[1]) / 20:.4f} ms")
