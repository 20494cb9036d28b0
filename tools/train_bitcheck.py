"""dL/dy (bit-exact) and the step's gradients of fixed batches through the
fused fast training kernel, with the library at argv[1], saved to argv[2]
(.npz) — for checking that a layout-only kernel change leaves results
unchanged: compare two such files with argv[3] = the other file."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2312_17241_b200 import _lib  # noqa: E402
import ctypes  # noqa: E402
_raw = ctypes.CDLL(sys.argv[1])
_lib._SIGS = {k: v for k, v in _lib._SIGS.items() if hasattr(_raw, k)}
_lib._LIB = _lib.load(sys.argv[1])
import paper_2312_17241_b200 as pg  # noqa: E402
from tests.golden_util import smooth_image  # noqa: E402

CFGS = {"c1": dict(n_f=2**12, n_c=2**14, n_p=4), "default": dict(),
        "sig4": dict(d=3, n_f=2**8, n_c=2**12, n_p=8, out_dim=4, out_sigmoid=True)}
out = {}
for name, kw in CFGS.items():
    m = pg.init_model(pg.HyperParams(**kw), seed=3)
    B = 20000
    if m.hyper.d == 2:
        st = pg.TrainState(m, smooth_image(128, 128), pg.TrainConfig(batch_size=B, seed=1), sampler="device")
    else:
        rng = np.random.default_rng(1)
        st = pg.FieldTrainState(m, rng.random((B, 3)).astype(np.float32),
                                rng.random((B, m.hyper.out_dim)).astype(np.float32), pg.TrainConfig(batch_size=B, seed=1))
    with torch.no_grad():   # deterministic, non-trivial state (steps would not be: reductions)
        g = torch.Generator(device="cuda").manual_seed(5)
        m.feats.copy_(torch.randn(m.feats.shape, device="cuda", generator=g) * 0.1)
    xs, tg = st.sample_batch()
    dy = torch.empty((xs.shape[0], 32), device="cuda")
    st.loss_sum.zero_()
    for t in (m.gmlp, m.gfeats, m.gconf):
        if t is not None:
            t.zero_()
    st.compute_grads(xs, tg, dy_out=dy)
    torch.cuda.synchronize()
    out[name + "_dy"] = dy.cpu().numpy()
    out[name + "_gmlp"] = m.gmlp.cpu().numpy()
    out[name + "_params"] = m.mlp_params.cpu().numpy()
np.savez(sys.argv[2], **out)
if len(sys.argv) > 3:
    other = np.load(sys.argv[3])
    for k in out:
        a, b = out[k], other[k]
        if k.endswith("_dy") or k.endswith("_params"):
            print(k, "bit-identical" if np.array_equal(a.view(np.uint32), b.view(np.uint32)) else
                  f"DIFFERS max {np.abs(a - b).max():.3e}")
        else:
            print(k, f"max rel {np.abs(a - b).max() / np.abs(b).max():.3e}")
