"""C1 step time of every training mode: fast (3xTF32 ping-pong), exact_mlp
(OpenBLAS-order FFMA), reference_order (+ BLAS-order weight gradients),
deterministic."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_17241_b200 as pg  # noqa: E402
from tests.golden_util import smooth_image  # noqa: E402

for name, kw in (("fast", {}), ("exact_mlp", dict(exact_mlp=True)), ("reference_order", dict(reference_order=True)),
                 ("deterministic", dict(deterministic=True))):
    st = pg.TrainState(pg.init_model(pg.HyperParams(n_f=2**12, n_c=2**14, n_p=4), seed=0), smooth_image(256, 256),
                       pg.TrainConfig(batch_size=1 << 18, seed=0), sampler="device", **kw)
    for _ in range(3):
        st.launch_step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        st.launch_step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: {ms:.3f} ms/step  {(1 << 18) / ms / 1e-3:.3g} samples/s", flush=True)
