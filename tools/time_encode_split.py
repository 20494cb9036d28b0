"""Time the stand-alone fused encode kernels at C1 with 2^18 samples (used
to evaluate a split-kernel training step)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200.encoding import encode_backward_device, encode_forward_device  # noqa: E402

B = 1 << 18
m = pg.init_model(pg.HyperParams(n_f=2**12, n_c=2**14, n_p=4), seed=0)
xs = torch.rand((B, 2), device="cuda", generator=torch.Generator("cuda").manual_seed(1))
y = torch.empty((B, 32), device="cuda")
dy = torch.randn((B, 32), device="cuda") * 1e-4


def timed(fn, n=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


print(f"encode fwd  {timed(lambda: encode_forward_device(m, xs, y)) * 1e3:.1f} us")
print(f"encode bwd  {timed(lambda: encode_backward_device(m, xs, dy)) * 1e3:.1f} us")
