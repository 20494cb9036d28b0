"""Time the C1 training step (2^18 samples) with the library at argv[1]
(A/B of kernel variants built into separate .so files)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2312_17241_b200 import _lib  # noqa: E402

import ctypes  # noqa: E402
_raw = ctypes.CDLL(sys.argv[1])
_lib._SIGS = {k: v for k, v in _lib._SIGS.items() if hasattr(_raw, k)}   # older builds lack newer entries
_lib._LIB = _lib.load(sys.argv[1])
import paper_2312_17241_b200 as pg  # noqa: E402
from tests.golden_util import smooth_image  # noqa: E402

import json  # noqa: E402
KW = json.loads(os.environ.get("CFG", '{"n_f": 4096, "n_c": 16384, "n_p": 4}'))   # default: C1
st = pg.TrainState(pg.init_model(pg.HyperParams(**KW), seed=0),
                   smooth_image(256, 256), pg.TrainConfig(batch_size=1 << 18, seed=0), sampler="device")
for _ in range(5):
    st.launch_step()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(20):
    st.launch_step()
e1.record()
torch.cuda.synchronize()
print(f"{sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}: {e0.elapsed_time(e1) / 20:.4f} ms/step, loss {st.loss_value():.6g}")
