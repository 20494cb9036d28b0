"""Per-phase cycle split of the fused training kernel (C1, 2^18 samples):
loads the PG_PHASE_PROF build (make -C paper_2312_17241_b200/csrc prof) and
prints, per phase, the share of CTA time spent between its barriers."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2312_17241_b200 import _lib  # noqa: E402

_lib._LIB = _lib.load(os.path.join(ROOT, "tools", "_prof", "libprobegrid_b200.so"))
import paper_2312_17241_b200 as pg  # noqa: E402
from tests.golden_util import smooth_image  # noqa: E402

EXACT = len(sys.argv) > 1 and sys.argv[1] == "exact"
NAMES = (["tile load", "encode fwd", "layer 1", "layer 2", "output+loss", "dW2", "delta2", "dW1",
          "delta1", "dW0", "dy", "encode bwd (+next-tile wait)"] if EXACT else
         ["stage next tile", "tile barrier (encode stragglers)", "layer 1", "layer 2", "output+loss",
          "dW2 + delta2", "delta2 store", "dW1 + dgrad2", "delta1 mask", "dW0 + dgrad1", "dy store",
          "fused encode bwd(t) + fwd(t+1)"])
READ = "pg_phase_prof_read" if EXACT else "pg_phase_prof_read_mma"
st = pg.TrainState(pg.init_model(pg.HyperParams(n_f=2**12, n_c=2**14, n_p=4), seed=0),
                   smooth_image(256, 256), pg.TrainConfig(batch_size=1 << 18, seed=0), sampler="device",
                   exact_mlp=EXACT)
for _ in range(5):
    st.launch_step()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
getattr(_lib._LIB, READ)(buf, 1)
for _ in range(10):
    st.launch_step()
torch.cuda.synchronize()
getattr(_lib._LIB, READ)(buf, 1)
v = np.array(buf[:12], dtype=np.float64)
tot = v.sum()
print(json.dumps({n: round(100 * x / tot, 2) for n, x in zip(NAMES, v)}, indent=1))
