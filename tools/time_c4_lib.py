import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2312_17241_b200 import _lib
_lib._LIB = _lib.load(sys.argv[1])
import paper_2312_17241_b200 as pg
import bench
hk = dict(d=3, n_f=2**8, n_c=2**16, n_p=8, n_max=2048, out_dim=4)
m = pg.init_model(pg.HyperParams(**hk), seed=0)
x, v = bench.field_points("c4", 1 << 20, 0) if hasattr(bench, "field_points") else (None, None)
st = pg.FieldTrainState(m, x, v, pg.TrainConfig(batch_size=1 << 18, seed=0))
for _ in range(3): st.launch_step()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(10): st.launch_step()
e1.record(); torch.cuda.synchronize()
print(sys.argv[2], "C4 ms/step", e0.elapsed_time(e1) / 10)
