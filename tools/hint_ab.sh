for H in 1 0; do echo HINTS=$H; PG_DECODE_L2_HINTS=$H python - <<'PY'
import torch, bench, paper_2312_17241_b200 as pg
from paper_2312_17241_b200.decode import decode_device
B=1<<24
xs=torch.rand((B,2),device="cuda",generator=torch.Generator("cuda").manual_seed(1234)); out=torch.empty((B,3),device="cuda")
for kw in (bench.C2, dict(n_f=2**16,n_c=2**16,n_p=16,n_max=8192)):
  _,inf=bench.inference_model(pg,pg.HyperParams(**kw))
  for mib in (32,96):
    inf.cell_budget=mib<<20; inf.invalidate_cells()
    for _ in range(3): decode_device(inf,xs,out,exact=False)
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): decode_device(inf,xs,out,exact=False)
    e1.record(); torch.cuda.synchronize()
    print(kw, mib, "%.3e"%(B*20/(e0.elapsed_time(e1)*1e-3)))
PY
done
