#!/bin/bash
# A/B of the decode variants / table budgets on one GPU (tools/decode_ab.py)
mkdir -p gpurun_out
rm -f gpurun_out/decode_ab_*.npy
python - <<'PY' > gpurun_out/decode_ab.log 2>&1
import torch, sys
sys.path.insert(0, ".")
import bench
for mib in (4, 32):
    s, g = bench.measure_l2(None, torch, table_mib=mib)
    print({"probe_table_mib": mib, "stream_gbs": s, "gather8_gbs": g, "gathers_per_s": g * 1e9 / 8})
PY
timeout 300 python tools/decode_ab.py default >> gpurun_out/decode_ab.log 2>&1
for k in 2 1; do
for b in 16384 32768 65536; do
  PG_DECODE_TABLE_KINDS=$k PG_DECODE_TABLE_BYTES=$b timeout 300 python tools/decode_ab.py tables_k${k}_$b tables >> gpurun_out/decode_ab.log 2>&1
done
done
cat gpurun_out/decode_ab.log
