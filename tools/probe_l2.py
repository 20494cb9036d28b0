"""The bench's L2 denominators on their own (for an ncu cross-check of the
coalesced stream probe: lts__t_bytes.sum.per_second)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

for mib in (8, 32):
    s, g = bench.measure_l2(None, torch, table_mib=mib)
    print(f"table {mib} MiB: L2 stream read {s:.0f} GB/s, random 8-B gathers {g:.0f} GB/s "
          f"({g * 1e9 / 8:.3e} gathers/s)")
