"""End-to-end decode through the drop-in numpy entry point, and the host-side
alternatives for feeding it (GPU box).  2^24 C2 queries per call.

  (a) decode_pixels(inf, numpy)            as shipped (exact and tcgen05)
  (b) numpy -> pinned staging (torch copy_) + HostDecoder streaming + copy out
  (c) cudaHostRegister the numpy buffers in place + HostDecoder streaming
  (d) the pinned-buffer HostDecoder alone (the bench's e2e, for reference)
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200.decode import HostDecoder  # noqa: E402

B = 1 << 24
_, inf = bench.inference_model(pg, pg.HyperParams(**bench.C2))
q = np.random.default_rng(1234).random((B, 2), dtype=np.float32)


def timeit(name, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    el = (time.perf_counter() - t0) / reps
    print(f"{name:58s} {el * 1e3:8.2f} ms  {B / el:.3e} q/s", flush=True)


timeit("(a) decode_pixels(inf, numpy) exact", lambda: pg.decode_pixels(inf, q))
timeit("(a) decode_pixels(inf, numpy, exact=False)", lambda: pg.decode_pixels(inf, q, exact=False))

hd = HostDecoder(inf)
px = torch.empty((B, 2)).pin_memory()
po = torch.empty((B, 3)).pin_memory()
out = np.empty((B, 3), np.float32)


def staged():
    px.copy_(torch.from_numpy(q))
    hd(px, po)
    torch.from_numpy(out).copy_(po)


timeit("(b) pinned staging + streaming decode", staged)
timeit("(d) pinned buffers, streaming decode only", lambda: hd(px, po))

cr = torch.cuda.cudart()
out2 = np.empty((B, 3), np.float32)


def registered():
    a = cr.cudaHostRegister(q.ctypes.data, q.nbytes, 0)
    b = cr.cudaHostRegister(out2.ctypes.data, out2.nbytes, 0)
    try:
        hd(torch.from_numpy(q), torch.from_numpy(out2))
    finally:
        cr.cudaHostUnregister(q.ctypes.data)
        cr.cudaHostUnregister(out2.ctypes.data)
    return a, b


try:
    t0 = time.perf_counter()
    cr.cudaHostRegister(q.ctypes.data, q.nbytes, 0)
    t1 = time.perf_counter()
    cr.cudaHostUnregister(q.ctypes.data)
    print(f"cudaHostRegister of 128 MiB: {(t1 - t0) * 1e3:.2f} ms")
    timeit("(c) cudaHostRegister in place + streaming decode", registered)
except Exception as e:  # noqa: BLE001
    print("(c) failed:", e)

t0 = time.perf_counter()
for _ in range(5):
    px.copy_(torch.from_numpy(q))
print(f"numpy -> pinned copy 128 MiB: {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms "
      f"(threads {torch.get_num_threads()})")
