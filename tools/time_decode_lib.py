"""Time the C2 headline decode (2^24 queries, tcgen05) with the library at
argv[1] (A/B of kernel variants built into separate .so files)."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2312_17241_b200 import _lib  # noqa: E402

_raw = ctypes.CDLL(sys.argv[1])
_lib._SIGS = {k: v for k, v in _lib._SIGS.items() if hasattr(_raw, k)}
_lib._LIB = _lib.load(sys.argv[1])
import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200.decode import decode_device  # noqa: E402

_, inf = bench.inference_model(pg, pg.HyperParams(**bench.C2), seed=0)
g = torch.Generator(device="cuda").manual_seed(1234)
xs = torch.rand((1 << 24, 2), generator=g, device="cuda")
out = torch.empty((1 << 24, 3), device="cuda")
for _ in range(3):
    decode_device(inf, xs, out, exact=False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    decode_device(inf, xs, out, exact=False)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"{sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}: {ms:.4f} ms, {(1 << 24) / ms / 1e-3:.4g} q/s")
if len(sys.argv) > 3 and sys.argv[3] == "stream":
    from paper_2312_17241_b200.decode import HostDecoder
    hx = xs.cpu().pin_memory()
    ho = torch.empty((1 << 24, 3)).pin_memory()
    hd = HostDecoder(inf, stream=True, stream_chunk=1 << 18)
    import time
    for _ in range(3):
        hd(hx, ho)
    t0 = time.perf_counter()
    for _ in range(5):
        hd(hx, ho)
    el = (time.perf_counter() - t0) / 5
    print(f"  stream e2e: {el * 1e3:.4f} ms, {(1 << 24) / el:.4g} q/s")
    os.environ["PG_DEBUG_STREAM_NOCOPY"] = "1"
    e0.record()
    for _ in range(5):
        hd(hx, ho)
    e1.record()
    torch.cuda.synchronize()
    print(f"  stream kernel only: {e0.elapsed_time(e1) / 5:.4f} ms (incl. host sync per call)")
    del os.environ["PG_DEBUG_STREAM_NOCOPY"]
if len(sys.argv) > 3 and sys.argv[3] == "exact":
    for kw, name in ((dict(exact=True), "exact reference-order"), (dict(exact=False, tensor=False), "FFMA")):
        for _ in range(2):
            decode_device(inf, xs, out, **kw)
        e0.record()
        for _ in range(5):
            decode_device(inf, xs, out, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"  {name}: {ms:.4f} ms, {(1 << 24) / ms / 1e-3:.4g} q/s")
