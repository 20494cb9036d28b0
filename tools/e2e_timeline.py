"""Timeline of the end-to-end host decode pipeline (same schedule as
pg_decode_host_f32: 3 streams, 2 slots, ramped chunks) rebuilt with torch
streams and events, to see where the e2e time goes: per chunk the H2D,
kernel and D2H start/end relative to the first H2D."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_17241_b200 as pg  # noqa: E402
from paper_2312_17241_b200.decode import decode_device  # noqa: E402

hyper = pg.HyperParams(**bench.C2)
_, inf = bench.inference_model(pg, hyper, seed=0)
B = bench.B_INFER
chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
hx = torch.rand((B, 2), generator=torch.Generator().manual_seed(1)).pin_memory()
ho = torch.empty((B, 3)).pin_memory()
dx = [torch.empty((chunk, 2), device="cuda") for _ in range(2)]
dout = [torch.empty((chunk, 3), device="cuda") for _ in range(2)]
si, sk, so = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def sizes():
    out, off = [], 0
    head = [chunk // 8, chunk // 4, chunk // 2]
    while off < B:
        n = head[len(out)] if len(out) < 3 else chunk
        rem = B - off
        if rem <= 2 * chunk and len(out) >= 3:   # halving tail
            n = max(rem // 2, chunk // 8) if rem > chunk // 8 else rem
        n = min(n, rem)
        out.append(n)
        off += n
    return out


def run(record):
    ev = []
    ev_in, ev_k, ev_out = [None, None], [None, None], [None, None]
    off = 0
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(si)
    for c, n in enumerate(sizes()):
        s = c & 1
        e = {k: torch.cuda.Event(enable_timing=True) for k in ("i0", "i1", "k0", "k1", "o0", "o1")}
        if c >= 2:
            si.wait_event(ev_k[s])
        e["i0"].record(si)
        with torch.cuda.stream(si):
            dx[s][:n].copy_(hx[off:off + n], non_blocking=True)
        e["i1"].record(si)
        ev_in[s] = e["i1"]
        sk.wait_event(ev_in[s])
        if c >= 2:
            sk.wait_event(ev_out[s])
        e["k0"].record(sk)
        with torch.cuda.stream(sk):
            decode_device(inf, dx[s][:n], dout[s][:n], exact=False)
        e["k1"].record(sk)
        ev_k[s] = e["k1"]
        so.wait_event(ev_k[s])
        e["o0"].record(so)
        with torch.cuda.stream(so):
            ho[off:off + n].copy_(dout[s][:n], non_blocking=True)
        e["o1"].record(so)
        ev_out[s] = e["o1"]
        ev.append((n, e))
        off += n
    torch.cuda.synchronize()
    if record:
        tot = t0.elapsed_time(ev[-1][1]["o1"])
        print(f"chunk {chunk}: total {tot:.3f} ms -> {B / tot / 1e-3:.4g} q/s")
        for n, e in ev:
            f = lambda k: t0.elapsed_time(e[k])
            print(f"  n={n:8d}  h2d {f('i0'):7.3f}-{f('i1'):7.3f}  kern {f('k0'):7.3f}-{f('k1'):7.3f} "
                  f"({f('k1') - f('k0'):6.3f})  d2h {f('o0'):7.3f}-{f('o1'):7.3f}")
    return ev


for _ in range(3):
    run(False)
run(True)
# kernel alone over the whole batch, for reference
xa = torch.empty((B, 2), device="cuda")
xa.copy_(hx)
oa = torch.empty((B, 3), device="cuda")
for _ in range(3):
    decode_device(inf, xa, oa, exact=False)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
decode_device(inf, xa, oa, exact=False)
b.record()
torch.cuda.synchronize()
print(f"one launch over all {B}: {a.elapsed_time(b):.3f} ms")
# chunked kernels alone (no copies in flight): tail effects vs DMA interference
for n in (1 << 19, 1 << 20, 1 << 21, 1 << 22):
    a.record()
    for lo in range(0, B, n):
        decode_device(inf, xa[lo:lo + n], oa[lo:lo + n], exact=False)
    b.record()
    torch.cuda.synchronize()
    print(f"chunks of {n}, kernels only: {a.elapsed_time(b):.3f} ms")
