#!/usr/bin/env python3
"""Benchmark of the learned-hash-probing hot path on B200 (BASELINE.json metric:
"encoded+MLP queries/sec and train samples/sec per GPU, % roofline").

Headline (``value``): encoded+MLP inference queries/s, whole job, on the
configs[1] workload (C2: 2-D gigapixel-style inference, 2^24 queries per GPU
per step, log2 n_f = 16, n_c = 2^16, N_p = 4, n_max = 8192, 16 levels, F = 2,
MLP [32, 64, 64, 3], fp16-stored tables).  A "step" = one fused decode of the
batch; inputs are resident in HBM and larger than L2 (128 MiB of
coordinates), tables stay L2-resident as in serving.  ``e2e`` = the same
metric through the C ABI's host-buffer decode (pinned host coordinates in,
pinned host outputs back, copies inside the timed region).  ``train`` = C1
training samples/s (256x256 image, n_f = 2^12, n_c = 2^14, N_p = 4, 2^18
samples per GPU per step, full step incl. both optimizers).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 runs under torchrun, one rank per GPU: queries shard across ranks with
no data-path collective (weak scaling); the training leg is data parallel
with one NCCL all-reduce per step.  Timing: CUDA events on the launching
stream, barrier + synchronize around the timed region, max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "encoded+MLP queries/sec and train samples/sec per GPU (1/2/4/8 B200), % roofline"
C2 = dict(n_f=2**16, n_c=2**16, n_p=4, n_max=8192)
C1 = dict(n_f=2**12, n_c=2**14, n_p=4)
B_INFER = 1 << 24
B_TRAIN = 1 << 18


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("bf16_tflops", 1590.0)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled every 20 ms through
    NVML (the library nvidia-smi reads) while the timed region runs."""

    def __init__(self, index):
        self.index, self.sm, self.mask, self.max_mhz = index, [], 0, None
        self._stop = threading.Event()
        self.err = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis else self.index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.nv = pynvml
        except Exception as e:  # pragma: no cover
            self.err = f"nvml unavailable: {e}"
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.mask |= int(get_reasons(self.h))
            except Exception as e:  # pragma: no cover
                self.err = str(e)
            time.sleep(0.02)

    def stop(self):
        if self.err and not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [self.err]}
        self._stop.set()
        self.thread.join(timeout=2)
        nv = self.nv
        bits = {nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap",
                nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                nv.nvmlClocksEventReasonHwPowerBrakeSlowdown: "hw_power_brake_slowdown"}
        reasons = sorted(n for bit, n in bits.items() if self.mask & bit)
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.sm)}


def ncu_traffic(kernel, units):
    """DRAM bytes per launch of `kernel` scaled to `units`, from the committed
    ncu capture summary (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            rec = json.load(f)[kernel]
        per_unit = (rec["dram_read_bytes"] + rec["dram_write_bytes"]) / rec["units_per_launch"]
        return per_unit * units
    except Exception:
        return None


# ------------------------------------------------------------------ config
def c2_config(world):
    """The workload both arms report (identical dicts: same_config)."""
    return {"workload": "C2 inference: 2-D probed hash grid decode, fused encode+MLP",
            "queries_per_gpu_per_step": B_INFER, "log2_n_f": 16, "n_c": 2**16, "n_p": 4,
            "n_levels": 16, "feature_dim": 2, "n_min": 16, "n_max": 8192, "mlp": [32, 64, 64, 3],
            "parallelism": f"query-sharded x{world}",
            "l2_policy": "inputs (128 MiB coords + 192 MiB outputs per GPU) larger than L2; "
                         "tables L2-resident"}


# ------------------------------------------------------------------ models
def inference_model(pg, hyper, seed=0):
    """conf ~ N(0,1) then full bake (uniform probes), features
    ~ 0.1 N(0,1), MLP from the reference init; fp16 downcast as to_inference."""
    import torch
    m = pg.init_model(hyper, seed=seed)
    rng = np.random.default_rng(seed)
    with torch.no_grad():
        m.feats.copy_(torch.from_numpy((rng.standard_normal(tuple(m.feats.shape)) * 0.1).astype(np.float32)))
        if m.probed:
            m.conf.copy_(torch.from_numpy(rng.standard_normal(tuple(m.conf.shape)).astype(np.float32)))
            m.rebake_all()
    return m, pg.to_inference(m)


def infer_bytes_per_query(hyper, n_probed, table_bytes_per_row):
    """Algorithmic bytes per query: coordinates in, 2^d feature
    rows per level, one baked byte per corner of each probed level, outputs."""
    C = 1 << hyper.d
    return (4 * hyper.d + hyper.n_levels * C * table_bytes_per_row + n_probed * C
            + 4 * hyper.out_dim)


def smem_baked_levels(hyper, n_probed, budget=65536):
    """Probed levels whose baked indices the decode kernel keeps bit-packed in
    shared memory (pg_decode_tc.cu plan_tables: automatic for N_p = 2, 4)."""
    lg = int(hyper.n_p).bit_length() - 1
    if lg not in (1, 2):
        return 0
    return min(n_probed, budget // (hyper.n_c * lg // 8))


def gathers_per_query(hyper, inf):
    """Random global gathers one C2 query issues in decode_umma_kernel: one
    16-byte record per level in the decode cell cache; else 2^d feature
    rows / probing ranges, plus 2^d baked bytes for probed levels whose
    baked indices are not in shared memory (the uncached probed levels,
    smallest first, within the 64 KB table budget)."""
    C = 1 << hyper.d
    cells = inf.cells()
    cached = [cells is not None and cells.off[lv] >= 0 for lv in range(hyper.n_levels)]
    probed_unc = [lv for lv in inf.probed if not cached[lv]]
    smem = smem_baked_levels(hyper, len(probed_unc))
    return sum(1 if c else C for c in cached) + C * (len(probed_unc) - smem)


def train_l2_ops_per_sample(hyper, n_probed):
    """Random L2 operations (gathers + reductions) one training sample issues
    in the fused step: forward 1 per dense/hashed corner, 2 per probed corner
    (baked byte + row or whole range); backward 1 reduction per dense/hashed
    corner, per probed corner the confidence row and probing range loads plus
    ceil(2 N_p / 4) feature and ceil(N_p / 4) confidence 16-byte reductions."""
    C, L, n_p = 1 << hyper.d, hyper.n_levels, hyper.n_p
    plain = L - n_probed
    fwd = C * (plain + 2 * n_probed)
    reds = -(-2 * n_p // 4) + -(-n_p // 4)
    bwd = C * (plain + n_probed * (2 + reds))
    return fwd + bwd


def train_bytes_per_sample(hyper, n_probed):
    """encode fwd + recompute-bwd bytes per training sample."""
    C, L, F, d, n_p = 1 << hyper.d, hyper.n_levels, hyper.feature_dim, hyper.d, hyper.n_p
    fwd = 4 * d + L * C * 4 * F + n_probed * C
    bwd = (4 * L * F + 4 * d + n_probed * C * (4 * n_p + 4 * F * n_p + 8 * F * n_p + 8 * n_p)
           + (L - n_probed) * C * 8 * F)
    return fwd + bwd


# ------------------------------------------------------------------ probes
def measure_l2(lib_call, torch, table_mib=8):
    """MEASURED L2 denominators: float4 streaming read over an L2-resident
    buffer and random 8-byte gathers from a table of the config's size."""
    from paper_2312_17241_b200 import _lib
    buf = torch.ones(table_mib * (1 << 20) // 4, dtype=torch.float32, device="cuda")
    sink = torch.zeros(1, device="cuda")
    reps = 50
    for _ in range(3):
        _lib.call("pg_probe_stream_read", _lib.ptr(buf), buf.numel() * 4, 2, _lib.ptr(sink), _lib.stream_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("pg_probe_stream_read", _lib.ptr(buf), buf.numel() * 4, reps, _lib.ptr(sink), _lib.stream_ptr())
    e1.record()
    torch.cuda.synchronize()
    stream_gbs = buf.numel() * 4 * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    entries = (table_mib * (1 << 20)) // 8
    nq = 1 << 26
    _lib.call("pg_probe_gather", _lib.ptr(buf), entries, nq, 7, _lib.ptr(sink), _lib.stream_ptr())
    e0.record()
    _lib.call("pg_probe_gather", _lib.ptr(buf), entries, nq, 9, _lib.ptr(sink), _lib.stream_ptr())
    e1.record()
    torch.cuda.synchronize()
    gather_gbs = nq * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9
    return stream_gbs, gather_gbs


# ------------------------------------------------------------------ CPU arm
class CpuDecode:
    """The reference's decode_pixels on the host: the reference's own compiled
    Cython core (oracle/_ref) when it was built, else the C port, driven by the
    oracle's restatement of model_io.decode_pixels; chunks of 16384 queries
    (model_io.py:45) spread over all host threads (the kernels release the
    GIL).  The model is built as bench.inference_model builds the GPU one."""

    def __init__(self, hyper, threads=None):
        from oracle import oracle as O
        self.O = O
        ref = O.reference_core_backend()
        self.kern, self.kind = (ref, "reference") if ref is not None else (O.CBackend, "port")
        om = O.init_model(O.Hyper(**hyper), seed=0)
        rng = np.random.default_rng(0)
        for L in om.levels:
            L.feats[:] = (rng.standard_normal(L.feats.shape) * 0.1).astype(np.float32)
        for L in om.levels:
            if L.conf is not None:
                L.conf[:] = rng.standard_normal(L.conf.shape).astype(np.float32)
                L.baked[:] = np.argmax(L.conf, axis=1)
        self.inf = O.to_inference(om)
        self.threads = threads or os.cpu_count() or 1

    def run(self, xs, budget_s=None):
        """Decode xs (all of it, or until budget_s); returns (queries, seconds)."""
        from concurrent.futures import ThreadPoolExecutor
        chunk = self.O.DECODE_CHUNK
        done = 0
        t0 = time.perf_counter()
        with ThreadPoolExecutor(self.threads) as ex:
            futs = [ex.submit(self.O.decode_pixels, self.inf, xs[lo:lo + chunk], self.kern)
                    for lo in range(0, xs.shape[0], chunk)]
            for lo, f in zip(range(0, xs.shape[0], chunk), futs):
                f.result()
                done += min(chunk, xs.shape[0] - lo)
                if budget_s is not None and time.perf_counter() - t0 > budget_s:
                    for g in futs:
                        g.cancel()
                    break
        return done, time.perf_counter() - t0


def cpu_decode_baseline(hyper, budget_s=15.0, sample=1 << 24, threads=None):
    """Bounded CPU sample of the headline workload (about budget_s seconds)."""
    cd = CpuDecode(hyper, threads)
    xs = np.random.default_rng(1234).random((sample, 2), dtype=np.float32)
    done, el = cd.run(xs, budget_s)
    return {"value": done / el, "unit": "queries/s", "cores": cd.threads, "kind": cd.kind,
            "sample": f"{done} of the same C2 queries (decode_pixels, {cd.O.DECODE_CHUNK}-query chunks, "
                      f"{cd.threads} threads, {el:.1f} s)"}


def cpu_train_baseline(budget_s=8.0):
    """Reference TrainState.step (C1, B=8192) on the host, median ms -> samples/s."""
    from oracle import oracle as O
    from tests.golden_util import smooth_image
    ref = O.reference_core_backend()
    kern, kind = (ref, "reference") if ref is not None else (O.CBackend, "port")
    st = O.TrainState(O.init_model(O.Hyper(**C1), 0), smooth_image(256, 256),
                      O.TrainCfg(batch_size=8192, seed=0), kern=kern)
    for _ in range(3):
        st.step()
    times = []
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < budget_s and len(times) < 400:
        a = time.perf_counter()
        st.step()
        times.append(time.perf_counter() - a)
    ms = float(np.median(times)) * 1e3
    return {"value": 8192 / (ms * 1e-3), "unit": "samples/s", "cores": 1, "kind": kind,
            "sample": f"{len(times)} TrainState.step at C1 B=8192, median {ms:.2f} ms "
                      "(encoding kernels single-threaded as shipped; BLAS threads for the MLP)"}


# ------------------------------------------------------------------ GPU arm
def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2312_17241_b200 as pg
    from paper_2312_17241_b200 import _lib
    from paper_2312_17241_b200.decode import HostDecoder, decode_device

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    hbm_peak, tensor_peak, peak_src = peaks()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------- inference (headline) ----------------
    hyper = pg.HyperParams(**C2)
    _, inf = inference_model(pg, hyper, seed=0)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    xs = torch.rand((B_INFER, 2), generator=g, device=dev)
    out = torch.empty((B_INFER, hyper.out_dim), device=dev)
    exact = args.exact
    for _ in range(args.warmup):
        decode_device(inf, xs, out, exact=exact)
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        decode_device(inf, xs, out, exact=exact)
    e1.record()
    torch.cuda.synchronize()
    barrier()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    clk = clocks.stop()
    ms_step = ms_total / args.steps
    qps = world * B_INFER / (ms_step * 1e-3)
    n_probed = len(inf.probed)
    bpq = infer_bytes_per_query(hyper, n_probed, table_bytes_per_row=2 * hyper.feature_dim)
    gpq = gathers_per_query(hyper, inf)
    achieved = B_INFER * bpq / (ms_step * 1e-3) / 1e9    # per GPU, per launch
    l2_stream, l2_gather = measure_l2(None, torch, table_mib=32)
    mlp_flops = 2 * sum(a * b for a, b in zip(inf.widths[:-1], inf.widths[1:]))

    # ---------------- raster-order queries (gigapixel-style image decode) ----------------
    # the same 2^24 queries as pixel centres of an 8192 x 2048 slab of an
    # 8192^2 image in raster order: neighbouring lanes share cells on the
    # coarse levels, the access pattern decode_image / decode_rect produce
    W_img, H_slab = 8192, B_INFER // 8192
    if os.environ.get("PG_BENCH_NO_RASTER"):
        W_img, H_slab = 8192, 1
    yy, xx = torch.meshgrid(torch.arange(H_slab, device=dev), torch.arange(W_img, device=dev),
                            indexing="ij")
    xs_r = torch.stack([(xx.reshape(-1).float() + 0.5) / W_img,
                        (yy.reshape(-1).float() + 0.5) / W_img], dim=1).contiguous()
    del xx, yy
    for _ in range(2):
        decode_device(inf, xs_r, out, exact=exact)
    e0.record()
    for _ in range(max(3, args.steps // 4)):
        decode_device(inf, xs_r, out, exact=exact)
    e1.record()
    torch.cuda.synchronize()
    raster_qps = world * B_INFER * max(3, args.steps // 4) / (e0.elapsed_time(e1) * 1e-3)
    del xs_r

    # ---------------- ablation: same decode, other MLP engines ----------------
    ablation = {}
    for name, kw in (("tcgen05_without_smem_baked_tables", dict(exact=False, smem_tables=False)),
                     ("cuda_core_fma", dict(exact=False, tensor=False)),
                     ("cuda_core_exact_reference_order", dict(exact=True))):
        for _ in range(2):
            decode_device(inf, xs, out, **kw)
        e0.record()
        for _ in range(max(3, args.steps // 4)):
            decode_device(inf, xs, out, **kw)
        e1.record()
        torch.cuda.synchronize()
        ablation[name] = B_INFER * max(3, args.steps // 4) / (e0.elapsed_time(e1) * 1e-3)

    # ---------------- e2e through the C ABI host-buffer decode ----------------
    hx = xs.cpu().pin_memory()
    ho = torch.empty((B_INFER, hyper.out_dim)).pin_memory()
    hd = HostDecoder(inf, chunk=1 << 21, exact=exact)
    torch.cuda.synchronize()
    for _ in range(max(1, args.warmup // 2)):
        hd(hx, ho)
    barrier()
    t0 = time.perf_counter()
    fallbacks = 0
    for _ in range(args.steps):
        hd(hx, ho)
        fallbacks += hd.fallbacks
    el = max_over_ranks(time.perf_counter() - t0)
    e2e_qps = world * B_INFER * args.steps / el
    e2e_launches = args.steps * (1 if hd.streaming else math.ceil(B_INFER / hd.chunk))

    # ---------------- e2e through the reference-facing numpy call ----------------
    # pg.decode_pixels(inf, numpy) is what a caller of the reference's
    # model_io.decode_pixels(inf, xs) switches to: numpy in, numpy out,
    # reference-order MLP by default (bit-identical), tcgen05 with exact=False
    q_np = hx.numpy()
    dropin = {}
    for name, ex in (("exact_reference_order", True), ("tcgen05", False)):
        pg.decode_pixels(inf, q_np, exact=ex)
        barrier()
        t0 = time.perf_counter()
        n_rep = max(3, args.steps // 4)
        for _ in range(n_rep):
            pg.decode_pixels(inf, q_np, exact=ex)
        dropin[name] = world * B_INFER * n_rep / max_over_ranks(time.perf_counter() - t0)

    # ---------------- training (C1, data parallel) ----------------
    train = run_train(args, pg, torch, dist, rank, world, dev, barrier, max_over_ranks, l2_stream,
                      l2_gather * 1e9 / 8)
    extra = {}
    if not args.quick:
        extra["train_c3"] = run_train_field(args, pg, torch, dist, rank, world, barrier, max_over_ranks, "c3",
                                            l2_stream)
        extra["train_c4"] = run_train_field(args, pg, torch, dist, rank, world, barrier, max_over_ranks, "c4",
                                            l2_stream)
        extra["train_c4_nerf"] = run_train_nerf(args, pg, torch, dist, rank, world, barrier, max_over_ranks,
                                                l2_stream)
        extra["train_c5"] = run_train_c5(args, pg, torch, dist, rank, world, barrier, max_over_ranks,
                                         l2_stream)
        if world == 1:
            extra["sweep_inference_c2_c5"] = run_sweep(args, pg, torch, decode_device)

    line = {
        "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (fp16-stored tables, fp32 math)", "data": "synthetic",
        "config": c2_config(world),
        "engine": {"kernel": "decode_umma_kernel", "probed_levels": n_probed,
                   "cell_cache_bytes": inf.cell_cache_bytes,
                   "cell_cached_levels": int(sum(1 for o in (inf.cells().off if inf.cells() else []) if o >= 0)),
                   "mlp_mode": ("exact (reference order, bit-identical)" if exact
                                else "tcgen05 kind::tf32 UMMA, 2-term split (fp32-level)")},
        "e2e": {"value": e2e_qps, "unit": "queries/s", "h2d_bytes_per_step": B_INFER * 2 * 4,
                "d2h_bytes_per_step": B_INFER * hyper.out_dim * 4,
                "host_fallback_pipelines": fallbacks,
                "dropin_decode_pixels_numpy_qps": dropin,
                "path": ("pg_decode_host_stream_cells_f32 (pinned host in/out; ONE decode launch fed 2^19-query "
                         "pieces by the copy engine through device flags, D2H of each piece on a stream wait "
                         "for its tile counter; 3 streams)" if hd.streaming else
                         "pg_decode_host_f32 (pinned host in/out; H2D, kernel, D2H on 3 event-ordered streams; "
                         "2^21-query chunks, ramped)")},
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak,
                     "binding_unit": "L1TEX/LSU random-gather issue and latency (ncu: issue 61%, L1TEX 66%, L2 34%, "
                                     "DRAM 3%, long-scoreboard stalls on the gathers; profiles/r02_*)",
                     "frac_by_unit": {"hbm": achieved / hbm_peak,
                                      "l2_stream": achieved / l2_stream,
                                      "random_gather_rate": qps / world * gpq / (l2_gather * 1e9 / 8)},
                     "traffic": ncu_traffic("decode_umma_kernel", B_INFER),
                     "kernel": "decode_umma_kernel", "bytes_per_query": bpq,
                     "peak_source": peak_src,
                     "l2_stream_read_gbs": l2_stream, "l2_random_gather_8B_gbs": l2_gather,
                     "frac_of_l2_stream": achieved / l2_stream,
                     "random_gathers_per_query": gpq,
                     "random_gather_rate_per_s": l2_gather * 1e9 / 8,
                     "frac_of_random_gather_rate": qps / world * gpq / (l2_gather * 1e9 / 8),
                     "mlp_tflops": qps / world * mlp_flops / 1e12,
                     "note": "table gathers are L2-resident: bytes are algorithmic gather bytes; "
                             "HBM streams only 20 B/query (coords + outputs). The binding limit is "
                             "the random-gather rate (pg_probe_gather, ~1 per SM per clock, measured "
                             "with 4-32 MiB tables, i.e. every gather an L1 miss): "
                             "random_gathers_per_query counts feature rows / probing ranges and baked "
                             "bytes not served from shared memory; the decode's coarse levels hit in "
                             "L1, so this fraction can exceed 1"},
        "clocks": clk,
        "ablation_queries_per_s": ablation,
        "raster_order_queries_per_s": raster_qps,
        "train": train,
        **extra,
    }
    return line, e2e_launches


def run_train(args, pg, torch, dist, rank, world, dev, barrier, max_over_ranks, l2_stream=None,
              l2_gather_rate=None):
    from tests.golden_util import smooth_image
    hyper = pg.HyperParams(**C1)
    model = pg.init_model(hyper, seed=0)
    img = smooth_image(256, 256)
    st = pg.TrainState(model, img, pg.TrainConfig(batch_size=B_TRAIN, seed=rank), sampler="device")
    dp = None
    if world > 1:
        from paper_2312_17241_b200.dist import DataParallel
        dp = DataParallel(st, dist)
    step = dp.launch_step if dp else st.launch_step
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    loss = st.loss_value()
    sps = world * B_TRAIN / (ms * 1e-3)
    n_probed = len(model.probed)
    bps = train_bytes_per_sample(hyper, n_probed)
    return {"metric": "train samples/s", "value": sps, "unit": "samples/s", "ms_per_step": ms,
            "config": {"workload": "C1 image fit step (fwd+bwd+dense Adam+lazy Adam/rebake)",
                       "samples_per_gpu_per_step": B_TRAIN, "image": "256x256 synthetic smooth",
                       "n_f": 2**12, "n_c": 2**14, "n_p": 4, "probed_levels": n_probed,
                       "sampler": "device", "parallelism": f"dp{world}"},
            "encode_bytes_per_sample": bps,
            "encode_algorithmic_gbs": B_TRAIN * bps / (ms * 1e-3) / 1e9,
            "encode_frac_of_l2_stream": (B_TRAIN * bps / (ms * 1e-3) / 1e9 / l2_stream) if l2_stream else None,
            "l2_random_ops_per_sample": train_l2_ops_per_sample(hyper, n_probed),
            "random_op_floor_ms": (train_l2_ops_per_sample(hyper, n_probed) * B_TRAIN / l2_gather_rate * 1e3
                                   if l2_gather_rate else None),
            "frac_of_random_op_floor": (train_l2_ops_per_sample(hyper, n_probed) * B_TRAIN / l2_gather_rate * 1e3 / ms
                                        if l2_gather_rate else None),
            "kernel": "train_mma_kernel (3xTF32 mma.sync MLP; exact_mlp=True selects the OpenBLAS-order FFMA kernel)",
            "traffic": ncu_traffic("train_mma_kernel", B_TRAIN),
            "last_loss": loss, "scaling": "weak"}


def run_train_c5(args, pg, torch, dist, rank, world, barrier, max_over_ranks, l2_stream=None):
    """configs[4] training side (C5): train samples/s of the unprobed hash grid
    (N_p = 1) against probed N_p = 2..16 at EQUAL feature-table size, on the
    shape of the reference's own overhead criterion (test_acceptance.py:227-256:
    n_f = 2^8, n_c = 2^12, B = 8192, step(N_p=16) <= 3.0 x step(N_p=1)), at the
    reference batch and at 2^18 samples per GPU; plus the default
    HyperParams() step (n_f = 2^6, N_p = 16)."""
    from paper_2312_17241_b200.dist import DataParallel
    from tests.golden_util import smooth_image
    img = smooth_image(256, 256)

    def one(hk, B):
        hyper = pg.HyperParams(**hk)
        st = pg.TrainState(pg.init_model(hyper, seed=0), img, pg.TrainConfig(batch_size=B, seed=rank),
                           sampler="device")
        step = DataParallel(st, dist).launch_step if world > 1 else st.launch_step
        ms = _time_steps(torch, step, max(5, args.steps), args.warmup, barrier, max_over_ranks)
        n_probed = len(st.model.probed)
        bps = train_bytes_per_sample(hyper, n_probed)
        r = {"n_f": hyper.n_f, "n_c": hyper.n_c, "n_p": hyper.n_p, "batch_per_gpu": B,
             "probed_levels": n_probed, "ms_per_step": ms, "samples_per_s": world * B / (ms * 1e-3),
             "encode_bytes_per_sample": bps, "encode_algorithmic_gbs": B * bps / (ms * 1e-3) / 1e9}
        if l2_stream:
            r["encode_frac_of_l2_stream"] = r["encode_algorithmic_gbs"] / l2_stream
        del st
        return r

    rows = []
    for B in (8192, B_TRAIN):
        for n_p in (1, 2, 4, 8, 16):
            rows.append(one(dict(n_f=2**8, n_c=2**12, n_p=n_p), B))
    env = {}
    for B in (8192, B_TRAIN):
        t = {r["n_p"]: r["ms_per_step"] for r in rows if r["batch_per_gpu"] == B}
        env[f"B{B}"] = {"step_np16_over_np1": t[16] / t[1], "bound": 3.0, "holds": t[16] / t[1] <= 3.0}
    default = one({}, B_TRAIN)
    return {"metric": "train samples/s", "unit": "samples/s",
            "config": {"workload": "C5 training: unprobed (N_p=1) vs probed at equal n_f",
                       "image": "256x256 synthetic smooth", "sampler": "device", "parallelism": f"dp{world}"},
            "points": rows, "overhead_envelope": env, "default_hyperparams_step": default}


def _time_steps(torch, step, steps, warmup, barrier, max_over_ranks):
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    barrier()
    return max_over_ranks(e0.elapsed_time(e1)) / steps


def field_points(kind, n, seed):
    """Synthetic 3-D training sets of SURVEY 8(d): C3 sphere SDF
    f(x) = |x - 0.5| - 0.3 with x ~ U[0,1)^3; C4 NeRF-style ray samples (rays
    from a radius-1.5 sphere around the centre, 64 uniform samples per ray
    inside [0.1, 0.9]^3) with an analytic (density, rgb) field."""
    rng = np.random.default_rng(seed)
    if kind == "c3":
        x = rng.random((n, 3), dtype=np.float32)
        v = (np.linalg.norm(x - 0.5, axis=1) - 0.3).astype(np.float32)[:, None]
        return x, v
    rays = n // 64
    d = rng.standard_normal((rays, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    origin = 0.5 + 1.5 * d
    t = np.sort(rng.random((rays, 64)), axis=1)
    pts = origin[:, None, :] - (0.6 + 1.8 * t)[:, :, None] * d[:, None, :]
    x = np.clip(pts.reshape(-1, 3), 0.1, 0.9).astype(np.float32)
    r2 = np.sum((x - 0.5) ** 2, axis=1, keepdims=True)
    v = np.concatenate([np.exp(-8.0 * r2), x], axis=1).astype(np.float32)
    return x, v


def run_train_field(args, pg, torch, dist, rank, world, barrier, max_over_ranks, kind, l2_stream=None):
    """C3 (3-D SDF, 2^22 points/step) or C4 (NeRF-style, N_p=8, out 4, 2^18
    samples/step) training step; data parallel under torchrun."""
    if kind == "c3":
        hk = dict(d=3, n_f=2**8, n_c=2**16, n_p=4, n_max=512, out_dim=1)
        B = 1 << 22
    else:
        hk = dict(d=3, n_f=2**8, n_c=2**16, n_p=8, n_max=2048, out_dim=4)
        B = 1 << 18
    hyper = pg.HyperParams(**hk)
    model = pg.init_model(hyper, seed=0)
    x, v = field_points(kind, 2 * B * world, seed=1)
    st = pg.FieldTrainState(model, x, v, pg.TrainConfig(batch_size=B, seed=rank))
    dp = None
    if world > 1:
        from paper_2312_17241_b200.dist import DataParallel
        dp = DataParallel(st, dist)
    steps = max(3, args.steps // 4)
    ms = _time_steps(torch, dp.launch_step if dp else st.launch_step, steps, args.warmup, barrier,
                     max_over_ranks)
    bps = train_bytes_per_sample(hyper, len(model.probed))
    return {"metric": "train samples/s", "value": world * B / (ms * 1e-3), "unit": "samples/s",
            "ms_per_step": ms, "steps": steps,
            "config": {"workload": f"{kind.upper()} 3-D field fit step", **hk,
                       "samples_per_gpu_per_step": B, "mlp": hyper.mlp_widths(),
                       "probed_levels": len(model.probed), "parallelism": f"dp{world}"},
            "encode_bytes_per_sample": bps, "encode_algorithmic_gbs": B * bps / (ms * 1e-3) / 1e9,
            "encode_frac_of_l2_stream": (B * bps / (ms * 1e-3) / 1e9 / l2_stream) if l2_stream else None,
            "last_loss": st.loss_value()}


def run_train_nerf(args, pg, torch, dist, rank, world, barrier, max_over_ranks, l2_stream=None):
    """C4 with the volume-compositing head: 2^12 rays x 64
    samples per GPU per step (2^18 samples), C4 encoding (N_p=8, out 4);
    targets rendered from an analytic field (soft ball of density, colour =
    position) through the same compositing.  Step = ray sampling, encode
    fwd, MLP + compositing + loss + backward, encode bwd, Adam, lazy Adam."""
    from paper_2312_17241_b200 import nerf
    hk = dict(d=3, n_f=2**8, n_c=2**16, n_p=8, n_max=2048, out_dim=4)
    R, S = 1 << 12, 64
    hyper = pg.HyperParams(**hk)
    model = pg.init_model(hyper, seed=0)
    o, d = nerf.orbit_rays(2 * R * world, seed=1)
    pts, deltas = nerf.sample_points(o, d, S)
    r = (pts - 0.5).norm(dim=1, keepdim=True)
    raw = torch.cat([12.0 * (0.3 - r) / 0.05, 4.0 * (pts - 0.5)], dim=1).contiguous()
    tgt = nerf.composite(raw, deltas, S)
    st = nerf.NerfTrainState(model, o, d, tgt, pg.TrainConfig(batch_size=R, seed=rank), n_samples=S)
    dp = None
    if world > 1:
        from paper_2312_17241_b200.dist import DataParallel
        dp = DataParallel(st, dist)
    steps = max(3, args.steps // 4)
    ms = _time_steps(torch, dp.launch_step if dp else st.launch_step, steps, args.warmup, barrier,
                     max_over_ranks)
    bps = train_bytes_per_sample(hyper, len(model.probed))
    gbs = R * S * bps / (ms * 1e-3) / 1e9
    return {"metric": "train rays/s", "value": world * R / (ms * 1e-3), "unit": "rays/s",
            "samples_per_s": world * R * S / (ms * 1e-3), "ms_per_step": ms, "steps": steps,
            "encode_bytes_per_sample": bps, "encode_algorithmic_gbs": gbs,
            "encode_frac_of_l2_stream": gbs / l2_stream if l2_stream else None,
            "config": {"workload": "C4 NeRF-style step with volume compositing", **hk,
                       "rays_per_gpu_per_step": R, "samples_per_ray": S, "mlp": hyper.mlp_widths(),
                       "probed_levels": len(model.probed), "parallelism": f"dp{world}",
                       "path": ("fused tensor-core step, one ray per 64-sample tile composited in-kernel "
                                "(pg_train_fused_f32 + PG_COMPOSITE)" if st.nerf_fused else
                                "generic encode kernels + pg_nerf_train_f32")},
            "last_loss": st.loss_value()}


def run_sweep(args, pg, torch, decode_device):
    """configs[1] / [4] sweep: decode q/s for log2 n_f in {14,16,18} x N_p in
    {2,4,8,16} (n_c = 2^16, n_max = 8192) and the unprobed N_p = 1 hash grid
    at equal table size (C5), 2^22 queries per call, tcgen05 path."""
    B = 1 << 22
    xs = torch.rand((B, 2), device="cuda", generator=torch.Generator("cuda").manual_seed(7))
    out = torch.empty((B, 3), device="cuda")
    res = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for lnf in (14, 16, 18):
        for n_p in (1, 2, 4, 8, 16):
            _, inf = inference_model(pg, pg.HyperParams(n_f=2**lnf, n_c=2**16, n_p=n_p, n_max=8192))
            for _ in range(3):
                decode_device(inf, xs, out, exact=False)
            e0.record()
            for _ in range(5):
                decode_device(inf, xs, out, exact=False)
            e1.record()
            torch.cuda.synchronize()
            res.append({"log2_n_f": lnf, "n_p": n_p, "probed_levels": len(inf.probed),
                        "queries_per_s": B * 5 / (e0.elapsed_time(e1) * 1e-3)})
            del inf
    return res


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU path on this host, rank 0
    only.  Every step decodes one full 2^24-query batch when the whole run
    fits in ~4 minutes at the rate the warm-up measured; otherwise each step
    is a bounded sample of the batch (stated in cpu_baseline.sample) and
    ms_per_step is the time of that sample."""
    if rank != 0:
        return None
    cd = CpuDecode(C2)
    xs = np.random.default_rng(1234).random((B_INFER, 2), dtype=np.float32)
    n_w, el_w = cd.run(xs[:1 << 20])                      # warm-up + rate estimate
    for _ in range(max(0, args.warmup - 1)):
        cd.run(xs[:1 << 20])
    rate = n_w / el_w
    per_step = B_INFER
    if args.steps * B_INFER / rate > 240.0:
        per_step = max(1 << 16, int(240.0 * rate / args.steps) // (1 << 14) * (1 << 14))
    times, n = [], 0
    for k in range(args.steps):
        lo = (k * per_step) % B_INFER
        done, el = cd.run(xs[lo:lo + per_step])
        times.append(el)
        n += done
    v = n / sum(times)
    sample = (f"every step the full {B_INFER}-query C2 batch" if per_step == B_INFER else
              f"every step a {per_step}-query slice of the {B_INFER}-query C2 batch")
    cb = {"value": v, "unit": "queries/s", "cores": cd.threads, "kind": cd.kind,
          "sample": f"{sample} (decode_pixels, {cd.O.DECODE_CHUNK}-query chunks on {cd.threads} threads)"}
    return {"metric": METRIC, "impl": "reference", "value": v, "unit": "queries/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.mean(times)) * 1e3, "queries_per_timed_step": per_step,
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": c2_config(world),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--exact", action="store_true", help="reference-order (bit-exact) MLP")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="headline + C1 train only")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))

    if args.impl == "reference":
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    # code-path check of the multi-rank bench on a one-GPU box (NOT a
    # measurement): PG_BENCH_SHARE_GPU=1 maps every rank to the visible GPUs
    # round-robin and PG_BENCH_DIST_BACKEND=gloo replaces NCCL (which refuses
    # two ranks on one device); the driver's N-GPU runs use neither
    if os.environ.get("PG_BENCH_SHARE_GPU") == "1":
        local_rank = local_rank % torch.cuda.device_count()
    if world > 1:
        torch.cuda.set_device(local_rank)
        backend = os.environ.get("PG_BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    line, _ = run_gpu(args, rank, world, local_rank)
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_decode_baseline(C2)
            line["train"]["cpu_baseline"] = cpu_train_baseline()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
