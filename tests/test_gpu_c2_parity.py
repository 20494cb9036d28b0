"""GPU parity at the headline configuration (BASELINE configs[1], SURVEY
8(d) C2): the decode the bench times — n_c = 2^16, n_max = 8192, the default
shared-memory table plan (bit-packed baked indices for the levels that fit
64 KB, whole-range global gathers for the rest) — against the oracle's
restatement of the reference's decode_pixels (model_io.py:292-311) on the
same tables, at every C2 sweep point the bench reports.

Bars: the exact engine (reference operation order, what `decode_pixels`
runs by default) is bit-exact; the tcgen05 engine within rtol 1e-5 /
atol 1e-6 (test_backends.py:139-148, mlp_infer_rows vs batched).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from tests.test_gpu_parity import _edge_points  # noqa: E402

N_Q = 1 << 17


def _c2_pair(log2_nf, n_p, seed=0):
    """Device model built exactly as bench.inference_model (conf ~ N(0,1),
    full bake, features ~ 0.1 N(0,1)) and the oracle model holding the same
    host tables."""
    import paper_2312_17241_b200 as pg
    kw = dict(n_f=2 ** log2_nf, n_c=2 ** 16, n_p=n_p, n_max=8192)
    m = pg.init_model(pg.HyperParams(**kw), seed=seed)
    rng = np.random.default_rng(seed)
    with torch.no_grad():
        m.feats.copy_(torch.from_numpy((rng.standard_normal(tuple(m.feats.shape)) * 0.1).astype(np.float32)))
        if m.probed:
            m.conf.copy_(torch.from_numpy(rng.standard_normal(tuple(m.conf.shape)).astype(np.float32)))
            m.rebake_all()
    om = O.init_model(O.Hyper(**kw), seed=seed)
    host = m.to_host()
    for L in om.levels:
        L.feats[:] = host["feats"][L.level]
        if L.conf is not None:
            L.conf[:] = host["conf"][L.level]
            L.baked[:] = host["baked"][L.level]
            # the device bake is the reference's strict '>' argmax
            np.testing.assert_array_equal(L.baked, np.argmax(L.conf, axis=1))
    for i in range(3):
        om.W[i][:] = host["W"][i]
        om.b[i][:] = host["b"][i]
    return pg.to_inference(m), O.to_inference(om)


@pytest.mark.parametrize("n_p", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("log2_nf", [14, 16, 18])
def test_c2_decode_default_plan_vs_oracle(log2_nf, n_p):
    from paper_2312_17241_b200.decode import decode_device
    inf, oinf = _c2_pair(log2_nf, n_p)
    q = _edge_points(N_Q, 2, np.float32, seed=log2_nf * 31 + n_p,
                     res_list=(16, 64, 322, 512, 1024, 4096, 8192))
    want = O.decode_pixels(oinf, q)
    xs = torch.from_numpy(q).cuda()
    exact = decode_device(inf, xs, exact=True).cpu().numpy()
    np.testing.assert_array_equal(exact, want)
    fast = decode_device(inf, xs, exact=False).cpu().numpy()     # the bench's engine and plan
    np.testing.assert_allclose(fast, want, rtol=1e-5, atol=1e-6)
    # the drop-in numpy entry point (pinned streaming path for large batches)
    import paper_2312_17241_b200 as pg
    np.testing.assert_array_equal(pg.decode_pixels(inf, q), want)


@pytest.mark.parametrize("kw", [dict(n_f=2 ** 16, n_c=2 ** 16, n_p=4, n_max=8192),
                                dict(n_f=2 ** 14, n_c=2 ** 16, n_p=16, n_max=8192),
                                dict(n_f=2 ** 18, n_c=2 ** 16, n_p=1, n_max=8192),
                                dict(n_f=2 ** 12, n_c=2 ** 14, n_p=8),
                                dict(d=3, n_f=2 ** 12, n_c=2 ** 12, n_p=4, out_dim=1),
                                dict(d=3, n_f=2 ** 10, n_c=2 ** 10, n_p=2, out_dim=4, out_sigmoid=True)])
@pytest.mark.parametrize("mib", [1, 32])
def test_decode_cell_cache_bit_identical(kw, mib):
    """The decode cell cache (pg_cells: per-cell records of the resolved
    corner rows of the coarsest levels) changes where rows are read from,
    not their values or the blend order: cached == uncached bit for bit,
    device and streaming host paths, at a small and the default budget."""
    import paper_2312_17241_b200 as pg
    from paper_2312_17241_b200.decode import HostDecoder, decode_device
    m = pg.init_model(pg.HyperParams(**kw), seed=2)
    rng = np.random.default_rng(4)
    with torch.no_grad():
        m.feats.copy_(torch.from_numpy((rng.standard_normal(tuple(m.feats.shape)) * 0.1).astype(np.float32)))
        if m.probed:
            m.conf.copy_(torch.from_numpy(rng.standard_normal(tuple(m.conf.shape)).astype(np.float32)))
            m.rebake_all()
    inf = pg.to_inference(m)
    inf.cell_budget = mib << 20
    d = inf.hyper.d
    q = _edge_points(1 << 16, d, np.float32, seed=9)
    xs = torch.from_numpy(q).cuda()
    plain = decode_device(inf, xs, exact=False, cells=False).cpu().numpy()
    cached = decode_device(inf, xs, exact=False).cpu().numpy()
    assert inf.cell_cache_bytes > 0
    np.testing.assert_array_equal(cached, plain)
    hx = torch.from_numpy(q).pin_memory()
    ho = torch.full((q.shape[0], inf.out_dim), float("nan")).pin_memory()
    HostDecoder(inf, stream=True, stream_chunk=1 << 14)(hx, ho)
    np.testing.assert_array_equal(ho.numpy(), plain)
    # the CUDA-core engines (reference order — decode_pixels' default — and FFMA)
    for kw2 in (dict(exact=True), dict(exact=False, tensor=False)):
        a = decode_device(inf, xs, cells=False, **kw2).cpu().numpy()
        np.testing.assert_array_equal(decode_device(inf, xs, **kw2).cpu().numpy(), a)
    ho2 = torch.full((q.shape[0], inf.out_dim), float("nan")).pin_memory()
    HostDecoder(inf, exact=True, chunk=1 << 14)(hx, ho2)        # chunked host path, exact engine
    np.testing.assert_array_equal(ho2.numpy(), decode_device(inf, xs, exact=True, cells=False).cpu().numpy())


@pytest.mark.parametrize("exact", [True, False])
def test_numpy_decode_pipeline_chunks(exact, monkeypatch):
    """decode_pixels(inf, numpy): the chunked host pipeline (pinned slots,
    H2D / kernel / D2H on three streams, host copies overlapped) returns
    exactly the device decode for batches of one, two and many chunks incl. a
    ragged tail, and still raises DomainViolation for a bad chunk."""
    import paper_2312_17241_b200 as pg
    from paper_2312_17241_b200 import decode as dec
    monkeypatch.setattr(dec, "HOST_CHUNK", 1 << 16)
    inf, _ = _c2_pair(16, 4)
    for n in ((1 << 16) + 5, 2 << 16, (7 << 16) + 12345):
        q = np.random.default_rng(n).random((n, 2)).astype(np.float32)
        got = pg.decode_pixels(inf, q, exact=exact)
        want = dec.decode_device(inf, torch.from_numpy(q).cuda(), exact=exact).cpu().numpy()
        np.testing.assert_array_equal(got, want)
    q[5 << 16, 0] = -0.5
    with pytest.raises(pg.DomainViolation):
        pg.decode_pixels(inf, q, exact=exact)
