"""The .cngp format on the GPU: device load of files written by the REAL
reference, device unpack/pack of the index blocks, decode bit-exact vs the
reference's decode_pixels of the same file, byte-identical round trips
(test_model_io.py TestSerializeRoundTrip, FORMAT.md)."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "cngp_files.npz"))
NAMES = ["np4", "np16", "np8_d3", "np2_sig_f4", "np1"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", NAMES)
def test_reference_file_device_load_and_decode(name):
    import paper_2312_17241_b200 as pg
    raw = bytes(GOLD[f"{name}_file"])
    inf = pg.deserialize(raw)
    # index blocks expanded on the device == the reference's unpack
    np.testing.assert_array_equal(inf.baked.cpu().numpy(), GOLD[f"{name}_baked"])
    got = pg.decode_pixels(inf, GOLD[f"{name}_xs"])          # exact (reference-order) decode
    want = GOLD[f"{name}_decode"]
    if inf.fast:
        np.testing.assert_array_equal(got, want)
    else:  # generic MLP shapes (F = 4, sigmoid): test_decode_generic_shape_matches_oracle bar
        np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-7)
    # the tensor-core decode of the same file
    from paper_2312_17241_b200.decode import decode_device
    fast = decode_device(inf, torch.from_numpy(GOLD[f"{name}_xs"]).cuda(), exact=False).cpu().numpy()
    np.testing.assert_allclose(fast, want, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("name", NAMES + ["format_example"])
def test_serialize_round_trip_byte_identical(name):
    import paper_2312_17241_b200 as pg
    raw = bytes(GOLD[f"{name}_file"])
    assert pg.serialize(pg.deserialize(raw)) == raw


@pytest.mark.parametrize("w", list(range(1, 9)))
def test_device_pack_unpack_matches_host(w):
    from paper_2312_17241_b200 import _lib
    from paper_2312_17241_b200 import model_io as mio
    rng = np.random.default_rng(w)
    for n_c in (1, 5, 8, 33, 1000, 4097):
        rows = 3
        e = rng.integers(0, 1 << w, size=(rows, n_c)).astype(np.uint8)
        nb = (n_c * w + 7) // 8
        de = torch.from_numpy(e).cuda()
        dp = torch.empty((rows, nb), dtype=torch.uint8, device="cuda")
        _lib.call("pg_pack_indices", _lib.ptr(de), rows, n_c, w, _lib.ptr(dp), _lib.stream_ptr())
        host = np.stack([np.frombuffer(mio.pack_indices(e[r], 1 << w), np.uint8) for r in range(rows)])
        np.testing.assert_array_equal(dp.cpu().numpy(), host)
        du = torch.empty((rows, n_c), dtype=torch.uint8, device="cuda")
        _lib.call("pg_unpack_indices", _lib.ptr(dp), rows, n_c, w, _lib.ptr(du), _lib.stream_ptr())
        np.testing.assert_array_equal(du.cpu().numpy(), e)


def test_trained_model_file_round_trip(tmp_path):
    """A model trained on the GPU serializes into a valid reference-format file
    whose decode equals the in-memory model's (test_model_io.py:107-112)."""
    import paper_2312_17241_b200 as pg
    from paper_2312_17241_b200 import model_io as mio
    hyper = pg.HyperParams(n_f=64, n_c=256, n_p=4, n_levels=4, n_min=4, n_max=16, n_neurons=16)
    img = np.random.default_rng(1).random((16, 16, 3)).astype(np.float32)
    res = pg.fit(img, hyper, pg.TrainConfig(steps=15, batch_size=128, seed=1))
    path = str(tmp_path / "m.cngp")
    n = pg.save(res.inference, path)
    assert n == mio.size_report(hyper).total_bytes
    clone = pg.load(path)
    xs = np.random.default_rng(2).random((64, 2)).astype(np.float32)
    np.testing.assert_array_equal(pg.decode_pixels(res.inference, xs), pg.decode_pixels(clone, xs))
    # serialize(Model) downcasts first, as the reference does (no image size)
    raw = pg.serialize(res.model)
    assert raw[:44] == open(path, "rb").read()[:44] and raw[52:] == open(path, "rb").read()[52:]


def test_gpu_sweep_small_grid(tmp_path):
    """run_sweep on the device (sweep.py:61-84): one fit per (configuration,
    seed), probed vs plain-hash rows, sizes from the file format."""
    import paper_2312_17241_b200 as pg
    from paper_2312_17241_b200.model_io import size_report
    img = np.random.default_rng(0).random((16, 16, 3)).astype(np.float32)
    base = pg.HyperParams(n_levels=4, n_min=4, n_max=16, n_neurons=16)
    grid = pg.expand_grid(base, [64], [256], [1, 4])
    seen = []
    pts = pg.run_sweep(img, grid, [0, 1], pg.TrainConfig(steps=20, batch_size=128), progress=seen.append)
    assert len(pts) == 4 and seen == pts
    assert [p.method for p in pts] == ["baseline", "baseline", "probed", "probed"]
    for p, (h, s) in zip(pts, [(h, s) for h in grid for s in (0, 1)]):
        assert p.size_bytes == size_report(h).total_bytes and p.seed == s
        assert np.isfinite(p.psnr_db) and p.psnr_db > 5.0
    again = pg.run_sweep(img, grid[:1], [0], pg.TrainConfig(steps=20, batch_size=128))
    assert abs(again[0].psnr_db - pts[0].psnr_db) < 1e-3   # same seeds (float atomics: not bit-reproducible)
    pg.write_csv(pts, str(tmp_path / "s.csv"))
    assert len(pg.pareto_front(pts)) >= 1


def _oracle_fit(img, kw, steps, batch, seed):
    """trainer.fit restated by the oracle: losses, then the PSNR of the fp16
    downcast decode of the full image (trainer.py:196-242)."""
    from oracle import oracle as O
    from paper_2312_17241_b200.sweep import psnr
    st = O.TrainState(O.init_model(O.Hyper(**kw), seed), img, O.TrainCfg(batch_size=batch, seed=seed))
    losses = [st.step() for _ in range(steps)]
    h, w = img.shape[:2]
    dec = O.decode_pixels(O.to_inference(st.model), O.grid_coords(w, h, 0, 0, w, h)).reshape(h, w, -1)
    return losses, psnr(img.astype(np.float64), np.clip(dec, 0.0, 1.0).astype(np.float64))


@pytest.mark.parametrize("base", [dict(n_levels=3, n_min=4, n_max=16, n_neurons=8),   # generic kernels
                                  dict(n_min=4, n_max=64)])                           # fused 16-level step
def test_gpu_sweep_matches_reference_fits(base):
    """Every job of a GPU sweep (probed and plain-hash rows, two seeds)
    against the reference's own fit restated by the oracle on the same
    image: final PSNR within 0.05 dB and losses within rtol 1e-4 / atol
    1e-7 — the reference's cross-backend bar (test_backends.py:174-191).
    The 16-level shape runs the fused step, whose default mode (3xTF32
    tensor-core MLP, float atomics) drifts past 1e-4 on this chaotic
    noise fit after ~5 steps; its loss curve is held to the bar in parity
    mode (reference_order + deterministic), its sweep PSNR in default mode."""
    import paper_2312_17241_b200 as pg
    img = np.random.default_rng(9).random((16, 16, 3)).astype(np.float32)
    steps, batch = 30, 128
    grid = pg.expand_grid(pg.HyperParams(**base), [32, 64], [64], [1, 4])
    cfg = pg.TrainConfig(steps=steps, batch_size=batch)
    pts = pg.run_sweep(img, grid, [0, 1], cfg)
    for p, (h, seed) in zip(pts, [(h, s) for h in grid for s in (0, 1)]):
        kw = dict(base, n_f=h.n_f, n_c=h.n_c, n_p=h.n_p)
        parity = dict(reference_order=True, deterministic=True) if "n_levels" not in base else {}
        res = pg.fit(img, h, pg.TrainConfig(steps=steps, batch_size=batch, seed=seed), **parity)
        losses, want_psnr = _oracle_fit(img, kw, steps, batch, seed)
        np.testing.assert_allclose(res.losses, losses, rtol=1e-4, atol=1e-7)
        assert res.final_psnr == pytest.approx(want_psnr, abs=0.05)
        assert p.psnr_db == pytest.approx(want_psnr, abs=0.05), (p, want_psnr)
