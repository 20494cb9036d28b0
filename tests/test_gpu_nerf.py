"""GPU: the NeRF-style compositing head through the C
ABI against the numpy restatement (oracle.composite_* / nerf_step_grads,
itself checked by finite differences in test_nerf_oracle.py), plus an
end-to-end fit of a synthetic radiance field."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402

KW = dict(d=3, out_dim=4, n_f=2**10, n_c=2**10, n_p=4, n_levels=16, n_min=4, n_max=64)


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _close(a, b, rel=1e-4):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    assert np.abs(a - b).max() <= rel * max(np.abs(b).max(), 1e-30), (np.abs(a - b).max(), np.abs(b).max())


@pytest.mark.parametrize("R,S", [(1000, 64), (37, 1), (5, 200), (0, 8)])
def test_composite_forward_vs_oracle(R, S):
    from paper_2312_17241_b200 import nerf
    rng = np.random.default_rng(R + S)
    raw = (rng.standard_normal((R * S, 4)) * 2).astype(np.float32)
    deltas = (rng.random(R * S) * 0.1).astype(np.float32)
    rgb, w = nerf.composite(torch.from_numpy(raw).cuda(), torch.from_numpy(deltas).cuda(), S, weights=True)
    orgb, ow = O.composite_forward(raw.reshape(R, S, 4).astype(np.float64), deltas.reshape(R, S).astype(np.float64))
    np.testing.assert_allclose(rgb.cpu().numpy(), orgb, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(w.cpu().numpy(), ow, rtol=1e-5, atol=1e-6)


def test_ray_samples_vs_oracle():
    """Slab entry/exit and midpoint samples: rays from outside, inside,
    grazing and missing the cube (fp32; products may round differently by
    an FMA, so 1e-6 absolute)."""
    from paper_2312_17241_b200 import nerf
    o, d = nerf.orbit_rays(4096, seed=3)
    o[:8] = torch.tensor([0.5, 0.5, 0.5], device="cuda")                     # inside
    d[8:16] = torch.tensor([1.0, 0.0, 0.0], device="cuda")                  # axis-aligned
    o[16:24] = torch.tensor([2.0, 2.0, 2.0], device="cuda")
    d[16:24] = torch.tensor([1.0, 0.0, 0.0], device="cuda")                 # misses
    pts, deltas = nerf.sample_points(o, d, 16)
    op, od = O.ray_samples(o.cpu().numpy(), d.cpu().numpy(), 16)
    np.testing.assert_allclose(pts.cpu().numpy(), op, atol=1e-6)
    np.testing.assert_allclose(deltas.cpu().numpy(), od, atol=1e-6)
    assert float(deltas[16 * 16:24 * 16].abs().max()) == 0.0
    assert float(pts.min()) >= 0.0 and float(pts.max()) <= 1.0


def _pair(seed=0):
    import paper_2312_17241_b200 as pg
    m = pg.init_model(pg.HyperParams(**KW), seed=seed)
    om = O.init_model(O.Hyper(**KW), seed=seed)
    rng = np.random.default_rng(seed + 3)
    for L in om.levels:    # a generic point: every level and probe matters
        L.feats[:] = (rng.standard_normal(L.feats.shape) * 0.5).astype(np.float32)
        if L.conf is not None:
            L.conf[:] = rng.standard_normal(L.conf.shape).astype(np.float32)
            L.baked[:] = np.argmax(L.conf, axis=1)
    m.load_host([L.feats for L in om.levels], {L.level: L.conf for L in om.levels if L.conf is not None},
                om.W, om.b)
    return m, om


@pytest.mark.parametrize("fused,R,S", [(False, 512, 16), (True, 128, 64), (False, 128, 64)])
def test_nerf_step_gradients_vs_oracle(fused, R, S):
    """One NeRF gradient pass: loss, dL/dy, MLP and table gradients against
    the numpy pass on the same rays — the generic path (encode kernels +
    pg_nerf_train_f32) and the fused tensor-core kernel with in-tile
    compositing (PG_COMPOSITE, one ray per 64-sample tile).  fp32 on both
    sides with different summation orders (FMA chains, 3xTF32, float
    atomics, warp scans), so bars are relative 1e-4 of each array's scale."""
    import paper_2312_17241_b200 as pg
    from paper_2312_17241_b200 import nerf
    m, om = _pair()
    o, d = nerf.orbit_rays(R, seed=5)
    tgt = torch.from_numpy(np.random.default_rng(6).random((R, 3)).astype(np.float32)).cuda()
    st = nerf.NerfTrainState(m, o, d, tgt, pg.TrainConfig(batch_size=R, seed=0), n_samples=S, fused=fused)
    assert st.nerf_fused == fused
    pts, tg = st.sample_batch()
    deltas, rgb = tg[0], tg[1]
    if fused:   # per-sample targets written by the sampling kernel (pg_ray_samples_targets_f32)
        t4 = tg[2].view(R, S, 4)
        assert torch.equal(t4[:, :, 0], deltas.view(R, S))
        assert torch.equal(t4[:, :, 1:], rgb[:, None, :].expand(R, S, 3))
    dy = torch.empty((R * S, 32), device="cuda")
    st.loss_sum.zero_()
    st.compute_grads(pts, tg, dy_out=dy)
    loss = float(st.loss_sum.item())
    oloss, ody = O.nerf_step_grads(om, pts.cpu().numpy(), deltas.cpu().numpy(), rgb.cpu().numpy(), S,
                                   st.scale)
    assert abs(loss - oloss) <= 1e-5 * oloss
    _close(dy.cpu().numpy(), ody)
    for i in range(3):
        _close(m.mlp.weight_grads[i].cpu().numpy(), om.Wg[i])
        _close(m.mlp.bias_grads[i].cpu().numpy(), om.bg[i])
    gf, gc = m.gfeats.cpu().numpy(), m.gconf.cpu().numpy()
    for L in om.levels:
        _close(gf[L.level], L.fgrad)
    for i, lv in enumerate(m.probed):
        _close(gc[i], om.levels[lv].cgrad)


def _scene(pts):
    """Analytic radiance field: a soft ball of density around the centre,
    colour = position."""
    r = np.linalg.norm(pts - 0.5, axis=-1)
    sigma_raw = 12.0 * (0.3 - r) / 0.05
    rgb_raw = 4.0 * (pts - 0.5)
    return np.concatenate([sigma_raw[..., None], rgb_raw], axis=-1)


@pytest.mark.parametrize("S", [32, 64])
def test_nerf_fit_synthetic_scene(S):
    """300 steps on 2^14 rays x S samples of an analytic scene rendered by
    the oracle (S = 64 runs the fused kernel): the photometric loss falls
    >= 10x and held-out rays render above 25 dB."""
    import paper_2312_17241_b200 as pg
    from paper_2312_17241_b200 import nerf
    o, d = nerf.orbit_rays(1 << 14, seed=1)
    pts, deltas = nerf.sample_points(o, d, S)
    raw = _scene(pts.cpu().numpy().astype(np.float64)).reshape(-1, S, 4)
    tgt, _ = O.composite_forward(raw, deltas.cpu().numpy().astype(np.float64).reshape(-1, S))
    m = pg.init_model(pg.HyperParams(d=3, out_dim=4, n_f=2**14, n_c=2**12, n_p=4, n_max=256), seed=0)
    st = nerf.NerfTrainState(m, o, d, tgt.astype(np.float32), pg.TrainConfig(batch_size=2048, seed=0),
                             n_samples=S)
    assert st.nerf_fused == (S == 64)
    losses = [st.step() for _ in range(300)]
    assert losses[-1] * 10 <= losses[0], (losses[0], losses[-1])
    ho, hd = nerf.orbit_rays(2048, seed=99)
    hp, hdel = nerf.sample_points(ho, hd, S)
    htgt, _ = O.composite_forward(_scene(hp.cpu().numpy().astype(np.float64)).reshape(-1, S, 4),
                                  hdel.cpu().numpy().astype(np.float64).reshape(-1, S))
    out = nerf.render(m, ho, hd, S).cpu().numpy()
    assert pg.psnr(htgt, out) >= 25.0, pg.psnr(htgt, out)


def test_nerf_rejects_wrong_heads():
    import paper_2312_17241_b200 as pg
    from paper_2312_17241_b200 import nerf
    m = pg.init_model(pg.HyperParams(d=3, out_dim=3, n_f=2**10, n_c=2**10, n_p=4), seed=0)
    o, d = nerf.orbit_rays(64)
    with pytest.raises(pg.InvalidHyperparameter):
        nerf.NerfTrainState(m, o, d, torch.zeros_like(o), pg.TrainConfig(batch_size=64), n_samples=4)
