"""Pin the CPU oracle (oracle/oracle.py + oracle/pg_oracle.c) against the real
reference: the golden vectors made by tests/golden/make_golden.py from
/root/reference, the reference's own known-answer tests, and — when
oracle/_ref holds the reference's compiled Cython core — live comparison."""

import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def fwd():
    return np.load(os.path.join(GOLD, "fwd_kernels.npz"))


@pytest.fixture(scope="module")
def bwd():
    return np.load(os.path.join(GOLD, "bwd_kernels.npz"))


@pytest.fixture(scope="module")
def traj():
    return np.load(os.path.join(GOLD, "model_traj.npz"))


def eq(a, b):
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("tag", ["float32", "float64"])
@pytest.mark.parametrize("d", [2, 3])
def test_forward_kernels_bit_exact_vs_golden(fwd, tag, d):
    k = f"{tag}_d{d}"
    xs = fwd[f"fwd_{k}_xs"]
    o, idx, w = O.CBackend.dense_fwd(xs, 8, fwd[f"fwd_{k}_dense_feats"])
    eq(idx, fwd[f"fwd_{k}_dense_idx"]); eq(w, fwd[f"fwd_{k}_dense_w"]); eq(o, fwd[f"fwd_{k}_dense_out"])
    o, idx, w = O.CBackend.hashed_fwd(xs, 33, 64, fwd[f"fwd_{k}_feats"], O.PRIMARY)
    eq(idx, fwd[f"fwd_{k}_hashed_idx"]); eq(w, fwd[f"fwd_{k}_hashed_w"]); eq(o, fwd[f"fwd_{k}_hashed_out"])
    o, base, row, w = O.CBackend.probed_fwd(xs, 21, 64, 32, 2, fwd[f"fwd_{k}_feats"],
                                            fwd[f"fwd_{k}_baked"], O.PRIMARY, O.AUX)
    eq(base, fwd[f"fwd_{k}_probed_base"]); eq(row, fwd[f"fwd_{k}_probed_row"])
    eq(w, fwd[f"fwd_{k}_probed_w"]); eq(o, fwd[f"fwd_{k}_probed_out"])
    o, base, row, w = O.CBackend.probed_fwd(xs, 322, 4096, 1 << 14, 2, fwd[f"fwd_{k}_feats2"],
                                            fwd[f"fwd_{k}_baked2"], O.PRIMARY, O.AUX)
    eq(base, fwd[f"fwd_{k}_p322_base"]); eq(row, fwd[f"fwd_{k}_p322_row"])
    eq(w, fwd[f"fwd_{k}_p322_w"]); eq(o, fwd[f"fwd_{k}_p322_out"])


@pytest.mark.parametrize("tag", ["float32", "float64"])
@pytest.mark.parametrize("F", [2, 4])
def test_backward_kernels_bit_exact_vs_golden(bwd, tag, F):
    k = f"bwd_{tag}_F{F}"
    dt = np.dtype(tag)
    g = np.zeros((64, F), dt)
    O.CBackend.indexed_bwd(bwd[f"{k}_up"], bwd[f"{k}_idx"], bwd[f"{k}_w"], g)
    eq(g, bwd[f"{k}_gidx"])
    rows_u, inv = O.CBackend.dedup_rows(bwd[f"{k}_row"], 32)
    eq(rows_u, bwd[f"{k}_rows_u"]); eq(inv, bwd[f"{k}_inv"])
    smu = O.softmax_rows(bwd[f"{k}_conf"][rows_u])
    eq(smu, bwd[f"{k}_smu"])
    gf = np.zeros((64, F), dt)
    gc = np.zeros_like(smu)
    O.CBackend.probed_bwd(bwd[f"{k}_up"], bwd[f"{k}_base"], inv, bwd[f"{k}_w"], smu,
                          bwd[f"{k}_feats"], gf, gc)
    eq(gf, bwd[f"{k}_gfeat"]); eq(gc, bwd[f"{k}_gconf_u"])


@pytest.mark.parametrize("tag", ["float32", "float64"])
def test_adam_rebake_bit_exact_vs_golden(bwd, tag):
    k = f"adam_{tag}"
    conf, m, v, baked = (bwd[f"{k}_{n}"].copy() for n in ("conf", "m", "v", "baked"))
    O.CBackend.adam_rebake_rows(conf, m, v, baked, bwd[f"{k}_rows_u"], bwd[f"{k}_g"],
                                5, 1e-2, 0.9, 0.99, 1e-15)
    eq(conf, bwd[f"{k}_conf_out"]); eq(m, bwd[f"{k}_m_out"]); eq(v, bwd[f"{k}_v_out"])
    eq(baked, bwd[f"{k}_baked_out"])


def test_mlp_bit_exact_vs_golden():
    g = np.load(os.path.join(GOLD, "mlp.npz"))
    W = [g[f"mlp_W{i}"] for i in range(3)]
    B = [g[f"mlp_b{i}"] for i in range(3)]
    eq(O.CBackend.mlp_infer_rows(g["mlp_x"], W, B), g["mlp_rows"])
    eq(O.CBackend.mlp_infer_rows(g["mlp_x"], W, B, True), g["mlp_rows_sig"])
    out, cache = O.mlp_forward(W, B, g["mlp_x"])
    eq(out, g["mlp_fwd"])
    Wg = [np.zeros_like(w) for w in W]
    Bg = [np.zeros_like(b) for b in B]
    dx = O.mlp_backward(W, Wg, Bg, cache, g["mlp_up"])
    eq(dx, g["mlp_dx"])
    for i in range(3):
        eq(Wg[i], g[f"mlp_Wg{i}"]); eq(Bg[i], g[f"mlp_bg{i}"])


def _small_hyper(traj):
    kv = {k: int(v) for k, v in traj["small_hyper"]}
    return O.Hyper(**kv)


def test_init_model_matches_reference(traj):
    m = O.init_model(_small_hyper(traj), seed=0)
    for i, L in enumerate(m.levels):
        eq(L.feats, traj[f"small_init_feats{i}"])
        if f"small_init_conf{i}" in traj:
            eq(L.conf, traj[f"small_init_conf{i}"]); eq(L.baked, traj[f"small_init_baked{i}"])
        else:
            assert L.conf is None
    for i, w in enumerate(m.W):
        eq(w, traj[f"small_init_W{i}"])


def test_c1_init_and_levels_match_reference(traj):
    from tests.golden_util import sha
    h = O.Hyper(n_f=2**12, n_c=2**14, n_p=4)
    m = O.init_model(h, seed=0)
    eq(np.array([[L.res, L.dense] for L in m.levels]), traj["c1_levels"])
    fp = []
    for i, L in enumerate(m.levels):
        fp.append(f"feats{i}:{sha(L.feats)}")
        if L.conf is not None:
            fp += [f"conf{i}:{sha(L.conf)}", f"baked{i}:{sha(L.baked)}"]
    fp += [f"W{i}:{sha(w)}" for i, w in enumerate(m.W)]
    assert fp == list(traj["c1_init_sha"])


def test_training_trajectory_bit_exact_small(traj):
    st = O.TrainState(O.init_model(_small_hyper(traj), seed=0), traj["small_img"],
                      O.TrainCfg(steps=30, batch_size=128, seed=0))
    losses = np.array([st.step() for _ in range(30)])
    eq(losses, traj["small_losses"])
    for i, L in enumerate(st.model.levels):
        eq(L.feats, traj[f"small_final_feats{i}"])
        if L.conf is not None:
            eq(L.conf, traj[f"small_final_conf{i}"]); eq(L.baked, traj[f"small_final_baked{i}"])
    for i in range(len(st.model.W)):
        eq(st.model.W[i], traj[f"small_final_W{i}"]); eq(st.model.b[i], traj[f"small_final_b{i}"])


def test_c1_five_steps_and_decode_bit_exact(traj):
    from tests.golden_util import sha, smooth_image
    h = O.Hyper(n_f=2**12, n_c=2**14, n_p=4)
    st = O.TrainState(O.init_model(h, seed=0), smooth_image(256, 256),
                      O.TrainCfg(steps=5, batch_size=8192, seed=0))
    losses = np.array([st.step() for _ in range(5)])
    eq(losses, traj["c1_losses"])
    fp = []
    for i, L in enumerate(st.model.levels):
        fp.append(f"feats{i}:{sha(L.feats)}")
        if L.conf is not None:
            fp.append(f"baked{i}:{sha(L.baked)}")
    assert fp == list(traj["c1_step5_sha"])
    inf = O.to_inference(st.model)
    eq(O.decode_pixels(inf, traj["c1_decode_xs"]), traj["c1_decode_out"])


# ---- reference known-answer tests (pkg/tests) restated against the oracle ----
def test_kat_spatial_hash():
    # test_indexing.py:133-137
    v = np.array([[[1, 2, 3]]])
    assert int(O._hash(v, O.PRIMARY)[0, 0]) == 2892625372


def test_kat_level_ladder():
    # test_indexing.py:36-42
    assert O.level_resolution(3, 16, 512, 16) == 32
    assert O.level_resolution(0, 16, 512, 16) == 16
    assert O.level_resolution(15, 16, 512, 16) == 512


def test_kat_bilinear_weights_and_corner_order():
    # test_indexing.py:94-100: t=(0.25, 0.5) in cell (0,0) of a 4-cell grid;
    # corners (0,0),(0,1),(1,0),(1,1) → dense rows v0 + 5*v1
    xs = np.array([[0.0625, 0.125]], np.float64)
    _, idx, w = O.CBackend.dense_fwd(xs, 4, np.zeros((25, 2)))
    assert idx[0].tolist() == [0, 5, 1, 6]
    np.testing.assert_allclose(w[0], [0.375, 0.375, 0.125, 0.125])
    # on-vertex point has unit weight on corner 0 (test_indexing.py:84-88)
    _, idx, w = O.CBackend.dense_fwd(np.array([[0.5, 0.25]]), 4, np.zeros((25, 2)))
    assert w[0].tolist() == [1.0, 0.0, 0.0, 0.0] and idx[0, 0] == 2 + 5 * 1


def test_kat_dense_vertex_row():
    # test_encoding.py:70-77 — vertex (2,1) on res 4 → row 2 + 5*1
    f = np.arange(50, dtype=np.float32).reshape(25, 2)
    out, idx, w = O.CBackend.dense_fwd(np.array([[0.5, 0.25]], np.float32), 4, f)
    eq(out[0], f[7])


def test_kat_hashed_vertex_row():
    # test_encoding.py:79-86
    f = np.arange(32, dtype=np.float32).reshape(16, 2)
    out, idx, w = O.CBackend.hashed_fwd(np.array([[0.25, 0.75]], np.float32), 4, 16, f, O.PRIMARY)
    h = (1 * 1) ^ ((3 * 2654435761) % 2**32)
    eq(out[0], f[h % 16])


def test_kat_argmax_ties():
    # test_codebooks.py:133-139 — strict '>' scan keeps the first maximum
    conf = np.array([[-1, 5, 5, 2], [0, 0, 0, 0], [0.1, 0.9, 0.3, 0.2]], np.float32)
    m = np.zeros_like(conf)
    v = np.zeros_like(conf)
    baked = np.zeros(3, np.uint8)
    O.CBackend.adam_rebake_rows(conf, m, v, baked, np.array([0, 1, 2], np.int32),
                                np.zeros_like(conf), 1, 0.0, 0.9, 0.99, 1e-15)
    assert baked.tolist() == [1, 0, 1]


# ---- live comparison with the reference's compiled core (oracle/_ref) ----
REF = O.reference_core_backend()


@pytest.mark.skipif(REF is None, reason="oracle/_ref not built (oracle/build_ref.sh)")
def test_live_reference_core_matches_oracle_training():
    h = O.Hyper(n_f=2**8, n_c=2**10, n_p=8, n_levels=8, n_max=128, n_neurons=16)
    img = np.random.default_rng(3).random((40, 40, 3)).astype(np.float32)
    a = O.TrainState(O.init_model(h, seed=1), img, O.TrainCfg(batch_size=512, seed=1))
    b = O.TrainState(O.init_model(h, seed=1), img, O.TrainCfg(batch_size=512, seed=1), kern=REF)
    for _ in range(8):
        assert a.step() == b.step()
    for La, Lb in zip(a.model.levels, b.model.levels):
        eq(La.feats, Lb.feats)
        if La.conf is not None:
            eq(La.conf, Lb.conf); eq(La.baked, Lb.baked)
    q = np.random.default_rng(4).random((700, 2)).astype(np.float32)
    inf = O.to_inference(a.model)
    eq(O.decode_pixels(inf, q), O.decode_pixels(inf, q, kern=REF))


@pytest.mark.skipif(REF is None, reason="oracle/_ref not built (oracle/build_ref.sh)")
@pytest.mark.parametrize("d", [2, 3])
def test_live_reference_core_matches_oracle_kernels(d):
    rng = np.random.default_rng(d)
    xs = rng.random((999, d)).astype(np.float32)
    feats = rng.standard_normal((1024, 2)).astype(np.float32)
    baked = rng.integers(0, 8, 512).astype(np.uint8)
    a = O.CBackend.probed_fwd(xs, 77, 1024, 512, 3, feats, baked, O.PRIMARY, O.AUX)
    b = REF.probed_fwd(xs, 77, 1024, 512, 3, feats, baked, O.PRIMARY, O.AUX)
    for x, y in zip(a, b):
        eq(x, y)


@pytest.mark.parametrize("K,fin,fout", [(8192, 64, 64), (8192, 32, 64), (8192, 64, 3), (128, 64, 64),
                                        (700, 64, 64), (702, 64, 64), (1000, 32, 64), (8492, 64, 4)])
def test_openblas_wgrad_order(K, fin, fout):
    """Pins the summation order of numpy's W_grad += a.T @ delta (OpenBLAS
    sgemm: K blocked by 448, last two blocks balanced, FMA chain per block)
    and of delta.sum(axis=0) (sequential) — the order pg_mlp_wgrad_blas_f32
    reproduces on the GPU (mlp.py:81-82)."""
    rng = np.random.default_rng(K + fin + fout)
    a = np.maximum(rng.standard_normal((K, fin)), 0).astype(np.float32)
    d = (rng.standard_normal((K, fout)) * 1e-3).astype(np.float32)
    gw0 = (rng.standard_normal((fin, fout)) * 1e-2).astype(np.float32)
    gb0 = (rng.standard_normal(fout) * 1e-2).astype(np.float32)
    gw, gb = gw0.copy(), gb0.copy()
    O.wgrad_blas(a, d, gw, gb)
    want_w, want_b = gw0.copy(), gb0.copy()
    want_w += a.T @ d
    want_b += d.sum(axis=0)
    eq(gw, want_w)
    eq(gb, want_b)
