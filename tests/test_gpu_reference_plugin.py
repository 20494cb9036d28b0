"""The REAL reference package driven through this repo's backend plug-in.

oracle/build_ref.sh stages the reference's own ``probegrid`` package (with
its compiled Cython core) into oracle/_ref/pkg (git-ignored; it travels to
the GPU box with the snapshot).  Here its seam (backends/__init__.py:12-50:
``_BACKENDS`` + ``set_backend``) receives ``paper_2312_17241_b200.backend``
as "cuda" — the four-line registration of INTEGRATION.md §1 — and the
reference's own orchestration runs on the sm_100a kernels: encoding.py's
encode_forward / encode_backward, trainer.py's TrainState.step and fit, and
model_io.py's decode_pixels.  Compared against the same orchestration on
the reference's Cython backend, with the reference's cross-backend bars
(test_backends.py:28-206): integer outputs and forwards bit-exact, gradients
rtol = atol = 1e-5, fit losses rtol 1e-4 / atol 1e-7, PSNR within 0.05 dB.
"""

import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REF_PKG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "pkg")


@pytest.fixture(scope="module")
def ref():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.isdir(os.path.join(REF_PKG, "probegrid")):
        pytest.skip("reference package not staged (oracle/build_ref.sh)")
    sys.path.insert(0, REF_PKG)
    import probegrid
    from probegrid import backends

    from paper_2312_17241_b200 import backend as cuda_backend
    backends._BACKENDS["cuda"] = cuda_backend
    assert "cython" in backends.available(), "reference core not compiled"
    yield probegrid
    backends.set_backend("cython")


def _run(ref, which, fn):
    from probegrid import backends
    prev = backends.name()
    backends.set_backend(which)
    try:
        return fn()
    finally:
        backends.set_backend(prev)


def _smooth(n=64):
    yy, xx = np.meshgrid((np.arange(n) + 0.5) / n, (np.arange(n) + 0.5) / n, indexing="ij")
    return np.stack([0.5 + 0.5 * np.sin(6 * np.pi * xx) * np.cos(4 * np.pi * yy), xx,
                     0.5 + 0.25 * np.sin(10 * np.pi * (xx + yy))], axis=2).astype(np.float32)


@pytest.mark.parametrize("kw", [dict(n_f=2**12, n_c=2**14, n_p=4), dict(),
                                dict(d=3, n_f=2**8, n_c=2**12, n_p=8, out_dim=1)])
def test_reference_encode_forward_backward_on_cuda(ref, kw):
    from probegrid.encoding import encode_backward, encode_forward
    from probegrid.model import HyperParams, init_model
    hyper = HyperParams(**kw)
    xs = np.random.default_rng(3).random((3000, hyper.d)).astype(np.float32)
    up = np.random.default_rng(4).standard_normal((3000, hyper.encoded_width)).astype(np.float32)

    def go():
        m = init_model(hyper, seed=0)
        y, traces = encode_forward(m, xs)
        encode_backward(m, traces, up)
        return m, y, traces

    mc, yc, tc = _run(ref, "cython", go)
    mg, yg, tg = _run(ref, "cuda", go)
    np.testing.assert_array_equal(yg, yc)
    for a, b in zip(tg, tc):
        assert a.kind == b.kind
        np.testing.assert_array_equal(a.weights, b.weights)
        for f in ("idx", "base", "row"):
            if getattr(b, f) is not None:
                np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    for a, b in zip(mg.levels, mc.levels):
        np.testing.assert_allclose(a.features.grads, b.features.grads, rtol=1e-5, atol=1e-5)
        if b.conf is not None:
            np.testing.assert_allclose(a.conf.grads, b.conf.grads, rtol=1e-5, atol=1e-5)


def test_reference_fit_on_cuda_matches_cython(ref):
    """test_backends.py:174-191 with the cuda backend in place of numpy."""
    from probegrid.model import HyperParams
    from probegrid.trainer import TrainConfig, fit
    img = np.random.default_rng(9).random((16, 16, 3)).astype(np.float32)
    hyper = HyperParams(n_f=32, n_c=64, n_p=4, n_levels=3, n_min=4, n_max=16, n_neurons=8)
    cfg = TrainConfig(steps=30, batch_size=128, seed=0)
    rc = _run(ref, "cython", lambda: fit(img, hyper, cfg))
    rg = _run(ref, "cuda", lambda: fit(img, hyper, cfg))
    np.testing.assert_allclose(rg.losses, rc.losses, rtol=1e-4, atol=1e-7)
    assert rg.final_psnr == pytest.approx(rc.final_psnr, abs=0.05)


def test_reference_trainstate_c1_on_cuda(ref):
    """30 reference TrainState.step calls at the C1 shape (smooth image,
    B = 8192) on the cuda backend track the Cython backend: losses rtol 1e-4,
    and the decode of the trained model through model_io.decode_pixels on
    the cuda backend equals the Cython backend's decode bit for bit."""
    from probegrid.model import HyperParams, init_model
    from probegrid.model_io import decode_pixels, to_inference
    from probegrid.trainer import TrainConfig, TrainState
    hyper = HyperParams(n_f=2**12, n_c=2**14, n_p=4)
    img = _smooth()

    def train():
        st = TrainState(init_model(hyper, seed=0), img, TrainConfig(batch_size=8192, seed=0))
        return st, [st.step() for _ in range(30)]

    stc, lc = _run(ref, "cython", train)
    stg, lg = _run(ref, "cuda", train)
    np.testing.assert_allclose(lg, lc, rtol=1e-4, atol=1e-7)
    inf = to_inference(stc.model, width=64, height=64)
    q = np.random.default_rng(5).random((20000, 2)).astype(np.float32)
    dc = _run(ref, "cython", lambda: decode_pixels(inf, q))
    dg = _run(ref, "cuda", lambda: decode_pixels(inf, q))
    np.testing.assert_array_equal(dg, dc)
