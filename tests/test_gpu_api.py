"""Drop-in API surface beyond the fused hot path, on the GPU: the standalone
MLP passes (mlp.py:55-85) and their ShapeMismatch errors, the reference's
LevelTrace view of an encode trace (encoding.py:22-30), StaleTrace
(encoding.py:103-109, 122-127; test_encoding.py:199-205), and the PNG
output of a decoded image (pngio.py:34-41)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402


class _Params:
    """The reference's MlpParams shape: numpy weights/biases + grads."""

    def __init__(self, W, B):
        self.weights, self.biases = W, B
        self.weight_grads = [np.zeros_like(w) for w in W]
        self.bias_grads = [np.zeros_like(b) for b in B]


@pytest.mark.parametrize("dtype,tol", [(np.float32, 1e-5), (np.float64, 1e-12)])
@pytest.mark.parametrize("widths", [[32, 64, 64, 3], [8, 16, 2], [5, 1]])
def test_standalone_mlp_vs_reference(widths, dtype, tol):
    from paper_2312_17241_b200.mlp import mlp_backward, mlp_forward
    rng = np.random.default_rng(len(widths))
    W = [rng.uniform(-1, 1, (a, b)).astype(dtype) for a, b in zip(widths[:-1], widths[1:])]
    B = [rng.uniform(-0.1, 0.1, b).astype(dtype) for b in widths[1:]]
    x = rng.standard_normal((777, widths[0])).astype(dtype)
    up = rng.standard_normal((777, widths[-1])).astype(dtype)
    p = _Params(W, B)
    out, cache = mlp_forward(p, x)
    want, ocache = O.mlp_forward(W, B, x)
    np.testing.assert_allclose(out, want, rtol=tol, atol=tol)
    dx = mlp_backward(p, cache, up)
    gW = [np.zeros_like(w) for w in W]
    gB = [np.zeros_like(b) for b in B]
    want_dx = O.mlp_backward(W, gW, gB, ocache, up)
    np.testing.assert_allclose(dx, want_dx, rtol=tol, atol=tol)
    for a, b in zip(p.weight_grads + p.bias_grads, gW + gB):
        np.testing.assert_allclose(a, b, rtol=tol, atol=tol * max(1.0, float(np.abs(b).max())))
    # gradients accumulate, as the reference's do
    mlp_backward(p, cache, up)
    np.testing.assert_allclose(p.weight_grads[0], 2 * gW[0], rtol=tol, atol=tol * max(1.0, float(np.abs(gW[0]).max())))
    # device tensors in -> device tensors out
    outd, cd = mlp_forward(p, torch.from_numpy(x).cuda())
    assert outd.is_cuda
    np.testing.assert_array_equal(outd.cpu().numpy(), out)


def test_standalone_mlp_shape_mismatch():
    import paper_2312_17241_b200 as pg
    from paper_2312_17241_b200.mlp import mlp_backward, mlp_forward
    p = _Params([np.ones((4, 3), np.float32)], [np.zeros(3, np.float32)])
    with pytest.raises(pg.ShapeMismatch):                     # mlp.py:57-60
        mlp_forward(p, np.ones((5, 3), np.float32))
    out, cache = mlp_forward(p, np.ones((5, 4), np.float32))
    with pytest.raises(pg.ShapeMismatch):                     # mlp.py:76-78
        mlp_backward(p, cache, np.ones((5, 2), np.float32))


def _tiny():
    import paper_2312_17241_b200 as pg
    return pg.HyperParams(n_f=16, n_c=8, n_p=4, n_levels=2, n_min=4, n_max=8, n_neurons=8, feature_dim=2)


def test_stale_trace_detected():
    """test_encoding.py:199-205 on the device model: replacing a level's
    table with a differently shaped array invalidates earlier traces."""
    import paper_2312_17241_b200 as pg
    m = pg.init_model(_tiny(), seed=0)
    y, traces = pg.encode_forward(m, np.array([[0.2, 0.8]]))
    m.levels[1].features.values = np.zeros((32, 2), dtype=np.float32)
    m.levels[1].features.grads = np.zeros((32, 2), dtype=np.float32)
    with pytest.raises(pg.StaleTrace):
        pg.encode_backward(m, traces, np.zeros_like(y))
    # a trace from another model, and an upstream of the wrong shape
    y2, tr2 = pg.encode_forward(m, np.array([[0.2, 0.8]]))
    other = pg.init_model(_tiny(), seed=0)
    with pytest.raises(pg.StaleTrace):
        pg.encode_backward(other, tr2, np.zeros_like(y2))
    with pytest.raises(pg.StaleTrace):
        pg.encode_backward(m, tr2, np.zeros((2, y2.shape[1]), np.float32))
    # same-shape replacement uploads the values and keeps traces valid
    new = np.full((16, 2), 0.25, np.float32)
    m.levels[1].features.values = new
    np.testing.assert_array_equal(m.levels[1].features.values.cpu().numpy(), new)
    pg.encode_backward(m, tr2, np.zeros_like(y2))


@pytest.mark.parametrize("kw", [dict(n_f=2**12, n_c=2**14, n_p=4), dict(n_f=2**10, n_c=2**10, n_p=1),
                                dict(d=3, n_f=2**8, n_c=2**12, n_p=8)])
def test_level_traces_match_reference(kw):
    """Iterating an encode trace yields the reference's LevelTrace per level
    (kind, weights, idx / base, row) — bit-exact against the oracle."""
    import paper_2312_17241_b200 as pg
    m = pg.init_model(pg.HyperParams(**kw), seed=0)
    om = O.init_model(O.Hyper(**kw), seed=0)
    xs = np.random.default_rng(1).random((999, m.hyper.d)).astype(np.float32)
    _, tr = pg.encode_forward(m, xs)
    _, otr = O.encode_forward(om, xs)
    assert len(tr) == len(otr)
    for a, b in zip(tr, otr):
        assert a.kind == b.kind
        np.testing.assert_array_equal(a.weights, b.w)
        for f in ("idx", "base", "row"):
            if getattr(b, f) is not None:
                np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    # the reference's lookup count (model_io.py:302-307)
    n = sum(t.weights.size for t in tr)
    assert n == 999 * (1 << m.hyper.d) * m.hyper.n_levels


def test_png_output_of_decoded_image(tmp_path):
    """save_image of a device-decoded image: the device quantisation equals
    the reference's numpy rule byte for byte, the file reads back with
    Pillow (the reference's reader) and with load_image."""
    import paper_2312_17241_b200 as pg
    from paper_2312_17241_b200.pngio import load_image, quantize, save_image
    m = pg.init_model(pg.HyperParams(n_f=2**10, n_c=2**10, n_p=4), seed=0)
    rng = np.random.default_rng(0)
    with torch.no_grad():
        m.feats.copy_(torch.from_numpy((rng.standard_normal(tuple(m.feats.shape))).astype(np.float32)))
    inf = pg.to_inference(m, 37, 23)
    img = pg.decode_image(inf)
    ref_u8 = np.rint(np.clip(img, 0.0, 1.0) * 255.0).astype(np.uint8)      # pngio.py:39
    np.testing.assert_array_equal(quantize(torch.from_numpy(img).cuda()), ref_u8)
    edge = np.array([[[-1.0, 0.0, 0.5 / 255], [1.5 / 255, 2.5 / 255, 1.0]],
                     [[2.0, np.float32(0.5), 254.5 / 255], [0.999, 1e-9, 0.4999 / 255]]], np.float32)
    np.testing.assert_array_equal(quantize(torch.from_numpy(edge).cuda()),
                                  np.rint(np.clip(edge, 0.0, 1.0) * 255.0).astype(np.uint8))
    path = str(tmp_path / "out.png")
    save_image(path, torch.from_numpy(img).cuda())
    from PIL import Image
    with Image.open(path) as im:
        np.testing.assert_array_equal(np.asarray(im.convert("RGB")), ref_u8)
    np.testing.assert_array_equal(load_image(path), ref_u8.astype(np.float32) / 255.0)
    # a Pillow-written PNG (adaptive filters) reads back identically
    p2 = str(tmp_path / "pil.png")
    Image.fromarray(ref_u8, mode="RGB").save(p2, format="PNG")
    np.testing.assert_array_equal(load_image(p2), ref_u8.astype(np.float32) / 255.0)
    with pytest.raises(pg.UnsupportedFormat):
        save_image(path, np.zeros((4, 4), np.float32))
