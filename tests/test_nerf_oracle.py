"""CPU: the volume-compositing restatement (oracle.composite_*) that the
NeRF-head kernels are checked against.  The reference has no renderer, so
this row is pinned by calculus instead: central finite differences in fp64
and closed-form limit cases."""
import numpy as np

from oracle import oracle as O


def _case(R=5, S=7, seed=0):
    rng = np.random.default_rng(seed)
    raw = rng.standard_normal((R, S, 4)) * 2.0
    deltas = rng.random((R, S)) * 0.3
    return raw, deltas


def test_composite_backward_matches_finite_differences():
    raw, deltas = _case()
    g = np.random.default_rng(1).standard_normal((raw.shape[0], 3))
    ana = O.composite_backward(raw, deltas, g)
    eps = 1e-6
    num = np.zeros_like(raw)
    for idx in np.ndindex(raw.shape):
        p, m = raw.copy(), raw.copy()
        p[idx] += eps
        m[idx] -= eps
        num[idx] = ((O.composite_forward(p, deltas)[0] - O.composite_forward(m, deltas)[0]) * g).sum() / (2 * eps)
    np.testing.assert_allclose(ana, num, rtol=1e-6, atol=1e-9)


def test_composite_limits():
    raw, deltas = _case(R=3, S=4, seed=2)
    # zero-length segments: nothing is rendered
    rgb, w = O.composite_forward(raw, np.zeros_like(deltas))
    assert np.all(rgb == 0) and np.all(w == 0)
    # an opaque first sample hides everything behind it
    raw2 = raw.copy()
    raw2[:, 0, 0] = 60.0
    rgb, w = O.composite_forward(raw2, np.ones_like(deltas))
    np.testing.assert_allclose(rgb, 1 / (1 + np.exp(-raw2[:, 0, 1:])), rtol=1e-12)
    np.testing.assert_allclose(w.sum(axis=1), 1.0, rtol=1e-12)
    # weights never exceed one in total
    rgb, w = O.composite_forward(raw, deltas)
    assert np.all(w >= 0) and np.all(w.sum(axis=1) <= 1 + 1e-12)
