"""tcgen05 building blocks: kind::tf32 UMMA GEMMs through TMEM against fp64
references — K-major shared-memory operands (the "RG" layout the fused
kernels use), M = 128 and M = 64 accumulators, single pass and the 2-term
(hi + lo) split."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _run(A, B, code):
    from paper_2312_17241_b200 import _lib
    tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    tD = torch.full((128, 64), np.nan, device="cuda")
    _lib.call("pg_selftest_umma_tf32", _lib.ptr(tA), _lib.ptr(tB), _lib.ptr(tD), code,
              _lib.stream_ptr())
    return tD.cpu().numpy()


def _scaled_err(D, ref, A, B, transpose_a=False):
    absA = np.abs(A.astype(np.float64))
    denom = (absA.T if transpose_a else absA) @ np.abs(B.astype(np.float64)).T \
        if not transpose_a else absA.T @ np.abs(B.astype(np.float64))
    return np.abs(D - ref) / denom


@pytest.mark.parametrize("split,tol", [(0, 3e-3), (1, 2e-6)])
def test_umma_kmajor_m128(split, tol):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(split)
    A = rng.standard_normal((128, 32)).astype(np.float32)
    # B exactly representable in tf32 (like the fp16-rounded inference MLP)
    B = rng.standard_normal((64, 32)).astype(np.float16).astype(np.float32)
    D = _run(A, B, split)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    err = np.abs(D - ref) / (np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64).T)
    print("mode0 max scaled error", err.max())
    assert err.max() <= tol


def test_umma_kmajor_k64():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(2)
    A = rng.standard_normal((128, 64)).astype(np.float16).astype(np.float32)
    B = rng.standard_normal((64, 64)).astype(np.float16).astype(np.float32)
    D = _run(A, B, 2 << 4)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    np.testing.assert_allclose(D, ref, rtol=1e-5, atol=1e-4)


def test_umma_kmajor_m64_layout():
    """D[64x64] = A[64x64] . B[64x64]^T with an M = 64 accumulator: row i of
    D lives in TMEM lane (i/16)*32 + i%16 (lanes 16..31 of each quarter unused)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(3)
    A = rng.standard_normal((64, 64)).astype(np.float16).astype(np.float32)
    B = rng.standard_normal((64, 64)).astype(np.float16).astype(np.float32)
    D = _run(A, B, 4 << 4)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    lanes = [(i // 16) * 32 + i % 16 for i in range(64)]
    np.testing.assert_allclose(D[lanes], ref, rtol=1e-5, atol=1e-4)


def test_umma_mn_major_operands():
    """MN-major shared-memory operands (the layout a weight-gradient GEMM
    with K = samples would read an activation tile in).  kind::f16 with an
    MN-major A (canonical no-swizzle layout: core matrix 8 K-rows x 16 B,
    LBO = K-group stride, SBO = MN-group stride, instruction-descriptor
    major bit) computes the product: the descriptor convention is right.
    kind::tf32 with the A or B major bit set writes zeros on this sm_100a
    for every layout tried (no-swizzle with both stride conventions, the
    128-byte-swizzled canonical atom): tf32 operands must be K-major, which
    is why the training kernel's weight-gradient GEMMs stay on mma.sync
    (DESIGN.md 4).  The test pins both behaviours."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(0)
    A = rng.standard_normal((128, 32)).astype(np.float16).astype(np.float32)
    B = rng.standard_normal((64, 32)).astype(np.float16).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    np.testing.assert_allclose(_run(A, B, 10 << 4), ref, rtol=1e-5, atol=1e-4)      # f16, A MN-major
    for code in (6 << 4, (6 << 4) | (1 << 1), (6 << 4) | (3 << 1), 8 << 4, (8 << 4) | (1 << 1)):
        D = _run(A, B, code)                                                        # tf32, MN-major
        ok = np.allclose(D, ref, rtol=1e-5, atol=1e-4)
        assert ok or not D.any(), f"code {code}: neither the product nor all-zero"
        print(f"tf32 MN-major variant code {code}: {'correct' if ok else 'all zeros'}")
