"""tcgen05 building blocks: one kind::tf32 UMMA GEMM through TMEM against an
fp64 reference (single pass at tf32 precision, 2-term split at ~fp32)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("split,tol", [(0, 3e-3), (1, 2e-6)])
def test_umma_tf32_gemm(split, tol):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2312_17241_b200 import _lib
    rng = np.random.default_rng(split)
    A = rng.standard_normal((128, 32)).astype(np.float32)
    # B exactly representable in tf32 (like the fp16-rounded inference MLP)
    B = rng.standard_normal((64, 32)).astype(np.float16).astype(np.float32)
    tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    tD = torch.zeros((128, 64), device="cuda")
    _lib.call("pg_selftest_umma_tf32", _lib.ptr(tA), _lib.ptr(tB), _lib.ptr(tD), split,
              _lib.stream_ptr())
    D = tD.cpu().numpy()
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    err = np.abs(D - ref) / (np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64).T)
    print("max scaled error", err.max())
    assert err.max() <= tol
