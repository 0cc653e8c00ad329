"""tcgen05 split-TF32 GEMM self-test (descriptor/layout/TMEM round trip)
against a float64 numpy product; tolerance 2e-6 relative to sum|x||w|."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("F,N,K", [(100, 48, 96), (128, 16, 8), (7, 33, 50), (64, 64, 100)])
def test_tc_split_tf32_gemm(F, N, K):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2603_21090_b200 import _lib
    L = _lib.lib()
    rng = np.random.default_rng(F * 1000 + N * 10 + K)
    W = rng.standard_normal((K, F)).astype(np.float32)
    X = rng.standard_normal((N, K)).astype(np.float32)
    dev = torch.device("cuda")
    tW, tX = torch.tensor(W, device=dev), torch.tensor(X, device=dev)
    tD = torch.zeros((N, F), dtype=torch.float32, device=dev)
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(L.stgn_debug_tc_gemm(F, N, K, tW.data_ptr(), tX.data_ptr(), tD.data_ptr(), 0,
                                    stream), "tc_gemm")
    ref = X.astype(np.float64) @ W.astype(np.float64)
    scale = np.abs(X).astype(np.float64) @ np.abs(W).astype(np.float64)
    err = np.max(np.abs(tD.cpu().numpy() - ref) / scale)
    assert err < 2e-6, f"split-TF32 relative error {err:.3e}"
