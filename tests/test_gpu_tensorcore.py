"""tcgen05 split-TF32 GEMM self-test (descriptor/layout/TMEM round trip)
against a float64 numpy product; tolerance 2e-6 relative to sum|x||w|.
Also checks the engine's three recompute kernels (bf16x3 128-row, split-TF32,
FFMA) against the reference fixtures."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [8, 40], ids=["smem-smem", "tmem-A"])
@pytest.mark.parametrize("F,N,K", [(100, 48, 96), (128, 16, 8), (7, 33, 50), (64, 64, 100)])
def test_tc_split_tf32_gemm(F, N, K, mode):
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
    # mode 8: both operands K-major in shared memory; 40: A (rows of X) in TMEM
    _lib.check(L.stgn_debug_tc_gemm(F, N, K, tW.data_ptr(), tX.data_ptr(), tD.data_ptr(), mode,
                                    stream), "tc_gemm")
    ref = X.astype(np.float64) @ W.astype(np.float64)
    scale = np.abs(X).astype(np.float64) @ np.abs(W).astype(np.float64)
    err = np.max(np.abs(tD.cpu().numpy() - ref) / scale)
    assert err < 2e-6, f"split-TF32 relative error {err:.3e}"


@pytest.mark.parametrize("name", ["c4_shape_tiny", "k2_sum_window", "selfloops_dups"])
def test_engine_tensor_core_path_vs_ffma(name):
    """Both recompute kernels meet the reference tolerances; the tcgen05 one is
    actually selected for these widths."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from golden_util import batches, case_setup, load
    from parity_util import assert_rows_close
    from paper_2603_21090_b200.engine import IncrementalEngine
    z = load("engine_" + name)
    cfg, params, stream = case_setup(z)
    n = int(z["node_count"])
    for tc in (True, "tf32", False):
        eng = IncrementalEngine(cfg, params, tensor_cores=tc)
        preds = []
        for b in batches(stream, cfg.batch_size):
            preds.extend(eng.process_batch_arrays(b.src, b.dst, b.t, b.feat).tolist())
        info = eng.info()
        # True selects the bf16x3 128-row kernel (all three cases have H = 2 and
        # a 4-padded k_in <= 224); "tf32" the split-TF32 kernel; False the FFMA kernel
        assert info["bf16x3"] == int(tc is True), (tc, info)
        assert info["tensor_cores"] == int(tc is not False), (tc, info)
        assert np.max(np.abs(np.array(preds) - z["preds"])) <= 1e-5
        assert_rows_close(eng.cache.h[:n].reshape(n, -1), z["h"].reshape(n, -1), f"h tc={tc}")
        assert_rows_close(eng.memory.states[:n], z["memory"], f"memory tc={tc}")
