"""Probe the tcgen05 GEMM variants with random inputs (developer tool)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_21090_b200 import _lib  # noqa: E402

L = _lib.lib()
dev = torch.device("cuda")


def run(F, N, K, W, X, mode=0):
    tW = torch.tensor(W.astype(np.float32), device=dev)
    tX = torch.tensor(X.astype(np.float32), device=dev)
    tD = torch.full((N, F), -1.0, dtype=torch.float32, device=dev)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(L.stgn_debug_tc_gemm(F, N, K, tW.data_ptr(), tX.data_ptr(), tD.data_ptr(), mode, s),
               "tc")
    torch.cuda.synchronize()
    return tD.cpu().numpy()


rng = np.random.default_rng(0)
for (F, N, K) in ((128, 16, 16), (100, 100, 96), (7, 33, 50)):
    W = rng.standard_normal((K, F))
    X = rng.standard_normal((N, K))
    ref = X @ W
    scale = np.abs(X) @ np.abs(W)
    for mode in (8, 8 + 32):
        if N > 16 and not (mode & 32) and N > 64:
            continue
        D = run(F, N, K, W, X, mode)
        err = np.max(np.abs(D - ref) / scale)
        print(f"F={F} N={N} K={K} mode={mode} max rel err {err:.3e}")
        if err > 1e-3:
            print(D[:3, :6], "\n", ref[:3, :6])
