"""Shared parity checks (tolerances stated once, used by every GPU test).

  integers (affected/direct sets, neighbour (nbr, eid) lists, rebuild
  decisions, counters): exact.
  memory, last_interaction, layer cache h, embeddings: per-row relative
  error ||x - ref|| / max(||ref||, ROW_FLOOR) <= REL_TOL (fp32 storage and
  accumulation against the float64 reference).
  predictions: |p - ref| <= PRED_ATOL.
"""

import numpy as np

REL_TOL = 1e-4
ROW_FLOOR = 1e-2
PRED_ATOL = 1e-5


def row_rel_err(x, ref):
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    x = x.reshape(x.shape[0], -1) if x.ndim > 1 else x.reshape(-1, 1)
    ref = ref.reshape(ref.shape[0], -1) if ref.ndim > 1 else ref.reshape(-1, 1)
    if x.size == 0:
        return 0.0
    num = np.linalg.norm(x - ref, axis=1)
    den = np.maximum(np.linalg.norm(ref, axis=1), ROW_FLOOR)
    return float(np.max(num / den))


def assert_rows_close(x, ref, what, tol=REL_TOL):
    err = row_rel_err(x, ref)
    assert err <= tol, f"{what}: max row-relative error {err:.3e} > {tol:.1e}"
    return err
