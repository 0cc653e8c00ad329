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


def check_delta_events(events_by_batch, mvn_by_batch, z, tol_rel=1e-9, tol_abs=1e-9):
    """Per batch: the same hit nodes in the same order, dn and nv exact; max_v,
    z_dev and bound to tol; the embedding to tol; max_value_norm_seen to tol.
    z_dev of an unchanged softmax is rounding noise in the reference (~1e-16:
    delta_embed's running sums), exact zero when re-evaluated, hence the
    absolute floor."""
    off = z["ev_off"]
    assert len(events_by_batch) == len(off) - 1
    for k, evs in enumerate(events_by_batch):
        lo, hi = int(off[k]), int(off[k + 1])
        assert [e["node"] for e in evs] == list(z["ev_node"][lo:hi]), f"batch {k}: hit nodes"
        assert [e["dn"] for e in evs] == list(z["ev_dn"][lo:hi])
        assert [e["nv"] for e in evs] == list(z["ev_nv"][lo:hi])
        for j, e in enumerate(evs):
            r = lo + j
            mv = z["ev_max_v"][r]
            assert abs(e["max_v"] - mv) <= tol_rel * max(mv, 1.0), (k, e["node"], "max_v")
            # an update that leaves the list empty (entries added and expired by the window
            # in the same batch) has no values (max_v = 0, bound = 0); the reference's z_dev
            # there is the rounding residue of Z after +s -s (1.0 when it stays > 0)
            if not (mv == 0.0 and e["max_v"] == 0.0):
                assert abs(e["z_dev"] - z["ev_z_dev"][r]) <= tol_abs, (k, e["node"], "z_dev")
            assert abs(e["bound"] - z["ev_bound"][r]) <= tol_abs * max(mv, 1.0) * e["dn"], \
                (k, e["node"], "bound")
            np.testing.assert_allclose(e["embedding"], z["ev_emb"][r], rtol=0,
                                       atol=tol_rel * max(1.0, float(np.abs(z["ev_emb"][r]).max())))
    np.testing.assert_allclose(np.array(mvn_by_batch), z["max_value_norm_seen"], rtol=tol_rel,
                               atol=0)

