"""Delta mode (S/engine.py:276-353): pin the oracle's classification to
fixtures the reference wrote with RunConfig(mode="delta")
(tests/golden/make_delta.py). Integers (sets, counters incl. embed_skip /
attn_hit / attn_miss, valid_at, versions, lists) must match exactly;
floats to 1e-9, because the reference applies hits with delta_embed's
running-sum updates while the oracle re-evaluates the same softmax. CPU only."""

import dataclasses

import numpy as np
import pytest

from golden_util import batches, case_setup, delta_cases, load
from oracle import stgn_oracle as orc

FLOAT_TOL = 1e-9


def run_oracle(name):
    z = load("delta_" + name)
    cfg, params, stream = case_setup(z)
    cfg = dataclasses.replace(cfg, mode="delta")
    o = orc.Oracle(cfg, params)
    keys = list(z["counter_keys"])
    preds, aff, dirs, kinds, counters = [], [], [], [], []
    o.events_by_batch, o.mvn_by_batch = [], []
    for b in batches(stream, cfg.batch_size):
        preds.extend(o.process_batch(b.src, b.dst, b.t, b.feat))
        o.events_by_batch.append(list(o.delta_events))
        o.mvn_by_batch.append(o.max_value_norm_seen)
        aff.extend(sorted(o.last_all))
        dirs.extend(sorted(o.last_direct))
        kinds.append({"none": 0, "partial": 1, "full": 2}[o.last_report["rebuild"]])
        counters.append([o.counters.get(k, 0) for k in keys])
    return z, o, preds, aff, dirs, kinds, counters


def test_delta_fixtures_present():
    assert {"tied_k1", "k2_fallback", "k1_window_adaptive", "k1_fixed_de0"} <= set(delta_cases())


@pytest.mark.parametrize("name", delta_cases())
def test_oracle_delta_mode_matches_reference(name):
    z, o, preds, aff, dirs, kinds, counters = run_oracle(name)
    assert np.array_equal(np.array(aff), z["affected"])
    assert np.array_equal(np.array(dirs), z["direct"])
    assert np.array_equal(np.array(kinds), z["rebuild_kind"])
    np.testing.assert_array_equal(np.array(counters, dtype=np.float64), z["counters"])
    np.testing.assert_allclose(np.array(preds), z["preds"], rtol=0, atol=FLOAT_TOL)
    n = int(z["node_count"])
    np.testing.assert_allclose(o.h[:n], z["h"], rtol=0, atol=FLOAT_TOL)
    np.testing.assert_allclose(o.mem[:n], z["memory"], rtol=0, atol=FLOAT_TOL)
    np.testing.assert_array_equal(o.valid_at[:n], z["valid_at"])
    np.testing.assert_array_equal(o.version[:n], z["version"])


def test_delta_fixtures_exercise_every_class():
    tot = {}
    for name in delta_cases():
        z = load("delta_" + name)
        keys = list(z["counter_keys"])
        c = z["counters"].sum(axis=0)
        for k in ("embed_skip", "attn_hit", "attn_miss"):
            tot[k] = tot.get(k, 0) + c[keys.index(k)]
    assert all(v > 0 for v in tot.values()), tot


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


@pytest.mark.parametrize("name", delta_cases())
def test_oracle_delta_bound_records_match_reference(name):
    z, o, *_ = run_oracle(name)
    check_delta_events(o.events_by_batch, o.mvn_by_batch, z, tol_rel=1e-9, tol_abs=1e-9)
