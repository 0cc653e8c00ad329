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
from parity_util import check_delta_events
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


@pytest.mark.parametrize("name", delta_cases())
def test_oracle_delta_bound_records_match_reference(name):
    z, o, *_ = run_oracle(name)
    check_delta_events(o.events_by_batch, o.mvn_by_batch, z, tol_rel=1e-9, tol_abs=1e-9)
