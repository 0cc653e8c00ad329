"""Pin the oracle (and the boundary types) to fixtures written by the
reference itself (tests/golden/make_golden.py). CPU only."""

import numpy as np
import pytest

from golden_util import GOLDEN, batches, case_setup, engine_cases, load, pipeline_cases
from oracle import stgn_oracle as orc
from paper_2603_21090_b200.config import Dims
from paper_2603_21090_b200.params import init_params
from paper_2603_21090_b200.streamio import generate_stream


@pytest.mark.parametrize("name", engine_cases())
def test_oracle_engine_matches_reference_bitwise(name):
    z = load("engine_" + name)
    cfg, params, stream = case_setup(z)
    o = orc.Oracle(cfg, params)
    preds, aff, dirs, kinds, cnts = [], [], [], [], []
    for b in batches(stream, cfg.batch_size):
        preds.extend(o.process_batch(b.src, b.dst, b.t, b.feat))
        aff.extend(sorted(o.last_all))
        dirs.extend(sorted(o.last_direct))
        kinds.append({"none": 0, "partial": 1, "full": 2}[o.last_report["rebuild"]])
        cnts.append(o.last_report["rebuild_nodes"])
    assert np.array_equal(np.array(aff), z["affected"])
    assert np.array_equal(np.array(dirs), z["direct"])
    assert np.array_equal(np.array(kinds), z["rebuild_kind"])
    assert np.array_equal(np.array(cnts), z["rebuild_cnt"])
    np.testing.assert_array_equal(np.array(preds), z["preds"])
    n = int(z["node_count"])
    assert o.node_count == n
    np.testing.assert_array_equal(o.mem[:n], z["memory"])
    np.testing.assert_array_equal(o.last[:n], z["last"])
    np.testing.assert_array_equal(o.version[:n], z["version"])
    np.testing.assert_array_equal(o.h[:n], z["h"])
    np.testing.assert_array_equal(o.valid_at[:n], z["valid_at"])
    for v in range(n):
        lst = o.neighbor_list(v)
        c = int(z["cache_cnt"][v])
        if c < 0:
            assert lst is None
            continue
        assert [x[0] for x in lst] == list(z["cache_nbr"][v, :c])
        assert [x[2] for x in lst] == list(z["cache_eid"][v, :c])
        assert [x[1] for x in lst] == list(z["cache_t"][v, :c])
    np.testing.assert_array_equal(o.full_reference(), z["full_reference"])
    assert o.tau == int(z["tau"])
    assert o.global_drift() == pytest.approx(float(z["global_drift"]), rel=1e-12, abs=0)


@pytest.mark.parametrize("name", pipeline_cases())
def test_oracle_pipeline_matches_reference_bitwise(name):
    z = load("pipeline_" + name)
    outs = orc.pipeline_many(z["qbase"], z["offsets"], z["payload"], z["feat"], z["dt"],
                             z["omega"], z["phi0"], z["wq"], z["wk"], z["wv"], z["wo"])
    for key, got in zip(("out", "scores", "values", "maxlog", "zsum", "qvecs"), outs):
        np.testing.assert_array_equal(got, z[key], err_msg=key)


def test_init_params_bit_identical():
    z = load("params_seed")
    for tag, dims in (("a", Dims(d_s=6, d_e=3, d_t=6, d_m=5, d_k=4, heads=2, layers=1)),
                      ("b", Dims(d_s=100, d_e=172, d_t=100, d_m=100, d_k=50, heads=2,
                                 layers=2))):
        for k, v in init_params(12345, dims).tensors().items():
            np.testing.assert_array_equal(v, z[f"{tag}_{k}"], err_msg=k)


def test_generate_stream_bit_identical():
    z = load("streams")
    kws = [dict(seed=0, n=50, m=400, attachment="uniform", d_e=3),
           dict(seed=1, n=100, m=1500, attachment="preferential", burstiness=2.0, d_e=4),
           dict(seed=2, n=2000, m=5000, attachment="preferential", d_e=0)]
    for i, kw in enumerate(kws):
        s = generate_stream(**kw)
        np.testing.assert_array_equal(s.src, z[f"s{i}_src"])
        np.testing.assert_array_equal(s.dst, z[f"s{i}_dst"])
        np.testing.assert_array_equal(s.t, z[f"s{i}_t"])
        np.testing.assert_array_equal(s.feat, z[f"s{i}_feat"])


def test_brute_force_matches_affected_on_golden():
    z = load("engine_k2_last_adaptive")
    cfg, params, stream = case_setup(z)
    o = orc.Oracle(cfg, params)
    for b in batches(stream, cfg.batch_size):
        o.process_batch(b.src, b.dst, b.t, b.feat)
        brute = orc.brute_force_affected(o, b.src, b.dst, cfg.fanout, cfg.dims.layers)
        assert brute == o.last_all
        assert len(o.last_all) <= 2 * len(b) * cfg.fanout ** cfg.dims.layers
