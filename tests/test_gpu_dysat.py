"""DySAT streaming inference (csrc/dysat.cuh through the C ABI) against the
float64 oracle (oracle/dysat_oracle.py). Parity is unpinned against the
reference (it ships no DySAT code); the oracle recomputes every node from the
raw edge history, independently of the device path's incremental state."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2603_21090_b200 import _lib
    _lib.lib()
    return torch


CASES = {
    "tc_d128": dict(n=300, d_in=16, d=128, heads_s=16, heads_t=16, window=4, fanout=8,
                    snapshot_len=40.0, max_snapshots=256, batch_size=50),
    "tc_d64": dict(n=200, d_in=10, d=64, heads_s=4, heads_t=4, window=3, fanout=6,
                   snapshot_len=25.0, max_snapshots=256, batch_size=40),
    "small": dict(n=60, d_in=12, d=32, heads_s=4, heads_t=2, window=3, fanout=5,
                  snapshot_len=12.0, max_snapshots=256, batch_size=16),
    "wide_heads": dict(n=50, d_in=20, d=64, heads_s=16, heads_t=8, window=1, fanout=31,
                       snapshot_len=30.0, max_snapshots=256, batch_size=24),
    "d_odd": dict(n=40, d_in=7, d=36, heads_s=3, heads_t=6, window=5, fanout=3,
                  snapshot_len=7.0, max_snapshots=256, batch_size=9),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("tc", [True, False])
def test_dysat_matches_oracle(cuda, name, tc):
    from oracle.dysat_oracle import DySATOracle
    from paper_2603_21090_b200.dysat import DySATConfig, DySATEngine, init_dysat_params
    from paper_2603_21090_b200.streamio import generate_stream
    cfg = DySATConfig(**CASES[name])
    params = init_dysat_params(3, cfg)
    st = generate_stream(7, cfg.n, 300, d_e=0, attachment="preferential")
    eng = DySATEngine(cfg, params, tensor_cores=tc, tc_min_rows=1)  # every launch on tcgen05
    dt = cfg.d // cfg.heads_t
    assert eng.tensor_cores == (tc and cfg.d in (64, 128) and dt in (8, 16, 32) and dt <= cfg.d // 4)
    orc = DySATOracle(cfg, params)
    assert np.allclose(eng.embeddings(), orc.emb, rtol=1e-4, atol=1e-4)
    B = cfg.batch_size
    worst = 0.0
    for lo in range(0, len(st), B):
        s, d, t = st.src[lo:lo + B], st.dst[lo:lo + B], st.t[lo:lo + B]
        p = eng.process_batch_arrays(s, d, t)
        q = orc.process_batch(s, d, t)
        worst = max(worst, float(np.max(np.abs(p - np.array(q)))))
        assert eng.last_affected == orc.last_affected
        assert eng.snapshot == orc.snapshot
        e, r = eng.embeddings(), orc.emb
        err = np.max(np.abs(e - r) / (1.0 + np.abs(r)))
        assert err < 1e-4, (lo, err)
    assert worst < 1e-5
    assert orc.snapshot >= 3  # the stream crossed several snapshot boundaries
    lists = orc.lists(orc.snapshot)
    for v in range(cfg.n):
        assert eng.neighbor_list(v) == lists[v], v


def test_dysat_full_recompute_equals_incremental(cuda):
    from paper_2603_21090_b200.dysat import DySATConfig, DySATEngine, init_dysat_params
    from paper_2603_21090_b200.streamio import generate_stream
    cfg = DySATConfig(**CASES["small"])
    eng = DySATEngine(cfg, init_dysat_params(1, cfg))
    st = generate_stream(2, cfg.n, 200, d_e=0)
    for lo in range(0, len(st), cfg.batch_size):
        eng.process_batch_arrays(st.src[lo:lo + cfg.batch_size], st.dst[lo:lo + cfg.batch_size],
                                 st.t[lo:lo + cfg.batch_size])
    before = eng.embeddings()
    eng.full_recompute()
    np.testing.assert_array_equal(eng.embeddings(), before)


def test_dysat_gap_longer_than_window(cuda):
    """Snapshots without edges between batches, some gaps longer than W."""
    from oracle.dysat_oracle import DySATOracle
    from paper_2603_21090_b200.dysat import DySATConfig, DySATEngine, init_dysat_params
    cfg = DySATConfig(**CASES["small"])   # W = 3, snapshot_len = 12
    p = init_dysat_params(4, cfg)
    eng, orc = DySATEngine(cfg, p), DySATOracle(cfg, p)
    rng = np.random.default_rng(0)
    t0 = 0.0
    for gap in (0.0, 13.0, 60.0, 5.0, 200.0, 24.0):
        t0 += gap
        s, d = rng.integers(0, cfg.n, 8), rng.integers(0, cfg.n, 8)
        t = t0 + np.sort(rng.uniform(0, 3, 8))
        a = eng.process_batch_arrays(s, d, t)
        b = orc.process_batch(s, d, t)
        np.testing.assert_allclose(a, b, atol=1e-5)
        t0 = float(t[-1])
        e, r = eng.embeddings(), orc.emb
        assert np.max(np.abs(e - r) / (1.0 + np.abs(r))) < 1e-4
    assert eng.snapshot == orc.snapshot


def test_dysat_rejects_bad_input(cuda):
    from paper_2603_21090_b200.config import ConfigError
    from paper_2603_21090_b200.dysat import DySATConfig, DySATEngine, init_dysat_params
    from paper_2603_21090_b200.edges import MonotonicityError
    cfg = DySATConfig(**CASES["small"])
    eng = DySATEngine(cfg, init_dysat_params(1, cfg))
    eng.process_batch_arrays([1], [2], [5.0])
    with pytest.raises(MonotonicityError):
        eng.process_batch_arrays([1], [2], [4.0])
    with pytest.raises(ValueError):
        eng.process_batch_arrays([1], [cfg.n], [6.0])
    with pytest.raises(ConfigError):
        DySATConfig(n=10, d=30, heads_s=4).validate()
