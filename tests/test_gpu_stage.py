"""Stage-level surface on the GPU (csrc/stage.cuh through the C ABI): the
reference's own unit tests of detect_affected, update_neighbor_cache and the
scheduler (T/test_engine.py:37-125, T/test_drift.py:147-190) pointed at this
engine, plus equivalences with the fused process_batch on random streams."""

import numpy as np
import pytest

from golden_util import random_params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2603_21090_b200 import _lib
    _lib.lib()
    return torch


def _dims(layers=1, heads=2):
    from paper_2603_21090_b200.config import Dims
    return Dims(d_s=6, d_e=3, d_t=6, d_m=5, d_k=4, heads=heads, layers=layers)


def make_engine(dims=None, seed=55, **cfg_kw):
    from paper_2603_21090_b200.config import RunConfig
    from paper_2603_21090_b200.engine import IncrementalEngine
    dims = dims or _dims()
    return IncrementalEngine(RunConfig(dims=dims, **cfg_kw), random_params(seed, dims))


def feed(eng, edges, batch_size=None):
    b = batch_size or eng.cfg.batch_size
    for i in range(0, len(edges), b):
        eng.process_batch(edges[i:i + b])


def e(src, dst, t, d_e=3):
    from paper_2603_21090_b200.edges import TemporalEdge
    return TemporalEdge(src, dst, t, np.zeros(d_e))


# --- T/test_engine.py:37-57 -------------------------------------------------------
def _path_engine(layers):
    eng = make_engine(_dims(layers), batch_size=4, fanout=10, nodes=4)
    feed(eng, [e(0, 1, 1.0), e(1, 2, 2.0), e(2, 3, 3.0)], batch_size=3)
    return eng


def test_path_graph_one_hop(cuda):
    eng = _path_engine(1)
    aff = eng.detect_affected(eng.stage_batch([e(0, 1, 4.0)]))
    assert aff.direct == {0, 1}
    assert aff.all == {0, 1, 2}


def test_path_graph_two_hops(cuda):
    eng = _path_engine(2)
    aff = eng.detect_affected(eng.stage_batch([e(0, 1, 4.0)]))
    assert aff.all == {0, 1, 2, 3}


def test_staging_mutates_nothing(cuda):
    eng = _path_engine(2)
    before = {v: eng.nbr_cache.get(v) for v in range(4)}
    m = eng.store.m
    pend = eng.stage_batch([e(0, 1, 4.0), e(3, 3, 4.0)])
    assert [p.edge_id for p in pend] == [m, m + 1]
    eng.detect_affected(pend)
    assert eng.store.m == m
    assert {v: eng.nbr_cache.get(v) for v in range(4)} == before


@pytest.mark.parametrize("layers,fanout,window", [(1, 2, np.inf), (1, 5, np.inf), (2, 2, np.inf),
                                                  (2, 5, np.inf), (2, 3, 20.0)])
def test_detect_affected_equals_process_batch(cuda, layers, fanout, window):
    """The staged (uncommitted) affected set equals the one the fused batch
    computes for the same edges, on random histories with self-loops and
    duplicates."""
    from paper_2603_21090_b200.edges import TemporalEdge
    dims = _dims(layers, heads=1)
    rng = np.random.default_rng(layers * 100 + fanout)
    for trial in range(12):
        n = int(rng.integers(4, 40))
        m = int(rng.integers(3, 80))
        hist = [TemporalEdge(int(rng.integers(0, n)), int(rng.integers(0, n)), float(t),
                             np.zeros(3)) for t in range(m)]
        b = int(rng.integers(1, 6))
        batch = [TemporalEdge(int(rng.integers(0, n)), int(rng.integers(0, n)), float(m + i),
                              np.zeros(3)) for i in range(b)]
        eng = make_engine(dims, seed=trial, batch_size=8, fanout=fanout, nodes=n, window=window)
        feed(eng, hist, 16)
        staged = eng.detect_affected(eng.stage_batch(batch))
        eng.process_batch(batch)
        got = eng.last_affected
        assert staged.direct == got.direct, trial
        assert staged.all == got.all, trial


# --- T/test_engine.py:80-125 ------------------------------------------------------
def test_insert_evict(cuda):
    from paper_2603_21090_b200.edges import NeighborEntry
    eng = make_engine(batch_size=4, fanout=3, nodes=8)
    feed(eng, [e(0, 1, 1.0), e(0, 2, 3.0), e(0, 3, 5.0)], batch_size=3)
    assert [x.t for x in eng.nbr_cache.get(0)] == [5.0, 3.0, 1.0]
    new = [NeighborEntry(4, 7.0, eng.store.m)]
    eng._pending.clear()
    eng.stage_batch([e(0, 4, 7.0)])
    rec = eng.update_neighbor_cache(0, new, {0, 4}, 7.0)
    assert [x.t for x in eng.nbr_cache.get(0)] == [7.0, 5.0, 3.0]
    assert [x.t for x in rec.expired] == [1.0]
    assert [x.t for x in rec.added] == [7.0]
    assert rec.updated == set()


def test_infinite_window_never_expires(cuda):
    eng = make_engine(batch_size=2, fanout=10, nodes=4)
    feed(eng, [e(0, 1, 1.0), e(0, 2, 1000.0)], batch_size=1)
    assert len(eng.nbr_cache.get(0)) == 2


def test_finite_window_marks_expired(cuda):
    from paper_2603_21090_b200.edges import NeighborEntry
    eng = make_engine(batch_size=1, fanout=10, nodes=4, window=5.0)
    feed(eng, [e(0, 1, 1.0)], batch_size=1)
    eng.stage_batch([e(0, 2, 10.0)])
    new = [NeighborEntry(2, 10.0, 1)]
    rec = eng.update_neighbor_cache(0, new, {0, 2}, 10.0)
    assert [x.t for x in rec.expired] == [1.0]
    assert [x.t for x in eng.nbr_cache.get(0)] == [10.0]


def test_fresh_node_keeps_exactly_new(cuda):
    from paper_2603_21090_b200.edges import NeighborEntry
    eng = make_engine(batch_size=2, fanout=5, nodes=4)
    eng.stage_batch([e(3, 1, 1.0), e(3, 2, 1.0)])
    new = [NeighborEntry(2, 1.0, 1), NeighborEntry(1, 1.0, 0)]
    rec = eng.update_neighbor_cache(3, new, {1, 2, 3}, 1.0)
    assert len(eng.nbr_cache.get(3)) == 2
    assert rec.expired == []
    assert eng.counters.get("nbr_miss") == 1


def test_updated_lists_direct_neighbours(cuda):
    """updated = the kept older entries whose neighbour is direct."""
    from paper_2603_21090_b200.edges import NeighborEntry
    eng = make_engine(batch_size=4, fanout=4, nodes=8)
    feed(eng, [e(0, 1, 1.0), e(0, 2, 2.0), e(0, 1, 3.0)], batch_size=3)
    m = eng.store.m
    eng.stage_batch([e(0, 5, 4.0)])
    rec = eng.update_neighbor_cache(0, [NeighborEntry(5, 4.0, m)], {0, 5, 1}, 4.0)
    assert rec.updated == {1}
    assert rec.expired == []
    assert [x.nbr for x in eng.nbr_cache.get(0)] == [5, 1, 2, 1]


def _ring_rows(eng, v):
    """(nbr, eid, t, payload, feat, basis) of v's cached list, newest first."""
    tab, L = eng._tab, eng.L
    k = int(tab.ring_ccnt[v])
    sl = [(int(tab.ring_head[v]) + j) % L for j in range(max(k, 0))]
    return (tab.ring_nbr[v][sl], tab.ring_eid[v][sl], tab.ring_t[v][sl], tab.ring_pay[v][:, sl],
            tab.ring_feat[v][sl], tab.ring_tb[v][sl])


@pytest.mark.parametrize("layers,window", [(1, np.inf), (2, np.inf), (2, 6.0)])
def test_stage_update_commit_equals_process_batch(cuda, layers, window):
    """The reference's process_batch stage order (S/engine.py:415-422):
    stage_batch -> detect_affected -> update_neighbor_cache on every affected
    node -> commit_pending leaves the same lists, records, store and frozen
    ring payloads as the fused batch."""
    from paper_2603_21090_b200.edges import NeighborEntry
    from paper_2603_21090_b200.streamio import generate_stream
    torch = cuda
    dims = _dims(layers)
    st = generate_stream(4, 30, 260, d_e=3)
    hist, tail = st.as_edges()[:200], st.as_edges()[200:]
    kw = dict(batch_size=12, fanout=4, nodes=30, window=window)
    a, b = make_engine(dims, **kw), make_engine(dims, **kw)
    feed(a, hist)
    feed(b, hist)
    for lo in range(0, len(tail), 12):
        batch = tail[lo:lo + 12]
        pend = a.stage_batch(batch)
        aff = a.detect_affected(pend)
        by_node = {}
        for pe in reversed(pend):
            by_node.setdefault(pe.src, []).append(NeighborEntry(pe.dst, pe.t, pe.edge_id))
            if pe.dst != pe.src:
                by_node.setdefault(pe.dst, []).append(NeighborEntry(pe.src, pe.t, pe.edge_id))
        recs = {v: a.update_neighbor_cache(v, by_node.get(v, []), aff.direct, batch[-1].t)
                for v in sorted(aff.all)}
        a.commit_pending()
        b.process_batch(batch)
        la = b.last_affected
        assert aff.all == la.all and aff.direct == la.direct
        for v in aff.all:
            assert recs[v].size == la.records[v].size, v
        for v in range(30):
            assert a.nbr_cache.get(v) == b.nbr_cache.get(v), v
            assert a.store.recent_upto(v, 100) == b.store.recent_upto(v, 100), v
        assert a.store.m == b.store.m
        if lo == 0:  # same pre-batch state: the frozen payloads agree bit for bit
            for v in range(30):
                for x, y in zip(_ring_rows(a, v), _ring_rows(b, v)):
                    assert torch.equal(x, y), v


def test_commit_keeps_uncached_nodes_uncached(cuda):
    eng = make_engine(batch_size=4, fanout=3, nodes=8)
    eng.stage_batch([e(5, 6, 1.0), e(5, 7, 2.0)])
    eng.commit_pending()
    assert eng.nbr_cache.get(5) is None
    assert [x.nbr for x in eng.store.recent_upto(5, 3)] == [7, 6]
    eng.process_batch([e(5, 1, 3.0)])
    assert [x.nbr for x in eng.nbr_cache.get(5)] == [1, 7, 6]


# --- T/test_drift.py:147-190 --------------------------------------------------------
def _drift_engine(**kw):
    from paper_2603_21090_b200.streamio import generate_stream
    dims = _dims()
    eng = make_engine(dims, seed=66, batch_size=5, fanout=4, nodes=20, **kw)
    st = generate_stream(2, 20, 150, d_e=3)
    feed(eng, st.as_edges(), 5)
    return eng


def test_full_rebuild_matches_reference(cuda):
    eng = _drift_engine()
    eng.scheduler.record_batch_changes({0: (1, 2)})
    eng.scheduler.note_affected({0})
    eng.scheduler.execute_rebuild(("full", None), eng)
    ref = eng.full_reference()
    n = ref.shape[0]
    np.testing.assert_array_equal(eng.cache.embeddings(n), ref)
    assert eng.scheduler.global_drift() == 0.0


def test_partial_rebuild_leaves_others_untouched(cuda):
    eng = _drift_engine()
    before = eng.cache.h.copy()
    eng.scheduler.execute_rebuild(("partial", {1, 2}), eng)
    for v in range(20):
        if v in (1, 2):
            continue
        np.testing.assert_array_equal(eng.cache.h[v], before[v])


def test_reset_after_any_rebuild(cuda):
    eng = _drift_engine()
    eng.scheduler.record_batch_changes({4: (5, 5)})
    eng.scheduler.note_affected({4})
    assert eng.scheduler.global_drift() > 0
    eng.scheduler.execute_rebuild(("partial", {4}), eng)
    assert eng.scheduler.global_drift() == 0.0
    assert eng.scheduler.tau == 0


def test_record_and_decide_follow_the_reference_rules(cuda):
    from paper_2603_21090_b200.edges import DriftContractError
    eng = _drift_engine(rebuild="never", gamma=0.5, delta_max=0.3, alpha=0.5)
    s = eng.scheduler
    s.reset()
    assert s.decide_rebuild(20) is None
    s.record_batch_changes({1: (1, 1), 2: (1, 4)})
    s.note_affected({1, 2, 3})
    assert s.tau == 1
    assert s.estimator(1) == 1.0 and s.estimator(2) == 0.25 and s.estimator(3) == 0.0
    assert s.global_drift() == pytest.approx(1.25 / 3)
    assert s.decide_rebuild(20) == ("partial", {1})
    assert s.decide_rebuild(2) == ("full", None)  # |drifted| >= alpha n
    s.record_batch_changes({})
    assert s.estimator(1) == 0.5  # lazy decay: gamma^(tau - touched)
    with pytest.raises(DriftContractError):
        s.record_batch_changes({5: (1, 0)})
    with pytest.raises(DriftContractError):
        s.execute_rebuild(None, eng)
