"""EdgeRing / form_batch (paper_2603_21090_b200/streaming.py) against the
reference EdgeQueue / form_batch contract, restated from the reference's own
tests (T/test_graph_store.py:19-80, T/test_batcher.py:24-45). CPU only."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2603_21090_b200.edges import FeatureDimError, TemporalEdge
from paper_2603_21090_b200.streaming import EdgeRing, form_batch


def edge(src, dst, t, d_e=0):
    return TemporalEdge(src, dst, t, np.zeros(d_e))


def test_enqueue_into_empty_and_full_rejects():
    q = EdgeRing(4, d_e=0, pinned=False)
    assert q.enqueue(edge(0, 1, 1.0)) is True and q.occupancy == 1
    for i in range(3):
        assert q.enqueue(edge(0, 1, float(i + 2)))
    assert q.enqueue(edge(0, 1, 9.0)) is False
    assert q.occupancy == 4


def test_feature_mismatch_is_error_not_false():
    q = EdgeRing(4, d_e=3, pinned=False)
    with pytest.raises(FeatureDimError):
        q.enqueue(edge(0, 1, 1.0, d_e=2))


def test_flush_order_partial_underfull_and_window():
    q = EdgeRing(16, d_e=0, pinned=False)
    for i in range(10):
        q.enqueue(edge(i, i + 1, float(i)))
    src, dst, t, _ = q.flush_batch(4)
    assert src.tolist() == [0, 1, 2, 3] and t.tolist() == [0.0, 1.0, 2.0, 3.0]
    assert q.occupancy == 6
    src, _, t, _ = q.flush_batch(10, before=7.0)
    assert t.tolist() == [4.0, 5.0, 6.0] and q.occupancy == 3
    assert len(q.flush_batch(600)[0]) == 3
    assert len(q.flush_batch(5)[0]) == 0


def test_form_batch_timestamp_staleness_and_empty():
    q = EdgeRing(64, d_e=0, pinned=False)
    for s, t in ((0, 1.0), (1, 2.0), (2, 3.0)):
        q.enqueue(edge(s, s + 1, t))
    b = form_batch(q, 3)
    assert b.t_batch == 3.0 and b.s_max == 2.0
    q.enqueue(edge(0, 1, 7.0))
    assert form_batch(q, 4).s_max == 0.0
    assert form_batch(q, 4) is None


@given(st.lists(st.tuples(st.booleans(), st.integers(1, 5)), max_size=60))
@settings(max_examples=100, deadline=None)
def test_fifo_roundtrip_against_list_oracle(ops):
    """Any interleaving of (vectorised) enqueues and flushes emits edges in
    exactly enqueue order, with reject-on-full taking a prefix."""
    q = EdgeRing(8, d_e=2, pinned=False)
    oracle, out, nxt = [], [], 0
    for is_enq, k in ops:
        if is_enq:
            src = np.arange(nxt, nxt + k)
            acc = q.enqueue_arrays(src, src + 1, src.astype(np.float64), np.ones((k, 2)) * src[:, None])
            oracle.extend(range(nxt, nxt + acc))
            nxt += k
        else:
            s, d, t, f = q.flush_batch(k)
            out.extend(s.tolist())
            assert (d == s + 1).all() and (t == s).all() and (f[:, 0] == s).all()
    out.extend(q.flush_batch(100)[0].tolist())
    assert out == oracle
