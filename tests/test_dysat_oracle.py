"""The DySAT oracle (test infrastructure) on hand-checkable cases, on CPU:
an isolated node's structural row is ELU(P_v), a single-snapshot window makes
the temporal softmax trivial (emb = v W_o + y), lists keep the L newest
entries of the snapshot only, and prediction uses the pre-batch embeddings."""

import math

import numpy as np

from oracle.dysat_oracle import DySATOracle, _elu
from paper_2603_21090_b200.dysat import DySATConfig, init_dysat_params


def _cfg(**kw):
    base = dict(n=6, d_in=5, d=8, heads_s=2, heads_t=2, window=1, fanout=2, snapshot_len=10.0,
                max_snapshots=16, batch_size=4)
    base.update(kw)
    return DySATConfig(**base)


def test_isolated_node_and_trivial_window():
    cfg = _cfg()
    p = init_dysat_params(0, cfg)
    o = DySATOracle(cfg, p)
    P = p.x @ p.w_s
    z = o.structural(0)
    np.testing.assert_allclose(z, _elu(P), rtol=1e-12)
    y = z + p.pos[0]
    np.testing.assert_allclose(o.emb, (y @ p.w_v) @ p.w_o + y, rtol=1e-12)


def test_lists_are_per_snapshot_newest_first():
    cfg = _cfg()
    o = DySATOracle(cfg, init_dysat_params(0, cfg))
    o.process_batch([0, 0, 0], [1, 2, 3], [1.0, 2.0, 3.0])
    assert o.lists(0)[0] == [3, 2]
    assert o.lists(0)[1] == [0]
    o.process_batch([4], [4], [15.0])        # next snapshot; a self-loop is one entry
    assert o.snapshot == 1
    assert o.lists(1)[4] == [4] and o.lists(1)[0] == []


def test_structural_attention_by_hand():
    cfg = _cfg(heads_s=1)
    p = init_dysat_params(1, cfg)
    o = DySATOracle(cfg, p)
    o.process_batch([0], [1], [1.0])
    P = p.x @ p.w_s
    e = np.array([p.a_self[0] @ P[0] + p.a_nbr[0] @ P[u] for u in (0, 1)])
    e = np.where(e > 0, e, 0.2 * e)
    a = np.exp(e - e.max())
    a /= a.sum()
    np.testing.assert_allclose(o.structural(0)[0], _elu(a[0] * P[0] + a[1] * P[1]), rtol=1e-12)


def test_prediction_uses_pre_batch_embeddings():
    cfg = _cfg()
    p = init_dysat_params(2, cfg)
    o = DySATOracle(cfg, p)
    e0 = o.emb.copy()
    got = o.process_batch([2], [3], [1.0])[0]
    x = p.w_pred[:cfg.d] @ e0[2] + p.w_pred[cfg.d:] @ e0[3] + p.b_pred
    assert got == 1.0 / (1.0 + math.exp(-x))
    assert o.last_affected == {2, 3}
