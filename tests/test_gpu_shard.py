"""The node-id-range-sharded engine (paper_2603_21090_b200/shard.py) against a
single engine on one GPU: all shards of a world run in one process
(ShardGroup: the same neighbour-feature and prediction-row exchanges as the
NCCL path, delivered in process). Scores, the affected sets, and every node's
memory and layer-cache rows (taken from its owner) must equal the single
engine's; the topology is replicated, so every shard's affected set is the
full one."""

import numpy as np
import pytest

from golden_util import batches, case_setup, load
from parity_util import PRED_ATOL, assert_rows_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2603_21090_b200 import _lib
    _lib.lib()
    return torch


@pytest.mark.parametrize("name,world", [("k2_last_adaptive", 2), ("k2_last_adaptive", 3),
                                        ("k1_fixed_de0", 2), ("c4_shape_tiny", 4)])
def test_sharded_engine_matches_single_engine(cuda, name, world):
    import dataclasses
    from paper_2603_21090_b200.engine import IncrementalEngine
    from paper_2603_21090_b200.shard import ShardGroup
    z = load("engine_" + name)
    cfg, params, stream = case_setup(z)
    n = int(z["node_count"])
    cfg = dataclasses.replace(cfg, nodes=max(cfg.nodes, n))
    single = IncrementalEngine(cfg, params)
    group = ShardGroup(cfg, params, world)
    for b in batches(stream, cfg.batch_size):
        p1 = single.process_batch_arrays(b.src, b.dst, b.t, b.feat)
        p2 = group.process_batch_arrays(b.src, b.dst, b.t, b.feat)
        assert np.max(np.abs(p1 - p2)) <= PRED_ATOL
        for sh in group.shards:
            assert sh.eng.last_affected.all == single.last_affected.all
            assert sh.eng.last_report.rebuild == single.last_report.rebuild
    n = cfg.nodes
    assert_rows_close(group.memory()[:n], single.memory.states[:n], "sharded memory")
    assert_rows_close(group.layers()[:n].reshape(n, -1), single.cache.h[:n].reshape(n, -1),
                      "sharded layer cache")
    # the reference's fixture too (the single engine is pinned to it elsewhere)
    nz = int(z["node_count"])
    assert_rows_close(group.layers()[:nz].reshape(nz, -1), z["h"].reshape(nz, -1), "vs reference")


def test_sharded_engine_keeps_only_its_payload_rows(cuda):
    import dataclasses
    from paper_2603_21090_b200.shard import ShardGroup
    z = load("engine_k2_last_adaptive")
    cfg, params, _ = case_setup(z)
    cfg = dataclasses.replace(cfg, nodes=max(cfg.nodes, int(z["node_count"])))
    group = ShardGroup(cfg, params, 2)
    for sh in group.shards:
        tab = sh.eng._tab
        assert tab.ring_pay.shape[0] == sh.hi - sh.lo
        assert tab.mem.shape[0] >= cfg.nodes  # small per-node state stays whole
