"""N>1 host logic on CPU (gloo, world_size 2): node-range sharding of the
full rebuild, the row all-gather, max-over-ranks timing, replica seeds.
The per-shard recompute is the oracle here (test infrastructure); on B200s
it is IncrementalEngine.rebuild_range over NCCL."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_21090_b200.dist import max_over_ranks, replica_seeds, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions():
    for n in (0, 1, 7, 100, 2_600_000):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
    assert list(replica_seeds(2, 4)) == [2, 3, 4, 5]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        here = os.path.dirname(os.path.abspath(__file__))
        sys.path.insert(0, here)
        sys.path.insert(0, os.path.dirname(here))
        from golden_util import batches, case_setup, load
        from oracle.stgn_oracle import Oracle
        from paper_2603_21090_b200.dist import sharded_rebuild

        z = load("engine_k2_wide_adaptive")
        cfg, params, stream = case_setup(z)
        cfg = cfg.with_(rebuild="never")
        orc = Oracle(cfg, params)       # every rank holds the same (replicated) state
        for b in batches(stream, cfg.batch_size):
            orc.process_batch(b.src, b.dst, b.t, b.feat)
        n = orc.node_count

        def recompute(lo, hi):
            if hi > lo:
                orc.rebuild_nodes(range(lo, hi))
            return torch.tensor(orc.h[lo:hi])

        rows = sharded_rebuild(recompute, n)
        ref = Oracle(cfg, params)
        for b in batches(stream, cfg.batch_size):
            ref.process_batch(b.src, b.dst, b.t, b.feat)
        ref.rebuild_nodes(None)
        ok = bool(np.array_equal(rows.numpy(), ref.h[:n]))
        t = max_over_ranks(1.0 + rank)
        out[rank] = (ok, t, rows.shape[0] == n)
    finally:
        dist.destroy_process_group()


def test_sharded_full_rebuild_world2():
    world = 2
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world,
                           start_method="spawn", join=True)
        res = dict(out)
    for r in range(world):
        ok, t, full = res[r]
        assert ok, f"rank {r}: sharded rebuild differs from the single-process rebuild"
        assert full
        assert t == 2.0  # max over ranks
