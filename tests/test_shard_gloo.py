"""Sharded-engine host logic on CPU (gloo, world sizes 2 and 3): node-id
ownership, the routing of the neighbour-feature (stack) exchange, and the
TorchComm all-to-all / all-gather the ShardedEngine runs over NCCL on B200s
(paper_2603_21090_b200/shard.py). The device phases are covered on the GPU by
tests/test_gpu_parity.py::test_sharded_engine_matches_single_engine."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_21090_b200.dist import shard_range
from paper_2603_21090_b200.shard import owners, stack_routes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bounds(n, world):
    return np.array([shard_range(n, world, r)[0] for r in range(world)] + [n])


def test_owners_and_routes():
    rng = np.random.default_rng(0)
    n, world = 97, 3
    b = _bounds(n, world)
    ids = np.arange(n)
    own = owners(b, ids)
    for r in range(world):
        lo, hi = shard_range(n, world, r)
        assert (own[lo:hi] == r).all()
    src, dst = rng.integers(0, n, 400), rng.integers(0, n, 400)
    for r in range(world):
        routes = stack_routes(b, r, src, dst)
        assert routes[r].size == 0
        for q in range(world):
            if q == r:
                continue
            # exactly r's endpoints of edges whose other end q owns
            want = set()
            for s_, d_ in zip(src, dst):
                if owners(b, [s_])[0] == r and owners(b, [d_])[0] == q:
                    want.add(int(s_))
                if owners(b, [d_])[0] == r and owners(b, [s_])[0] == q:
                    want.add(int(d_))
            assert set(routes[q].tolist()) == want
            assert (np.diff(routes[q]) > 0).all()


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_21090_b200.shard import TorchComm
        comm = TorchComm()
        n, width = 50, 6
        b = _bounds(n, world)
        rng = np.random.default_rng(7)   # the same batch on every rank
        src, dst = rng.integers(0, n, 64), rng.integers(0, n, 64)
        # every node's "stack" is a known function of its id
        table = torch.arange(n, dtype=torch.float32)[:, None] * 10 + torch.arange(width)
        routes = stack_routes(b, rank, src, dst)
        sends_n = [torch.from_numpy(rt).to(torch.int32) for rt in routes]
        sends_r = [table[torch.from_numpy(rt)] for rt in routes]
        got_n = comm.all_to_all(sends_n)
        got_r = comm.all_to_all(sends_r)
        ok = True
        need = set()
        for s_, d_ in zip(src, dst):  # stacks this rank needs: others' ends of its edges
            os_, od = owners(b, [s_])[0], owners(b, [d_])[0]
            if od == rank and os_ != rank:
                need.add(int(s_))
            if os_ == rank and od != rank:
                need.add(int(d_))
        got = set()
        for q in range(world):
            for k, v in enumerate(got_n[q].tolist()):
                got.add(v)
                ok &= owners(b, [v])[0] == q
                ok &= bool(torch.equal(got_r[q][k], table[v]))
        ok &= got == need
        # variable-size all-gather
        mine = torch.full((rank + 2, 3), float(rank))
        allg = comm.all_gather(mine)
        ok &= [a.shape[0] for a in allg] == [q + 2 for q in range(world)]
        ok &= all(bool((a == q).all()) for q, a in enumerate(allg))
        out[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


def _run(world):
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    return [out[r] for r in range(world)]


def test_stack_exchange_gloo_world2():
    assert all(_run(2))


def test_stack_exchange_gloo_world3():
    assert all(_run(3))
