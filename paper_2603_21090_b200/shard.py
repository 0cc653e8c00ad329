"""Node-range-sharded incremental engine (BASELINE north_star:
"million-node graphs are partitioned by node-id range across the GPUs of one
box; cross-shard frontier and neighbour-feature exchange over NCCL").

The reference has no multi-GPU code (PAPER.md:2389-2393 lists it as future
work); this is the B200 design for the same per-batch semantics
(S/engine.py:400-438), one engine per rank:

  * Ownership. Rank r owns node ids [lo_r, hi_r) (dist.shard_range). It keeps
    the frozen payload rows of its nodes' neighbour rings (ring_pay, the time
    basis and the edge features: ~12 KB of the ~14 KB per node at C4) and is
    the only rank that recomputes their embeddings.
  * Replicated topology. Every rank ingests every edge into the ring metadata
    (neighbour ids, times, edge ids), the append-only store and the drift
    estimators, which are small (~200 B per node). The K-hop affected set,
    the change records and the rebuild decisions are therefore computed
    identically on every rank without a per-hop frontier exchange.
  * Neighbour-feature exchange (before a batch). A ring entry of node v
    freezes the pre-batch stack [s_u || h_u,0 .. h_u,K-2] of the other end u
    (S/engine_base.py:88-106, 124-129), and v's message reads s_u
    (S/engine_base.py:193-247). For every edge whose endpoints have different
    owners, each owner sends its endpoint's stack to the other owner:
    one all-to-all (NCCL all_to_all_single with per-rank splits).
  * Prediction exchange (mid-batch). predict_link needs the final-layer
    embeddings of both endpoints (S/engine.py:425-426); each rank computes its
    owned direct nodes' rows, an all-gather completes the set on every rank,
    and every rank then finishes the batch (scores, memory commit, drift,
    rebuild of its own nodes) identically.

The batch runs in two device phases around that exchange
(stgn_engine_batch_phase). Exchanges go through a `Comm`: TorchComm over
torch.distributed (NCCL on the B200 box; gloo in the CPU tests), or the
in-process ShardGroup driver that runs all shards of a world on one device
(the parity test against a single engine).
"""

from __future__ import annotations

import numpy as np

from .dist import shard_range


# ---------------------------------------------------------------------------
class TorchComm:
    """Exchanges over torch.distributed (one process per GPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_to_all(self, chunks):
        """chunks[r]: tensor sent to rank r (same trailing shape and dtype on
        every rank); returns the tensors received from each rank."""
        import torch
        dist = self.dist
        dev = chunks[0].device
        tail = tuple(chunks[0].shape[1:])
        counts = torch.tensor([c.shape[0] for c in chunks], dtype=torch.int64, device=dev)
        recv_counts = torch.empty_like(counts)
        dist.all_to_all_single(recv_counts, counts, group=self.group)
        rc = [int(x) for x in recv_counts.tolist()]
        width = int(np.prod(tail)) if tail else 1
        send = torch.cat([c.reshape(c.shape[0], width) for c in chunks], 0)
        recv = torch.empty((sum(rc), width), dtype=send.dtype, device=dev)
        # uneven splits: NCCL on the B200 box, gloo in the CPU tests
        dist.all_to_all_single(recv, send, rc, [c.shape[0] for c in chunks], group=self.group)
        out, o = [], 0
        for n in rc:
            out.append(recv[o:o + n].reshape((n,) + tail))
            o += n
        return out

    def all_gather(self, t):
        """Variable first dimension: returns every rank's tensor."""
        import torch
        dist = self.dist
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        ns = [torch.empty_like(n) for _ in range(self.world)]
        dist.all_gather(ns, n, group=self.group)
        ns = [int(x.item()) for x in ns]
        cap = max(ns) if ns else 0
        pad = torch.zeros((cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[:t.shape[0]] = t
        out = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(out, pad, group=self.group)
        return [o[:k] for o, k in zip(out, ns)]


# ---------------------------------------------------------------------------
def owners(bounds: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """Rank owning each node id (bounds = [lo_0, lo_1, ..., n])."""
    return np.searchsorted(bounds, np.asarray(ids), side="right") - 1


def stack_routes(bounds, rank: int, src, dst):
    """Per destination rank, the sorted unique nodes of `rank` whose stacks the
    destination needs: endpoints owned by `rank` of edges whose other end
    another rank owns."""
    src, dst = np.asarray(src, dtype=np.int64), np.asarray(dst, dtype=np.int64)
    os_, od = owners(bounds, src), owners(bounds, dst)
    world = len(bounds) - 1
    out = []
    for r in range(world):
        if r == rank:
            out.append(np.zeros(0, dtype=np.int64))
            continue
        a = src[(os_ == rank) & (od == r)]
        b = dst[(od == rank) & (os_ == r)]
        out.append(np.unique(np.concatenate([a, b])))
    return out


class ShardedEngine:
    """One rank's shard of the incremental engine: IncrementalEngine's batch
    surface (process_batch_arrays returns the batch's scores, identical on
    every rank) with node-id-range ownership; see the module docstring."""

    def __init__(self, cfg, params, rank: int, world: int, comm=None, **kw):
        from .config import ConfigError
        from .engine import IncrementalEngine
        if cfg.nodes <= 0:
            raise ConfigError("a sharded engine needs cfg.nodes (the node-id range to split)")
        if cfg.mode == "delta":
            raise ConfigError("delta mode is single-engine only")
        self.rank, self.world, self.comm = rank, world, comm
        self.n = cfg.nodes
        self.lo, self.hi = shard_range(self.n, world, rank)
        self.bounds = np.array([shard_range(self.n, world, r)[0] for r in range(world)] + [self.n])
        self.eng = IncrementalEngine(cfg, params, shard=(self.lo, self.hi), **kw)
        self.cfg, self.params, self.dims = cfg, params, params.dims

    # -- neighbour-feature exchange ------------------------------------------
    def stack_sends(self, src, dst):
        """(nodes, stacks) per destination rank: the pre-batch stacks
        [s_u | h_u,0 .. h_u,K-2] of this rank's endpoints on cross-shard edges."""
        torch = self.eng._torch
        routes = stack_routes(self.bounds, self.rank, src, dst)
        out = []
        for nodes in routes:
            idx = torch.from_numpy(nodes).to(self.eng.device)
            out.append((idx.to(torch.int32), self.eng.gather_stacks(idx)))
        return out

    def stack_recv(self, received):
        """Write the other owners' stacks into this rank's ghost rows."""
        torch = self.eng._torch
        nodes = [n for n, _ in received if n.shape[0]]
        if not nodes:
            return
        rows = torch.cat([r for n, r in received if n.shape[0]], 0)
        self.eng.scatter_stacks(torch.cat(nodes, 0).to(torch.int64), rows)

    # -- the two device phases around the prediction exchange -----------------
    def phase1(self, src, dst, t, feat=None):
        self.eng.batch_phase1(src, dst, t, feat)
        return self.eng.dpred_export()

    def phase2(self, gathered):
        self.eng.dpred_import(gathered)
        return self.eng.batch_phase2()

    def process_batch_arrays(self, src, dst, t, feat=None):
        """One batch on this rank, exchanges through self.comm (collective: every
        rank calls it with the same batch)."""
        torch = self.eng._torch
        sends = self.stack_sends(src, dst)
        got_n = self.comm.all_to_all([n for n, _ in sends])
        w = self.eng.stack_width
        got_r = self.comm.all_to_all([r.reshape(-1, w) for _, r in sends])
        self.stack_recv(list(zip(got_n, got_r)))
        nodes, rows = self.phase1(src, dst, t, feat)
        all_n = self.comm.all_gather(nodes)
        all_r = self.comm.all_gather(rows)
        return self.phase2((torch.cat(all_n, 0), torch.cat(all_r, 0)))

    # -- owned views ----------------------------------------------------------
    def owned_layers(self):
        """(lo, hi, h[lo:hi]) of this rank's nodes."""
        return self.lo, self.hi, self.eng.cache.h[self.lo:self.hi]

    def owned_memory(self):
        return self.lo, self.hi, self.eng.memory.states[self.lo:self.hi]


class ShardGroup:
    """All shards of a world in one process (one device): runs each batch's
    phases and exchanges in lockstep. Used to check the sharded protocol
    against a single engine on one GPU; on a multi-GPU box each rank runs a
    ShardedEngine with a TorchComm instead."""

    def __init__(self, cfg, params, world: int, **kw):
        self.shards = [ShardedEngine(cfg, params, r, world, None, **kw) for r in range(world)]
        self.world = world

    def process_batch_arrays(self, src, dst, t, feat=None):
        import torch
        sends = [sh.stack_sends(src, dst) for sh in self.shards]
        for r, sh in enumerate(self.shards):
            sh.stack_recv([sends[q][r] for q in range(self.world)])
        parts = [sh.phase1(src, dst, t, feat) for sh in self.shards]
        gathered = (torch.cat([p[0] for p in parts], 0), torch.cat([p[1] for p in parts], 0))
        preds = [sh.phase2(gathered) for sh in self.shards]
        for p in preds[1:]:
            if not np.array_equal(p, preds[0]):
                raise RuntimeError("shards disagree on the batch scores")
        return preds[0]

    def layers(self):
        """(n, K, d) layer cache assembled from the owners."""
        return np.concatenate([sh.owned_layers()[2] for sh in self.shards], 0)

    def memory(self):
        return np.concatenate([sh.owned_memory()[2] for sh in self.shards], 0)
