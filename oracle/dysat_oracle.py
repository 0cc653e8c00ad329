"""ORACLE — test infrastructure, NOT product code.

Float64 numpy restatement of the DySAT streaming-inference model stated in
paper_2603_21090_b200/dysat.py (structural GAT over per-snapshot neighbour
lists, temporal self-attention over the last W snapshots). Only tests/ and
bench.py's CPU-baseline leg use it, as the checker / timed CPU baseline.

Parity unpinned: the reference ships no DySAT code (PAPER.md:1905-1912,
2266-2267 report results only), so nothing outside this repo pins this
restatement; it is written from the model definition, computed the slow,
obvious way (full recompute of every node from the raw edge history on
request), independently of the device path's incremental bookkeeping.
"""

from __future__ import annotations

import math

import numpy as np


def _elu(x):
    return np.where(x > 0, x, np.expm1(np.minimum(x, 0)))


class DySATOracle:
    def __init__(self, cfg, params):
        self.cfg, self.p = cfg, params
        self.P = np.asarray(params.x, np.float64) @ np.asarray(params.w_s, np.float64)
        self.edges: list = []        # (src, dst, t) in arrival order
        self.snapshot = 0
        self.t_now = -math.inf
        self.last_affected: set = set()
        self._z_hist: dict = {}      # snapshot j -> (n, d) structural outputs (final lists)
        self.emb = self._embeddings()

    # -- model --------------------------------------------------------------------
    def lists(self, k):
        """Per node: its L most recent entries of snapshot k, newest first."""
        L, n = self.cfg.fanout, self.cfg.n
        out = [[] for _ in range(n)]
        for s, d, t in reversed(self.edges):
            if math.floor(t / self.cfg.snapshot_len) != k:
                continue
            if len(out[s]) < L:
                out[s].append(d)
            if d != s and len(out[d]) < L:
                out[d].append(s)
        return out

    def structural(self, k):
        cfg, P = self.cfg, self.P
        H, dh = cfg.heads_s, cfg.d // cfg.heads_s
        a_s, a_n = np.asarray(self.p.a_self), np.asarray(self.p.a_nbr)
        Z = np.zeros((cfg.n, cfg.d))
        for v, lst in enumerate(self.lists(k)):
            us = [v] + lst
            for h in range(H):
                blk = slice(h * dh, (h + 1) * dh)
                e = np.array([a_s[h] @ P[v, blk] + a_n[h] @ P[u, blk] for u in us])
                e = np.where(e > 0, e, 0.2 * e)
                a = np.exp(e - e.max())
                a /= a.sum()
                Z[v, blk] = sum(a[i] * P[u, blk] for i, u in enumerate(us))
        return _elu(Z)

    def _embeddings(self):
        cfg, p = self.cfg, self.p
        k = self.snapshot
        j0 = max(0, k - cfg.window + 1)
        Y = []
        for j in range(j0, k + 1):
            z = self.structural(j) if j == k else self._z_hist[j]
            Y.append(z + np.asarray(p.pos)[j])
        Y = np.stack(Y, 1)                                   # (n, nw, d)
        q = Y[:, -1] @ p.w_q
        K = Y @ p.w_k
        V = Y @ p.w_v
        Ht, dt = cfg.heads_t, cfg.d // cfg.heads_t
        o = np.zeros((cfg.n, cfg.d))
        for g in range(Ht):
            blk = slice(g * dt, (g + 1) * dt)
            lg = np.einsum("nc,njc->nj", q[:, blk], K[:, :, blk]) / math.sqrt(dt)
            a = np.exp(lg - lg.max(1, keepdims=True))
            a /= a.sum(1, keepdims=True)
            o[:, blk] = np.einsum("nj,njc->nc", a, V[:, :, blk])
        return o @ p.w_o + Y[:, -1]

    def predict(self, u, v):
        d = self.cfg.d
        w = np.asarray(self.p.w_pred)
        x = w[:d] @ self.emb[u] + w[d:] @ self.emb[v] + self.p.b_pred
        return 1.0 / (1.0 + math.exp(-x))

    # -- stream ---------------------------------------------------------------------
    def process_batch(self, src, dst, t):
        """Predict each snapshot segment's edges from the current embeddings,
        then apply them (recomputing every node from scratch)."""
        out = []
        aff: set = set()
        i = 0
        B = len(src)
        while i < B:
            k = math.floor(t[i] / self.cfg.snapshot_len)
            while self.snapshot < k:  # roll: finalise the snapshot's structural rows
                self._z_hist[self.snapshot] = self.structural(self.snapshot)
                self.snapshot += 1
                self.emb = self._embeddings()
            j = i
            while j < B and math.floor(t[j] / self.cfg.snapshot_len) == k:
                j += 1
            out.extend(self.predict(int(src[q]), int(dst[q])) for q in range(i, j))
            self.edges.extend((int(src[q]), int(dst[q]), float(t[q])) for q in range(i, j))
            aff = {int(x) for x in src[i:j]} | {int(x) for x in dst[i:j]}
            self.emb = self._embeddings()
            i = j
        self.t_now = float(t[-1]) if B else self.t_now
        self.last_affected = aff
        return out
