"""ORACLE — test infrastructure, NOT product code.

CPU restatement (float64, numpy + numba) of the reference's exact-mode
incremental path, used only by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, always as the checker or
the timed CPU baseline and never as the thing measured or shipped.

What it restates (reference = /root/reference/pkg/src/streamtgn, "S/"):
  attention pipeline  S/kernels/pipeline_numba.py:15-111 (same per-scalar
                      accumulation order, so results are bitwise equal to
                      the reference's numba kernel)
  process_batch       S/engine.py:400-438 (exact mode)
    stage / freeze    S/engine_base.py:88-106, S/state.py:118-127
    grouping          S/engine.py:170-180
    affected set      S/engine.py:182-212
    neighbour cache   S/engine.py:216-243, S/graph_store.py:189-198
    run_pipeline      S/engine_base.py:139-189
    predict_link      S/kernels/reference.py:183-186
    commit + memory   S/engine_base.py:108-116, 193-247; S/engine.py:357-372
    drift / rebuild   S/drift.py:16-96, S/engine.py:385-396, 440-453
  full_reference      S/engine.py:374-381
  delta mode          S/engine.py:276-331 classification (embed_skip /
                      attn_hit / attn_miss, AttnState stamps from
                      _build_attn_state :247-274); a hit's delta_embed
                      update (:43-118) is evaluated as the same softmax
                      over the same frozen-payload key rows, so hits agree
                      with the reference to rounding, not bitwise;
                      the per-hit error-bound record DeltaEvent(bound =
                      |dN|/|N| * max_v * z_dev) of _apply_delta (:333-353)
                      and max_value_norm_seen (:255-261, :349) follow from
                      the log-partition (log Z) of each node's last state
                      build and the value-row norms of the recompute

Pinning: tests/test_golden_oracle.py checks this module against fixtures
written by the reference itself (tests/golden/make_golden.py) — bitwise
for integers and predictions/embeddings/memory, on every fixture.
"""

from __future__ import annotations

import math

import numpy as np

try:  # numba keeps the CPU baseline at the reference's own speed
    from numba import njit
except ImportError:  # pragma: no cover - the image ships numba
    def njit(*a, **k):
        def wrap(f):
            return f
        return wrap if not (a and callable(a[0])) else a[0]


# ---------------------------------------------------------------------------
# attention pipeline (flat layout of the reference operator)
# ---------------------------------------------------------------------------

@njit(cache=False)
def _proj_kv(payload, feat, phi, e, idx, l, h, wk, wv, kvec, values):
    d = payload.shape[2]
    d_e = feat.shape[1]
    d_t = phi.shape[1]
    d_k = wk.shape[3]
    for b in range(d_k):
        ak = 0.0
        av = 0.0
        for a in range(d):
            x = payload[idx, l, a]
            ak += x * wk[l, h, a, b]
            av += x * wv[l, h, a, b]
        for a in range(d_e):
            x = feat[idx, a]
            ak += x * wk[l, h, d + a, b]
            av += x * wv[l, h, d + a, b]
        for a in range(d_t):
            x = phi[e, a]
            ak += x * wk[l, h, d + d_e + a, b]
            av += x * wv[l, h, d + d_e + a, b]
        kvec[b] = ak
        values[idx, l, h, b] = av


@njit(cache=False)
def _attend_nodes(qbase, offsets, payload, feat, dt, omega, phi0, wq, wk, wv, wo,
                  out, scores, values, maxlog, zsum, qvecs, cap):
    n_nodes, d = qbase.shape
    K, H, q_in, d_k = wq.shape
    d_t = phi0.shape[0]
    half = omega.shape[0]
    scale = 1.0 / np.sqrt(d_k)
    amp = np.sqrt(1.0 / d_t)
    x = np.empty(q_in)
    q = np.empty(d_k)
    kvec = np.empty(d_k)
    phi = np.empty((cap, d_t))
    lg = np.empty(cap)
    cat = np.empty(H * d_k)
    for i in range(n_nodes):
        lo = offsets[i]
        E = offsets[i + 1] - lo
        for e in range(E):
            for f in range(half):
                ang = omega[f] * dt[lo + e]
                phi[e, 2 * f] = amp * np.cos(ang)
                phi[e, 2 * f + 1] = amp * np.sin(ang)
        for l in range(K):
            for j in range(d):
                x[j] = qbase[i, j] if l == 0 else out[i, l - 1, j]
            for j in range(d_t):
                x[d + j] = phi0[j]
            for c in range(H * d_k):
                cat[c] = 0.0
            for h in range(H):
                for b in range(d_k):
                    acc = 0.0
                    for a in range(q_in):
                        acc += x[a] * wq[l, h, a, b]
                    q[b] = acc
                    qvecs[i, l, h, b] = acc
                if E == 0:
                    continue
                top = -np.inf
                for e in range(E):
                    _proj_kv(payload, feat, phi, e, lo + e, l, h, wk, wv, kvec, values)
                    s = 0.0
                    for b in range(d_k):
                        s += q[b] * kvec[b]
                    s *= scale
                    lg[e] = s
                    if s > top:
                        top = s
                maxlog[i, l, h] = top
                z = 0.0
                for e in range(E):
                    w = np.exp(lg[e] - top)
                    scores[lo + e, l, h] = w
                    z += w
                zsum[i, l, h] = z
                for b in range(d_k):
                    acc = 0.0
                    for e in range(E):
                        acc += scores[lo + e, l, h] * values[lo + e, l, h, b]
                    cat[h * d_k + b] = acc / z
            for j in range(d):
                acc = 0.0
                for c in range(H * d_k):
                    acc += cat[c] * wo[l, c, j]
                out[i, l, j] = acc


def pipeline_many(qbase, offsets, payload, feat, dt, omega, phi0, wq, wk, wv, wo):
    """Operator contract of the reference's kernels.pipeline_many
    (S/kernels/__init__.py:42-44): returns (out, scores, values, maxlog,
    zsum, qvecs), scores in the max-scaled frame, empty rows -> 0 / -inf."""
    N, d = qbase.shape
    K, H, _, d_k = wq.shape
    E_tot = payload.shape[0]
    out = np.zeros((N, K, d))
    scores = np.zeros((E_tot, K, H))
    values = np.zeros((E_tot, K, H, d_k))
    maxlog = np.full((N, K, H), -np.inf)
    zsum = np.zeros((N, K, H))
    qvecs = np.zeros((N, K, H, d_k))
    if N:
        cap = max(1, int(np.max(np.diff(offsets))) if E_tot else 1)
        _attend_nodes(np.ascontiguousarray(qbase, dtype=np.float64),
                      np.ascontiguousarray(offsets, dtype=np.int64),
                      np.ascontiguousarray(payload, dtype=np.float64),
                      np.ascontiguousarray(feat, dtype=np.float64),
                      np.ascontiguousarray(dt, dtype=np.float64),
                      omega, phi0, wq, wk, wv, wo,
                      out, scores, values, maxlog, zsum, qvecs, cap)
    return out, scores, values, maxlog, zsum, qvecs


def time_encode(dt, omega):
    """phi(dt) = sqrt(1/d_t) * interleaved [cos w_f dt, sin w_f dt]
    (S/kernels/reference.py:21-29)."""
    d_t = 2 * omega.shape[0]
    out = np.empty(d_t)
    ang = omega * dt
    out[0::2] = np.cos(ang)
    out[1::2] = np.sin(ang)
    out *= np.sqrt(1.0 / d_t)
    return out


def _phi_matrix(dts, omega):
    d_t = 2 * omega.shape[0]
    ang = np.outer(dts, omega)
    out = np.empty((dts.shape[0], d_t))
    out[:, 0::2] = np.cos(ang)
    out[:, 1::2] = np.sin(ang)
    out *= np.sqrt(1.0 / d_t)
    return out


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def predict_link(hu, hv, p):
    return float(_sigmoid(p.w_pred @ np.concatenate([hu, hv]) + p.b_pred))


# ---------------------------------------------------------------------------
# the exact-mode engine
# ---------------------------------------------------------------------------

class _Lists:
    """Append-only per-node adjacency (store) — S/graph_store.py:102-198."""

    def __init__(self):
        self.per_node: dict[int, list[tuple[int, float, int]]] = {}

    def append(self, v, nbr, t, eid):
        self.per_node.setdefault(v, []).append((nbr, t, eid))

    def recent(self, v, limit):
        lst = self.per_node.get(v)
        if not lst:
            return []
        return lst[::-1][:limit]


class Oracle:
    """Float64 restatement of IncrementalEngine (exact mode) + rebuild.

    Neighbour entries are (nbr, t, eid) tuples, newest first.
    """

    def __init__(self, cfg, params):
        cfg.validate()
        if cfg.mode not in ("exact", "delta"):
            raise ValueError(f"unknown mode {cfg.mode}")
        self.delta = cfg.mode == "delta"
        self.attn: dict[int, tuple] = {}  # delta mode: node -> (mem_version, t_ref) of its AttnState
        self.logz: dict[int, np.ndarray] = {}  # delta mode: node -> log Z per head of that state
        self.max_value_norm_seen = 0.0
        self.delta_events: list[dict] = []
        self.cfg, self.p = cfg, params
        dm = params.dims
        self.K, self.d, self.L = dm.layers, dm.d, cfg.fanout
        cap = max(cfg.nodes, 16)
        self.mem = np.zeros((cap, dm.d_s))
        self.last = np.zeros(cap)
        self.version = np.zeros(cap, dtype=np.int64)
        self.h = np.zeros((cap, self.K, self.d))
        self.valid = np.zeros(cap, dtype=bool)
        self.valid_at = np.full(cap, -np.inf)
        self.n_mem = cfg.nodes
        self.store = _Lists()
        self.store_n = 0
        self.m = 0
        self.t_now = -np.inf
        self.feats = np.zeros((0, dm.d_e))
        self.stacks = np.zeros((0, 2, self.K, self.d))
        self.src_of = np.zeros(0, dtype=np.int64)
        self.cache: dict[int, list] = {}
        self._pending: dict = {}
        self.phi0 = time_encode(0.0, params.omega)
        self.batch_index = 0
        self.counters: dict[str, float] = {}
        self.totals: dict[str, float] = {}
        # drift scheduler state (S/drift.py:26-96)
        self.tau = 0
        self.acc: dict[int, float] = {}
        self.touched: dict[int, int] = {}
        self.cum: set[int] = set()
        self.last_direct: set[int] = set()
        self.last_all: set[int] = set()
        self.last_sizes: dict[int, int] = {}
        self.last_report = None
        self.last_pred_h: dict[int, np.ndarray] = {}

    # -- bookkeeping --------------------------------------------------------
    @property
    def node_count(self):
        return max(self.store_n, self.n_mem, self.cfg.nodes)

    def _grow(self, n):
        cap = self.mem.shape[0]
        if n > cap:
            new = max(n, 2 * cap, 16)
            def g(a, fill=0):
                out = np.full((new,) + a.shape[1:], fill, dtype=a.dtype)
                out[:cap] = a
                return out
            self.mem, self.last, self.version = g(self.mem), g(self.last), g(self.version)
            self.h, self.valid = g(self.h), g(self.valid)
            self.valid_at = g(self.valid_at, -np.inf)
        self.n_mem = max(self.n_mem, n)

    def _count(self, key, v=1):
        self.counters[key] = self.counters.get(key, 0) + v
        self.totals[key] = self.totals.get(key, 0) + v

    def _stack(self, v):
        st = np.zeros((self.K, self.d))
        st[0, :self.p.dims.d_s] = self.mem[v]
        for j in range(1, self.K):
            st[j] = self.h[v, j - 1]
        return st

    # -- pipeline over a node list (S/engine_base.py:139-189) ---------------
    def _pipeline(self, ids, lists, pending, count=True, full=False):
        p = self.p
        dm = p.dims
        N = len(ids)
        offs = np.zeros(N + 1, dtype=np.int64)
        offs[1:] = np.cumsum([len(x) for x in lists])
        E = int(offs[-1])
        qbase = np.zeros((N, self.d))
        if N:
            qbase[:, :dm.d_s] = self.mem[np.asarray(ids, dtype=np.int64)]
        payload = np.zeros((E, self.K, self.d))
        feat = np.zeros((E, dm.d_e))
        dt = np.empty(E)
        pos = 0
        for v, lst in zip(ids, lists):
            t_ref = lst[0][1] if lst else 0.0
            for (nbr, t, eid) in lst:
                dt[pos] = t_ref - t
                if eid < self.m:
                    side = 1 if self.src_of[eid] == v else 0
                    payload[pos] = self.stacks[eid, side]
                    feat[pos] = self.feats[eid]
                else:
                    s, d_, _, f, st_s, st_d = pending[eid]
                    payload[pos] = st_d if v == s else st_s
                    feat[pos] = f
                pos += 1
        if count:
            self._count("rows_gathered", N)
            per_node = dm.heads * dm.query_in * dm.d_k + dm.heads * dm.d_k * dm.d
            per_entry = dm.heads * (2 * dm.key_in * dm.d_k + 2 * dm.d_k)
            self._count("macs_attention", dm.layers * (N * per_node + E * per_entry))
        res = pipeline_many(qbase, offs, payload, feat, dt, p.omega, self.phi0,
                            p.w_q, p.w_k, p.w_v, p.w_o)
        return (res, offs) if full else res[0]

    def _state_stats(self, res, offs, i):
        """(log Z per head, max value-row norm) of row i of a layer-0 pipeline
        result: _log_z / _max_value_norm (S/engine.py:121-134) of the state
        _build_attn_state (:247-274) would build from it."""
        _, _, values, maxlog, zsum, _ = res
        lo, hi = int(offs[i]), int(offs[i + 1])
        H = zsum.shape[2]
        lz = np.array([np.log(zsum[i, 0, h]) + maxlog[i, 0, h] if zsum[i, 0, h] > 0 else -np.inf
                       for h in range(H)])
        mv = 0.0
        if hi > lo:
            mv = float(np.max(np.linalg.norm(values[lo:hi, 0], axis=-1)))
        return lz, mv

    def _recompute(self, ids, valid_at, count=True, keep_states=True, hits=None, sizes=None):
        lists = [self.cache.get(v) or [] for v in ids]
        track = self.delta and self.K == 1
        res, offs = self._pipeline(ids, lists, self._pending, count, full=True)
        out = res[0]
        for i, v in enumerate(ids):
            self.h[v] = out[i]
            self.valid[v] = True
            self.valid_at[v] = valid_at
            if track and (keep_states or hits):
                lz, mv = self._state_stats(res, offs, i)
                self.max_value_norm_seen = max(self.max_value_norm_seen, mv)
                if hits:  # _apply_delta: the bound record of this update
                    old = self.logz.get(v, np.full(len(lz), -np.inf))
                    z_dev = 0.0
                    for h in range(len(lz)):
                        if np.isfinite(lz[h]):
                            ratio = np.exp(old[h] - lz[h]) if np.isfinite(old[h]) else 0.0
                            z_dev = max(z_dev, abs(1.0 - ratio))
                    nv = max(len(lists[i]), 1)
                    self.delta_events.append(dict(
                        node=v, embedding=out[i, self.K - 1].copy(),
                        bound=(sizes[v] / nv) * mv * z_dev, dn=sizes[v], nv=nv, max_v=mv,
                        z_dev=z_dev))
                self.logz[v] = lz
        if keep_states:
            self._stamp(ids)
        return out

    def _stamp(self, ids):
        """Delta mode, single layer: the AttnState (mem_version, t_ref) that
        _build_attn_state (S/engine.py:247-274) leaves behind."""
        if self.delta and self.K == 1:
            for v in ids:
                lst = self.cache.get(v) or []
                self.attn[v] = (int(self.version[v]), lst[0][1] if lst else 0.0)

    def _delta_stage(self, ids, direct, sizes, t_batch, compute):
        """S/engine.py:276-319: skip / attn_hit / attn_miss per node of A."""
        K = self.K
        out = np.zeros((len(ids), K, self.d))
        hits, misses, pos = [], [], {}
        for i, v in enumerate(ids):
            pos[v] = i
            if v not in direct and sizes[v] == 0 and self.valid[v]:
                self._count("embed_skip")
                out[i] = self.h[v]
                continue
            lst = self.cache.get(v) or []
            t_ref = lst[0][1] if lst else 0.0
            if K == 1 and self.valid[v] and self.attn.get(v) == (int(self.version[v]), t_ref):
                hits.append(v)
                self._count("attn_hit")
            else:
                misses.append(v)
                self._count("attn_miss")
        if compute:
            for lst, cnt in ((misses, True), (hits, False)):
                if lst:
                    res = self._recompute(lst, t_batch, count=cnt, keep_states=cnt,
                                          hits=not cnt, sizes=sizes)
                    for j, v in enumerate(lst):
                        out[pos[v]] = res[j]
        else:
            self._stamp(misses)
        computed = set(hits) | set(misses)
        for v in ids:
            if v in direct:
                self._count("embed_predict")
            elif v in computed:
                self._count("embed_refresh")
        return out

    # -- the batch -----------------------------------------------------------
    def process_batch(self, src, dst, t, feat, compute=True):
        """Arrays in, list of prediction floats out (S/engine.py:400-438).

        compute=False is a fast-forward used only to position the CPU
        baseline deep in a stream: topology, caches, memory and drift are
        updated exactly, the attention recomputes are skipped (their cost
        depends on topology only, their values feed nothing but h)."""
        if self.delta and not compute:
            raise ValueError("compute=False fast-forward is exact-mode only")
        self._compute = compute
        self.counters = {}
        self.delta_events = []
        self.last_pred_h = {}
        src = np.asarray(src, dtype=np.int64)
        dst = np.asarray(dst, dtype=np.int64)
        t = np.asarray(t, dtype=np.float64)
        feat = np.asarray(feat, dtype=np.float64).reshape(len(src), self.p.dims.d_e)
        B = len(src)
        if B == 0:
            self.last_report = dict(index=self.batch_index, edges=0, t_batch=self.t_now,
                                    direct=0, affected=0, rebuild="none", rebuild_nodes=0)
            return []
        prev = self.t_now
        for x in t:
            if x < prev:
                raise ValueError(f"batch edge at t={x} precedes committed history t={prev}")
            prev = x
        self.batch_index += 1
        t_batch = float(t[-1])
        K, L = self.K, self.L
        self._grow(int(max(src.max(), dst.max())) + 1)
        # stage: edge ids + frozen pre-batch stacks
        m0 = self.m
        self._pending = {}
        for i in range(B):
            s, d_ = int(src[i]), int(dst[i])
            self._pending[m0 + i] = (s, d_, float(t[i]), feat[i], self._stack(s), self._stack(d_))
        # group: per endpoint, newest first; self-loop -> one entry
        new: dict[int, list] = {}
        for i in range(B - 1, -1, -1):
            s, d_, ti = int(src[i]), int(dst[i]), float(t[i])
            new.setdefault(s, []).append((d_, ti, m0 + i))
            if d_ != s:
                new.setdefault(d_, []).append((s, ti, m0 + i))
        direct = set(new)

        def base_of(w):
            b = self.cache.get(w)
            return self.store.recent(w, L) if b is None else b

        # affected set: K hops over distinct ids of the post-insertion top-L
        A = set(direct)
        frontier = sorted(direct)
        for _ in range(K):
            nxt = []
            for w in frontier:
                for (u, _, _) in (new.get(w, []) + base_of(w))[:L]:
                    if u not in A:
                        A.add(u)
                        nxt.append(u)
            frontier = nxt
        # stage 1: neighbour cache (+ change-record sizes)
        sizes = {}
        for v in sorted(A):
            nv = new.get(v, [])
            cached = self.cache.get(v)
            if cached is None:
                self._count("nbr_miss")
                merged = nv + self.store.recent(v, L)
                expired = 0
            else:
                self._count("nbr_hit")
                merged = nv + cached
                expired = max(0, len(merged) - L)
            kept = merged[:L]
            n_new = min(len(nv), len(kept))
            if math.isfinite(self.cfg.window):
                cut = t_batch - self.cfg.window
                keep2 = [x for x in kept if x[1] >= cut]
                expired += len(kept) - len(keep2)
                kept = keep2
                n_new = min(n_new, len(kept))
            upd = {x[0] for x in kept[n_new:] if x[0] in direct}
            sizes[v] = len(nv) + expired + len(upd)
            self.cache[v] = kept
        # stages 2-4: recompute sorted(A) with pre-batch memory
        ids = sorted(A)
        if self.delta:
            out = self._delta_stage(ids, direct, sizes, t_batch, compute)
        else:
            out = self._recompute(ids, t_batch) if compute else np.zeros((len(ids), K, self.d))
            for v in ids:
                self._count("embed_predict" if v in direct else "embed_refresh")
        hK = {v: out[i, K - 1] for i, v in enumerate(ids)}
        preds = [predict_link(hK[int(src[i])], hK[int(dst[i])], self.p) for i in range(B)]
        self.last_pred_h = {v: hK[v].copy() for v in direct}
        # stage 5: commit
        for i in range(B):
            s, d_, ti = int(src[i]), int(dst[i]), float(t[i])
            eid = self.m
            self.store.append(s, d_, ti, eid)
            if d_ != s:
                self.store.append(d_, s, ti, eid)
            _, _, _, f, st_s, st_d = self._pending[eid]
            if eid >= self.src_of.shape[0]:
                cap = max(16, 2 * self.src_of.shape[0])
                def g(a):
                    out = np.zeros((cap,) + a.shape[1:], dtype=a.dtype)
                    out[:eid] = a[:eid]
                    return out
                self.feats, self.stacks, self.src_of = g(self.feats), g(self.stacks), g(self.src_of)
            self.feats[eid] = f
            self.stacks[eid, 0], self.stacks[eid, 1] = st_s, st_d
            self.src_of[eid] = s
            self.m += 1
            self.t_now = ti
            self.store_n = max(self.store_n, s + 1, d_ + 1)
        self._pending = {}
        dlist = self._memory_step(src, dst, t, feat)
        if dlist:
            if compute:
                self._recompute(dlist, t_batch)
            else:
                self._stamp(dlist)
            self._count("embed_refresh", len(dlist))
        changes = {}
        for v in A:
            lst = self.cache.get(v)
            if sizes[v] > 0 and lst:
                changes[v] = (sizes[v], len(lst))
        self.tau += 1
        for v, (dn, nv) in changes.items():
            self.acc[v] = self._decayed(v) + dn / nv
            self.touched[v] = self.tau
        self.cum.update(A)
        kind, cnt = self._rebuild_policy()
        self._count("direct", len(direct))
        self._count("affected", len(A))
        self.last_direct, self.last_all, self.last_sizes = direct, A, sizes
        self.last_report = dict(index=self.batch_index, edges=B, t_batch=t_batch,
                                direct=len(direct), affected=len(A),
                                rebuild=kind, rebuild_nodes=cnt)
        return preds

    # S/engine_base.py:193-247 — same numpy ops so the bits match
    def _memory_step(self, src, dst, t, feat):
        p = self.p
        dm = p.dims
        B = len(src)
        M = 2 * B
        owners = np.empty(M, dtype=np.int64)
        owners[0::2], owners[1::2] = src, dst
        others = np.empty(M, dtype=np.int64)
        others[0::2], others[1::2] = dst, src
        times = np.repeat(t, 2)
        rows = np.empty((M, dm.msg_in))
        rows[:, :dm.d_s] = self.mem[owners]
        rows[:, dm.d_s:2 * dm.d_s] = self.mem[others]
        rows[:, 2 * dm.d_s:2 * dm.d_s + dm.d_e] = np.repeat(feat, 2, axis=0)
        rows[:, 2 * dm.d_s + dm.d_e:] = _phi_matrix(times - self.last[owners], p.omega)
        m_src = rows @ p.w_msg_src.T + p.b_msg_src
        m_dst = rows @ p.w_msg_dst.T + p.b_msg_dst
        side_src = np.zeros(M, dtype=bool)
        side_src[0::2] = True
        msgs = np.where(side_src[:, None], m_src, m_dst)
        self._count("messages", M)
        self._count("macs_gru", M * dm.d_m * dm.msg_in)
        groups: dict[int, list] = {}
        for r in range(M):
            groups.setdefault(int(owners[r]), []).append((msgs[r], float(times[r])))
        dlist = sorted(groups)
        agg = np.zeros((len(dlist), dm.d_m))
        mode = self.cfg.aggregator
        for j, v in enumerate(dlist):
            g = groups[v]
            if mode == "mean":
                agg[j] = sum(mm for mm, _ in g) / len(g)
            elif mode == "sum":
                tot = np.zeros_like(g[0][0])
                for mm, _ in g:
                    tot = tot + mm
                agg[j] = tot
            else:
                best = g[0]
                for c in g[1:]:
                    if c[1] >= best[1]:
                        best = c
                agg[j] = best[0]
        prev = self.mem[dlist]
        z = _sigmoid(agg @ p.w_z.T + prev @ p.u_z.T + p.b_z)
        r = _sigmoid(agg @ p.w_r.T + prev @ p.u_r.T + p.b_r)
        cand = np.tanh(agg @ p.w_h.T + (r * prev) @ p.u_h.T + p.b_h)
        self.mem[dlist] = (1.0 - z) * cand + z * prev
        self.version[dlist] = self.batch_index
        for v in dlist:
            self.last[v] = max(tt for _, tt in groups[v])
        self._count("gru_steps", len(dlist))
        self._count("macs_gru", len(dlist) * 3 * (dm.d_s * dm.d_m + dm.d_s * dm.d_s))
        return dlist

    # -- drift + rebuild (S/drift.py:16-96, S/engine.py:385-396, 440-453) ----
    def _decayed(self, v):
        a = self.acc.get(v, 0.0)
        if a == 0.0:
            return 0.0
        return a * self.cfg.gamma ** (self.tau - self.touched[v])

    def global_drift(self):
        if not self.cum:
            return 0.0
        return sum(self._decayed(v) for v in self.cum) / len(self.cum)

    def _rebuild_policy(self):
        cfg = self.cfg
        if cfg.rebuild == "never":
            return "none", 0
        if cfg.rebuild == "fixed":
            if cfg.rebuild_interval < 1 or self.batch_index % cfg.rebuild_interval:
                return "none", 0
            kind, nodes = "full", None
        else:
            if self.global_drift() <= cfg.delta_max:
                return "none", 0
            drifted = {v for v in self.cum if self._decayed(v) > cfg.delta_max}
            n = self.node_count
            kind, nodes = ("partial", drifted) if len(drifted) < cfg.alpha * n else ("full", None)
        cnt = self.rebuild_nodes(sorted(nodes) if kind == "partial" else None)
        self.tau = 0
        self.acc.clear()
        self.touched.clear()
        self.cum.clear()
        self._count("rebuilds")
        return kind, cnt

    def rebuild_nodes(self, nodes):
        ids = sorted(nodes) if nodes is not None else list(range(self.node_count))
        if not ids:
            return 0
        self._grow(max(ids) + 1)
        for v in ids:
            if self.cache.get(v) is None:
                self.cache[v] = self.store.recent(v, self.L)
        self._pending = {}
        if getattr(self, "_compute", True):
            self._recompute(ids, self.t_now if self.m else 0.0)
        else:
            self._stamp(ids)
        self._count("rebuild_pipelines", len(ids))
        return len(ids)

    def full_reference(self):
        ids = list(range(self.node_count))
        self._grow(len(ids))
        lists = [self.cache[v] if self.cache.get(v) is not None
                 else self.store.recent(v, self.L) for v in ids]
        self._pending = {}
        out = self._pipeline(ids, lists, {})
        return out[:, self.K - 1, :]

    def embeddings(self, n=None):
        n = self.node_count if n is None else n
        self._grow(n)
        return self.h[:n, self.K - 1, :]

    def neighbor_list(self, v):
        lst = self.cache.get(v)
        return None if lst is None else list(lst)


def brute_force_affected(oracle: Oracle, src, dst, fanout, layers):
    """Independent K-hop closure over the committed store (S/runner.py:33-54)."""
    direct = set(int(x) for x in src) | set(int(x) for x in dst)
    A = set(direct)
    frontier = sorted(direct)
    for _ in range(layers):
        nxt = []
        for w in frontier:
            for (u, _, _) in oracle.store.recent(w, fanout):
                if u not in A:
                    A.add(u)
                    nxt.append(u)
        frontier = nxt
    return A
