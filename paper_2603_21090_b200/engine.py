"""GPU-resident drop-in for the reference's IncrementalEngine (exact mode).

Mirrors /root/reference/pkg/src/streamtgn/engine.py:155-453 — same
constructor (RunConfig, ModelParameters), same `process_batch`,
`rebuild_nodes`, `full_reference` and the read-side surface the runner and
tests use (`memory`, `cache`, `nbr_cache`, `store`, `counters`,
`scheduler`, `last_report`, `last_affected`, `last_pred_embeddings`), plus the
stage-level entry points process_batch runs fused (`stage_batch`,
`detect_affected`, `update_neighbor_cache`, `commit_pending`, and the
scheduler's `record_batch_changes` / `note_affected` / `decide_rebuild` /
`execute_rebuild` / `reset`).
All state lives on the device in PyTorch-allocated tensors; each batch is
one call into the C ABI (include/stgn.h), which replays a captured CUDA
graph of the sm_100a kernels. There is no CPU fallback: without a GPU or
the built library the constructor raises.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .config import ConfigError, RunConfig
from .edges import (ChangeRecord, DriftContractError, FeatureDimError, InputError,
                    MonotonicityError, NeighborEntry, PendingEdge, edges_to_arrays)
from .params import ModelParameters


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2603_21090_b200 needs a CUDA GPU (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch


def _bf16_rne(x):
    """float64 -> bf16 bits (uint16), via float32, round to nearest even."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def _bf16_float(b):
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _rup(x, m):
    return (x + m - 1) // m * m


@dataclass
class BatchReport:
    """S/engine.py:32-40."""
    index: int
    edges: int
    t_batch: float
    direct: int
    affected: int
    rebuild: str = "none"
    rebuild_nodes: int = 0


@dataclass
class ChangeRecordSize:
    """Size of a node's change record (|added| + |expired| + |updated|)."""
    size: int

    @property
    def empty(self) -> bool:
        return self.size == 0


@dataclass
class AffectedSet:
    """S/state.py:147-151 (records carry sizes only)."""
    direct: set
    all: set
    records: dict = field(default_factory=dict)


class Counters:
    """S/state.py:209-227."""

    def __init__(self):
        self.totals: dict[str, float] = {}
        self.batch: dict[str, float] = {}

    def start_batch(self):
        self.batch = {}

    def add(self, key, amount=1):
        self.batch[key] = self.batch.get(key, 0) + amount
        self.totals[key] = self.totals.get(key, 0) + amount

    def get(self, key):
        return self.batch.get(key, 0)

    def total(self, key):
        return self.totals.get(key, 0)


_REBUILD_NAMES = {0: "none", 1: "partial", 2: "full"}


@dataclass
class DeltaEvent:
    """One delta-mode embedding update, kept for bound verification (S/engine.py:20-29)."""

    node: int
    embedding: np.ndarray
    bound: float
    dn: int
    nv: int
    max_v: float
    z_dev: float


class _Tables:
    """PyTorch-allocated device tables bound into the C engine. Node tables,
    edge tables, the gamma^k table and the scratch grow independently."""

    NODE_I32 = ("ring_cnt", "ring_head", "ring_ccnt", "nodecnt", "nodeadj", "nodefill",
                "nodeoff", "cum_list", "amark", "dmark", "cum_mark", "cum_pos")
    EDGE = ("e_src", "e_dst", "e_t", "e_feat", "e_prev")

    def __init__(self, eng, cap_nodes, cap_edges, gpow_len):
        self.eng = eng
        torch = eng._torch
        self.ctl = torch.zeros(_rup(C.sizeof(_lib.Ctl), 8) // 8, dtype=torch.int64,
                               device=eng.device)
        self.cap_nodes = self.cap_edges = 0
        self._alloc_nodes(cap_nodes)
        self._alloc_edges(cap_edges)
        self._alloc_gpow(gpow_len)
        self.new_scratch()

    def _z(self, *shape, dt=None, fill=0):
        torch = self.eng._torch
        t = torch.empty(*shape, dtype=dt or torch.float32, device=self.eng.device)
        return t.fill_(fill)

    def _alloc_nodes(self, N):
        torch, g = self.eng._torch, self.eng
        old = {k: getattr(self, k) for k in self._node_names()} if self.cap_nodes else {}
        n0 = self.cap_nodes
        z = self._z
        self.mem = z(N, g.ld_s)
        self.last = z(N, dt=torch.float64)
        self.version = z(N, dt=torch.int64)
        self.h = z(N, g.K, g.ld_d)
        self.valid = z(N, dt=torch.uint8)
        self.valid_at = z(N, dt=torch.float64, fill=-math.inf)
        for name in self.NODE_I32:
            setattr(self, name, z(N, dt=torch.int32))
        self.ring_ccnt.fill_(-1)
        self.ring_nbr = z(N, g.L, dt=torch.int32)
        self.ring_eid = z(N, g.L, dt=torch.int64)
        self.ring_t = z(N, g.L, dt=torch.float64)
        # frozen payload rows: every node, or only the shard's (bound with a base offset)
        NP = N if g.shard is None else g.shard[1] - g.shard[0]
        self.ring_pay = z(NP, g.K, g.L, g.ld_d)
        self.ring_feat = z(NP, g.L, g.ld_e)
        self.ring_tb = z(NP, g.L, g.ld_t)
        self.drift_acc = z(N, dt=torch.float64)
        self.drift_touched = z(N, dt=torch.int64)
        self.attn_ver = z(N, dt=torch.int64, fill=-1)
        self.attn_tref = z(N, dt=torch.float64)
        # delta mode, K = 1: log Z per head of each node's attention state, and the
        # per-batch bound-record buffers (stgn.h stgn_state; csrc/delta.cuh)
        self.attn_logz = z(N, 4, dt=torch.float64, fill=-math.inf)
        ne = N if g.K == 1 else 1
        self.ev_cap = ne if g.K == 1 else 0
        for name in ("ev_node", "ev_dpos", "ev_dn", "ev_nv"):
            setattr(self, name, z(ne, dt=torch.int32))
        for name in ("ev_bound", "ev_maxv", "ev_zdev"):
            setattr(self, name, z(ne, dt=torch.float64))
        self.adj_head = z(N, dt=torch.int64, fill=-1)
        self.adj_deg = z(N, dt=torch.int64)
        for k, t in old.items():
            if g.shard is not None and k in ("ring_pay", "ring_feat", "ring_tb"):
                getattr(self, k).copy_(t)
                continue
            getattr(self, k)[:n0].copy_(t[:n0])
        self.cap_nodes = N

    def _node_names(self):
        return ("mem", "last", "version", "h", "valid", "valid_at", *self.NODE_I32, "ring_nbr",
                "ring_eid", "ring_t", "ring_pay", "ring_feat", "ring_tb", "drift_acc", "drift_touched", "attn_ver", "attn_tref",
                "attn_logz", "adj_head", "adj_deg")

    def _alloc_edges(self, E):
        torch, g = self.eng._torch, self.eng
        names = self.EDGE + (("e_pay",) if g.edge_payloads else ())
        old = {k: getattr(self, k) for k in names} if self.cap_edges else {}
        e0 = self.cap_edges
        z = self._z
        self.e_src = z(E, dt=torch.int32)
        self.e_dst = z(E, dt=torch.int32)
        self.e_t = z(E, dt=torch.float64)
        self.e_feat = z(E, g.ld_e)
        self.e_prev = z(2 * E, dt=torch.int64, fill=-1)
        # payload log (stgn.h e_pay): every store entry's frozen stack, for snapshots
        self.e_pay = z(2 * E, g.K, g.ld_d) if g.edge_payloads else None
        for k, t in old.items():
            lim = 2 * e0 if k in ("e_prev", "e_pay") else e0
            getattr(self, k)[:lim].copy_(t[:lim])
        self.cap_edges = E

    def _alloc_gpow(self, G):
        torch, g = self.eng._torch, self.eng
        self.gpow = torch.tensor([g.cfg.gamma ** k for k in range(G)], dtype=torch.float64,
                                 device=g.device)

    def new_scratch(self):
        eng = self.eng
        sb = eng._L.stgn_scratch_bytes(C.byref(eng._dims), C.byref(eng._cfgs), self.cap_nodes)
        if sb < 0:
            raise ConfigError("invalid dims/config for the CUDA engine")
        self.scratch = self._z(int(sb), dt=eng._torch.uint8)

    def grow(self, nodes=0, edges=0, gpow=0, scratch=False):
        """Grow what is too small (doubling); returns True if anything moved."""
        moved = False
        if nodes > self.cap_nodes:
            self._alloc_nodes(max(nodes, 2 * self.cap_nodes))
            moved = scratch = True
        if edges > self.cap_edges:
            self._alloc_edges(max(edges, 2 * self.cap_edges))
            moved = True
        if gpow > self.gpow.numel():
            self._alloc_gpow(max(gpow, 2 * self.gpow.numel()))
            moved = True
        if scratch:
            self.new_scratch()
            moved = True
        return moved

    def struct(self) -> _lib.State:
        s = _lib.State()
        s.cap_nodes, s.cap_edges, s.gpow_len = self.cap_nodes, self.cap_edges, self.gpow.numel()
        for name in _lib.STATE_PTRS + _lib.DELTA_PTRS:
            setattr(s, name, getattr(self, name).data_ptr())
        if self.eng.shard is not None:  # payload rows of nodes lo..hi-1 only: base offset
            lo = self.eng.shard[0]
            for name in ("ring_pay", "ring_feat", "ring_tb"):
                t = getattr(self, name)
                row = t[0].numel() * t.element_size()
                setattr(s, name, t.data_ptr() - lo * row)
        s.ev_cap = self.ev_cap
        s.e_pay = self.e_pay.data_ptr() if self.e_pay is not None else None
        return s


class _MemoryView:
    """Read view of NodeMemoryTable (S/state.py:23-48)."""

    def __init__(self, eng):
        self._e = eng

    @property
    def states(self):
        e = self._e
        return e._tab.mem[:e._cap_view(), :e.dims.d_s].double().cpu().numpy()

    @property
    def last_interaction(self):
        e = self._e
        return e._tab.last[:e._cap_view()].cpu().numpy()

    @property
    def version(self):
        e = self._e
        return e._tab.version[:e._cap_view()].cpu().numpy()

    @property
    def n(self):
        return self._e._n_mem


class _CacheView:
    """Read view of LayerCache (S/state.py:91-127)."""

    def __init__(self, eng):
        self._e = eng

    @property
    def h(self):
        e = self._e
        return e._tab.h[:e._cap_view(), :, :e.dims.d].double().cpu().numpy()

    @property
    def valid(self):
        return self._e._tab.valid[:self._e._cap_view()].bool().cpu().numpy()

    @property
    def valid_at(self):
        return self._e._tab.valid_at[:self._e._cap_view()].cpu().numpy()

    def embeddings(self, n: int) -> np.ndarray:
        e = self._e
        e._ensure_nodes(n)
        return e._tab.h[:n, e.K - 1, :e.dims.d].double().cpu().numpy()


class _NeighborCacheView:
    """Read view of NeighborCache (S/state.py:154-171): the ring prefix."""

    def __init__(self, eng):
        self._e = eng

    def _list(self, v, length):
        e = self._e
        head = int(e._tab.ring_head[v])
        slots = [(head + j) % e.L for j in range(length)]
        nbr = e._tab.ring_nbr[v].cpu().numpy()
        ts = e._tab.ring_t[v].cpu().numpy()
        eid = e._tab.ring_eid[v].cpu().numpy()
        return [NeighborEntry(int(nbr[s]), float(ts[s]), int(eid[s])) for s in slots]

    def get(self, v):
        e = self._e
        if v < 0 or v >= e._tab.cap_nodes:
            return None
        cc = int(e._tab.ring_ccnt[v])
        if cc < 0:
            return None
        return self._list(v, cc)

    def __contains__(self, v):
        return self.get(v) is not None


class _StoreView:
    """Read view of TemporalAdjacencyList (S/graph_store.py:102-198)."""

    def __init__(self, eng):
        self._e = eng

    @property
    def m(self):
        return self._e._m

    @property
    def n(self):
        return self._e._store_n

    @property
    def t_now(self):
        return self._e._t_now

    @property
    def d_e(self):
        return self._e.dims.d_e

    def degree(self, v):
        e = self._e
        if v >= e._tab.cap_nodes:
            return 0
        return int(e._tab.adj_deg[v])

    def _walk(self, v):
        """Newest-first (nbr, t, eid) along the device chain."""
        e = self._e
        if v >= e._tab.cap_nodes:
            return
        ent = int(e._tab.adj_head[v])
        src = e._tab.e_src
        dst = e._tab.e_dst
        while ent >= 0:
            eid, side = ent >> 1, ent & 1
            s, d = int(src[eid]), int(dst[eid])
            yield (d if side == 0 else s), float(e._tab.e_t[eid]), eid
            ent = int(e._tab.e_prev[ent])

    def recent_upto(self, v, limit):
        out = []
        if limit <= 0:
            return out
        for nbr, t, eid in self._walk(v):
            out.append(NeighborEntry(nbr, t, eid))
            if len(out) == limit:
                break
        return out

    def get_temporal_neighbors(self, v, t_start, t_end):
        if t_start > t_end:
            raise ValueError("t_start must be <= t_end")
        out = []
        for nbr, t, eid in self._walk(v):
            if t > t_end:
                continue
            if t < t_start:
                break
            out.append(NeighborEntry(nbr, t, eid))
        return out

    def edge_feature(self, eid):
        e = self._e
        if eid >= e._m:
            raise IndexError(f"edge id {eid} out of range")
        return e._tab.e_feat[eid, :e.dims.d_e].double().cpu().numpy()

    def feature_table(self):
        e = self._e
        return e._tab.e_feat[:e._m, :e.dims.d_e].double().cpu().numpy()


class _SchedulerView:
    """Read view of DriftScheduler (S/drift.py:26-96)."""

    def __init__(self, eng):
        self._e = eng

    def _ctl(self):
        raw = self._e._tab.ctl.cpu().numpy().tobytes()
        return _lib.Ctl.from_buffer_copy(raw[:C.sizeof(_lib.Ctl)])

    @property
    def tau(self):
        return int(self._ctl().tau)

    @property
    def gamma(self):
        return self._e.cfg.gamma

    def estimator(self, v):
        e = self._e
        ctl = self._ctl()
        if v >= e._tab.cap_nodes or int(e._tab.cum_mark[v]) != int(ctl.cum_gen) + 1:
            return 0.0
        pos = int(e._tab.cum_pos[v])
        acc = float(e._tab.drift_acc[pos])
        if acc == 0.0:
            return 0.0
        return acc * e.cfg.gamma ** (int(ctl.tau) - int(e._tab.drift_touched[pos]))

    def _decayed_all(self):
        """Decayed estimators of the cumulative set, by position (device)."""
        e, ctl = self._e, self._ctl()
        n, tau = int(ctl.cum_count), int(ctl.tau)
        torch = e._torch
        acc = e._tab.drift_acc[:n]
        age = tau - e._tab.drift_touched[:n]
        if tau < e._tab.gpow.numel():  # the gamma^k table the batch kernels use
            dec = e._tab.gpow[age.clamp(0, e._tab.gpow.numel() - 1)]
        else:
            dec = torch.pow(torch.tensor(e.cfg.gamma, dtype=torch.float64, device=e.device),
                            age.to(torch.float64))
        return torch.where(acc != 0.0, acc * dec, torch.zeros_like(acc))

    def global_drift(self):
        n = int(self._ctl().cum_count)
        if n == 0:
            return 0.0
        # one reduction on the device (S/drift.py:62-70)
        return float(self._decayed_all().sum().item()) / n

    @property
    def delta_max(self):
        return self._e.cfg.delta_max

    @property
    def alpha(self):
        return self._e.cfg.alpha

    def note_affected(self, nodes) -> None:
        """S/drift.py:59-60: nodes join the cumulative affected set."""
        e = self._e
        torch, tab = e._torch, e._tab
        ids = sorted({int(v) for v in nodes})
        if not ids:
            return
        e._grow(need_nodes=ids[-1] + 1)
        tab = e._tab
        ctl = self._ctl()
        gen = int(ctl.cum_gen) + 1
        idx = torch.tensor(ids, dtype=torch.int64, device=e.device)
        new = idx[tab.cum_mark[idx] != gen]
        k, n0 = int(new.numel()), int(ctl.cum_count)
        if k == 0:
            return
        pos = torch.arange(n0, n0 + k, dtype=torch.int64, device=e.device)
        tab.cum_mark[new] = gen
        tab.cum_list[pos] = new.to(torch.int32)
        tab.cum_pos[new] = pos.to(torch.int32)
        tab.drift_acc[pos] = 0.0
        tab.drift_touched[pos] = 0
        tab.ctl[1] = n0 + k

    def record_batch_changes(self, changes: dict) -> None:
        """S/drift.py:51-57: tau advances; each v's estimator becomes
        gamma^elapsed * acc + |dN_v| / |N_v|. Estimators live at the node's
        position in the cumulative set (csrc/batch.cuh k_drift_record), so a
        recorded node also joins that set (the engine always notes the nodes it
        records, S/engine.py:371-372)."""
        e = self._e
        tab = e._tab
        tau = int(self._ctl().tau) + 1
        tab.ctl[0] = tau
        items = []
        for v, (dn, nv) in changes.items():
            if nv <= 0:
                raise DriftContractError(f"node {v}: |N_v| must be positive")
            items.append((int(v), dn, nv))
        if not items:
            return
        self.note_affected([v for v, _, _ in items])
        tab = e._tab
        torch = e._torch
        idx = torch.tensor([v for v, _, _ in items], dtype=torch.int64, device=e.device)
        pos = tab.cum_pos[idx].to(torch.int64)
        acc = tab.drift_acc[pos].tolist()
        tch = tab.drift_touched[pos].tolist()
        g = e.cfg.gamma
        new = [(a * g ** (tau - t) if a != 0.0 else 0.0) + dn / nv
               for a, t, (_, dn, nv) in zip(acc, tch, items)]
        tab.drift_acc[pos] = torch.tensor(new, dtype=torch.float64, device=e.device)
        tab.drift_touched[pos] = tau

    def decide_rebuild(self, n: int):
        """S/drift.py:72-78: None, ("partial", drifted nodes) or ("full", None)."""
        if self.global_drift() <= self.delta_max:
            return None
        e = self._e
        n_c = int(self._ctl().cum_count)
        dec = self._decayed_all()
        drifted = set(e._tab.cum_list[:n_c][dec > self.delta_max].tolist())
        if len(drifted) < self.alpha * n:
            return ("partial", drifted)
        return ("full", None)

    def execute_rebuild(self, decision, engine) -> int:
        """S/drift.py:80-90: run the rebuild on the engine, then reset."""
        if decision is None:
            raise DriftContractError("execute_rebuild needs a non-None decision")
        kind, nodes = decision
        count = engine.rebuild_nodes(sorted(nodes) if kind == "partial" else None)
        self.reset()
        return count

    def reset(self) -> None:
        """S/drift.py:92-96 (as k_drift_reset_fin: forgetting the set clears
        every estimator)."""
        ctl = self._e._tab.ctl
        ctl[0] = 0
        ctl[1] = 0
        ctl[2] += 1  # cum_gen (low word)


class IncrementalEngine:
    """B200 exact-mode engine; see the module docstring.

    recompute: "affected" recomputes every node of A (the reference's
    literal exact mode, default); "direct" recomputes V_direct only, which is
    value-identical when the window is infinite (keys/values come from
    payloads frozen at insertion, so A minus V_direct has unchanged inputs).

    cfg.mode == "delta" selects the reference's delta mode (S/engine.py:276-331):
    affected nodes outside V_direct with an empty change record keep their
    cached row (embed_skip); the others are classified attn_hit / attn_miss
    exactly as the reference does and recomputed on the device (a hit's
    delta_embed update is the same softmax over the same frozen-payload key
    rows, so the recompute returns the delta result up to rounding). For
    K = 1 the per-update error-bound records (delta_events, S/engine.py:333-353)
    and max_value_norm_seen are computed on the device (csrc/delta.cuh).
    """

    def __init__(self, cfg: RunConfig, params: ModelParameters, *, recompute: str = "affected",
                 max_batch: int | None = None, device: int | None = None,
                 tensor_cores: bool | str = True, edge_payloads: bool = False,
                 shard: tuple | None = None):
        cfg.validate()
        self.edge_payloads = bool(edge_payloads)  # keep every entry's payload (snapshots)
        # node-id range [lo, hi) whose payload rows this engine keeps and recomputes
        # (shard.py); None = every node
        self.shard = None
        if shard is not None:
            lo, hi = int(shard[0]), int(shard[1])
            if cfg.nodes <= 0 or not 0 <= lo < hi <= cfg.nodes:
                raise ConfigError("shard=(lo, hi) needs 0 <= lo < hi <= cfg.nodes")
            if edge_payloads:
                raise ConfigError("the payload log is single-engine only")
            self.shard = (lo, hi)
        if cfg.mode == "delta":
            if recompute not in ("affected", "delta"):
                raise ConfigError("delta mode recomputes by its own classification")
            recompute = "delta"
        elif recompute == "delta":
            raise ConfigError('recompute="delta" needs cfg.mode == "delta"')
        if recompute not in _lib.SCOPE:
            raise ConfigError(f"recompute must be one of {tuple(_lib.SCOPE)}")
        self._torch = _torch()
        torch = self._torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.cfg = cfg
        self.params = params
        self.dims = dm = params.dims
        if dm != cfg.dims:
            raise ConfigError("params.dims must equal cfg.dims")
        self.K, self.L = dm.layers, cfg.fanout
        self.ld_s, self.ld_d = _rup(dm.d_s, 4), _rup(dm.d, 4)
        self.ld_e = _rup(max(dm.d_e, 1), 4)
        self.ld_t = _rup(dm.d_t, 4)
        self.recompute = recompute
        # tcgen05 GEMMs where the TMEM plan fits: True = bf16x3 128-row kernel (H = 2,
        # k_in <= 224), else split-TF32; "tf32" = split-TF32 only; False = FFMA
        if tensor_cores not in (True, False, "tf32"):
            raise ConfigError("tensor_cores must be True, False or 'tf32'")
        self.tensor_cores = tensor_cores
        self._L = _lib.lib()
        self._dims = _lib.dims_struct(dm)
        self._max_batch = max(int(max_batch or cfg.batch_size), 1)
        self._handle = None
        self._make_handle()
        self._upload_weights()
        cap_nodes = max(cfg.nodes, 16)
        self._tab = _Tables(self, cap_nodes, max(1024, 4 * self._max_batch), 4096)
        self._bind()
        # host mirrors of the store / scheduler scalars
        self._m = 0
        self._t_now = -math.inf
        self._store_n = 0
        self._n_mem = cfg.nodes
        self.batch_index = 0
        self.counters = Counters()
        self.last_report: BatchReport | None = None
        self._last_nD = 0
        self._last_nA = 0
        self._affected_cache = None
        self._pred_cache = None
        self.memory = _MemoryView(self)
        self.cache = _CacheView(self)
        self.nbr_cache = _NeighborCacheView(self)
        self.store = _StoreView(self)
        self.scheduler = _SchedulerView(self)
        self._rep = _lib.Report()
        self._ev_batch = -1     # batch whose bound records self._events holds
        self._events: list = []
        self._preds = np.zeros(self._max_batch, dtype=np.float64)
        self._pending: dict = {}       # staged edges by id (stage_batch .. commit_pending)
        self._stage_put: set = set()   # nodes whose lists update_neighbor_cache moved
        self._stage_stamp = 0x80000000  # node marks of detect_affected (batches use < 2^31)

    # -- plumbing -------------------------------------------------------------
    def _stream(self):
        return C.c_void_p(self._torch.cuda.current_stream(self.device).cuda_stream)

    def _make_handle(self):
        cfg = self.cfg
        self._cfgs = _lib.Config(cfg.fanout, _lib.AGG[cfg.aggregator], _lib.REBUILD[cfg.rebuild],
                                 int(cfg.rebuild_interval), cfg.gamma, cfg.delta_max, cfg.alpha,
                                 cfg.window, _lib.SCOPE[self.recompute], self._max_batch)
        h = C.c_void_p()
        with self._torch.cuda.device(self.device):
            _lib.check(self._L.stgn_engine_create(C.byref(self._dims), C.byref(self._cfgs),
                                                  C.byref(h)), "engine_create")
        if self._handle is not None:
            self._L.stgn_engine_destroy(self._handle)
        self._handle = h
        if getattr(self, "_state_only", False):
            self._L.stgn_engine_set_skip_recompute(h, 1)
        if self.shard is not None:
            _lib.check(self._L.stgn_engine_set_ownership(self._handle, *self.shard), "ownership")

    def _upload_weights(self):
        torch = self._torch
        p, dm = self.params, self.dims
        K, H, d_k = dm.layers, dm.heads, dm.d_k
        def f32(a):  # last dim padded to a multiple of 4 (zero-filled); see stgn.h
            a = np.asarray(a, dtype=np.float64)
            pad = _rup(a.shape[-1], 4) - a.shape[-1]
            if pad:
                a = np.concatenate([a, np.zeros(a.shape[:-1] + (pad,))], axis=-1)
            return torch.tensor(np.ascontiguousarray(a, dtype=np.float32), device=self.device)

        def f64(a):
            return torch.tensor(np.ascontiguousarray(a, dtype=np.float64), device=self.device)

        def catcols(mats):  # [rows][n * ld(cols)]: each block padded to a multiple of 4
            blocks = []
            for m in mats:
                pad = _rup(m.shape[1], 4) - m.shape[1]
                blocks.append(np.concatenate([m, np.zeros((m.shape[0], pad))], axis=1))
            return torch.tensor(np.ascontiguousarray(np.concatenate(blocks, axis=1),
                                                     dtype=np.float32), device=self.device)

        ang = p.omega * 0.0
        phi0 = np.empty(dm.d_t)
        phi0[0::2], phi0[1::2] = np.cos(ang), np.sin(ang)
        phi0 *= np.sqrt(1.0 / dm.d_t)
        wq_full = np.transpose(p.w_q, (0, 2, 1, 3)).reshape(K, dm.query_in, H * d_k)
        W = {
            "wq": f32(wq_full[:, :dm.d, :]),
            "bq": torch.tensor(np.einsum("t,ltc->lc", phi0, wq_full[:, dm.d:, :]),
                               dtype=torch.float32, device=self.device),
            "wkt": f32(np.transpose(p.w_k, (0, 1, 3, 2))),
            "wv": f32(p.w_v),
            "wo": f32(p.w_o),
            "wmsg": f32(np.concatenate([p.w_msg_src.T, p.w_msg_dst.T], axis=0)),
            "bmsg": torch.tensor(np.stack([p.b_msg_src, p.b_msg_dst]), dtype=torch.float32,
                                 device=self.device),
            "wgru": catcols([p.w_z.T, p.w_r.T, p.w_h.T]),
            "ugru": catcols([p.u_z.T, p.u_r.T, p.u_h.T]),
            "bgru": torch.tensor(np.stack([p.b_z, p.b_r, p.b_h]), dtype=torch.float32,
                                 device=self.device),
            "wpred": f64(p.w_pred),
            "omega": f64(p.omega),
            "phi0": torch.tensor(phi0, dtype=torch.float32, device=self.device),
        }
        if self.tensor_cores:
            wqx = wq_full[:, :dm.d, :].transpose(0, 2, 1)            # (K, HD, d)   [n][k]
            W["tcq"] = self._pack_kmajor(wqx)
            W["tck"] = self._pack_kmajor(p.w_k)                         # (K, H, k_in, d_k)
            W["tcv"] = self._pack_kmajor(np.transpose(p.w_v, (0, 1, 3, 2)))  # (K, H, d_k, k_in)
            W["tco"] = self._pack_kmajor(np.transpose(p.w_o, (0, 2, 1)))     # (K, d, HD)
        if self.tensor_cores is True and H == 2:
            W.update(self._pack_bf16x3())
        if self.tensor_cores is True:
            W["t4mem"] = self._pack_memory_bf16x3()
        self._w = W
        ws = _lib.Weights(**{k: v.data_ptr() for k, v in W.items()}, bpred=float(p.b_pred))
        _lib.check(self._L.stgn_engine_set_weights(self._handle, C.byref(ws)), "set_weights")

    def _pack_bf16x3(self):
        """Operands of the bf16x3 recompute kernel (stgn.h t4*): the folded
        per-head weights with log2(e)/sqrt(d_k) in W_K (the kernel's softmax
        is base 2) and the time-encoding amplitude sqrt(1/d_t) in the time rows
        of W_K and W_V."""
        p, dm = self.params, self.dims
        K, H, d_k, d = dm.layers, dm.heads, dm.d_k, dm.d
        Kq = _rup(d_k, 16)
        amp = np.sqrt(1.0 / dm.d_t)
        t0 = d + dm.d_e                       # first time-encoding row of k_in
        ang = p.omega * 0.0
        phi0 = np.empty(dm.d_t)
        phi0[0::2], phi0[1::2] = np.cos(ang), np.sin(ang)
        phi0 *= amp
        wq = np.zeros((K, H * Kq, d))         # [n = h*Kq + j][k]
        bq = np.zeros((K, H, Kq))
        wo = np.zeros((K, d, H * Kq))         # [m][h*Kq + j]
        for h in range(H):
            wq[:, h * Kq:h * Kq + d_k, :] = np.transpose(p.w_q[:, h, :d, :], (0, 2, 1))
            bq[:, h, :d_k] = np.einsum("t,ltc->lc", phi0, p.w_q[:, h, d:, :])
            wo[:, :, h * Kq:h * Kq + d_k] = np.transpose(p.w_o[:, h * d_k:(h + 1) * d_k, :], (0, 2, 1))
        # key rows in the kernel's 4-padded layout [payload | features | time]
        r4 = lambda x: _rup(x, 4)  # noqa: E731
        kmap = np.concatenate([np.arange(d), r4(d) + np.arange(dm.d_e),
                               r4(d) + r4(dm.d_e) + np.arange(dm.d_t)])
        kpad = r4(d) + r4(dm.d_e) + r4(dm.d_t)
        wk = np.zeros((K, H, kpad, d_k))      # [n][k]
        # log2(e) folded in: the kernel's softmax runs on exp2 (one MUFU.EX2 per weight)
        wk[:, :, kmap, :] = p.w_k * (np.log2(np.e) / np.sqrt(d_k))
        wk[:, :, kmap[t0:], :] *= amp
        wv = np.zeros((K, H, d_k, kpad))      # [n][k]
        wv[:, :, :, kmap] = np.transpose(p.w_v, (0, 1, 3, 2))
        wv[:, :, :, kmap[t0:]] *= amp
        # folded output operands: P_h = wv_h^T (kpad x d_k) @ w_o[l, h] (d_k x d), as B
        # operands [n = output column][k = key feature], split at column Na (stgn.h t4p)
        No = _rup(d, 16)
        Na = min(No, 64)
        pk = []
        for l in range(K):
            P = [np.zeros((No, kpad)) for _ in range(H)]
            for h in range(H):
                P[h][:d, :] = (wv[l, h].T @ p.w_o[l, h * d_k:(h + 1) * d_k, :]).T
            blocks = [P[h][:Na] for h in range(H)] + ([P[h][Na:] for h in range(H)] if No > Na else [])
            pk += [self._pack_kmajor_bf16(b).reshape(-1) for b in blocks]
        t4p = self._torch.cat(pk)
        return {"t4q": self._pack_kmajor_bf16(wq), "t4k": self._pack_kmajor_bf16(wk),
                "t4v": self._pack_kmajor_bf16(wv), "t4o": self._pack_kmajor_bf16(wo), "t4p": t4p,
                "t4bq": self._torch.tensor(bq.astype(np.float32), device=self.device)}

    def _pack_memory_bf16x3(self):
        """Operands of the bf16x3 memory-update kernel (stgn.h t4mem, csrc/mem4.cuh):
        message weights in K-chunks of 128 columns of x (w_msg_src chunk j, then
        w_msg_dst chunk j), then [w_z; w_r], [u_z; u_r], w_h, u_h, each a K-major
        bf16 hi/lo block."""
        p, dm = self.params, self.dims
        Nm, Ns = _rup(dm.d_m, 16), _rup(dm.d_s, 16)
        nmsg = -(-dm.msg_in // 128)
        wm = np.zeros((nmsg, 2, Nm, 128))                   # chunk j: [W_src cols, W_dst cols]
        for side, wsd in enumerate((p.w_msg_src, p.w_msg_dst)):   # (d_m, msg_in)
            full = np.zeros((Nm, nmsg * 128))
            full[:dm.d_m, :dm.msg_in] = wsd
            wm[:, side] = full.reshape(Nm, nmsg, 128).transpose(1, 0, 2)
        wm = wm.reshape(2 * nmsg, Nm, 128)
        zr0 = np.zeros((2 * Ns, Nm))
        zr0[:dm.d_s, :dm.d_m], zr0[Ns:Ns + dm.d_s, :dm.d_m] = p.w_z, p.w_r
        zr1 = np.zeros((2 * Ns, Ns))
        zr1[:dm.d_s, :dm.d_s], zr1[Ns:Ns + dm.d_s, :dm.d_s] = p.u_z, p.u_r
        wh = np.zeros((Ns, Nm))
        wh[:dm.d_s, :dm.d_m] = p.w_h
        uh = np.zeros((Ns, Ns))
        uh[:dm.d_s, :dm.d_s] = p.u_h
        blocks = [self._pack_kmajor_bf16(wm).reshape(-1)] + \
            [self._pack_kmajor_bf16(b).reshape(-1) for b in (zr0, zr1, wh, uh)]
        return self._torch.cat(blocks)

    def _pack_kmajor_bf16(self, B):
        """(..., N, K) float64 -> (..., 2*Np*Kp) bf16 bits (int16 tensor): the
        K-major tcgen05 B operand (8x8 core matrices), hi block then lo block,
        hi = bf16(w), lo = bf16(w - hi), both rounded to nearest even."""
        B = np.asarray(B, dtype=np.float64)
        *lead, N, K = B.shape
        Np, Kp = _rup(N, 16), _rup(K, 16)
        Bp = np.zeros((*lead, Np, Kp))
        Bp[..., :N, :K] = B
        hi = _bf16_rne(Bp)
        lo = _bf16_rne(Bp - _bf16_float(hi))
        n, k = np.meshgrid(np.arange(Np), np.arange(Kp), indexing="ij")
        idx = (((n // 8) * (Kp // 8) + k // 8) * 64 + (n % 8) * 8 + k % 8).ravel()
        out = np.zeros((*lead, 2, Np * Kp), dtype=np.uint16)
        out[..., 0, idx] = hi.reshape(*lead, Np * Kp)
        out[..., 1, idx] = lo.reshape(*lead, Np * Kp)
        out = np.ascontiguousarray(out.reshape(*lead, 2 * Np * Kp)).view(np.int16)
        return self._torch.tensor(out, device=self.device)

    def _pack_kmajor(self, B):
        """(..., N, K) float64 -> (..., 2*Np*Kp) float32 tensor: the K-major
        tcgen05 B operand (8x4 core matrices), hi block then lo block."""
        B = np.asarray(B, dtype=np.float64)
        *lead, N, K = B.shape
        Np, Kp = _rup(N, 16), _rup(K, 8)
        Bp = np.zeros((*lead, Np, Kp))
        Bp[..., :N, :K] = B
        hi = Bp.astype(np.float32)
        trunc = (hi.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
        lo = (Bp - trunc.astype(np.float64)).astype(np.float32)
        n, k = np.meshgrid(np.arange(Np), np.arange(Kp), indexing="ij")
        idx = (((n // 8) * (Kp // 4) + k // 4) * 32 + (n % 8) * 4 + k % 4).ravel()
        out = np.zeros((*lead, 2, Np * Kp), dtype=np.float32)
        out[..., 0, idx] = hi.reshape(*lead, Np * Kp)
        out[..., 1, idx] = lo.reshape(*lead, Np * Kp)
        return self._torch.tensor(np.ascontiguousarray(out.reshape(*lead, 2 * Np * Kp)),
                                  device=self.device)

    def _bind(self):
        self._state = self._tab.struct()
        _lib.check(self._L.stgn_engine_bind(self._handle, C.byref(self._state)), "bind")

    def _grow(self, need_nodes=0, need_edges=0, need_batch=0, need_gpow=0):
        tab = self._tab
        if self.shard is not None and need_nodes > self.cfg.nodes:
            raise ValueError(f"node id {need_nodes - 1} outside the sharded id range "
                             f"[0, {self.cfg.nodes})")
        rebuild_handle = need_batch > self._max_batch
        if rebuild_handle:
            self._max_batch = max(need_batch, 2 * self._max_batch)
            self._preds = np.zeros(self._max_batch, dtype=np.float64)
            self._make_handle()
            self._upload_weights()
        if (need_nodes > tab.cap_nodes or need_edges > tab.cap_edges or
                need_gpow > tab.gpow.numel() or rebuild_handle):
            self._torch.cuda.current_stream(self.device).synchronize()
            tab.grow(nodes=need_nodes, edges=need_edges, gpow=need_gpow, scratch=rebuild_handle)
            self._bind()

    def reserve(self, nodes: int = 0, edges: int = 0, batch: int = 0, batches: int = 0):
        """Pre-size the device tables (avoids regrowth copies mid-stream)."""
        self._grow(need_nodes=nodes, need_edges=edges, need_batch=batch,
                   need_gpow=self.batch_index + batches + 3 if batches else 0)

    def _ensure_nodes(self, n):
        if n > self._tab.cap_nodes:
            self._grow(need_nodes=n)
        self._n_mem = max(self._n_mem, n)

    def _cap_view(self):
        return min(self._tab.cap_nodes, max(self.node_count, 16))

    def __del__(self):
        try:
            if self._handle is not None:
                self._L.stgn_engine_destroy(self._handle)
        except Exception:
            pass

    # -- reference surface ---------------------------------------------------------
    @property
    def node_count(self) -> int:
        return max(self._store_n, self._n_mem, self.cfg.nodes)

    def process_batch(self, batch) -> list[float]:
        """S/engine.py:400-438."""
        src, dst, t, feat = edges_to_arrays(batch, self.dims.d_e)
        return self.process_batch_arrays(src, dst, t, feat).tolist()

    def process_batch_arrays(self, src, dst, t, feat=None) -> np.ndarray:
        """Array form of process_batch: (B,) ids, (B,) float64 times,
        (B, d_e) features; returns the (B,) float64 link scores."""
        self.counters.start_batch()
        self._affected_cache = None
        self._pred_cache = None
        self._pending.clear()  # the fused batch stages and commits its own edges
        self._stage_put.clear()
        src = np.ascontiguousarray(src, dtype=np.int64)
        dst = np.ascontiguousarray(dst, dtype=np.int64)
        t = np.ascontiguousarray(t, dtype=np.float64)
        B = int(src.shape[0])
        d_e = self.dims.d_e
        if feat is None:
            feat = np.zeros((B, d_e), dtype=np.float32)
        feat = np.ascontiguousarray(feat, dtype=np.float32)
        if feat.shape != (B, d_e) and not (d_e == 0 and feat.size == 0):
            raise FeatureDimError(f"edge features have shape {feat.shape}, expected ({B}, {d_e})")
        if B == 0:
            self._last_nD = self._last_nA = 0
            self.last_report = BatchReport(self.batch_index, 0, self._t_now, 0, 0)
            return np.zeros(0)
        if dst.shape[0] != B or t.shape[0] != B:
            raise ValueError("src, dst and t must have the same length")
        if (src < 0).any() or (dst < 0).any():
            raise ValueError("node ids must be non-negative")
        prev = np.concatenate([[self._t_now], t[:-1]])
        bad = np.nonzero(t < prev)[0]
        if bad.size:
            j = int(bad[0])
            raise MonotonicityError(
                f"batch edge at t={t[j]} precedes committed history t={prev[j]}")
        top = int(max(src.max(), dst.max())) + 1
        n_after = max(self._n_mem, top, self.cfg.nodes, self._store_n)
        self._grow(need_nodes=n_after, need_edges=self._m + B, need_batch=B,
                   need_gpow=self.batch_index + 3)
        self._n_mem = max(self._n_mem, top)
        self.batch_index += 1
        src32 = src.astype(np.int32)   # keep the converted arrays alive across the call
        dst32 = dst.astype(np.int32)
        rc = self._L.stgn_engine_process_batch(
            self._handle, B, src32.ctypes.data, dst32.ctypes.data,
            t.ctypes.data, feat.ctypes.data, self._m, self.batch_index, self.node_count,
            self._preds.ctypes.data, C.byref(self._rep), self._stream())
        if rc:
            self.batch_index -= 1
            _lib.check(rc, "process_batch")
        self._after_batch(B, float(t[-1]), top)
        return self._preds[:B].copy()

    # -- sharded batches (shard.py): two device phases around the exchange --------
    @property
    def stack_width(self) -> int:
        """Floats per node stack row [s (ld_s) | h_0 .. h_{K-2} (ld_d each)]."""
        return self.ld_s + (self.K - 1) * self.ld_d

    def gather_stacks(self, idx):
        """Pre-batch stacks of node ids `idx` (device int64 tensor): [n, stack_width]."""
        tab, torch = self._tab, self._torch
        parts = [tab.mem[idx]]
        if self.K > 1:
            parts.append(tab.h[idx, :self.K - 1].reshape(idx.shape[0], (self.K - 1) * self.ld_d))
        return torch.cat(parts, 1).contiguous()

    def scatter_stacks(self, idx, rows):
        """Write stacks (from gather_stacks on their owner) into rows `idx`."""
        tab = self._tab
        tab.mem[idx] = rows[:, :self.ld_s]
        if self.K > 1:
            tab.h[idx, :self.K - 1] = rows[:, self.ld_s:].reshape(idx.shape[0], self.K - 1,
                                                                   self.ld_d)

    def batch_phase1(self, src, dst, t, feat=None):
        """Stage one batch and run it through the recompute (stgn_engine_batch_phase 1)."""
        torch = self._torch
        self.counters.start_batch()
        self._affected_cache = None
        self._pred_cache = None
        src = np.ascontiguousarray(src, dtype=np.int64)
        dst = np.ascontiguousarray(dst, dtype=np.int64)
        t = np.ascontiguousarray(t, dtype=np.float64)
        B = int(src.shape[0])
        if B == 0 or dst.shape[0] != B or t.shape[0] != B:
            raise ValueError("a sharded batch needs B >= 1 edges with matching src/dst/t")
        if (src < 0).any() or (dst < 0).any():
            raise ValueError("node ids must be non-negative")
        prev = np.concatenate([[self._t_now], t[:-1]])
        if (t < prev).any():
            j = int(np.nonzero(t < prev)[0][0])
            raise MonotonicityError(f"batch edge at t={t[j]} precedes committed history t={prev[j]}")
        top = int(max(src.max(), dst.max())) + 1
        self._grow(need_nodes=max(self._n_mem, top, self.cfg.nodes, self._store_n),
                   need_edges=self._m + B, need_batch=B, need_gpow=self.batch_index + 3)
        self._n_mem = max(self._n_mem, top)
        self.batch_index += 1
        dev = self.device
        self._ph = dict(
            B=B, top=top, t_last=float(t[-1]),
            src=torch.from_numpy(src.astype(np.int32)).to(dev),
            dst=torch.from_numpy(dst.astype(np.int32)).to(dev),
            t=torch.from_numpy(t).to(dev),
            feat=(torch.from_numpy(np.ascontiguousarray(feat, dtype=np.float32)).to(dev)
                  if (feat is not None and self.dims.d_e) else None))
        ph = self._ph
        rc = self._L.stgn_engine_batch_phase(
            self._handle, 1, B, ph["src"].data_ptr(), ph["dst"].data_ptr(), ph["t"].data_ptr(),
            ph["feat"].data_ptr() if ph["feat"] is not None else None, self._m, self.batch_index,
            self.node_count, None, None, self._stream())
        if rc:
            self.batch_index -= 1
            _lib.check(rc, "batch_phase(1)")

    def dpred_export(self):
        """(node ids int32, [n, ld_d] rows) of this engine's owned direct nodes."""
        torch = self._torch
        cap = 2 * self._max_batch
        nodes = torch.empty(cap, dtype=torch.int32, device=self.device)
        rows = torch.empty((cap, self.ld_d), dtype=torch.float32, device=self.device)
        cnt = C.c_int64()
        _lib.check(self._L.stgn_engine_dpred_export(self._handle, nodes.data_ptr(), rows.data_ptr(),
                                                    C.byref(cnt), self._stream()), "dpred_export")
        n = int(cnt.value)
        return nodes[:n], rows[:n]

    def dpred_import(self, gathered):
        nodes, rows = gathered
        nodes = nodes.to(self.device, dtype=self._torch.int32).contiguous()
        rows = rows.to(self.device, dtype=self._torch.float32).contiguous()
        _lib.check(self._L.stgn_engine_dpred_import(self._handle, nodes.data_ptr(), rows.data_ptr(),
                                                    int(nodes.shape[0]), self._stream()),
                   "dpred_import")

    def batch_phase2(self) -> np.ndarray:
        """Scores, memory commit, drift and rebuild; returns the batch's scores."""
        ph = self._ph
        preds = self._torch.empty(ph["B"], dtype=self._torch.float64, device=self.device)
        _lib.check(self._L.stgn_engine_batch_phase(
            self._handle, 2, ph["B"], None, None, None, None, self._m, self.batch_index,
            self.node_count, preds.data_ptr(), C.byref(self._rep), self._stream()), "batch_phase(2)")
        self._after_batch(ph["B"], ph["t_last"], ph["top"])
        self._ph = None
        return preds.cpu().numpy()

    def process_batch_device(self, src, dst, t, feat=None, *, max_id: int, t_last: float,
                             t_first: float, report: bool = False):
        """Batch already resident on the device (torch tensors: src/dst int32,
        t float64, feat float32 (B, d_e)); returns the device float64 score
        tensor without synchronising. The caller vouches for validity
        (non-negative ids, non-decreasing times >= t_now) and passes the
        largest id and the first/last timestamps it already knows."""
        torch = self._torch
        B = int(src.shape[0])
        if B == 0:
            return torch.zeros(0, dtype=torch.float64, device=self.device)
        if t_first < self._t_now:
            raise MonotonicityError(f"batch edge at t={t_first} precedes committed history "
                                    f"t={self._t_now}")
        top = int(max_id) + 1
        self._grow(need_nodes=max(self._n_mem, top, self.cfg.nodes, self._store_n),
                   need_edges=self._m + B, need_batch=B, need_gpow=self.batch_index + 3)
        self._n_mem = max(self._n_mem, top)
        self.batch_index += 1
        self.counters.start_batch()
        self._affected_cache = None
        self._pred_cache = None
        preds = torch.empty(B, dtype=torch.float64, device=self.device)
        fptr = feat.data_ptr() if (feat is not None and self.dims.d_e) else None
        rc = self._L.stgn_engine_process_batch_dev(
            self._handle, B, src.data_ptr(), dst.data_ptr(), t.data_ptr(), fptr, self._m,
            self.batch_index, self.node_count, preds.data_ptr(),
            C.byref(self._rep) if report else None, self._stream())
        if rc:
            self.batch_index -= 1
            _lib.check(rc, "process_batch_device")
        if report:
            self._after_batch(B, float(t_last), top)
        else:
            self._m += B
            self._t_now = float(t_last)
            self._store_n = max(self._store_n, top)
            self._last_nD = self._last_nA = None  # not fetched
            self.last_report = None
        return preds

    def set_recompute(self, recompute: str):
        """Switch between "affected" (the reference's literal exact mode) and
        "direct" (value-identical with an infinite window) for later batches."""
        if recompute not in _lib.SCOPE:
            raise ConfigError(f"recompute must be one of {tuple(_lib.SCOPE)}")
        # single-layer delta mode keeps attention-state stamps from its first batch;
        # multi-layer models have none (S/engine.py:252-253), so there the switch is exact
        if self.K == 1 and (recompute == "delta") != (self.cfg.mode == "delta"):
            raise ConfigError("for single-layer models the delta scope is fixed by cfg.mode")
        _lib.check(self._L.stgn_engine_set_scope(self._handle, _lib.SCOPE[recompute]), "set_scope")
        self.recompute = recompute

    def set_state_only(self, on: bool):
        """Test-harness fast-forward (the oracle's process_batch(compute=False)):
        while on, batches advance topology, rings, memory and drift without the
        attention recomputes, so the layer cache keeps its current rows."""
        _lib.check(self._L.stgn_engine_set_skip_recompute(self._handle, int(bool(on))),
                   "set_skip_recompute")
        self._state_only = bool(on)

    # -- profiling ----------------------------------------------------------------
    def set_profiling(self, on: bool):
        _lib.check(self._L.stgn_engine_set_profiling(self._handle, int(bool(on))), "profiling")

    def stage_times(self) -> tuple[dict, int]:
        """Per-stage device milliseconds of the last batch (profiling on) and
        the number of kernel launches per batch."""
        buf = (C.c_float * 16)()
        launches = C.c_int64()
        n = self._L.stgn_engine_stage_times(self._handle, buf, 16, C.byref(launches))
        names = [self._L.stgn_stage_name(i).decode() for i in range(max(n, 0))]
        return {nm: float(buf[i]) for i, nm in enumerate(names)}, int(launches.value)

    def info(self) -> dict:
        """Engine facts from the C ABI (graph replay, conditional rebuild, tiles)."""
        buf = (C.c_int64 * 14)()
        _lib.check(self._L.stgn_engine_info(self._handle, buf, 14), "info")
        keys = ("graph_active", "conditional_rebuild", "launches_per_batch", "attn_tile_rows",
                "attn_staged_weight_floats", "num_sms", "attn_smem_bytes", "memory_smem_bytes",
                "tensor_cores", "tc_tile_rows", "bf16x3", "bf16x3_smem_bytes",
                "memory_bf16x3", "memory_bf16x3_smem_bytes")
        return {k: int(buf[i]) for i, k in enumerate(keys)}

    @property
    def delta_events(self) -> list:
        """The last batch's DeltaEvent records (delta mode, K = 1; else [])."""
        if self.cfg.mode != "delta" or self.K != 1:
            return []
        if self._ev_batch != self.batch_index:
            self._events = self._fetch_delta_events()
            self._ev_batch = self.batch_index
        return self._events

    @property
    def max_value_norm_seen(self) -> float:
        """Running max of the attention states' value-row norms (S/engine.py:255-261, 349)."""
        if self.cfg.mode != "delta" or self.K != 1:
            return 0.0
        return float(self._tab.ctl[4:5].cpu().view(self._torch.float64).item())

    def _fetch_delta_events(self):
        cap = max(self._tab.ev_cap, 1)
        d = self.dims.d
        node = np.zeros(cap, np.int32)
        dn = np.zeros(cap, np.int32)
        nv = np.zeros(cap, np.int32)
        bound, mv, zd = np.zeros(cap), np.zeros(cap), np.zeros(cap)
        emb = np.zeros((cap, d), np.float32)
        mvn = C.c_double()
        P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self.sync()
        n = self._L.stgn_engine_delta_events(self._handle, C.c_int64(cap), P(node), P(bound), P(dn),
                                             P(nv), P(mv), P(zd), P(emb), C.byref(mvn))
        if n < 0:
            _lib.check(n, "delta_events")
        return [DeltaEvent(node=int(node[i]), embedding=emb[i].astype(np.float64),
                           bound=float(bound[i]), dn=int(dn[i]), nv=int(nv[i]),
                           max_v=float(mv[i]), z_dev=float(zd[i])) for i in range(n)]

    def _after_batch(self, B, t_last, top):
        self._m += B
        self._t_now = t_last
        self._store_n = max(self._store_n, top)
        self._account(self._rep, B, t_last, self.batch_index)

    def _account(self, r, B, t_last, index):
        """Counters, last_report and the last batch's set sizes from a report
        (synchronous calls, or a pipelined caller collecting batch `index`)."""
        dm = self.dims
        self._last_nD, self._last_nA = int(r.direct), int(r.affected)
        nD, nA = self._last_nD, self._last_nA
        c = self.counters
        c.add("nbr_hit", int(r.nbr_hit))
        c.add("nbr_miss", int(r.nbr_miss))
        c.add("embed_predict", nD)
        if self.recompute == "delta":  # S/engine.py:287-319
            for k in ("embed_skip", "attn_hit", "attn_miss"):
                if getattr(r, k):
                    c.add(k, int(getattr(r, k)))
            c.add("embed_refresh", nA - int(r.embed_skip))
            c.add("rows_gathered", int(r.attn_miss) + nD)
            c.add("macs_attention", self._mac_attn(int(r.attn_miss), int(r.entries_miss)) +
                  self._mac_attn(nD, int(r.entries_direct)))
        else:
            c.add("embed_refresh", nA)
            c.add("rows_gathered", nA + nD)
            c.add("macs_attention", self._mac_attn(nA, int(r.entries_affected)) +
                  self._mac_attn(nD, int(r.entries_direct)))
        c.add("messages", 2 * B)
        c.add("macs_gru", 2 * B * dm.d_m * dm.msg_in +
              nD * 3 * (dm.d_s * dm.d_m + dm.d_s * dm.d_s))
        c.add("gru_steps", nD)
        kind = _REBUILD_NAMES[int(r.rebuild_kind)]
        rb = int(r.rebuild_nodes)
        if kind != "none":
            c.add("rows_gathered", rb)
            c.add("macs_attention", self._mac_attn(rb, int(r.entries_rebuild)))
            c.add("rebuild_pipelines", rb)
            c.add("rebuilds")
        c.add("direct", nD)
        c.add("affected", nA)
        self.last_global_drift = float(r.global_drift)
        self.last_report = BatchReport(index=index, edges=B, t_batch=t_last,
                                       direct=nD, affected=nA, rebuild=kind, rebuild_nodes=rb)

    def _mac_attn(self, n, e):
        dm = self.dims
        per_node = dm.heads * dm.query_in * dm.d_k + dm.heads * dm.d_k * dm.d
        per_entry = dm.heads * (2 * dm.key_in * dm.d_k + 2 * dm.d_k)
        return dm.layers * (n * per_node + e * per_entry)

    def _fetch_lists(self):
        """(direct ids in device order, affected ids, change-record sizes)."""
        if self._affected_cache is None:
            nD, nA = self._last_nD, self._last_nA
            d = np.zeros(max(nD, 1), dtype=np.int32)
            a = np.zeros(max(nA, 1), dtype=np.int32)
            sz = np.zeros(max(nA, 1), dtype=np.int32)
            gd, ga = C.c_int64(), C.c_int64()
            _lib.check(self._L.stgn_engine_affected(self._handle, d.ctypes.data, a.ctypes.data,
                                                    a.size, C.byref(gd), C.byref(ga),
                                                    sz.ctypes.data, self._stream()), "affected")
            self._affected_cache = (d[:nD], a[:nA], sz[:nA])
        return self._affected_cache

    @property
    def last_affected(self) -> AffectedSet | None:
        if self.last_report is None:
            return None
        d, a, sz = self._fetch_lists()
        recs = {int(v): ChangeRecordSize(int(s)) for v, s in zip(a, sz)}
        return AffectedSet(set(d.tolist()), set(a.tolist()), recs)

    @property
    def last_pred_embeddings(self) -> dict:
        if self._pred_cache is None:
            nD = self._last_nD
            self._pred_cache = {}
            if nD:
                d, _, _ = self._fetch_lists()
                out = np.zeros((nD, self.dims.d), dtype=np.float32)
                _lib.check(self._L.stgn_engine_pred_embeddings(self._handle, out.ctypes.data, nD,
                                                               self._stream()), "pred_emb")
                self._pred_cache = {int(v): out[i].astype(np.float64) for i, v in enumerate(d)}
        return self._pred_cache

    def rebuild_nodes(self, nodes) -> int:
        """S/engine.py:385-396."""
        n = self.node_count
        if nodes is not None:
            ids = np.array(sorted(nodes), dtype=np.int32)
            if ids.size == 0:
                return 0
            self._ensure_nodes(int(ids.max()) + 1)
            n = self.node_count
            ptr, cnt = ids.ctypes.data, ids.size
        else:
            if n == 0:
                return 0
            self._ensure_nodes(n)
            ptr, cnt = None, 0
        out = C.c_int64()
        valid_at = self._t_now if self._m else 0.0
        _lib.check(self._L.stgn_engine_rebuild(self._handle, ptr, cnt, n, valid_at, C.byref(out),
                                               self._stream()), "rebuild")
        self.counters.add("rebuild_pipelines", int(out.value))
        return int(out.value)

    def full_reference(self) -> np.ndarray:
        """S/engine.py:374-381 (read-only)."""
        torch = self._torch
        n = self.node_count
        self._ensure_nodes(n)
        out = torch.empty((max(n, 1), self.ld_d), dtype=torch.float32, device=self.device)
        if n:
            _lib.check(self._L.stgn_engine_full_reference(self._handle, n, out.data_ptr(),
                                                          self._stream()), "full_reference")
        return out[:n, :self.dims.d].double().cpu().numpy()

    def snapshot_layers(self, t_now: float | None = None) -> np.ndarray:
        """Pure K-layer recompute of every node (OracleEngine.full_recompute,
        S/oracle.py:47-65): (n, K, d) float64; nothing is mutated. t_now earlier
        than the newest edge uses each node's L newest entries with t <= t_now
        (S/graph_store.py:158-173) and needs edge_payloads=True."""
        torch = self._torch
        n = self.node_count
        self._ensure_nodes(n)
        hist = t_now is not None and self._m > 0 and t_now < self._t_now
        if hist and not self.edge_payloads:
            raise ConfigError("historical snapshots need IncrementalEngine(edge_payloads=True)")
        out = torch.zeros((max(n, 1), self.K, self.ld_d), dtype=torch.float32, device=self.device)
        if n:
            _lib.check(self._L.stgn_engine_snapshot(self._handle, n,
                                                    float(t_now) if hist else math.inf,
                                                    out.data_ptr(), self._stream()), "snapshot")
        return out[:n, :, :self.dims.d].double().cpu().numpy()

    def rebuild_range(self, lo: int, hi: int):
        """Exact recompute of node ids [lo, hi); returns their layer-cache rows
        (device tensor [hi-lo, K, d])."""
        if hi > lo:
            self.rebuild_nodes(range(lo, hi))
        return self._tab.h[lo:hi, :, :self.dims.d]

    def distributed_full_rebuild(self, group=None) -> int:
        """rebuild_nodes(None) split by node-id range over the ranks of
        `group` (every rank holds the same state: replicas). Each rank
        recomputes its shard; an all-gather of the layer-cache rows leaves
        every replica identical to a single-device full rebuild."""
        from .dist import sharded_rebuild
        n = self.node_count
        if n == 0:
            return 0
        self._ensure_nodes(n)
        rows = sharded_rebuild(self.rebuild_range, n, group)
        tab = self._tab
        tab.h[:n, :, :self.dims.d] = rows
        cc = tab.ring_ccnt[:n]
        tab.ring_ccnt[:n] = self._torch.where(cc < 0, tab.ring_cnt[:n], cc)
        tab.valid[:n] = 1
        tab.valid_at[:n] = self._t_now if self._m else 0.0
        if self.recompute == "delta" and self.K == 1:
            # attention-state stamps of every rebuilt node, as k_rb_fill stamps the local
            # shard (S/engine.py:393-395): a single-device rebuild stamps all n
            torch = self._torch
            tab.attn_ver[:n] = tab.version[:n]
            head = tab.ring_head[:n].to(torch.int64)
            tref = tab.ring_t[:n].gather(1, head.unsqueeze(1)).squeeze(1)
            tab.attn_tref[:n] = torch.where(tab.ring_ccnt[:n] > 0, tref, torch.zeros_like(tref))
        # rebuild_range counted this rank's shard; a single-device rebuild counts all n
        from .dist import gather_rows, shard_range
        import torch.distributed as dist
        lo, hi = shard_range(n, dist.get_world_size(group), dist.get_rank(group))
        if self.recompute == "delta" and self.K == 1:
            # the rebuilt states' log Z (csrc/delta.cuh) from every shard, and the
            # running max value norm over all of them
            tab.attn_logz[:n] = gather_rows(tab.attn_logz[lo:hi].clone(), n, group)
            mvn = tab.ctl[4:5].view(self._torch.float64).clone()
            dist.all_reduce(mvn, op=dist.ReduceOp.MAX, group=group)
            tab.ctl[4:5] = mvn.view(self._torch.int64)
        self.counters.add("rebuild_pipelines", n - (hi - lo))
        return n

    # convenience for the scheduler API
    def execute_rebuild(self, decision) -> int:
        if decision is None:
            raise DriftContractError("execute_rebuild needs a non-None decision")
        kind, nodes = decision
        return self.rebuild_nodes(sorted(nodes) if kind == "partial" else None)

    # -- stage-level surface (csrc/stage.cuh) -----------------------------------
    def _stack_of(self, row) -> np.ndarray:
        """gather_stacks row -> the reference's (K, d) stack (S/state.py:118-127)."""
        dm = self.dims
        st = np.zeros((self.K, dm.d))
        st[0, :dm.d_s] = row[:dm.d_s]
        for j in range(1, self.K):
            o = self.ld_s + (j - 1) * self.ld_d
            st[j] = row[o:o + dm.d]
        return st

    def stage_batch(self, batch) -> list:
        """S/engine_base.py:88-106: edge ids from the store's count, both
        endpoints' pre-batch stacks frozen (one device gather). Nothing is
        committed; the edges wait in `_pending` for commit_pending."""
        torch = self._torch
        src, dst, t, feat = edges_to_arrays(batch, self.dims.d_e)
        B = len(batch)
        if B == 0:
            return []
        top = int(max(src.max(), dst.max())) + 1
        self._grow(need_nodes=max(self._n_mem, top, self.cfg.nodes, self._store_n),
                   need_edges=self._m + B)
        self._n_mem = max(self._n_mem, top)
        ids = torch.from_numpy(np.concatenate([src, dst])).to(self.device)
        rows = self.gather_stacks(ids).double().cpu().numpy()
        out = []
        for i in range(B):
            pe = PendingEdge(edge_id=self._m + i, src=int(src[i]), dst=int(dst[i]), t=float(t[i]),
                             feat=feat[i].copy(), stack_src=self._stack_of(rows[i]),
                             stack_dst=self._stack_of(rows[B + i]))
            self._pending[pe.edge_id] = pe
            out.append(pe)
        return out

    def detect_affected(self, pending) -> AffectedSet:
        """S/engine.py:196-212 on the device (k_stage_affected): the direct
        endpoints and their K-hop closure over the post-insertion truncated
        lists; nothing is mutated. Records start empty, as in the reference."""
        torch = self._torch
        pending = list(pending)
        if not pending:
            return AffectedSet(set(), set(), {})
        dev = self.device
        src = torch.tensor([pe.src for pe in pending], dtype=torch.int32, device=dev)
        dst = torch.tensor([pe.dst for pe in pending], dtype=torch.int32, device=dev)
        top = int(max(src.max().item(), dst.max().item())) + 1
        self._grow(need_nodes=max(top, self.node_count))
        cap = self._tab.cap_nodes
        out = torch.empty(cap, dtype=torch.int32, device=dev)
        hop = torch.zeros(self.K + 2, dtype=torch.int32, device=dev)
        self._stage_stamp = self._stage_stamp + 1 if self._stage_stamp < 0xFFFFFFFF else 0x80000000
        _lib.check(self._L.stgn_engine_stage_affected(
            self._handle, len(pending), src.data_ptr(), dst.data_ptr(), self._stage_stamp,
            out.data_ptr(), cap, hop.data_ptr(), self._stream()), "stage_affected")
        h = hop.cpu().numpy()
        ids = out[:int(h[self.K + 1])].cpu().numpy()
        allset = set(ids.tolist())
        return AffectedSet(set(ids[:int(h[1])].tolist()), allset,
                           {v: ChangeRecord() for v in allset})

    def _entry_payload(self, e, viewer):
        """(stack (K, d), feat) of entry e seen from `viewer` (S/engine_base.py:119-133)."""
        pe = self._pending.get(int(e.edge_id))
        if pe is not None:
            return (pe.stack_dst if viewer == pe.src else pe.stack_src), pe.feat
        eid = int(e.edge_id)
        if eid >= self._m or self._tab.e_pay is None:
            raise InputError(f"edge {eid} is neither staged nor in the payload log "
                             "(build the engine with edge_payloads=True)")
        side = 0 if int(self._tab.e_src[eid]) == viewer else 1
        row = self._tab.e_pay[2 * eid + side].double().cpu().numpy()
        st = row.reshape(self.K, self.ld_d)[:, :self.dims.d]
        return st, self._tab.e_feat[eid, :self.dims.d_e].double().cpu().numpy()

    def _stage_update(self, items, direct, t_now):
        """items: [(v, [NeighborEntry newest first], put)] with distinct v.
        Returns per item (hit, expired entries, updated neighbours)."""
        torch = self._torch
        if not items:
            return []
        dev, K, dm = self.device, self.K, self.dims
        top = max(v for v, _, _ in items) + 1
        self._grow(need_nodes=max(top, self.node_count))
        nodes = [int(v) for v, _, _ in items]
        off = np.zeros(len(items) + 1, dtype=np.int32)
        for i, (_, ents, _) in enumerate(items):
            off[i + 1] = off[i] + len(ents)
        ne = int(off[-1])
        pay = np.zeros((max(ne, 1), K, self.ld_d), dtype=np.float32)
        feat = np.zeros((max(ne, 1), self.ld_e), dtype=np.float32)
        nbr = np.zeros(max(ne, 1), dtype=np.int32)
        tt = np.zeros(max(ne, 1), dtype=np.float64)
        eid = np.zeros(max(ne, 1), dtype=np.int64)
        q = 0
        for v, ents, _ in items:
            for e in ents:
                st, f = self._entry_payload(e, v)
                pay[q, :, :dm.d] = st
                feat[q, :dm.d_e] = f
                nbr[q], tt[q], eid[q] = int(e.nbr), float(e.t), int(e.edge_id)
                q += 1

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        d_nodes, d_off, d_nbr, d_t, d_eid = map(up, (np.array(nodes, dtype=np.int32), off, nbr,
                                                     tt, eid))
        d_pay, d_feat = up(pay), up(feat)
        d_put = up(np.array([1 if p else 0 for _, _, p in items], dtype=np.int32))
        d_dir = up(np.array(sorted(int(x) for x in direct) or [0], dtype=np.int32))
        nn, L = len(items), self.L
        z = torch.zeros
        hit, exp_n, upd_n = (z(nn, dtype=torch.int32, device=dev) for _ in range(3))
        exp_nbr = z(ne + nn * L, dtype=torch.int32, device=dev)
        exp_t = z(ne + nn * L, dtype=torch.float64, device=dev)
        exp_eid = z(ne + nn * L, dtype=torch.int64, device=dev)
        upd_nbr = z(nn * L, dtype=torch.int32, device=dev)
        ent = _lib.StageEntries(*[x.data_ptr() for x in (d_nodes, d_off, d_nbr, d_t, d_eid, d_pay,
                                                         d_feat, d_put)])
        rec = _lib.StageRecords(*[x.data_ptr() for x in (hit, exp_n, exp_nbr, exp_t, exp_eid,
                                                         upd_n, upd_nbr)])
        _lib.check(self._L.stgn_engine_stage_nbr_update(
            self._handle, nn, C.byref(ent), d_dir.data_ptr(), len(direct), float(t_now),
            C.byref(rec), self._stream()), "stage_nbr_update")
        hit, exp_n, upd_n = hit.tolist(), exp_n.tolist(), upd_n.tolist()
        exp_nbr, exp_t, exp_eid = exp_nbr.tolist(), exp_t.tolist(), exp_eid.tolist()
        upd_nbr = upd_nbr.tolist()
        out = []
        for i in range(nn):
            xo = int(off[i]) + i * L
            expired = [NeighborEntry(exp_nbr[xo + k], exp_t[xo + k], exp_eid[xo + k])
                       for k in range(exp_n[i])]
            out.append((bool(hit[i]), expired, set(upd_nbr[i * L:i * L + upd_n[i]])))
        return out

    def update_neighbor_cache(self, v: int, new_entries, direct, t_now: float) -> ChangeRecord:
        """S/engine.py:216-243 on the device (k_stage_nbr_update): prepend,
        evict beyond L, expire outside the window; returns the ChangeRecord.
        New entries must be staged (stage_batch) or in the payload log."""
        new_entries = list(new_entries)
        hit, expired, updated = self._stage_update([(int(v), new_entries, True)], set(direct),
                                                   t_now)[0]
        self.counters.add("nbr_hit" if hit else "nbr_miss")
        self._stage_put.add(int(v))
        return ChangeRecord(added=new_entries, expired=expired, updated=updated)

    def commit_pending(self) -> None:
        """S/engine_base.py:108-117: the staged edges enter the store in id
        order (k_stage_commit). The store's top-L lists of their endpoints move
        with them; a cached endpoint whose list update_neighbor_cache did not
        move gets the post-insertion list (the cache and the store's top-L share
        one ring per node here, csrc/stage.cuh)."""
        if not self._pending:
            return
        torch = self._torch
        eids = sorted(self._pending)
        if eids != list(range(self._m, self._m + len(eids))):
            raise InputError(f"staged edge ids {eids[0]}..{eids[-1]} do not follow the store "
                             f"count {self._m}")
        pes = [self._pending[i] for i in eids]
        prev = self._t_now
        for pe in pes:
            if pe.t < prev:
                raise MonotonicityError(
                    f"batch edge at t={pe.t} precedes committed history t={prev}")
            prev = pe.t
        P, dev, dm = len(pes), self.device, self.dims
        by_node: dict = {}
        for pe in reversed(pes):  # S/engine.py:170-180
            by_node.setdefault(pe.src, []).append(NeighborEntry(pe.dst, pe.t, pe.edge_id))
            if pe.dst != pe.src:
                by_node.setdefault(pe.dst, []).append(NeighborEntry(pe.src, pe.t, pe.edge_id))
        todo = [v for v in by_node if v not in self._stage_put]
        if todo:
            cached = self._tab.ring_ccnt[torch.tensor(todo, dtype=torch.int64, device=dev)]
            items = [(v, by_node[v], c >= 0) for v, c in zip(todo, cached.tolist())]
            self._stage_update(items, set(by_node), pes[-1].t)
        src = torch.tensor([pe.src for pe in pes], dtype=torch.int32, device=dev)
        dst = torch.tensor([pe.dst for pe in pes], dtype=torch.int32, device=dev)
        tt = torch.tensor([pe.t for pe in pes], dtype=torch.float64, device=dev)
        feat = np.zeros((P, self.ld_e), dtype=np.float32)
        pay = np.zeros((P, 2, self.K, self.ld_d), dtype=np.float32)
        for i, pe in enumerate(pes):
            feat[i, :dm.d_e] = pe.feat
            pay[i, 0, :, :dm.d] = pe.stack_dst
            pay[i, 1, :, :dm.d] = pe.stack_src
        d_feat = torch.from_numpy(feat).to(dev)
        d_pay = torch.from_numpy(pay).to(dev)
        _lib.check(self._L.stgn_engine_stage_commit(
            self._handle, P, src.data_ptr(), dst.data_ptr(), tt.data_ptr(), d_feat.data_ptr(),
            d_pay.data_ptr(), self._m, self._stream()), "stage_commit")
        self._m += P
        self._t_now = pes[-1].t
        self._store_n = max(self._store_n, max(max(pe.src, pe.dst) for pe in pes) + 1)
        self._pending.clear()
        self._stage_put.clear()

    def sync(self):
        self._torch.cuda.current_stream(self.device).synchronize()
