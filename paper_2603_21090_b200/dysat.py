"""DySAT incremental inference on the B200 engine.

The reference only reports DySAT results (PAPER.md:1905-1912, 2266-2267:
"structural and temporal self-attention over graph snapshots"); it ships no
DySAT code, so the model below is this repo's statement of DySAT (Sankar et
al., WSDM 2020) for streaming inference, and parity is pinned only to the
float64 restatement in oracle/dysat_oracle.py ("parity unpinned" against the
reference).

Model (one structural layer, one temporal layer, as DySAT's default):
  snapshots   edge (u, v, t) belongs to snapshot k = floor(t / snapshot_len);
              node v's list in snapshot k = its L most recent entries of that
              snapshot, newest first (a self-loop contributes one entry)
  structural  P = X W_s (static node features X); per head h (d / H_s wide)
                e_vu = LeakyReLU(a_self,h . P_v,h + a_nbr,h . P_u,h, 0.2)
                over u in [v] + list_k(v) (self first); alpha = softmax(e)
                z_v^k = ELU(concat_h sum_u alpha_vu P_u,h)
  temporal    y_j = z_v^j + pos[j] for the snapshots j = max(0, k-W+1) .. k;
              per head g (d / H_t wide): a_j = softmax_j(q_g . k_j,g / sqrt(d/H_t))
              with q = y_k W_q, k_j = y_j W_k, v_j = y_j W_v;
              emb_v = concat_g sum_j a_j v_j,g W_o + y_k
  prediction  sigmoid(w_pred . [emb_u || emb_v] + b_pred) with the embeddings
              before the edges are applied (predict, then update)

Incremental rule: a batch changes z^k only of its endpoints (the structural
layer reads static P and the endpoints' lists), so the affected set of a batch
is exactly its endpoints; their temporal outputs are recomputed from the
cached key/value rows of the earlier snapshots. A snapshot boundary
(roll) clears the lists and recomputes every node (all z^k become the
self-only ELU(P_v)): that is DySAT's O(|V|) step.

Device layout and kernels: csrc/dysat.cuh; C ABI: stgn_dysat_* (include/stgn.h).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .config import ConfigError


@dataclass(frozen=True)
class DySATConfig:
    n: int                      # node count (node features are per node)
    d_in: int = 64              # node-feature width
    d: int = 128                # model width
    heads_s: int = 8            # structural heads
    heads_t: int = 8            # temporal heads
    window: int = 8             # temporal window W (snapshots)
    fanout: int = 20            # L: most recent entries per node per snapshot
    snapshot_len: float = 1000.0
    max_snapshots: int = 4096   # positional-embedding rows
    batch_size: int = 600

    def validate(self):
        ok = (self.n > 0 and self.d_in > 0 and self.d > 0 and self.heads_s > 0 and
              self.heads_t > 0 and self.d % self.heads_s == 0 and self.d % self.heads_t == 0 and
              1 <= self.window <= 32 and 1 <= self.fanout <= 31 and self.snapshot_len > 0 and
              self.max_snapshots > 0 and self.batch_size > 0 and self.heads_s <= 32)
        if not ok:
            raise ConfigError(f"invalid DySAT config {self}")


@dataclass
class DySATParams:
    x: np.ndarray        # (n, d_in) node features
    w_s: np.ndarray      # (d_in, d)
    a_self: np.ndarray   # (H_s, d / H_s)
    a_nbr: np.ndarray    # (H_s, d / H_s)
    pos: np.ndarray      # (max_snapshots, d)
    w_q: np.ndarray      # (d, d)
    w_k: np.ndarray
    w_v: np.ndarray
    w_o: np.ndarray
    w_pred: np.ndarray   # (2 d,)
    b_pred: float


def init_dysat_params(seed: int, cfg: DySATConfig) -> DySATParams:
    """Seeded Glorot-normal weights, unit-normal features (synthetic model)."""
    rng = np.random.default_rng(seed)

    def glorot(a, b):
        return rng.standard_normal((a, b)) * math.sqrt(2.0 / (a + b))
    dh = cfg.d // cfg.heads_s
    return DySATParams(
        x=rng.standard_normal((cfg.n, cfg.d_in)),
        w_s=glorot(cfg.d_in, cfg.d),
        a_self=rng.standard_normal((cfg.heads_s, dh)) * math.sqrt(1.0 / dh),
        a_nbr=rng.standard_normal((cfg.heads_s, dh)) * math.sqrt(1.0 / dh),
        pos=rng.standard_normal((cfg.max_snapshots, cfg.d)) * 0.1,
        w_q=glorot(cfg.d, cfg.d), w_k=glorot(cfg.d, cfg.d), w_v=glorot(cfg.d, cfg.d),
        w_o=glorot(cfg.d, cfg.d),
        w_pred=rng.standard_normal(2 * cfg.d) * math.sqrt(1.0 / cfg.d),
        b_pred=float(rng.standard_normal()))


def _kmajor_bf16(B):
    """(N, K) float64 -> (2 N K,) uint16 viewed as int16: the K-major tcgen05 B
    operand (8x8 core matrices), hi block then lo block (engine._pack_kmajor_bf16)."""
    from .engine import _bf16_float, _bf16_rne
    N, K = B.shape
    hi = _bf16_rne(B)
    lo = _bf16_rne(B - _bf16_float(hi))
    n, k = np.meshgrid(np.arange(N), np.arange(K), indexing="ij")
    idx = (((n // 8) * (K // 8) + k // 8) * 64 + (n % 8) * 8 + k % 8).ravel()
    out = np.zeros((2, N * K), dtype=np.uint16)
    out[0, idx] = hi.ravel()
    out[1, idx] = lo.ravel()
    return out.reshape(-1).view(np.int16)


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("DySATEngine needs a CUDA device (no CPU fallback)")
    return torch


class DySATEngine:
    """Snapshot-stream DySAT inference on one GPU: process_batch predicts the
    batch's links from the current embeddings, then applies the edges and
    recomputes the affected nodes (the endpoints); a batch crossing snapshot
    boundaries is split there and each boundary rolls the snapshot (every
    node recomputed). full_recompute() recomputes every node in place (the
    baseline the incremental path is measured against)."""

    def __init__(self, cfg: DySATConfig, params: DySATParams, device=None,
                 tensor_cores: bool = True, tc_min_rows: int = 64 * 128):
        cfg.validate()
        torch = self._torch = _torch()
        self.cfg, self.params = cfg, params
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self._L = _lib.lib()
        n, d = cfg.n, cfg.d
        self.ld = ld = (d + 3) // 4 * 4
        dev = self.device

        def f32(a, rows, cols):
            t = torch.zeros((rows, cols), dtype=torch.float32, device=dev)
            a = np.asarray(a, dtype=np.float64).reshape(rows, -1)
            t[:, :a.shape[1]] = torch.from_numpy(a.astype(np.float32)).to(dev)
            return t
        # P = X W_s (fp64 on the host, once, then fp32: the static projected features)
        P = np.asarray(params.x, dtype=np.float64) @ np.asarray(params.w_s, dtype=np.float64)
        dh = d // cfg.heads_s
        Ph = P.reshape(n, cfg.heads_s, dh)
        self.P = f32(P, n, ld)
        self.ss = f32(np.einsum("nhc,hc->nh", Ph, params.a_self), n, cfg.heads_s)
        self.sn = f32(np.einsum("nhc,hc->nh", Ph, params.a_nbr), n, cfg.heads_s)
        self.pos = f32(params.pos, cfg.max_snapshots, ld)
        self.wq, self.wk = f32(params.w_q, d, ld), f32(params.w_k, d, ld)
        self.wv, self.wo = f32(params.w_v, d, ld), f32(params.w_o, d, ld)
        self.wpred = torch.from_numpy(np.asarray(params.w_pred, dtype=np.float64)).to(dev)
        # tcgen05 B operands of the temporal GEMMs (d = 64 / 128): W^T as K-major bf16
        # hi | lo blocks (csrc/dysat.cuh k_dy_temporal_tc); None -> the FFMA kernel
        dt = d // cfg.heads_t
        self.tensor_cores = tensor_cores and d in (64, 128) and dt in (8, 16, 32) and dt <= d // 4
        self.tc_min_rows = int(tc_min_rows)
        self.wtc = (torch.from_numpy(np.stack([_kmajor_bf16(np.asarray(w, np.float64).T)
                                               for w in (params.w_q, params.w_k, params.w_v,
                                                         params.w_o)])).to(dev)
                    if self.tensor_cores else None)
        i32 = torch.int32
        self.lst_nbr = torch.zeros((n, cfg.fanout), dtype=i32, device=dev)
        self.lst_head = torch.zeros(n, dtype=i32, device=dev)
        self.lst_cnt = torch.zeros(n, dtype=i32, device=dev)
        self.hist_k = torch.zeros((n, cfg.window, ld), dtype=torch.float32, device=dev)
        self.hist_v = torch.zeros((n, cfg.window, ld), dtype=torch.float32, device=dev)
        self.emb = torch.zeros((n, ld), dtype=torch.float32, device=dev)
        self.mark = torch.zeros(n, dtype=i32, device=dev)
        self.chunk = min(n, 1 << 16)
        rows = max(self.chunk, 2 * cfg.batch_size)
        self.rows = torch.zeros((rows, ld), dtype=torch.float32, device=dev)
        self.work = torch.zeros(2 * cfg.batch_size + 8, dtype=i32, device=dev)
        self.preds = torch.zeros(cfg.batch_size, dtype=torch.float64, device=dev)
        self.snapshot = 0
        self.t_now = -math.inf
        self._stamp = 0
        self.last_affected: set = set()
        self._s = _lib.DySAT()
        self._fill()
        self._check(self._L.stgn_dysat_recompute_all(C.byref(self._s), self._stream()), "init")

    def _stream(self):
        return C.c_void_p(self._torch.cuda.current_stream(self.device).cuda_stream)

    def _check(self, rc, what):
        _lib.check(rc, "dysat_" + what)

    def _fill(self):
        c, s = self.cfg, self._s
        s.d_in, s.d, s.heads_s, s.heads_t = c.d_in, c.d, c.heads_s, c.heads_t
        s.window, s.fanout, s.ld = c.window, c.fanout, self.ld
        s.n, s.snapshot, s.pos_len, s.chunk = c.n, self.snapshot, c.max_snapshots, self.chunk
        s.max_batch = c.batch_size
        for name in ("P", "ss", "sn", "lst_nbr", "lst_head", "lst_cnt", "hist_k", "hist_v", "emb",
                     "mark", "work", "rows", "pos", "wq", "wk", "wv", "wo", "wpred"):
            setattr(s, name, getattr(self, name).data_ptr())
        s.bpred = float(self.params.b_pred)
        s.wtc = self.wtc.data_ptr() if self.wtc is not None else None
        # a batch's ~2B rows fill few 128-row tiles: below this the 16-row FFMA tiles win
        s.tc_min_rows = self.tc_min_rows

    # -- batches ----------------------------------------------------------------
    def _roll_to(self, k):
        """Advance to snapshot k (each boundary recomputes every node). Only the
        last W snapshots are ever read, so a gap longer than the window starts
        rolling at k - W (the skipped snapshots have empty lists either way)."""
        if k >= self.cfg.max_snapshots:
            raise ConfigError("snapshot index beyond max_snapshots")
        if k - self.snapshot > self.cfg.window:
            self.snapshot = k - self.cfg.window
        while self.snapshot < k:
            self.snapshot += 1
            if self.snapshot >= self.cfg.max_snapshots:
                raise ConfigError("snapshot index beyond max_snapshots")
            self._s.snapshot = self.snapshot
            self._check(self._L.stgn_dysat_roll(C.byref(self._s), self._stream()), "roll")

    def process_batch_arrays(self, src, dst, t) -> np.ndarray:
        from .edges import MonotonicityError
        torch = self._torch
        src = np.ascontiguousarray(src, dtype=np.int64)
        dst = np.ascontiguousarray(dst, dtype=np.int64)
        t = np.ascontiguousarray(t, dtype=np.float64)
        B = src.shape[0]
        if B == 0:
            self.last_affected = set()
            return np.zeros(0)
        if B > self.cfg.batch_size:
            raise ConfigError(f"batch of {B} edges > batch_size {self.cfg.batch_size}")
        if (src < 0).any() or (dst < 0).any() or (src >= self.cfg.n).any() or (dst >= self.cfg.n).any():
            raise ValueError("node ids must lie in [0, n)")
        prev = np.concatenate([[self.t_now], t[:-1]])
        if (t < prev).any():
            j = int(np.nonzero(t < prev)[0][0])
            raise MonotonicityError(f"batch edge at t={t[j]} precedes committed history t={prev[j]}")
        snap = np.floor(t / self.cfg.snapshot_len).astype(np.int64)
        out = np.zeros(B)
        aff: set = set()
        lo = 0
        while lo < B:
            k = int(snap[lo])
            hi = lo + int(np.searchsorted(snap[lo:], k, side="right"))
            self._roll_to(k)
            s32 = torch.from_numpy(src[lo:hi].astype(np.int32)).to(self.device)
            d32 = torch.from_numpy(dst[lo:hi].astype(np.int32)).to(self.device)
            self._stamp = self._stamp % 0x7FFFFFFF + 1
            na = C.c_int32()
            self._check(self._L.stgn_dysat_batch(C.byref(self._s), hi - lo, s32.data_ptr(),
                                                 d32.data_ptr(), self._stamp,
                                                 self.preds.data_ptr(), C.byref(na),
                                                 self._stream()), "batch")
            out[lo:hi] = self.preds[:hi - lo].cpu().numpy()
            aff = set(self.work[:na.value].cpu().tolist())
            lo = hi
        self.t_now = float(t[-1])
        self.last_affected = aff
        return out

    def process_batch_device(self, src32, dst32, t_last: float, snap: int):
        """Device-resident batch (bench): int32 ids on the device, all in one
        snapshot `snap`; no host synchronisation."""
        self._roll_to(snap)
        self._stamp = self._stamp % 0x7FFFFFFF + 1
        self._check(self._L.stgn_dysat_batch(C.byref(self._s), int(src32.shape[0]),
                                             src32.data_ptr(), dst32.data_ptr(), self._stamp,
                                             self.preds.data_ptr(), None, self._stream()),
                    "batch")
        self.t_now = t_last

    def full_recompute(self):
        """Every node's structural and temporal outputs at the current snapshot
        (the non-incremental baseline; values identical to the incremental state)."""
        self._check(self._L.stgn_dysat_recompute_all(C.byref(self._s), self._stream()),
                    "recompute_all")

    def embeddings(self) -> np.ndarray:
        return self.emb[:, :self.cfg.d].double().cpu().numpy()

    def neighbor_list(self, v: int) -> list:
        c = int(self.lst_cnt[v])
        h = int(self.lst_head[v])
        row = self.lst_nbr[v].cpu().tolist()
        return [row[(h + j) % self.cfg.fanout] for j in range(c)]
