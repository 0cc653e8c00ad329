"""Ingestion and asynchronous batched streaming.

  EdgeRing        <- EdgeQueue (S/graph_store.py:45-92): fixed-capacity FIFO
                     with reject-on-full backpressure and the time-window
                     flush filter, stored struct-of-arrays in pinned host
                     memory so a formed batch is copied to the GPU without an
                     intermediate buffer.
  form_batch      <- S/batcher.py:33-40: t_batch = newest member, s_max = the
                     staleness gap to the oldest.
  StreamingEngine    the north star's "relaxed-order batched streaming on CUDA
                     streams": batch i+1's host-to-device copy (copy stream)
                     and batch i-1's score read-back overlap batch i's graph on
                     the engine stream. Results come back in submission order;
                     the engine state evolves exactly as with process_batch
                     (same batches, same order), only the host waits less.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .edges import FeatureDimError, MonotonicityError


def _host_array(shape, dtype, pinned):
    if pinned:
        import torch
        tdt = {np.int32: torch.int32, np.float64: torch.float64, np.float32: torch.float32}[dtype]
        return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
    return np.empty(shape, dtype=dtype)


class EdgeRing:
    """Fixed-capacity FIFO of edges, struct of arrays (pinned when a GPU is
    present). Semantics of the reference EdgeQueue: enqueue returns False and
    leaves the ring unchanged when full; a feature-length mismatch raises."""

    def __init__(self, capacity: int, d_e: int, pinned: bool | None = None):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        if pinned is None:
            try:
                import torch
                pinned = torch.cuda.is_available()
            except ImportError:
                pinned = False
        self.capacity, self.d_e = int(capacity), int(d_e)
        self.src = _host_array(capacity, np.int32, pinned)
        self.dst = _host_array(capacity, np.int32, pinned)
        self.t = _host_array(capacity, np.float64, pinned)
        self.feat = _host_array((capacity, max(d_e, 1)), np.float32, pinned)
        self._head = 0
        self._size = 0

    def __len__(self) -> int:
        return self._size

    @property
    def occupancy(self) -> int:
        return self._size

    def enqueue(self, edge) -> bool:
        """One TemporalEdge (S/graph_store.py:60-71)."""
        feat = np.asarray(edge.feat, dtype=np.float64).reshape(-1)
        if feat.shape[0] != self.d_e:
            raise FeatureDimError(f"edge feature has length {feat.shape[0]}, expected {self.d_e}")
        if self._size == self.capacity:
            return False
        i = (self._head + self._size) % self.capacity
        self.src[i], self.dst[i], self.t[i] = edge.src, edge.dst, edge.t
        if self.d_e:
            self.feat[i, :self.d_e] = feat
        self._size += 1
        return True

    def enqueue_arrays(self, src, dst, t, feat=None) -> int:
        """Vectorised enqueue; returns how many edges were accepted (a prefix)."""
        src, dst, t = np.asarray(src), np.asarray(dst), np.asarray(t)
        if feat is None and self.d_e:
            raise FeatureDimError(f"edge features missing, expected width {self.d_e}")
        if feat is not None and self.d_e and np.asarray(feat).shape[-1] != self.d_e:
            raise FeatureDimError(f"edge features have width {np.asarray(feat).shape[-1]}, "
                                  f"expected {self.d_e}")
        n = min(int(src.shape[0]), self.capacity - self._size)
        p = (self._head + self._size) % self.capacity
        first = min(n, self.capacity - p)
        for (lo, hi), (a, b) in (((p, p + first), (0, first)), ((0, n - first), (first, n))):
            if hi <= lo:
                continue
            self.src[lo:hi], self.dst[lo:hi], self.t[lo:hi] = src[a:b], dst[a:b], t[a:b]
            if self.d_e and feat is not None:
                self.feat[lo:hi, :self.d_e] = np.asarray(feat)[a:b]
        self._size += n
        return n

    def flush_batch(self, max_count: int, before: float | None = None):
        """Remove and return up to max_count oldest edges (S/graph_store.py:73-92)
        as contiguous arrays (src, dst, t, feat); `before` stops at the first
        edge with t >= before so FIFO order is kept."""
        n = max(0, min(int(max_count), self._size))
        if before is not None and n:
            idx = (self._head + np.arange(n)) % self.capacity
            late = np.nonzero(self.t[idx] >= before)[0]
            if late.size:
                n = int(late[0])
        idx = (self._head + np.arange(n)) % self.capacity
        out = (self.src[idx], self.dst[idx], self.t[idx], self.feat[idx, :self.d_e])
        self._head = (self._head + n) % self.capacity
        self._size -= n
        return out


@dataclass
class Batch:
    """S/batcher.py:17-30 (array form)."""
    src: np.ndarray
    dst: np.ndarray
    t: np.ndarray
    feat: np.ndarray
    t_batch: float
    s_max: float

    def __len__(self) -> int:
        return int(self.src.shape[0])


def form_batch(ring: EdgeRing, batch_size: int) -> Batch | None:
    """S/batcher.py:33-40: flush up to batch_size edges; None when empty."""
    src, dst, t, feat = ring.flush_batch(batch_size)
    if src.shape[0] == 0:
        return None
    return Batch(src, dst, t, feat, float(t.max()), float(t.max() - t.min()))


class StreamingEngine:
    """Pipelined driver of an IncrementalEngine.

    submit(src, dst, t[, feat]) validates a batch on the host (ids >= 0,
    non-decreasing times, no earlier than anything submitted before), copies
    it from pinned host memory into one of `depth` device slots on an upload
    stream (after the graph that last read that slot), enqueues the batch
    graph on the engine's stream behind the upload, and reads the scores back
    into pinned memory on a download stream. Nothing blocks unless `depth`
    batches are in flight. results() / drain() return (batch number, scores)
    in submission order.
    """

    def __init__(self, engine, depth: int = 3, max_batch: int | None = None):
        import torch
        self.eng, self.torch = engine, torch
        self.depth = max(2, int(depth))
        B = int(max_batch or engine.cfg.batch_size)
        dev, d_e = engine.device, engine.dims.d_e
        self.B, self.d_e = B, d_e
        self.up = torch.cuda.Stream(device=dev)
        self.down = torch.cuda.Stream(device=dev)

        def host(*shape, dt):
            return torch.empty(*shape, dtype=dt, pin_memory=True)

        def devb(*shape, dt):
            return torch.empty(*shape, dtype=dt, device=dev)

        self._h = [dict(src=host(B, dt=torch.int32), dst=host(B, dt=torch.int32),
                        t=host(B, dt=torch.float64), feat=host(B, max(d_e, 1), dt=torch.float32),
                        preds=host(B, dt=torch.float64)) for _ in range(self.depth)]
        self._d = [dict(src=devb(B, dt=torch.int32), dst=devb(B, dt=torch.int32),
                        t=devb(B, dt=torch.float64), feat=devb(B, max(d_e, 1), dt=torch.float32))
                   for _ in range(self.depth)]
        # per-slot copy of the batch's result block (counters): device copy on the engine
        # stream right behind the batch, read back with the scores
        nres = int(engine._L.stgn_batch_result_bytes())
        self._res_d = [devb(nres, dt=torch.uint8) for _ in range(self.depth)]
        self._res_h = [host(nres, dt=torch.uint8) for _ in range(self.depth)]
        self._meta = [None] * self.depth     # (edges, t_last, batch index) of the slot's batch
        self._used = [None] * self.depth   # event on the engine stream: slot's graph enqueued
        self._done = [None] * self.depth   # event on the download stream: scores in pinned memory
        self._pending = []                 # (batch number, slot, n), submission order
        self._ready = []
        self._t_last = -np.inf
        self.submitted = 0

    def submit(self, src, dst, t, feat=None) -> int:
        torch, eng = self.torch, self.eng
        src, dst = np.asarray(src), np.asarray(dst)
        t = np.asarray(t, dtype=np.float64)
        n = int(src.shape[0])
        if n == 0:
            return -1
        if n > self.B:
            raise ValueError(f"batch of {n} edges exceeds the streaming slot size {self.B}")
        if (src < 0).any() or (dst < 0).any():
            raise ValueError("node ids must be non-negative")
        t_floor = max(self._t_last, eng._t_now)
        if t[0] < t_floor or (n > 1 and (np.diff(t) < 0).any()):
            raise MonotonicityError(f"batch edge precedes committed history t={t_floor}")
        k = self.submitted % self.depth
        if self._done[k] is not None:      # the slot's previous batch must be read back first
            self._collect(until_slot=k)
        h, d = self._h[k], self._d[k]
        h["src"][:n] = torch.from_numpy(src.astype(np.int32, copy=False))
        h["dst"][:n] = torch.from_numpy(dst.astype(np.int32, copy=False))
        h["t"][:n] = torch.from_numpy(t)
        has_feat = bool(self.d_e) and feat is not None
        if has_feat:
            h["feat"][:n, :self.d_e] = torch.from_numpy(np.asarray(feat, dtype=np.float32))
        main = torch.cuda.current_stream(eng.device)
        if self._used[k] is not None:
            self.up.wait_event(self._used[k])
        with torch.cuda.stream(self.up):
            for key in ("src", "dst", "t"):
                d[key][:n].copy_(h[key][:n], non_blocking=True)
            if has_feat:
                d["feat"][:n].copy_(h["feat"][:n], non_blocking=True)
            uploaded = torch.cuda.Event()
            uploaded.record(self.up)
        main.wait_event(uploaded)
        preds = eng.process_batch_device(
            d["src"][:n], d["dst"][:n], d["t"][:n], d["feat"][:n, :self.d_e] if has_feat else None,
            max_id=int(max(src.max(), dst.max())), t_first=float(t[0]), t_last=float(t[-1]))
        import ctypes as C
        from . import _lib
        _lib.check(eng._L.stgn_engine_result_copy(
            eng._handle, C.c_void_p(self._res_d[k].data_ptr()), 1,
            C.c_void_p(main.cuda_stream)), "result_copy")
        self._meta[k] = (n, float(t[-1]), eng.batch_index)
        used = torch.cuda.Event()
        used.record(main)
        self._used[k] = used
        self.down.wait_event(used)
        with torch.cuda.stream(self.down):
            h["preds"][:n].copy_(preds, non_blocking=True)
            self._res_h[k].copy_(self._res_d[k], non_blocking=True)
            done = torch.cuda.Event()
            done.record(self.down)
        preds.record_stream(self.down)
        self._done[k] = done
        self._t_last = float(t[-1])
        self._pending.append((self.submitted, k, n))
        self.submitted += 1
        return self.submitted - 1

    def _pop(self):
        import ctypes as C
        from . import _lib
        num, slot, n = self._pending.pop(0)
        self._done[slot].synchronize()
        self._ready.append((num, self._h[slot]["preds"][:n].numpy().copy()))
        self._done[slot] = None
        # the batch's counters and report (S/runner.py:73-77), in submission order
        eng = self.eng
        rep = _lib.Report()
        _lib.check(eng._L.stgn_report_from_result(C.c_void_p(self._res_h[slot].data_ptr()),
                                                  C.byref(rep)), "report")
        edges, t_last, index = self._meta[slot]
        eng.counters.start_batch()
        eng._account(rep, edges, t_last, index)
        if num != self.submitted - 1:  # the device-side lists belong to a later batch
            eng._last_nD = eng._last_nA = None
        return slot

    def _collect(self, until_slot):
        while self._pending:
            if self._pop() == until_slot:
                return

    def results(self):
        """Scores of every batch whose read-back has completed (non-blocking)."""
        while self._pending and self._done[self._pending[0][1]].query():
            self._pop()
        out, self._ready = self._ready, []
        return out

    def drain(self):
        """Block until every submitted batch is done; return the remaining scores."""
        while self._pending:
            self._pop()
        out, self._ready = self._ready, []
        return out
