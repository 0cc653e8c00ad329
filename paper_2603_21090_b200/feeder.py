"""Device-resident edge streams: upload a whole stream (or a window of it) to
HBM once and feed it to the engine batch by batch with no host round trip
per batch (each batch is one CUDA-graph replay on the engine stream; the
host only enqueues). This is the fast-forward used to bring the engine to
the C3/C4 state (30M edges) and the replay harness of the benchmarks.

The per-batch facts process_batch_device needs from the host (largest id,
first/last timestamp) are computed once, vectorised, here; the stream's
validity (non-negative ids, non-decreasing times) is checked once for the
whole window, so the per-batch checks of process_batch_arrays
(S/engine.py:408-413) hold for every batch fed from it.
"""

from __future__ import annotations

import numpy as np

from .edges import MonotonicityError


class DeviceStream:
    def __init__(self, eng, edges, batch: int, lo: int = 0, hi: int | None = None):
        torch = eng._torch
        hi = len(edges) if hi is None else min(hi, len(edges))
        if batch < 1:
            raise ValueError("batch must be >= 1")
        self.eng, self.B, self.lo, self.hi = eng, int(batch), int(lo), int(hi)
        src = np.asarray(edges.src[lo:hi])
        dst = np.asarray(edges.dst[lo:hi])
        t = np.ascontiguousarray(edges.t[lo:hi], dtype=np.float64)
        if src.size and (src.min() < 0 or dst.min() < 0):
            raise ValueError("node ids must be non-negative")
        if t.size > 1 and (np.diff(t) < 0).any():
            raise MonotonicityError("stream timestamps decrease")
        dev = eng.device
        self.src = torch.from_numpy(src.astype(np.int32)).to(dev)
        self.dst = torch.from_numpy(dst.astype(np.int32)).to(dev)
        self.t = torch.from_numpy(t).to(dev)
        d_e = eng.dims.d_e
        self.feat = (torch.from_numpy(np.ascontiguousarray(edges.feat[lo:hi], dtype=np.float32)).to(dev)
                     if d_e else None)
        starts = np.arange(0, hi - lo, self.B)
        mx = np.maximum(src, dst)
        self.max_id = np.maximum.reduceat(mx, starts) if starts.size else np.zeros(0, np.int64)
        self.t_first = t[starts] if starts.size else np.zeros(0)
        ends = np.minimum(starts + self.B, hi - lo) - 1
        self.t_last = t[ends] if starts.size else np.zeros(0)
        self.n_batches = int(starts.size)

    def batch(self, k: int, report: bool = False):
        """Feed batch k of the window; returns the device score tensor."""
        a = k * self.B
        b = min(a + self.B, self.hi - self.lo)
        f = self.feat[a:b] if self.feat is not None else None
        return self.eng.process_batch_device(
            self.src[a:b], self.dst[a:b], self.t[a:b], f, max_id=int(self.max_id[k]),
            t_first=float(self.t_first[k]), t_last=float(self.t_last[k]), report=report)

    def run(self, k0: int = 0, k1: int | None = None, report_last: bool = True):
        """Feed batches k0..k1-1 back to back; only the last one reports."""
        k1 = self.n_batches if k1 is None else min(k1, self.n_batches)
        out = None
        for k in range(k0, k1):
            out = self.batch(k, report=report_last and k == k1 - 1)
        return out
