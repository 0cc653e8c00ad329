"""Bounded-staleness harness on the B200 path (S/batcher.py:43-83,
S/oracle.py:112-125): the stream replayed strictly one edge at a time through
the full-recompute engine is the ground truth; the incremental engine at each
batch size is compared with it edge by edge.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .engine import IncrementalEngine
from .full_engine import OracleEngine
from .streaming import Batch


def batches_of(stream, batch_size: int):
    """S/batcher.py:43-48: arrival-order batches over an in-memory stream
    (EdgeArrays)."""
    for i in range(0, len(stream), batch_size):
        c = stream.slice(i, i + batch_size)
        yield Batch(c.src, c.dst, c.t, c.feat, float(c.t.max()), float(c.t.max() - c.t.min()))


def replay_sequential(stream, cfg, params):
    """S/oracle.py:112-125: per-edge predictions of the stream as batch-size-1
    batches of the full-recompute engine (a full snapshot after every edge when
    K > 1, whose payloads read the layer cache). Returns (preds, engine)."""
    import dataclasses
    eng = OracleEngine(dataclasses.replace(cfg, batch_size=1), params)
    snap = params.dims.layers > 1
    preds = []
    for i in range(len(stream)):
        p, _ = eng.apply_batch_arrays(stream.src[i:i + 1], stream.dst[i:i + 1],
                                      stream.t[i:i + 1], stream.feat[i:i + 1], snapshot=snap)
        preds.extend(np.asarray(p).tolist())
    return preds, eng


@dataclass
class StalenessReport:
    """S/batcher.py:51-55."""
    batch_size: int
    max_dev: float
    mean_dev: float


def compare_sequential_vs_batched(stream, batch_sizes, cfg, params, seq_preds=None):
    """S/batcher.py:57-83: (reports, slope of max deviation against batch
    size). `seq_preds` reuses an earlier replay_sequential result."""
    import dataclasses
    seq = np.asarray(seq_preds if seq_preds is not None else replay_sequential(stream, cfg, params)[0])
    reports = []
    for b in batch_sizes:
        eng = IncrementalEngine(dataclasses.replace(cfg, batch_size=b), params)
        preds = []
        for batch in batches_of(stream, b):
            preds.extend(eng.process_batch_arrays(batch.src, batch.dst, batch.t, batch.feat).tolist())
        dev = np.abs(np.asarray(preds) - seq)
        reports.append(StalenessReport(batch_size=b, max_dev=float(dev.max()) if dev.size else 0.0,
                                       mean_dev=float(dev.mean()) if dev.size else 0.0))
    if len(reports) >= 2:
        xs = np.array([r.batch_size for r in reports], dtype=np.float64)
        slope = float(np.polyfit(xs, np.array([r.max_dev for r in reports]), 1)[0])
    else:
        slope = 0.0
    return reports, slope
