"""Full-recomputation engine on the B200 path: the reference's OracleEngine
(S/oracle.py:35-108), the TGL-style baseline the paper's incremental speed-ups
are quoted against ("index refresh").

Every batch: predictions from pre-batch memory for the batch endpoints over
the post-insertion neighbour lists, the memory update, then an exact
recompute of every node (the same recompute kernel as the incremental path,
over all node ids). Predictions equal IncrementalEngine's in exact mode (the
reference pins incremental == oracle bitwise, T/test_engine.py:262-273), so
the batch step reuses it and adds the O(n) refresh.

full_recompute(t_now) is pure, as the reference's (stgn_engine_snapshot: every
layer of every node into a fresh buffer). A t_now earlier than the newest edge
rebuilds each node's list from the append-only store (the L newest entries with
t <= t_now) and the engine's payload log of every entry's frozen stack, which
this engine keeps (edge_payloads=True). apply_batch_full refreshes the layer
cache like the reference's. A finite neighbour-cache window is refused: the
reference's oracle lists ignore it, the incremental batch path does not.
"""

from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass

import numpy as np

from .config import ConfigError, RunConfig
from .engine import IncrementalEngine
from .params import ModelParameters


@dataclass
class EngineSnapshot:
    """S/oracle.py:17-32."""
    embeddings: np.ndarray   # (n, d) final layer
    layers: np.ndarray       # (n, K, d)
    memory: np.ndarray       # (n, d_s)
    last_interaction: np.ndarray
    timestamp: float

    def dump(self) -> str:
        lines = [f"snapshot t={self.timestamp!r} n={self.embeddings.shape[0]}"]
        for v in range(self.embeddings.shape[0]):
            lines.append(f"node {v} " + " ".join(f"{x:.17g}" for x in self.embeddings[v]))
        return "\n".join(lines) + "\n"


class OracleEngine:
    """S/oracle.py:35: recomputes every node's embedding after each batch."""

    def __init__(self, cfg: RunConfig, params: ModelParameters, **kw):
        if math.isfinite(cfg.window):
            raise ConfigError("the full-recompute engine reads the store's top-L lists; "
                              "a finite neighbour-cache window is not supported")
        # drift-aware rebuilds are moot when every batch rebuilds everything
        kw.setdefault("edge_payloads", True)
        self._eng = IncrementalEngine(dataclasses.replace(cfg, rebuild="never"), params, **kw)
        self.cfg, self.params = cfg, params
        self.last_pred_embeddings: dict[int, np.ndarray] = {}

    # reference surface shared with the incremental engine
    @property
    def node_count(self) -> int:
        return self._eng.node_count

    @property
    def memory(self):
        return self._eng.memory

    @property
    def cache(self):
        return self._eng.cache

    @property
    def store(self):
        return self._eng.store

    @property
    def counters(self):
        return self._eng.counters

    @property
    def batch_index(self) -> int:
        return self._eng.batch_index

    def full_recompute(self, t_now: float | None = None) -> EngineSnapshot:
        """K-layer attention for every node; pure (S/oracle.py:47-65)."""
        return self._snapshot(t_now, self._eng.snapshot_layers(t_now))

    def _refresh(self) -> EngineSnapshot:
        """apply_batch_full's snapshot: the full recompute written to the layer cache."""
        self._eng.rebuild_nodes(None)
        return self._snapshot()

    def _snapshot(self, t_now=None, layers=None) -> EngineSnapshot:
        eng = self._eng
        n = eng.node_count
        if layers is None:
            layers = eng.cache.h[:n].copy()
        ts = t_now if t_now is not None else (eng.store.t_now if eng.store.m else 0.0)
        return EngineSnapshot(embeddings=layers[:, -1, :].copy(), layers=layers,
                              memory=eng.memory.states[:n].copy(),
                              last_interaction=eng.memory.last_interaction[:n].copy(),
                              timestamp=float(ts))

    def apply_batch_full(self, batch, snapshot: bool = True):
        """S/oracle.py:67-96: (predictions, snapshot) for one batch."""
        preds = self._eng.process_batch(batch)
        self.last_pred_embeddings = dict(self._eng.last_pred_embeddings)
        if not batch:
            return [], self._snapshot()
        if not snapshot:
            return preds, self._snapshot()
        return preds, self._refresh()

    def apply_batch_arrays(self, src, dst, t, feat=None, snapshot: bool = True):
        """Array form of apply_batch_full (no TemporalEdge objects)."""
        preds = self._eng.process_batch_arrays(src, dst, t, feat)
        self.last_pred_embeddings = dict(self._eng.last_pred_embeddings)
        if not snapshot or len(preds) == 0:
            return preds, self._snapshot()
        return preds, self._refresh()
