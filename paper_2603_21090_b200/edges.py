"""Boundary types for edges and adjacency entries, plus the error classes
the reference raises on this path.

  TemporalEdge, NeighborEntry  <- /root/reference/pkg/src/streamtgn/graph_store.py:24-42
  MonotonicityError, FeatureDimError <- graph_store.py:16-21
  InputError        <- engine_base.py:30
  KernelInputError  <- kernels/reference.py:17
  DriftContractError <- drift.py:9
  PendingEdge       <- engine_base.py:50-58
  ChangeRecord      <- state.py:131-140
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np


class FeatureDimError(ValueError):
    """Edge feature vector does not match the configured d_e."""


class MonotonicityError(ValueError):
    """Edge timestamp is older than an already-inserted one."""


class InputError(ValueError):
    """Out-of-range ids or malformed arrays at the engine boundary."""


class KernelInputError(ValueError):
    """Operator-level shape / contract violation."""


class DriftContractError(ValueError):
    """Drift scheduler misuse (|N_v| <= 0, execute without a decision)."""


@dataclass(frozen=True)
class TemporalEdge:
    src: int
    dst: int
    t: float
    feat: np.ndarray

    def __post_init__(self):
        if self.src < 0 or self.dst < 0:
            raise ValueError("node ids must be non-negative")


class NeighborEntry(NamedTuple):
    """One adjacency entry seen from a node: other endpoint, time, edge id."""

    nbr: int
    t: float
    edge_id: int


@dataclass
class PendingEdge:
    """A staged batch edge (S/engine_base.py:50-58): its id, endpoints, time,
    features and the (K, d) pre-batch stacks frozen for both endpoints."""

    edge_id: int
    src: int
    dst: int
    t: float
    feat: np.ndarray
    stack_src: np.ndarray
    stack_dst: np.ndarray


@dataclass
class ChangeRecord:
    """Per-node neighbourhood delta of one update (S/state.py:131-140)."""

    added: list = field(default_factory=list)
    expired: list = field(default_factory=list)
    updated: set = field(default_factory=set)

    @property
    def size(self) -> int:
        return len(self.added) + len(self.expired) + len(self.updated)

    @property
    def empty(self) -> bool:
        return self.size == 0


def edges_to_arrays(batch, d_e: int):
    """list[TemporalEdge] -> (src int64, dst int64, t float64, feat (B, d_e) float64).

    Raises FeatureDimError on a feature-length mismatch (the reference
    raises it on insertion, graph_store.py:128-130)."""
    B = len(batch)
    src = np.fromiter((e.src for e in batch), dtype=np.int64, count=B)
    dst = np.fromiter((e.dst for e in batch), dtype=np.int64, count=B)
    t = np.fromiter((e.t for e in batch), dtype=np.float64, count=B)
    feat = np.zeros((B, d_e), dtype=np.float64)
    for i, e in enumerate(batch):
        f = np.asarray(e.feat, dtype=np.float64)
        if f.shape != (d_e,):
            raise FeatureDimError(
                f"edge feature has length {f.size}, expected {d_e}")
        feat[i] = f
    return src, dst, t, feat
