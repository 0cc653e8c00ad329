"""Helpers to rebuild configs/params/streams from the golden fixtures."""

from __future__ import annotations

import glob
import os

import numpy as np

from paper_2603_21090_b200.config import Dims, RunConfig
from paper_2603_21090_b200.params import ModelParameters
from paper_2603_21090_b200.streamio import EdgeArrays

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
DIM_KEYS = ("d_s", "d_e", "d_t", "d_x", "d_m", "d_k", "heads", "layers")


def engine_cases():
    return sorted(os.path.basename(p)[len("engine_"):-4]
                  for p in glob.glob(os.path.join(GOLDEN, "engine_*.npz")))


def delta_cases():
    return sorted(os.path.basename(p)[len("delta_"):-4]
                  for p in glob.glob(os.path.join(GOLDEN, "delta_*.npz")))


def pipeline_cases():
    return sorted(os.path.basename(p)[len("pipeline_"):-4]
                  for p in glob.glob(os.path.join(GOLDEN, "pipeline_*.npz")))


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))


def case_setup(z):
    dims = Dims(**{k: int(v) for k, v in zip(DIM_KEYS, z["dims"])})
    cfg = RunConfig(dims=dims, batch_size=int(z["batch_size"]), fanout=int(z["fanout"]),
                    nodes=int(z["nodes"]), aggregator=str(z["aggregator"]),
                    rebuild=str(z["rebuild"]), rebuild_interval=int(z["rebuild_interval"]),
                    gamma=float(z["gamma"]), delta_max=float(z["delta_max"]),
                    alpha=float(z["alpha"]), window=float(z["window"]))
    tensors = {k[len("param_"):]: v for k, v in z.items() if k.startswith("param_")}
    b_pred = float(tensors.pop("b_pred")[0])
    params = ModelParameters(dims=dims, b_pred=b_pred, **tensors)
    stream = EdgeArrays(z["src"], z["dst"], z["t"], z["feat"].reshape(len(z["src"]), dims.d_e))
    return cfg, params, stream


def batches(stream: EdgeArrays, B: int):
    for lo in range(0, len(stream), B):
        yield stream.slice(lo, min(lo + B, len(stream)))


def random_params(seed, dims):
    """init_params with random biases, as the reference's tests/conftest.py:18-26
    and tests/golden/make_golden.py:random_params (same draw order)."""
    from paper_2603_21090_b200.params import init_params
    p = init_params(seed, dims)
    rng = np.random.default_rng(seed + 1)
    for name, t in p.tensors().items():
        if name.startswith("b_") and name != "b_pred":
            t[...] = rng.standard_normal(t.shape)
    p.b_pred = float(rng.standard_normal())
    return p
