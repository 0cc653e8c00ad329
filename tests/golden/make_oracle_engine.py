"""Fixture of the reference's full-recompute OracleEngine (S/oracle.py:35-108)
on the stream/params of an existing engine fixture (run in the build
container, where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_oracle_engine.py

Writes oracle_engine_<case>.npz: per-batch predictions of apply_batch_full
and the final snapshot (layers, memory, last_interaction, timestamp).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

from make_golden import ENGINE_CASES, random_params  # noqa: E402
from streamtgn.config import Dims, RunConfig  # noqa: E402
from streamtgn.graph_store import TemporalEdge  # noqa: E402
from streamtgn.oracle import OracleEngine  # noqa: E402
from streamtgn.params import init_params  # noqa: E402
from streamtgn.streamio import generate_stream  # noqa: E402


def main(cases=("k2_last_adaptive", "k1_fixed_de0")):
    for name, dkw, ckw, pseed, rnd, skw, B in ENGINE_CASES:
        if name not in cases:
            continue
        dims = Dims(**dkw)
        cfg = RunConfig(dims=dims, batch_size=B, **ckw)
        params = random_params(pseed, dims) if rnd else init_params(pseed, dims)
        stream = generate_stream(**skw)
        eng = OracleEngine(cfg, params)
        preds = []
        snap = None
        for i in range(0, len(stream), B):
            p, snap = eng.apply_batch_full(stream[i:i + B])
            preds.extend(p)
        # pure historical snapshots (full_recompute(t_now), S/oracle.py:40-65) at a
        # few times inside the stream, plus the current-state one
        ts = np.array([e.t for e in stream])
        t_hist = np.array([ts[len(ts) // 7], ts[len(ts) // 2], ts[-B - 1], ts[-1] + 1.0])
        hist = [eng.full_recompute(float(t)).layers for t in t_hist]
        np.savez_compressed(os.path.join(HERE, f"oracle_engine_{name}.npz"),
                            preds=np.array(preds), layers=snap.layers, memory=snap.memory,
                            last=snap.last_interaction, timestamp=np.array([snap.timestamp]),
                            t_hist=t_hist, hist_layers=np.stack(hist))
        print(name, len(preds), snap.layers.shape)


if __name__ == "__main__":
    main()
