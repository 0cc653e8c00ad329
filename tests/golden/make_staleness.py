"""Fixture of the reference's bounded-staleness harness (S/batcher.py:57-83,
S/oracle.py:112-125): strict B=1 sequential replay vs the incremental engine
at several batch sizes (run in the build container):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_staleness.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

from make_golden import random_params  # noqa: E402
from streamtgn.batcher import batches_of, compare_sequential_vs_batched  # noqa: E402
from streamtgn.config import Dims, RunConfig  # noqa: E402
from streamtgn.engine import IncrementalEngine  # noqa: E402
from streamtgn.oracle import replay_sequential  # noqa: E402
from streamtgn.streamio import generate_stream  # noqa: E402

CASES = {"k1": (Dims(d_s=6, d_e=3, d_t=6, d_m=5, d_k=4, heads=2, layers=1), 3),
         "k2": (Dims(d_s=6, d_e=3, d_t=6, d_m=5, d_k=4, heads=2, layers=2), 5)}
BATCH_SIZES = [1, 4, 16, 50]


def main():
    for name, (dims, seed) in CASES.items():
        cfg = RunConfig(dims=dims, batch_size=8, fanout=4, nodes=30)
        params = random_params(seed, dims)
        stream = generate_stream(seed=seed, n=30, m=200, attachment="preferential", d_e=3)
        seq, _ = replay_sequential(stream, cfg, params)
        out = {"seq": np.array(seq), "batch_sizes": np.array(BATCH_SIZES)}
        for b in BATCH_SIZES:
            eng = IncrementalEngine(cfg.with_(batch_size=b), params)
            preds = []
            for batch in batches_of(stream, b):
                preds.extend(eng.process_batch(batch.edges))
            out[f"b{b}"] = np.array(preds)
        reports, slope = compare_sequential_vs_batched(stream, BATCH_SIZES, cfg, params)
        out["max_dev"] = np.array([r.max_dev for r in reports])
        out["mean_dev"] = np.array([r.mean_dev for r in reports])
        out["slope"] = np.array([slope])
        np.savez_compressed(os.path.join(HERE, f"staleness_{name}.npz"), **out)
        print(name, out["max_dev"], slope)


if __name__ == "__main__":
    main()
