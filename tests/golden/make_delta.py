"""Write delta-mode engine fixtures by running the REFERENCE itself with
RunConfig(mode="delta") (S/engine.py:276-353). Same record layout as
make_golden.py's engine_<name>.npz, plus the delta-mode counters
embed_skip / attn_hit / attn_miss; saved as delta_<name>.npz.

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_delta.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg  # noqa: E402  (puts the reference on sys.path)
from streamtgn.graph_store import TemporalEdge  # noqa: E402

SMALL = dict(d_s=6, d_e=3, d_t=6, d_m=5, d_k=4, heads=2)


def tied_stream():
    """The reference's test_delta_hits_with_tied_timestamps stream
    (T/test_engine.py:332-345): 4 edges per integer tick on 12 nodes."""
    rng = np.random.default_rng(0)
    out = []
    for tick in range(30):
        for _ in range(4):
            u, v = rng.integers(0, 12, size=2)
            out.append(TemporalEdge(int(u), int(v), float(tick), rng.standard_normal(3)))
    return out


DELTA_CASES = [
    # (name, dims kwargs, cfg kwargs, params seed, random biases, stream, batch size)
    ("tied_k1", dict(SMALL, layers=1), dict(fanout=6, nodes=12), 4, True, "tied", 4),
    ("near_oracle_k1", dict(SMALL, layers=1), dict(fanout=6, nodes=12), 4, True,
     dict(seed=17, n=12, m=160, d_e=3), 4),
    ("skip_k1", dict(SMALL, layers=1), dict(fanout=4, nodes=10), 5, True,
     dict(seed=19, n=10, m=120, d_e=3), 2),
    ("k2_fallback", dict(SMALL, layers=2), dict(fanout=4, nodes=15), 6, True,
     dict(seed=23, n=15, m=120, d_e=3), 4),
    ("k1_window_adaptive", dict(SMALL, layers=1),
     dict(fanout=5, nodes=80, window=4.0, rebuild="adaptive", gamma=0.9, delta_max=0.5,
          alpha=0.1), 8, True,
     dict(seed=31, n=80, m=1200, attachment="preferential", burstiness=2.0, d_e=3), 12),
    ("k1_fixed_de0", dict(d_s=8, d_e=0, d_t=8, d_m=8, d_k=4, heads=2, layers=1),
     dict(fanout=10, nodes=0, rebuild="fixed", rebuild_interval=7), 11, False,
     dict(seed=12, n=200, m=1500, attachment="preferential", d_e=0), 20),
]


def main():
    mg.COUNTER_KEYS = mg.COUNTER_KEYS + ("embed_skip", "attn_hit", "attn_miss")
    orig = mg.handmade_stream
    for name, dkw, ckw, pseed, rb, skw, B in DELTA_CASES:
        if skw == "tied":
            mg.handmade_stream = lambda d_e: tied_stream()
            skw_use = "handmade"
        else:
            mg.handmade_stream = orig
            skw_use = skw
        mg.run_engine_case("delta_" + name, dkw, dict(ckw, mode="delta"), pseed, rb, skw_use, B)
        src = os.path.join(HERE, f"engine_delta_{name}.npz")
        z = dict(np.load(src))
        os.remove(src)
        np.savez_compressed(os.path.join(HERE, f"delta_{name}.npz"), **z)
        c = z["counters"].sum(axis=0)
        keys = list(z["counter_keys"])
        print(f"  delta_{name}: " + ", ".join(f"{k}={int(c[keys.index(k)])}"
                                              for k in ("embed_skip", "attn_hit", "attn_miss")))


if __name__ == "__main__":
    main()
