"""Digest fixtures of the reference generator at scale (run in the build
container, where /root/reference exists):

    python tests/golden/make_stream_digests.py

Writes stream_digests.json: sha256 over int64 [src; dst; bits(t)] of
streamtgn.streamio.generate_stream (S/streamio.py:86-145) for d_e = 0
streams, including the first 100K edges of the C3/C4 shape (n = 2.6M,
seed 2). tests/test_streamio_native.py checks the native generator
(csrc/gen.cpp) against them.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from streamtgn.streamio import generate_stream  # noqa: E402

CASES = [dict(seed=2, n=2_600_000, m=100_000, attachment="preferential", d_e=0),
         dict(seed=7, n=300, m=20_000, attachment="preferential", burstiness=3.0, d_e=0),
         dict(seed=5, n=1000, m=20_000, attachment="uniform", burstiness=2.0, d_e=0)]


def digest(src, dst, t):
    a = np.stack([np.asarray(src, dtype=np.int64), np.asarray(dst, dtype=np.int64),
                  np.asarray(t, dtype=np.float64).view(np.int64)])
    return hashlib.sha256(a.tobytes()).hexdigest()


def main():
    out = []
    for kw in CASES:
        s = generate_stream(**kw)
        out.append(dict(kw=kw, sha256=digest([e.src for e in s], [e.dst for e in s],
                                             [e.t for e in s])))
    with open(os.path.join(HERE, "stream_digests.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("stream_digests.json written")


if __name__ == "__main__":
    main()
