"""Native stream generator (csrc/gen.cpp, stgn_generate_stream) against the
reference generator S/streamio.py:86-145: digests the reference produced at
the C3/C4 shape (tests/golden/stream_digests.json) and edge-for-edge
equality with the Python loop on mixed cases. CPU only (host code)."""

import json
import os

import numpy as np
import pytest

from paper_2603_21090_b200.streamio import generate_stream

HERE = os.path.dirname(os.path.abspath(__file__))


def _digest(s):
    import hashlib
    a = np.stack([s.src, s.dst, s.t.view(np.int64)])
    return hashlib.sha256(a.tobytes()).hexdigest()


@pytest.mark.parametrize("case", json.load(open(os.path.join(HERE, "golden", "stream_digests.json"))),
                         ids=lambda c: f"seed{c['kw']['seed']}_n{c['kw']['n']}")
def test_native_matches_reference_digest(case):
    s = generate_stream(**case["kw"], native=True)
    assert _digest(s) == case["sha256"]


@pytest.mark.parametrize("kw", [
    dict(seed=0, n=2, m=3000, attachment="preferential"),          # constant retries
    dict(seed=11, n=3, m=5000, attachment="uniform", burstiness=4.0),
    dict(seed=3, n=50_000, m=30_000, attachment="preferential", burstiness=1.5),
    dict(seed=9, n=(1 << 33) + 7, m=4000, attachment="uniform"),  # 64-bit Lemire branch
    dict(seed=1, n=1, m=1, attachment="uniform"),
])
def test_native_equals_python_loop(kw):
    if kw["n"] < 2:
        with pytest.raises(ValueError):
            generate_stream(**kw, d_e=0, native=True)
        return
    a = generate_stream(**kw, d_e=0, native=True)
    b = generate_stream(**kw, d_e=0, native=False)
    np.testing.assert_array_equal(a.src, b.src)
    np.testing.assert_array_equal(a.dst, b.dst)
    np.testing.assert_array_equal(a.t, b.t)
    assert a.feat.shape == b.feat.shape == (kw["m"], 0)


def test_native_rejects_features():
    with pytest.raises(ValueError):
        generate_stream(0, 10, 10, d_e=3, native=True)
