"""Edge-stream formats and the deterministic synthetic generator.

  generate_stream  <- /root/reference/pkg/src/streamtgn/streamio.py:86-145
      Same RNG (numpy PCG64 default_rng) and the same draw sequence, so a
      given seed yields the reference's edges exactly (pinned by
      tests/golden/streams.npz, made by the reference itself).
  CSV format       <- streamio.py:15-79 ("# streamtgn-edges v1 d_e=<k>")

The generator returns struct-of-arrays (src, dst, t, feat) because the
engine ingests arrays; `as_edges` converts to the reference's
list[TemporalEdge] when a caller wants objects.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from .edges import TemporalEdge

HEADER_PREFIX = "# streamtgn-edges v1 d_e="
_EPOCH_TICKS = 50
_HOT_FRACTION = 0.1


class StreamParseError(ValueError):
    def __init__(self, line_no: int, message: str):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


@dataclass
class EdgeArrays:
    src: np.ndarray   # int64 (m,)
    dst: np.ndarray   # int64 (m,)
    t: np.ndarray     # float64 (m,)
    feat: np.ndarray  # float64 (m, d_e)

    def __len__(self) -> int:
        return int(self.src.shape[0])

    def slice(self, lo: int, hi: int) -> "EdgeArrays":
        return EdgeArrays(self.src[lo:hi], self.dst[lo:hi], self.t[lo:hi], self.feat[lo:hi])

    def as_edges(self) -> list[TemporalEdge]:
        return [TemporalEdge(int(s), int(d), float(t), f.copy())
                for s, d, t, f in zip(self.src, self.dst, self.t, self.feat)]

    @staticmethod
    def from_edges(edges, d_e: int) -> "EdgeArrays":
        from .edges import edges_to_arrays
        return EdgeArrays(*edges_to_arrays(edges, d_e))


def generate_stream(seed: int, n: int, m: int, attachment: str = "uniform",
                    burstiness: float = 1.0, d_e: int = 4,
                    native: bool | None = None) -> EdgeArrays:
    """Integer-tick synthetic stream; alternating cold/hot epochs of 50 ticks
    (hot epochs draw endpoints from the first 10% of ids when bursty), and
    degree-biased destinations under `preferential` (p = 0.8).

    native (default: when d_e == 0) runs the C generator of the in-tree
    library (csrc/gen.cpp), which replays numpy's PCG64 draws and yields the
    same edges as the loop below (tests/test_streamio_native.py); streams with
    edge features always use the loop (numpy's normal sampler is not
    restated natively)."""
    if native is None:
        native = d_e == 0
    if native and d_e != 0:
        raise ValueError("the native generator covers d_e = 0 streams only")
    if native:
        return _generate_native(seed, n, m, attachment, burstiness)
    if n < 2:
        raise ValueError("need at least 2 nodes")
    if m < 1:
        raise ValueError("need at least 1 edge")
    if attachment not in ("uniform", "preferential"):
        raise ValueError(f"unknown attachment {attachment!r}")
    if burstiness < 1.0:
        raise ValueError("burstiness must be >= 1")
    rng = np.random.default_rng(seed)
    rate_hi = 4.0 * burstiness / (burstiness + 1.0)
    rate_lo = 4.0 / (burstiness + 1.0)
    hot = max(2, int(n * _HOT_FRACTION))
    bursty = burstiness > 1.0
    pref = attachment == "preferential"

    src = np.empty(m, dtype=np.int64)
    dst = np.empty(m, dtype=np.int64)
    ts = np.empty(m, dtype=np.float64)
    feat = np.empty((m, d_e), dtype=np.float64)
    pool = np.empty(2 * m, dtype=np.int64)  # one slot per incident endpoint
    integers, uniform01, normal = rng.integers, rng.random, rng.standard_normal

    k = 0
    tick = 0
    carry = 0.0
    while k < m:
        is_hot = (tick // _EPOCH_TICKS) % 2 == 1
        carry += rate_hi if is_hot else rate_lo
        count = int(carry)
        carry -= count
        span = hot if (is_hot and bursty) else n
        for _ in range(count):
            if k >= m:
                break
            s = int(integers(0, span))
            if pref and k > 0 and uniform01() < 0.8:
                d = int(pool[int(integers(0, 2 * k))])
            else:
                d = int(integers(0, span))
            retry = 0
            while d == s and retry < 8:
                d = int(integers(0, span))
                retry += 1
            feat[k] = normal(d_e)
            src[k], dst[k], ts[k] = s, d, float(tick)
            pool[2 * k], pool[2 * k + 1] = s, d
            k += 1
        tick += 1
    return EdgeArrays(src, dst, ts, feat)


def _check_gen_args(n, m, attachment, burstiness):
    if n < 2:
        raise ValueError("need at least 2 nodes")
    if m < 1:
        raise ValueError("need at least 1 edge")
    if attachment not in ("uniform", "preferential"):
        raise ValueError(f"unknown attachment {attachment!r}")
    if burstiness < 1.0:
        raise ValueError("burstiness must be >= 1")


def _generate_native(seed, n, m, attachment, burstiness) -> EdgeArrays:
    import ctypes as C

    from . import _lib
    _check_gen_args(n, m, attachment, burstiness)
    st = np.random.default_rng(seed).bit_generator.state
    mask = (1 << 64) - 1
    s, inc = st["state"]["state"], st["state"]["inc"]
    rs = np.array([s >> 64, s & mask, inc >> 64, inc & mask, st["has_uint32"], st["uinteger"]],
                  dtype=np.uint64)
    src = np.empty(m, dtype=np.int64)
    dst = np.empty(m, dtype=np.int64)
    ts = np.empty(m, dtype=np.float64)
    vp = C.c_void_p
    rc = _lib.lib().stgn_generate_stream(vp(rs.ctypes.data), int(n), int(m),
                                         int(attachment == "preferential"), float(burstiness),
                                         vp(src.ctypes.data), vp(dst.ctypes.data),
                                         vp(ts.ctypes.data), None)
    _lib.check(rc, "stgn_generate_stream")
    return EdgeArrays(src, dst, ts, np.empty((m, 0), dtype=np.float64))


def _read_stream_native(path, sort):
    import ctypes as C

    from . import _lib
    try:
        L = _lib.lib()
    except OSError:
        return None
    m, d_e, bad = C.c_int64(), C.c_int64(), C.c_int64()
    bpath = os.fsencode(path)
    rc = L.stgn_read_stream(bpath, int(sort), 0, C.byref(m), C.byref(d_e), None, None, None, None,
                            C.byref(bad))
    if rc not in (_lib.STGN_OK, _lib.STGN_ERR_CAPACITY):
        return None
    n, k = int(m.value), int(d_e.value)
    src = np.empty(n, dtype=np.int64)
    dst = np.empty(n, dtype=np.int64)
    ts = np.empty(n, dtype=np.float64)
    feat = np.empty((n, k), dtype=np.float64)
    vp = C.c_void_p
    rc = L.stgn_read_stream(bpath, int(sort), n, C.byref(m), C.byref(d_e), vp(src.ctypes.data),
                            vp(dst.ctypes.data), vp(ts.ctypes.data),
                            vp(feat.ctypes.data) if k else None, C.byref(bad))
    if rc != _lib.STGN_OK:
        return None
    return EdgeArrays(src, dst, ts, feat), k


def serialize_stream(edges: EdgeArrays, d_e: int) -> str:
    lines = [f"{HEADER_PREFIX}{d_e}"]
    for s, d, t, f in zip(edges.src, edges.dst, edges.t, edges.feat):
        lines.append(",".join([str(int(s)), str(int(d)), repr(float(t))]
                              + [repr(float(x)) for x in f]))
    return "\n".join(lines) + "\n"


def write_stream(edges: EdgeArrays, d_e: int, path: str) -> None:
    with open(path, "w") as fh:
        fh.write(serialize_stream(edges, d_e))


def read_stream(path: str, sort: bool = False, native: bool = True) -> tuple[EdgeArrays, int]:
    """S/streamio.py:53-79. The native reader (csrc/gen.cpp) parses plain
    files; anything it declines (format errors, unusual spellings) is re-read
    by the Python parser below, so results and errors are the reference's."""
    if native:
        got = _read_stream_native(path, sort)
        if got is not None:
            return got
    with open(path) as fh:
        header = fh.readline().rstrip("\n")
        if not header.startswith(HEADER_PREFIX):
            raise StreamParseError(1, f"bad header {header!r}")
        try:
            d_e = int(header[len(HEADER_PREFIX):])
        except ValueError:
            raise StreamParseError(1, "d_e is not an integer") from None
        rows = []
        prev = -np.inf
        ordered = True
        for line_no, line in enumerate(fh, start=2):
            line = line.strip()
            if not line:
                continue
            parts = line.split(",")
            if len(parts) != 3 + d_e:
                raise StreamParseError(line_no, f"expected {3 + d_e} fields, got {len(parts)}")
            try:
                s, d, t = int(parts[0]), int(parts[1]), float(parts[2])
                f = [float(x) for x in parts[3:]]
            except ValueError as exc:
                raise StreamParseError(line_no, str(exc)) from None
            if s < 0 or d < 0:
                raise StreamParseError(line_no, "negative node id")
            if t < prev:
                if not sort:
                    raise StreamParseError(
                        line_no, f"timestamp {t} decreases (previous {prev}); use --sort")
                ordered = False
            prev = max(prev, t)
            rows.append((s, d, t, f))
    if sort and not ordered:
        rows.sort(key=lambda r: r[2])
    m = len(rows)
    out = EdgeArrays(np.array([r[0] for r in rows], dtype=np.int64),
                     np.array([r[1] for r in rows], dtype=np.int64),
                     np.array([r[2] for r in rows], dtype=np.float64),
                     np.array([r[3] for r in rows], dtype=np.float64).reshape(m, d_e))
    return out, d_e
