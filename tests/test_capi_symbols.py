"""CPU-side checks of the boundary: the library loads without a GPU, exports
every symbol include/stgn.h declares, and the ctypes structures match the
header's layouts."""

import ctypes as C
import os
import re

import pytest

from paper_2603_21090_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header():
    with open(os.path.join(ROOT, "include", "stgn.h")) as fh:
        return fh.read()


def test_header_declares_exactly_the_bound_symbols():
    declared = set(re.findall(r"\b(stgn_[a-z0-9_]+)\s*\(", _header()))
    assert declared == set(_lib.EXPORTS)


def test_library_loads_and_exports():
    L = _lib.lib()
    for name in _lib.EXPORTS:
        assert hasattr(L, name), name
    assert b"sm_100a" in L.stgn_version()


def test_scratch_sizing_and_validation():
    from paper_2603_21090_b200.config import Dims
    L = _lib.lib()
    d = _lib.dims_struct(Dims(d_s=100, d_e=0, d_t=100, d_m=100, d_k=50, heads=2, layers=2))
    cfg = _lib.Config(10, 1, 0, 0, 0.9, 0.5, 0.1, float("inf"), 0, 600)
    assert L.stgn_scratch_bytes(C.byref(d), C.byref(cfg), 2_600_000) > 2_600_000 * 4
    bad = _lib.dims_struct(Dims(d_s=100, d_e=0, d_t=100, d_m=100, d_k=50, heads=2, layers=2))
    bad.d_t = 7
    assert L.stgn_scratch_bytes(C.byref(bad), C.byref(cfg), 10) == -1


def test_struct_layouts_match_header():
    assert C.sizeof(_lib.Dims) == 8 * 4
    assert C.sizeof(_lib.Config) == 4 * 4 + 4 * 8 + 2 * 4
    assert C.sizeof(_lib.Ctl) == 8 + 8 + 4 + 4 + 6 * 8
    assert C.sizeof(_lib.Report) == 12 * 8 + 8 + 4 * 8 + 3 * 8
    assert C.sizeof(_lib.State) == 3 * 8 + (len(_lib.STATE_PTRS) + len(_lib.DELTA_PTRS)) * 8 + 8 + 8
    hdr = _header()
    state_block = hdr[hdr.index("typedef struct {\n  int64_t cap_nodes"):]
    state_block = state_block[:state_block.index("} stgn_state;")]
    state_block = re.sub(r"/\*.*?\*/", "", state_block, flags=re.S)
    names = re.findall(r"\*\s*([a-z_0-9]+)", state_block)
    assert tuple(names) == _lib.STATE_PTRS + _lib.DELTA_PTRS + ("e_pay",)


def test_engine_refuses_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_21090_b200.config import Dims, RunConfig
    from paper_2603_21090_b200.engine import IncrementalEngine
    from paper_2603_21090_b200.params import init_params
    dims = Dims()
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        IncrementalEngine(RunConfig(dims=dims), init_params(0, dims))
