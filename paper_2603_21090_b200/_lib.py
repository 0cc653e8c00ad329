"""ctypes binding of the C ABI in include/stgn.h (the in-tree _stgn.so).

There is no fallback: if the library or a GPU is missing, `lib()` raises.
"""

from __future__ import annotations

import ctypes as C
import os

from .config import ConfigError
from .edges import InputError, KernelInputError, MonotonicityError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_stgn.so")

STGN_OK, STGN_ERR_INVALID, STGN_ERR_BOUNDS, STGN_ERR_CUDA, STGN_ERR_CAPACITY, STGN_ERR_ORDER = range(6)
AGG = {"mean": 0, "last": 1, "sum": 2}
REBUILD = {"never": 0, "fixed": 1, "adaptive": 2}
SCOPE = {"affected": 0, "direct": 1, "delta": 2}

# Symbols include/stgn.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = (
    "stgn_version", "stgn_last_error", "stgn_scratch_bytes", "stgn_engine_create", "stgn_engine_destroy",
    "stgn_engine_set_weights", "stgn_engine_bind", "stgn_engine_process_batch",
    "stgn_engine_process_batch_dev", "stgn_engine_rebuild", "stgn_engine_full_reference",
    "stgn_engine_affected", "stgn_engine_pred_embeddings", "stgn_pipeline_many",
    "stgn_engine_set_profiling", "stgn_engine_stage_times", "stgn_stage_name",
    "stgn_engine_info", "stgn_debug_tc_gemm", "stgn_generate_stream",
    "stgn_debug_a4_prof", "stgn_debug_a4_cta", "stgn_engine_set_scope", "stgn_read_stream",
    "stgn_engine_set_skip_recompute", "stgn_engine_delta_events", "stgn_batch_result_bytes",
    "stgn_engine_result_copy", "stgn_report_from_result", "stgn_engine_snapshot",
    "stgn_engine_set_ownership", "stgn_engine_batch_phase", "stgn_engine_dpred_export",
    "stgn_engine_dpred_import", "stgn_engine_stage_affected", "stgn_engine_stage_nbr_update",
    "stgn_engine_stage_commit", "stgn_dysat_batch", "stgn_dysat_recompute_all", "stgn_dysat_roll",
)


class Dims(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("d_s", "d_e", "d_t", "d_x", "d_m", "d_k", "heads", "layers")]


class Config(C.Structure):
    _fields_ = [("fanout", C.c_int32), ("aggregator", C.c_int32), ("rebuild", C.c_int32),
                ("rebuild_interval", C.c_int32), ("gamma", C.c_double),
                ("delta_max", C.c_double), ("alpha", C.c_double), ("window", C.c_double),
                ("scope", C.c_int32), ("max_batch", C.c_int32)]


class Weights(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in
                ("wq", "bq", "wkt", "wv", "wo", "wmsg", "bmsg", "wgru", "ugru", "bgru", "wpred",
                 "omega", "phi0")] + [("bpred", C.c_double)] + \
               [(n, C.c_void_p) for n in ("tcq", "tck", "tcv", "tco", "t4q", "t4k", "t4v", "t4o",
                                          "t4bq", "t4mem", "t4p")]


class Ctl(C.Structure):
    _fields_ = [("tau", C.c_int64), ("cum_count", C.c_int64), ("cum_gen", C.c_uint32),
                ("pad0", C.c_uint32), ("reserved", C.c_int64 * 6)]


STATE_PTRS = (
    "mem", "last", "version", "h", "valid", "valid_at", "ring_cnt", "ring_head", "ring_ccnt",
    "ring_nbr", "ring_eid", "ring_t", "ring_pay", "ring_feat", "ring_tb", "amark", "dmark", "nodecnt",
    "nodeadj", "nodefill", "nodeoff", "drift_acc", "drift_touched", "cum_mark", "cum_list",
    "cum_pos", "attn_ver", "attn_tref",
    "e_src", "e_dst", "e_t", "e_feat", "e_prev", "adj_head", "adj_deg", "gpow", "ctl", "scratch",
)


DELTA_PTRS = ("attn_logz", "ev_node", "ev_dpos", "ev_dn", "ev_nv", "ev_bound", "ev_maxv",
              "ev_zdev")


class StageEntries(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("nodes", "off", "nbr", "t", "eid", "pay", "feat", "put")]


class StageRecords(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("hit", "exp_n", "exp_nbr", "exp_t", "exp_eid", "upd_n",
                                           "upd_nbr")]


class DySAT(C.Structure):
    _fields_ = ([(n, C.c_int32) for n in ("d_in", "d", "heads_s", "heads_t", "window", "fanout",
                                          "ld", "max_batch")] +
                [(n, C.c_int64) for n in ("n", "snapshot", "pos_len", "chunk")] +
                [(n, C.c_void_p) for n in ("P", "ss", "sn", "lst_nbr", "lst_head", "lst_cnt",
                                           "hist_k", "hist_v", "emb", "mark", "work", "rows",
                                           "pos", "wq", "wk", "wv", "wo", "wpred")] +
                [("bpred", C.c_double), ("wtc", C.c_void_p), ("tc_min_rows", C.c_int64)])


class State(C.Structure):
    _fields_ = [("cap_nodes", C.c_int64), ("cap_edges", C.c_int64), ("gpow_len", C.c_int64)] + \
               [(n, C.c_void_p) for n in STATE_PTRS + DELTA_PTRS] + [("ev_cap", C.c_int64),
                                                                    ("e_pay", C.c_void_p)]


class Report(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("direct", "affected", "nbr_hit", "nbr_miss", "entries_affected",
                 "entries_direct", "rebuild_kind", "rebuild_nodes", "entries_rebuild", "tau",
                 "cum_count", "changed")] + [("global_drift", C.c_double)] + \
               [(n, C.c_int64) for n in ("embed_skip", "attn_hit", "attn_miss", "entries_miss")] + \
               [("reserved", C.c_int64 * 3)]


_LIB = None


def lib():
    """Load _stgn.so (building it first if the sources are newer)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        from .build import build
        build()
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    P = C.POINTER
    L.stgn_version.restype = C.c_char_p
    L.stgn_last_error.restype = C.c_char_p
    L.stgn_scratch_bytes.restype = i64
    L.stgn_scratch_bytes.argtypes = [P(Dims), P(Config), i64]
    L.stgn_engine_create.argtypes = [P(Dims), P(Config), P(vp)]
    L.stgn_engine_destroy.argtypes = [vp]
    L.stgn_engine_set_weights.argtypes = [vp, P(Weights)]
    L.stgn_engine_bind.argtypes = [vp, P(State)]
    L.stgn_engine_process_batch.argtypes = [vp, i32, vp, vp, vp, vp, i64, i64, i64, vp,
                                            P(Report), vp]
    L.stgn_engine_process_batch_dev.argtypes = [vp, i32, vp, vp, vp, vp, i64, i64, i64, vp,
                                                P(Report), vp]
    L.stgn_engine_rebuild.argtypes = [vp, vp, i64, i64, dbl, P(i64), vp]
    L.stgn_engine_full_reference.argtypes = [vp, i64, vp, vp]
    L.stgn_engine_snapshot.argtypes = [vp, i64, dbl, vp, vp]
    L.stgn_engine_set_ownership.argtypes = [vp, i32, i32]
    L.stgn_engine_batch_phase.argtypes = [vp, i32, i32, vp, vp, vp, vp, i64, i64, i64, vp, vp, vp]
    L.stgn_engine_dpred_export.argtypes = [vp, vp, vp, vp, vp]
    L.stgn_engine_dpred_import.argtypes = [vp, vp, vp, i64, vp]
    L.stgn_engine_stage_affected.argtypes = [vp, i32, vp, vp, C.c_uint32, vp, i64, vp, vp]
    L.stgn_engine_stage_nbr_update.argtypes = [vp, i32, P(StageEntries), vp, i32, dbl,
                                               P(StageRecords), vp]
    L.stgn_engine_stage_commit.argtypes = [vp, i32, vp, vp, vp, vp, vp, i64, vp]
    L.stgn_dysat_batch.argtypes = [P(DySAT), i32, vp, vp, C.c_uint32, vp, vp, vp]
    L.stgn_dysat_recompute_all.argtypes = [P(DySAT), vp]
    L.stgn_dysat_roll.argtypes = [P(DySAT), vp]
    L.stgn_engine_affected.argtypes = [vp, vp, vp, i64, P(i64), P(i64), vp, vp]
    L.stgn_engine_pred_embeddings.argtypes = [vp, vp, i64, vp]
    L.stgn_pipeline_many.argtypes = [P(Dims), i64, i64] + [vp] * 18
    L.stgn_engine_set_profiling.argtypes = [vp, C.c_int]
    L.stgn_engine_stage_times.argtypes = [vp, vp, C.c_int, P(i64)]
    L.stgn_stage_name.restype = C.c_char_p
    L.stgn_batch_result_bytes.restype = i64
    L.stgn_stage_name.argtypes = [C.c_int]
    L.stgn_engine_info.argtypes = [vp, vp, C.c_int]
    L.stgn_debug_tc_gemm.argtypes = [C.c_int, C.c_int, C.c_int, vp, vp, vp, C.c_int, vp]
    L.stgn_debug_a4_prof.argtypes = [vp, C.c_int]
    L.stgn_debug_a4_cta.argtypes = [vp, C.c_int]
    L.stgn_engine_set_scope.argtypes = [vp, C.c_int]
    L.stgn_engine_set_skip_recompute.argtypes = [vp, C.c_int]
    L.stgn_read_stream.argtypes = [C.c_char_p, i32, i64, P(i64), P(i64), vp, vp, vp, vp, P(i64)]
    L.stgn_generate_stream.argtypes = [vp, i64, i64, i32, dbl, vp, vp, vp, vp]
    for name in EXPORTS:
        if name not in ("stgn_version", "stgn_last_error", "stgn_scratch_bytes",
                        "stgn_stage_name", "stgn_batch_result_bytes"):
            getattr(L, name).restype = C.c_int
    _LIB = L
    return L


def check(rc: int, what: str = "") -> None:
    if rc == STGN_OK:
        return
    msg = f"{what}: stgn error {rc}"
    if rc == STGN_ERR_INVALID:
        raise ConfigError(msg)
    if rc == STGN_ERR_BOUNDS:
        raise InputError(msg)
    if rc == STGN_ERR_ORDER:
        raise MonotonicityError(msg)
    if rc == STGN_ERR_CAPACITY:
        raise KernelInputError(msg + " (capacity)")
    detail = _LIB.stgn_last_error().decode() if _LIB is not None else ""
    raise RuntimeError(f"{msg} (CUDA failure: {detail})")


def dims_struct(dims) -> Dims:
    return Dims(dims.d_s, dims.d_e, dims.d_t, dims.d_x, dims.d_m, dims.d_k, dims.heads,
                dims.layers)
