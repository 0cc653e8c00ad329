"""Operator-level drop-in for the reference's `kernels.pipeline_many`
(/root/reference/pkg/src/streamtgn/kernels/__init__.py:42-44; contract in
kernels/pipeline_numpy.py:21-72): same arguments, same six outputs, float64
numpy in and out, computed by the sm_100a attention kernel through
`stgn_pipeline_many` (include/stgn.h). No CPU fallback.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .config import Dims
from .edges import KernelInputError

BACKEND = "cuda"


def pipeline_many(qbase, offsets, payload, feat, dt, omega, phi0, wq, wk, wv, wo):
    """K-layer multi-head temporal attention for N nodes over flat entries.

    Returns (out (N,K,d), scores (E,K,H), values (E,K,H,d_k),
    maxlog (N,K,H), zsum (N,K,H), qvecs (N,K,H,d_k)) as float64.
    """
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("pipeline_many needs a CUDA GPU; there is no CPU fallback")
    qbase = np.asarray(qbase, dtype=np.float64)
    N, d = qbase.shape
    K, H, q_in, d_k = wq.shape
    E = int(np.asarray(payload).shape[0])
    d_e = int(np.asarray(feat).reshape(E, -1).shape[1]) if E else int(wk.shape[2] - d - phi0.shape[0])
    d_t = int(phi0.shape[0])
    if q_in != d + d_t or wk.shape != (K, H, d + d_e + d_t, d_k) or wo.shape != (K, H * d_k, d):
        raise KernelInputError("pipeline_many: inconsistent shapes")
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    if offsets.shape != (N + 1,) or (N and int(offsets[-1]) != E):
        raise KernelInputError("pipeline_many: offsets must have N+1 entries ending at E")
    dims = Dims(d_s=d, d_e=d_e, d_t=d_t, d_x=0, d_m=1, d_k=d_k, heads=H, layers=K)
    dev = torch.device("cuda", torch.cuda.current_device())

    def f32(a, shape):
        return torch.tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(shape)),
                            device=dev)

    t_q = f32(qbase, (N, d))
    t_off = torch.tensor(offsets, device=dev)
    t_pay = f32(payload, (E, K, d))
    t_feat = f32(feat, (E, d_e))
    t_dt = torch.tensor(np.ascontiguousarray(dt, dtype=np.float64).reshape(E), device=dev)
    t_om = torch.tensor(np.ascontiguousarray(omega, dtype=np.float64), device=dev)
    t_phi0 = f32(phi0, (d_t,))
    t_wq, t_wk, t_wv, t_wo = f32(wq, wq.shape), f32(wk, wk.shape), f32(wv, wv.shape), f32(wo, wo.shape)
    out = torch.zeros((N, K, d), dtype=torch.float32, device=dev)
    scores = torch.zeros((E, K, H), dtype=torch.float32, device=dev)
    values = torch.zeros((E, K, H, d_k), dtype=torch.float32, device=dev)
    maxlog = torch.full((N, K, H), -np.inf, dtype=torch.float32, device=dev)
    zsum = torch.zeros((N, K, H), dtype=torch.float32, device=dev)
    qvecs = torch.zeros((N, K, H, d_k), dtype=torch.float32, device=dev)
    ds = _lib.dims_struct(dims)
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    _lib.check(_lib.lib().stgn_pipeline_many(
        C.byref(ds), N, E, p(t_q), p(t_off), p(t_pay), p(t_feat), p(t_dt), p(t_om), p(t_phi0),
        p(t_wq), p(t_wk), p(t_wv), p(t_wo), p(out), p(scores), p(values), p(maxlog), p(zsum),
        p(qvecs), stream), "pipeline_many")
    return tuple(x.double().cpu().numpy() for x in (out, scores, values, maxlog, zsum, qvecs))
