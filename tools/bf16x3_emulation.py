"""Numerical study behind the bf16x3 choice (DESIGN.md §3/§4): emulate the
recompute kernel's folded GEMM chain with fp32, split-TF32 and bf16x3
arithmetic on inputs captured from the oracle at C4 widths and compare with
the float64 pipeline (row-relative embedding error, prediction error).

    python tools/bf16x3_emulation.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.stgn_oracle import Oracle, pipeline_many
import oracle.stgn_oracle as so
from paper_2603_21090_b200.config import Dims, RunConfig
from paper_2603_21090_b200.params import init_params
from paper_2603_21090_b200.streamio import generate_stream
dims = Dims(d_s=100, d_e=0, d_t=100, d_m=100, d_k=50, heads=2, layers=2)
cfg = RunConfig(dims=dims, batch_size=600, fanout=10, nodes=20000, aggregator="last", rebuild="never")
p = init_params(0, dims)
st = generate_stream(2, 20000, 600*60, attachment="preferential", d_e=0)
o = Oracle(cfg, p)
cap = {}
orig = Oracle._pipeline
def hook(self, ids, lists, pending):
    # capture inputs by re-running the marshal part
    cap['args'] = (ids, lists, pending)
    return orig(self, ids, lists, pending)
Oracle._pipeline = hook
captured = None
orig_pm = so.pipeline_many
def pm(*a):
    global captured
    captured = a
    return orig_pm(*a)
so.pipeline_many = pm
for lo in range(0, len(st), 600):
    o.process_batch(st.src[lo:lo+600], st.dst[lo:lo+600], st.t[lo:lo+600], st.feat[lo:lo+600])
qbase, offs, payload, feat, dt, omega, phi0, wq, wk, wv, wo = captured
print('N', qbase.shape, 'E', payload.shape, 'mean E', payload.shape[0]/qbase.shape[0])
ref = orig_pm(*captured)[0]

def split(x, kind):
    x = x.astype(np.float32)
    if kind == 'bf16':
        def rb(v):
            u = v.astype(np.float32).view(np.uint32).astype(np.uint64)
            u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
            return u.astype(np.uint32).view(np.float32)
    elif kind == 'tf32':
        def rb(v):
            u = v.astype(np.float32).view(np.uint32)
            return (u & 0xFFFFE000).view(np.float32)
    hi = rb(x); lo = rb((x - hi).astype(np.float32))
    return hi.astype(np.float64), lo.astype(np.float64)

def gemm(x, w, kind):
    if kind == 'fp32':
        return (x.astype(np.float32).astype(np.float64) @ w.astype(np.float32).astype(np.float64)).astype(np.float32).astype(np.float64)
    xh, xl = split(x, kind); wh, wl = split(w, kind)
    return (xh @ wh + xh @ wl + xl @ wh).astype(np.float32).astype(np.float64)

def emu(kind):
    N, d = qbase.shape
    K, H, q_in, d_k = wq.shape
    k_in = wk.shape[2]
    x = qbase.copy()
    out_all = np.zeros((N, K, d))
    t_ref_dt = dt
    # phi
    ang = np.outer(dt, omega); phi = np.empty((len(dt), 2*len(omega))); phi[:,0::2]=np.cos(ang); phi[:,1::2]=np.sin(ang); phi *= np.sqrt(1/(2*len(omega)))
    phi = phi.astype(np.float32).astype(np.float64)
    for l in range(K):
        cs = []
        for h in range(H):
            b = phi0 @ wq[l,h][d:]
            q = gemm(x, wq[l,h][:d], kind) + b.astype(np.float32)
            qt = gemm(q, wk[l,h].T, kind) / np.sqrt(d_k)   # (N, k_in)
            kin = np.concatenate([payload[:, l, :], feat, phi], axis=1).astype(np.float32).astype(np.float64)
            ub = np.zeros((N, k_in))
            for i in range(N):
                a, bnd = offs[i], offs[i+1]
                if bnd == a: continue
                lg = kin[a:bnd] @ qt[i]
                w = np.exp(lg - lg.max()); w /= w.sum()
                ub[i] = w @ kin[a:bnd]
            cs.append(gemm(ub, wv[l,h], kind))
        c = np.concatenate(cs, axis=1)
        x = gemm(c, wo[l], kind)
        out_all[:, l] = x
    return out_all

for kind in ['fp32', 'tf32', 'bf16']:
    e = emu(kind)
    for l in range(2):
        r = ref[:, l]; d_ = e[:, l] - r
        nr = np.maximum(np.linalg.norm(r, axis=1), 1e-2)
        rel = np.linalg.norm(d_, axis=1) / nr
        print(kind, 'layer', l, 'max row rel', rel.max(), 'p99', np.percentile(rel, 99), 'median', np.median(rel))
rng = np.random.default_rng(0)
e = emu('bf16')
N = ref.shape[0]
iu = rng.integers(0, N, 5000); iv = rng.integers(0, N, 5000)
def pred(h):
    z = np.concatenate([h[iu, -1], h[iv, -1]], axis=1) @ p.w_pred + p.b_pred
    return 1/(1+np.exp(-z))
print('pred max abs diff bf16', np.abs(pred(e) - pred(ref)).max(), 'h norm median', np.median(np.linalg.norm(ref[:, -1], axis=1)))
