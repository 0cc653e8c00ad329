// Delta mode (cfg.mode = "delta"), K = 1: the statistics of each node's
// attention state and the error-bound record of every attn_hit update.
//
// Reference: _build_attn_state S/engine.py:247-274 keeps, per node, the
// softmax state of its last exact evaluation and raises max_value_norm_seen
// to the largest value-row norm ||kin_e W_V[0,h]||; _apply_delta :333-353
// updates a hit's state in place and records
//   DeltaEvent(node, embedding, bound = |dN|/|N| * max_v * z_dev, dn, nv, max_v, z_dev)
// with z_dev = max_h |1 - Z_old/Z_new| (delta_embed :43-118, _log_z :121-127)
// and max_v the largest value norm of the updated state (:130-134).
//
// The B200 path recomputes hits exactly (csrc/batch.cuh k_delta_classify), so
// Z_old is the log-partition kept from the node's last state build
// (attn_logz, written here for every state-building row: misses, hits, the
// post-commit refresh of V_direct, rebuilds) and Z_new is the hit row's own.
// One 128-thread block per row: the row's key rows kin_e = [payload | feat |
// phi(t_ref - t_e)] in shared memory, value norms (per-entry W_V projection,
// the one quantity the folded recompute never forms), q = x W_Q + b, the
// folded key q~_h = W_K,h q_h / sqrt(d_k), logits and log Z in float64.
#pragma once

#include "batch.cuh"

#define DS_THREADS 128

static inline size_t delta_state_smem(const Geo& g) {
  return sizeof(float) * ((size_t)g.d + g.HD + (size_t)g.H * g.k_in + (size_t)g.L * g.k_in +
                          2 * (size_t)g.L * g.H + 8);
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // non-negative doubles order like their bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            (unsigned long long)__double_as_longlong(v));
}

// mode 0: the batch's delta rows (clist[0, nC): V_direct first, which are also
//         evaluated with post-batch memory mem_new[r], whose state is the one kept);
//         runs after the recompute, before the memory commit.
// mode 1: a rebuild list (list[0, n), list NULL = node ids 0..n-1; n = *count_ptr
//         or count_const), with committed memory.
__global__ void __launch_bounds__(DS_THREADS)
k_delta_state(Geo g, StateView st, Scratch s, EngW w, const int32_t* list,
              const int32_t* count_ptr, int count_const, int mode) {
  extern __shared__ float dsm[];
  float* x = dsm;                      // [d]
  float* q = x + g.d;                  // [HD]
  float* qt = q + g.HD;                // [H][k_in]
  float* kin = qt + g.H * g.k_in;      // [L][k_in]
  float* lg = kin + g.L * g.k_in;      // [L][H]
  float* nrm = lg + g.L * g.H;         // [L][H] value norm^2
  __shared__ double s_lz[8];
  __shared__ float s_maxv;
  const int tid = threadIdx.x;
  const int N = mode == 0 ? s.res->nC : (count_ptr ? *count_ptr : count_const);
  const int nD = mode == 0 ? s.res->nD : 0;
  const float inv_sqrt_dk = (float)(1.0 / sqrt((double)g.d_k));
  double* mvn = reinterpret_cast<double*>(&st.ctl->reserved[1]);
  for (int r = blockIdx.x; r < N; r += gridDim.x) {
    const int v = mode == 0 ? s.clist[r] : (list ? list[r] : r);
    const int cc = st.ring_ccnt[v];
    const int E = cc >= 0 ? cc : st.ring_cnt[v];
    const int hd = st.ring_head[v];
    const double tref = E > 0 ? st.ring_t[(int64_t)v * g.L + hd] : 0.0;
    for (int o = tid; o < E * g.k_in; o += DS_THREADS) {
      const int e = o / g.k_in, c = o - e * g.k_in;
      int slot = hd + e;
      if (slot >= g.L) slot -= g.L;
      const int64_t rs = (int64_t)v * g.L + slot;
      float val;
      if (c < g.d) {
        val = st.ring_pay[((int64_t)v * g.K * g.L + slot) * g.ld_d + c];  // layer 0
      } else if (c < g.d + g.d_e) {
        val = st.ring_feat[rs * g.ld_e + (c - g.d)];
      } else {
        const int p = c - g.d - g.d_e;
        float sv, cv;
        phase_sincos(w.omega[p >> 1], tref - st.ring_t[rs], &sv, &cv);
        val = ((p & 1) ? sv : cv) * g.phi_amp;
      }
      kin[e * g.k_in + c] = val;
    }
    for (int o = tid; o < E * g.H; o += DS_THREADS) nrm[o] = 0.f;
    __syncthreads();
    // value rows v_{e,h} = kin_e W_V[0,h] (d_k each): squared norms
    for (int o = tid; o < E * g.H * g.d_k; o += DS_THREADS) {
      const int j = o % g.d_k, eh = o / g.d_k, h = eh % g.H, e = eh / g.H;
      const float* wv = w.wv + (int64_t)h * g.k_in * w.ld_dk + j;
      const float* kr = kin + e * g.k_in;
      float acc = 0.f;
      for (int c = 0; c < g.k_in; ++c) acc = fmaf(kr[c], wv[(int64_t)c * w.ld_dk], acc);
      atomicAdd(&nrm[eh], acc * acc);
    }
    __syncthreads();
    if (tid == 0) {
      float m = 0.f;
      for (int o = 0; o < E * g.H; ++o) m = fmaxf(m, sqrtf(nrm[o]));
      s_maxv = m;
    }
    const bool direct = mode == 0 && r < nD;
    const int npass = direct ? 2 : 1;
    for (int pass = 0; pass < npass; ++pass) {
      const float* xs = pass == 0 ? st.mem + (int64_t)v * g.ld_s : s.mem_new + (int64_t)r * g.ld_s;
      for (int c = tid; c < g.d; c += DS_THREADS) x[c] = c < g.d_s ? xs[c] : 0.f;
      __syncthreads();
      for (int j = tid; j < g.HD; j += DS_THREADS) {  // q = [x | phi(0)] W_Q (layer 0)
        float acc = w.bq[j];
        for (int c = 0; c < g.d; ++c) acc = fmaf(x[c], w.wq[(int64_t)c * w.ld_hd + j], acc);
        q[j] = acc;
      }
      __syncthreads();
      for (int o = tid; o < g.H * g.k_in; o += DS_THREADS) {  // q~_h = W_K,h q_h / sqrt(d_k)
        const int h = o / g.k_in, c = o - h * g.k_in;
        float acc = 0.f;
        for (int j = 0; j < g.d_k; ++j)
          acc = fmaf(w.wkt[((int64_t)h * g.d_k + j) * w.ld_kin + c], q[h * g.d_k + j], acc);
        qt[o] = acc * inv_sqrt_dk;
      }
      __syncthreads();
      for (int o = tid; o < E * g.H; o += DS_THREADS) {
        const int e = o / g.H, h = o - e * g.H;
        const float* kr = kin + e * g.k_in;
        const float* qh = qt + h * g.k_in;
        float acc = 0.f;
        for (int c = 0; c < g.k_in; ++c) acc = fmaf(kr[c], qh[c], acc);
        lg[o] = acc;
      }
      __syncthreads();
      if (tid < g.H) {  // log Z = max + log sum exp (-inf for an empty state)
        const int h = tid;
        double m = -INFINITY;
        for (int e = 0; e < E; ++e) m = fmax(m, (double)lg[e * g.H + h]);
        double z = 0.0;
        for (int e = 0; e < E; ++e) z += exp((double)lg[e * g.H + h] - m);
        s_lz[h] = E > 0 ? m + log(z) : -INFINITY;
      }
      __syncthreads();
      if (tid == 0) {
        double* lz_node = st.attn_logz + (int64_t)v * 4;
        if (mode == 0 && pass == 0 && (s.c_info[r] & 1)) {  // attn_hit: the update's record
          double zdev = 0.0;
          for (int h = 0; h < g.H; ++h) {
            if (isfinite(s_lz[h])) {
              const double old = lz_node[h];
              const double ratio = isfinite(old) ? exp(old - s_lz[h]) : 0.0;
              zdev = fmax(zdev, fabs(1.0 - ratio));
            }
          }
          const int dn = s.c_info[r] >> 1, nv = E > 1 ? E : 1;
          const int64_t idx =
              (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(&st.ctl->reserved[0]), 1ull);
          if (idx < st.ev_cap) {
            st.ev_node[idx] = v;
            st.ev_dpos[idx] = direct ? r : -1;
            st.ev_dn[idx] = dn;
            st.ev_nv[idx] = nv;
            st.ev_maxv[idx] = (double)s_maxv;
            st.ev_zdev[idx] = zdev;
            st.ev_bound[idx] = ((double)dn / (double)nv) * (double)s_maxv * zdev;
          }
        }
        if (pass == npass - 1)
          for (int h = 0; h < g.H; ++h) lz_node[h] = s_lz[h];
        if (pass == 0) atomic_max_nonneg(mvn, (double)s_maxv);
      }
      __syncthreads();
    }
  }
}

// embeddings of the batch's records: direct hits from the pre-batch-memory
// rows (dpred), the others from the final layer of h
__global__ void k_delta_ev_gather(Geo g, StateView st, Scratch s, const int32_t* node,
                                  const int32_t* dpos, int n, float* out) {
  GRID_STRIDE(o, (int64_t)n * g.d) {
    const int i = (int)(o / g.d), c = (int)(o % g.d);
    const float* src = dpos[i] >= 0 ? s.dpred + (int64_t)dpos[i] * g.ld_d
                                    : st.h + ((int64_t)node[i] * g.K + (g.K - 1)) * g.ld_d;
    out[o] = src[c];
  }
}
