// K-layer temporal attention recompute (the hot kernel).
//
// Restates the reference's per-node pipeline (S/kernels/pipeline_numba.py:15-111,
// spec S/kernels/reference.py:120-180) for a tile of T nodes per CTA:
//
//   x_0 = [s_v || 0_dx]            x_l = out_{l-1}
//   q_h   = [x_l || phi(0)] W_Q[l,h]                        (tile GEMM)
//   qk_h  = W_K[l,h] q_h / sqrt(d_k)        (k_in-vector;    tile GEMM)
//   logit_{e,h} = qk_h . kin_e,   kin_e = [payload_e,l || feat_e || phi(t_ref - t_e)]
//   ubar_h = sum_e softmax_e(logit) kin_e   (online softmax, one warp per node)
//   c_h   = ubar_h W_V[l,h]                                   (tile GEMM)
//   out_l = [c_1..c_H] W_O[l]                                 (tile GEMM)
//
// The key/value projections are folded into the query side and the
// softmax-weighted input average (q.(kin W_K) = (W_K q).kin and
// sum_e a_e (kin_e W_V) = (sum_e a_e kin_e) W_V), which is the same
// function with 5.5x fewer FLOPs at C4 widths; per-entry keys/values
// are only materialised for the operator-level API (STATS).
#pragma once

#include "common.cuh"

struct AttnWeights {
  const float *wq, *wkt, *wv, *wo;   // packed, see stgn.h
  const double* omega;
  const float* phi0;
};

// ---- node sources ------------------------------------------------------------

struct RingSrc {
  // node list
  const int32_t* list;       // nullptr -> node = index
  const int32_t* count_ptr;  // device count (nullable)
  int64_t count_const;
  int use_store;             // uncached nodes read the store top-L (full_reference)
  // state
  const float* mem;
  float* h;
  uint8_t* valid;
  double* valid_at;
  const int32_t *ring_cnt, *ring_head, *ring_ccnt;
  const double* ring_t;
  const float *ring_pay, *ring_feat;
  const float* ring_tb;           // [node][L][ld_t] time basis of the slot timestamps
  // outputs / side effects
  const double* valid_at_ptr;   // device value (hdr->t_batch) or nullptr
  double valid_at_const;
  int write_valid;
  float* final_out;             // nullable: write last layer to final_out[idx] instead of h
  float* layers_out;            // nullable: write every layer l to layers_out[idx][l] instead of h
                                // (pure snapshot recompute, full_recompute)
  float* dpred;                 // nullable: copy last layer of idx < *dpred_count into dpred[idx]
  const int32_t* dpred_count;
  unsigned long long* e_count;  // nullable: sum of entry counts
  // Fused pre/post pass (engine batch path): rows [0, *pre_n) are list[idx]
  // with pre-batch memory, rows [*pre_n, *pre_n + *post_n) are list[idx - pre_n]
  // (the direct set) with post-batch memory mem_post[idx - pre_n]. Pre rows
  // with idx < *post_n (direct nodes) only feed dpred; everything else writes h.
  int fused;
  const int32_t *pre_n, *post_n;
  const float* mem_post;
  unsigned long long* e_count_post;

  __device__ int64_t count() const {
    if (fused) return (int64_t)pre_n[0] + post_n[0];
    return count_ptr ? (int64_t)count_ptr[0] : count_const;
  }
  int own_lo, own_hi;            // node-id shard (own_hi <= own_lo: all): other rows are skipped
  __device__ int node(int64_t idx) const {
    int v;
    if (fused) {
      const int p = pre_n[0];
      v = list[idx < p ? idx : idx - p];
    } else {
      v = list ? list[idx] : (int)idx;
    }
    if (own_hi > own_lo && (v < own_lo || v >= own_hi)) return -1;
    return v;
  }
};

struct FlatSrc {
  int64_t N;
  const int64_t* offsets;
  const float *qbase, *payload, *feat;
  const double* dt;
  float *out, *scores, *values, *maxlog, *zsum, *qvecs;
};

// ---- tile GEMM: C[T][N] = alpha * A[T][kd] (smem) x W[kd][N] (global) -------
// Each thread owns 4 consecutive rows of one column; rows of A beyond the
// tile are zero so T is padded to a multiple of 4.
__device__ __forceinline__ void tile_gemm(const float* __restrict__ A, int lda, int T, int kd,
                                          const float* __restrict__ W, int ldw, int N,
                                          float* __restrict__ C, int ldc, float alpha,
                                          bool accumulate = false) {
  const int groups = T >> 2;
  for (int o = threadIdx.x; o < groups * N; o += blockDim.x) {
    const int n = o % N;
    const int i0 = (o / N) << 2;
    const float* a0 = A + (int64_t)i0 * lda;
    float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
    const float* wp = W + n;
#pragma unroll 4
    for (int k = 0; k < kd; ++k) {
      const float w = __ldg(wp + (int64_t)k * ldw);
      c0 = fmaf(a0[k], w, c0);
      c1 = fmaf(a0[lda + k], w, c1);
      c2 = fmaf(a0[2 * lda + k], w, c2);
      c3 = fmaf(a0[3 * lda + k], w, c3);
    }
    float* cp = C + (int64_t)i0 * ldc + n;
    if (accumulate) {
      cp[0] += alpha * c0;
      cp[ldc] += alpha * c1;
      cp[2 * ldc] += alpha * c2;
      cp[3 * ldc] += alpha * c3;
    } else {
      cp[0] = alpha * c0;
      cp[ldc] = alpha * c1;
      cp[2 * ldc] = alpha * c2;
      cp[3 * ldc] = alpha * c3;
    }
  }
}

template <int MAXA>
__device__ __forceinline__ void load_kin(float (&kin)[MAXA], const Geo& g, const float* pay,
                                         const float* feat, double dt, const double* omega,
                                         int lane) {
#pragma unroll
  for (int k = 0; k < MAXA; ++k) {
    const int a = lane + 32 * k;
    float v = 0.f;
    if (a < g.d) {
      v = pay[a];
    } else if (a < g.d + g.d_e) {
      v = feat[a - g.d];
    } else if (a < g.k_in) {
      v = phi_component(omega, a - g.d - g.d_e, dt, g.phi_amp);
    }
    kin[k] = v;
  }
}

// Smem floats needed for a tile of T nodes.
static inline int64_t attn_smem_floats(const Geo& g, int T, bool stats) {
  int64_t f = (int64_t)T * g.q_in + (int64_t)T * g.HD + (int64_t)T * g.H * g.k_in +
              (int64_t)T * g.HD;
  if (stats) f += (int64_t)STGN_WARPS * g.k_in;
  return f;
}

#define TMAX 64

template <int MAXA, int MAXH, bool FLAT>
__global__ void __launch_bounds__(STGN_THREADS)
attn_kernel(Geo g, AttnWeights w, RingSrc rs, FlatSrc fs, int T) {
  extern __shared__ float4 smem4[];
  float* X = reinterpret_cast<float*>(smem4);      // [T][q_in]
  float* Q = X + (int64_t)T * g.q_in;              // [T][HD]
  float* U = Q + (int64_t)T * g.HD;                // [T][H][k_in]
  float* Cc = U + (int64_t)T * g.H * g.k_in;       // [T][HD]
  float* kbuf = Cc + (int64_t)T * g.HD;            // [WARPS][k_in] (FLAT only)
  __shared__ int s_node[TMAX];
  __shared__ int s_E[TMAX];
  __shared__ int s_head[TMAX];
  __shared__ int64_t s_lo[TMAX];
  __shared__ double s_tref[TMAX];

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t N = FLAT ? fs.N : rs.count();
  const int64_t ntiles = cdiv(N, T);
  const int UK = g.H * g.k_in;
  int64_t dpred_n = 0;
  if (!FLAT && rs.dpred) dpred_n = rs.dpred_count[0];

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * T;
    // ---- tile metadata
    for (int i = threadIdx.x; i < T; i += blockDim.x) {
      const int64_t idx = base + i;
      int node = -1, E = 0, head = 0;
      int64_t lo = 0;
      double tref = 0.0;
      if (idx < N) {
        if (FLAT) {
          node = (int)idx;
          lo = fs.offsets[idx];
          E = (int)(fs.offsets[idx + 1] - lo);
        } else {
          node = rs.node(idx);
          if (node >= 0) {
            const int cc = rs.ring_ccnt[node];
            E = cc >= 0 ? cc : (rs.use_store ? rs.ring_cnt[node] : 0);
            head = rs.ring_head[node];
            if (E > 0) tref = rs.ring_t[(int64_t)node * g.L + head];
            if (rs.e_count && E) atomicAdd(rs.e_count, (unsigned long long)E);
          }
        }
      }
      s_node[i] = node;
      s_E[i] = E;
      s_head[i] = head;
      s_lo[i] = lo;
      s_tref[i] = tref;
    }
    __syncthreads();
    // ---- layer-0 query input [x0 || phi0]
    for (int o = threadIdx.x; o < T * g.q_in; o += blockDim.x) {
      const int i = o / g.q_in, j = o % g.q_in;
      const int node = s_node[i];
      float v = 0.f;
      if (node >= 0) {
        if (j >= g.d) v = w.phi0[j - g.d];
        else if (FLAT) v = fs.qbase[(int64_t)node * g.d + j];
        else if (j < g.d_s) v = rs.mem[(int64_t)node * g.ld_s + j];
      }
      X[o] = v;
    }
    __syncthreads();

    for (int l = 0; l < g.K; ++l) {
      const float* wq = w.wq + (int64_t)l * g.q_in * g.HD;
      const float* wkt = w.wkt + (int64_t)l * g.H * g.d_k * g.k_in;
      const float* wv = w.wv + (int64_t)l * g.H * g.k_in * g.d_k;
      const float* wo = w.wo + (int64_t)l * g.HD * g.d;
      // q = x W_Q
      tile_gemm(X, g.q_in, T, g.q_in, wq, g.HD, g.HD, Q, g.HD, 1.f);
      __syncthreads();
      if (FLAT) {
        for (int o = threadIdx.x; o < T * g.HD; o += blockDim.x) {
          const int i = o / g.HD, c = o % g.HD;
          if (s_node[i] >= 0) fs.qvecs[((int64_t)s_node[i] * g.K + l) * g.HD + c] = Q[o];
        }
      }
      // qk_h = (W_K[l,h] q_h) / sqrt(d_k)
      for (int hh = 0; hh < g.H; ++hh)
        tile_gemm(Q + hh * g.d_k, g.HD, T, g.d_k, wkt + (int64_t)hh * g.d_k * g.k_in, g.k_in,
                  g.k_in, U + hh * g.k_in, UK, g.inv_sqrt_dk);
      __syncthreads();

      // ---- per-node online softmax over the entries (one warp per node)
      for (int i = warp; i < T; i += STGN_WARPS) {
        const int node = s_node[i];
        const int E = s_E[i];
        float* Ui = U + (int64_t)i * UK;
        float qk[MAXH][MAXA], ub[MAXH][MAXA], mx[MAXH], zs[MAXH];
#pragma unroll
        for (int hh = 0; hh < MAXH; ++hh) {
          mx[hh] = -INFINITY;
          zs[hh] = 0.f;
#pragma unroll
          for (int k = 0; k < MAXA; ++k) {
            const int a = lane + 32 * k;
            qk[hh][k] = (hh < g.H && a < g.k_in) ? Ui[hh * g.k_in + a] : 0.f;
            ub[hh][k] = 0.f;
          }
        }
        for (int e = 0; e < E; ++e) {
          const float *pay, *ft;
          double dt;
          int64_t gidx = 0;
          if (FLAT) {
            gidx = s_lo[i] + e;
            pay = fs.payload + (gidx * g.K + l) * g.d;
            ft = fs.feat + gidx * g.d_e;
            dt = fs.dt[gidx];
          } else {
            int slot = s_head[i] + e;
            if (slot >= g.L) slot -= g.L;
            pay = rs.ring_pay + (((int64_t)node * g.K + l) * g.L + slot) * g.ld_d;
            ft = rs.ring_feat + ((int64_t)node * g.L + slot) * g.ld_e;
            dt = s_tref[i] - rs.ring_t[(int64_t)node * g.L + slot];
          }
          float kin[MAXA];
          load_kin<MAXA>(kin, g, pay, ft, dt, w.omega, lane);
#pragma unroll
          for (int hh = 0; hh < MAXH; ++hh) {
            if (hh < g.H) {
              float part = 0.f;
#pragma unroll
              for (int k = 0; k < MAXA; ++k) part = fmaf(qk[hh][k], kin[k], part);
              const float logit = warp_sum(part);
              if (FLAT && lane == 0) fs.scores[(gidx * g.K + l) * g.H + hh] = logit;
              const float nm = fmaxf(mx[hh], logit);
              const float sc = expf(mx[hh] - nm);
              const float p = expf(logit - nm);
              zs[hh] = zs[hh] * sc + p;
#pragma unroll
              for (int k = 0; k < MAXA; ++k) ub[hh][k] = fmaf(p, kin[k], ub[hh][k] * sc);
              mx[hh] = nm;
            }
          }
          if (FLAT) {  // per-entry values for the operator API
            float* kb = kbuf + warp * g.k_in;
#pragma unroll
            for (int k = 0; k < MAXA; ++k) {
              const int a = lane + 32 * k;
              if (a < g.k_in) kb[a] = kin[k];
            }
            __syncwarp();
            for (int o = lane; o < g.HD; o += 32) {
              const int hh = o / g.d_k, b = o % g.d_k;
              const float* wcol = wv + (int64_t)hh * g.k_in * g.d_k + b;
              float acc = 0.f;
              for (int a = 0; a < g.k_in; ++a) acc = fmaf(kb[a], __ldg(wcol + (int64_t)a * g.d_k), acc);
              fs.values[((gidx * g.K + l) * g.H + hh) * g.d_k + b] = acc;
            }
            __syncwarp();
          }
        }
#pragma unroll
        for (int hh = 0; hh < MAXH; ++hh) {
          if (hh < g.H) {
            const float inv = E > 0 ? 1.f / zs[hh] : 0.f;
#pragma unroll
            for (int k = 0; k < MAXA; ++k) {
              const int a = lane + 32 * k;
              if (a < g.k_in) Ui[hh * g.k_in + a] = ub[hh][k] * inv;
            }
          }
        }
        if (FLAT && node >= 0) {
          __syncwarp();
          if (lane < g.H) {
            float mv = -INFINITY, zv = 0.f;
#pragma unroll
            for (int hh = 0; hh < MAXH; ++hh)
              if (hh == lane) { mv = mx[hh]; zv = zs[hh]; }
            fs.maxlog[((int64_t)node * g.K + l) * g.H + lane] = mv;
            fs.zsum[((int64_t)node * g.K + l) * g.H + lane] = zv;
          }
          // rescale raw logits into the max-scaled frame
          for (int o = lane; o < E * g.H; o += 32) {
            const int e = o / g.H, hh = o % g.H;
            float mv = 0.f;
#pragma unroll
            for (int q = 0; q < MAXH; ++q)
              if (q == hh) mv = mx[q];
            float* sp = fs.scores + ((s_lo[i] + e) * g.K + l) * g.H + hh;
            *sp = expf(*sp - mv);
          }
        }
      }
      __syncthreads();
      // c_h = ubar_h W_V[l,h]
      for (int hh = 0; hh < g.H; ++hh)
        tile_gemm(U + hh * g.k_in, UK, T, g.k_in, wv + (int64_t)hh * g.k_in * g.d_k, g.d_k,
                  g.d_k, Cc + hh * g.d_k, g.HD, 1.f);
      __syncthreads();
      // out_l = c W_O -> X[:, :d] (next layer's query input)
      tile_gemm(Cc, g.HD, T, g.HD, wo, g.d, g.d, X, g.q_in, 1.f);
      __syncthreads();
      // write out_l
      for (int o = threadIdx.x; o < T * g.d; o += blockDim.x) {
        const int i = o / g.d, j = o % g.d;
        const int node = s_node[i];
        if (node < 0) continue;
        const float v = X[(int64_t)i * g.q_in + j];
        if (FLAT) {
          fs.out[((int64_t)node * g.K + l) * g.d + j] = v;
        } else {
          const int64_t idx = base + i;
          const bool last = (l == g.K - 1);
          if (rs.layers_out) {
            rs.layers_out[(idx * g.K + l) * g.ld_d + j] = v;
          } else if (rs.final_out) {  // read-only recompute (full_reference)
            if (last) rs.final_out[idx * g.ld_d + j] = v;
          } else {
            rs.h[((int64_t)node * g.K + l) * g.ld_d + j] = v;
          }
          if (last && rs.dpred && idx < dpred_n) rs.dpred[idx * g.ld_d + j] = v;
        }
      }
      if (!FLAT && rs.write_valid && l == g.K - 1) {
        for (int i = threadIdx.x; i < T; i += blockDim.x) {
          const int node = s_node[i];
          if (node < 0) continue;
          rs.valid[node] = 1;
          rs.valid_at[node] = rs.valid_at_ptr ? rs.valid_at_ptr[0] : rs.valid_at_const;
        }
      }
      __syncthreads();
    }
  }
}
