// Engine-side K-layer temporal attention recompute (the hot kernel, v2).
//
// Same function as attn_kernel (attn.cuh; reference S/kernels/pipeline_numba.py:15-111)
// restructured for latency and throughput on sm_100a:
//  * persistent grid of one 512-thread CTA per SM; the node list is cut into
//    one wave of row tiles (T = ceil(N / grid) rounded to 4, <= 32), so even
//    a ~1K-node direct set spreads over every SM;
//  * the phi(0) half of the query input is constant, so it is folded into a
//    per-layer bias (q = x W_Q[:d] + phi0 W_Q[d:]) and the Q GEMM has K = d;
//  * dense steps are R4 register-blocked FFMA GEMMs (gemm.cuh) over
//    shared-memory activations, weights from L1/L2;
//  * the tile's frozen payload rows (all layers) are prefetched into L2 at
//    tile start, so the per-node online-softmax walk does not wait on HBM;
//  * the time encoding reduces the angle in float64 and evaluates sin/cos
//    pairs in float32 on the SFU, one frequency per lane.
#pragma once

#include "attn.cuh"
#include "gemm.cuh"

struct EngW {
  const float *wq, *bq, *wkt, *wv, *wo;  // packed (stgn.h)
  const double* omega;
  int ld_hd, ld_kin, ld_dk, ld_d;        // padded row strides
};

#define A2_TMAX 64       // static metadata capacity; the runtime cap is tmax
#define A2_THREADS 512
#define A2_WARPS (A2_THREADS / 32)
#define A2_MAXI 4

static inline int64_t attn2_row_floats(const Geo& g) { return g.d + 2 * g.HD + g.H * g.k_in; }

// Largest weight block one GEMM of a layer stages at once.
static inline int64_t attn2_wsm_full(const Geo& g) {
  const int64_t ld_hd = round_up(g.HD, 4), ld_kin = round_up(g.k_in, 4);
  const int64_t ld_dk = round_up(g.d_k, 4), ld_d = round_up(g.d, 4);
  int64_t m = (int64_t)g.d * ld_hd;
  m = m > (int64_t)g.H * g.d_k * ld_kin ? m : (int64_t)g.H * g.d_k * ld_kin;
  m = m > (int64_t)g.H * g.k_in * ld_dk ? m : (int64_t)g.H * g.k_in * ld_dk;
  m = m > (int64_t)g.HD * ld_d ? m : (int64_t)g.HD * ld_d;
  return m;
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Key input element a of one ring entry: [payload_l || feat || phi(dt)] (the
// reference's kin_row, S/engine_base.py:135-137).
__device__ __forceinline__ float a2_key(const Geo& g, const EngW& w, const float* pay,
                                        const float* ft, double dt, int a) {
  if (a < g.d) return pay[a];
  if (a < g.d + g.d_e) return ft[a - g.d];
  const int p = a - g.d - g.d_e;
  float sv, cv;
  phase_sincos(w.omega[p >> 1], dt, &sv, &cv);
  return ((p & 1) ? sv : cv) * g.phi_amp;
}

// GEN = 1: any widths (d, d_e, d_t, H): the walk keeps no per-lane register
// arrays; one head at a time, the query is read from shared memory and the
// value accumulator lives in a per-warp row of the (then idle) weight stage.
template <int KF, int MAXH, int GEN = 0>
__global__ void __launch_bounds__(A2_THREADS, 1)
attn2_kernel(Geo g, EngW w, RingSrc rs, int tmax, int wsm_floats) {
  constexpr int KP = 4;  // payload elements per lane (d <= 128)
  constexpr int KT = 2;  // frequencies per lane (d_t / 2 <= 64)
  extern __shared__ float4 smem4[];
  float* X = reinterpret_cast<float*>(smem4);           // R4 [T][d]
  float* Q = X + tmax * g.d;                             // R4 [T][HD]
  float* U = Q + tmax * g.HD;                            // R4 [T][H*k_in]
  float* Cc = U + tmax * g.H * g.k_in;                   // R4 [T][HD]
  float* Wsm = Cc + tmax * g.HD;                         // staged weight rows
  __shared__ int s_node[A2_TMAX];
  __shared__ int s_E[A2_TMAX];
  __shared__ int s_head[A2_TMAX];
  __shared__ double s_tref[A2_TMAX];
  __shared__ int s_mode[A2_TMAX];  // 0 write h, 1 direct pre-pass (dpred only), 2 post-memory row

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int64_t N = rs.count();
  if (N <= 0) return;
  int T = (int)round_up(cdiv(N, gridDim.x), 4);
  if (T > tmax) T = tmax;
  const int64_t ntiles = cdiv(N, T);
  const int UK = g.H * g.k_in;
  const int64_t pre_rows = rs.fused ? (int64_t)rs.pre_n[0] : N;
  const int64_t d_rows = rs.fused ? (int64_t)rs.post_n[0] : 0;
  const int pay_lines = (g.d * 4 + 127) / 128;
  const int feat_lines = g.d_e ? (g.d_e * 4 + 127) / 128 : 0;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * T;
    if (tid < A2_TMAX) {  // warps 0-1
      const int i = tid;
      const int64_t idx = base + i;
      int node = -1, E = 0, head = 0, mode = 0;
      double tref = 0.0;
      if (i < T && idx < N) {
        node = rs.node(idx);
        if (rs.fused) mode = idx >= pre_rows ? 2 : (idx < d_rows ? 1 : 0);
        const int cc = node >= 0 ? rs.ring_ccnt[node] : 0;
        E = node < 0 ? 0 : (cc >= 0 ? cc : (rs.use_store ? rs.ring_cnt[node] : 0));
        head = node >= 0 ? rs.ring_head[node] : 0;
        if (E > 0) tref = rs.ring_t[(int64_t)node * g.L + head];
      }
      s_node[i] = node;
      s_E[i] = E;
      s_head[i] = head;
      s_tref[i] = tref;
      s_mode[i] = mode;
      if (rs.e_count) {
        unsigned long long e_pre = mode == 2 ? 0ull : (unsigned long long)E;
        unsigned long long e_post = mode == 2 ? (unsigned long long)E : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          e_pre += __shfl_xor_sync(0xffffffffu, e_pre, o);
          e_post += __shfl_xor_sync(0xffffffffu, e_post, o);
        }
        if (lane == 0 && e_pre) atomicAdd(rs.e_count, e_pre);
        if (lane == 0 && e_post && rs.e_count_post) atomicAdd(rs.e_count_post, e_post);
      }
    }
    __syncthreads();
    // L2 prefetch of every payload / feature row the tile will read
    {
      const int per_entry = g.K * pay_lines + feat_lines;
      const int total = T * g.L * per_entry;
      for (int x = tid; x < total; x += A2_THREADS) {
        const int i = x / (g.L * per_entry);
        const int rem = x % (g.L * per_entry);
        const int e = rem / per_entry;
        const int q = rem % per_entry;
        const int node = s_node[i];
        if (node < 0 || e >= s_E[i]) continue;
        int slot = s_head[i] + e;
        if (slot >= g.L) slot -= g.L;
        const char* p;
        if (q < g.K * pay_lines) {
          const int l = q / pay_lines, ln = q % pay_lines;
          p = reinterpret_cast<const char*>(rs.ring_pay + (((int64_t)node * g.K + l) * g.L + slot) * g.ld_d) + ln * 128;
        } else {
          p = reinterpret_cast<const char*>(rs.ring_feat + ((int64_t)node * g.L + slot) * g.ld_e) + (q - g.K * pay_lines) * 128;
        }
        prefetch_l2(p);
      }
    }
    // x_0 = [s_v || 0_dx]
    for (int o = tid; o < T * g.d; o += A2_THREADS) {
      const int i = o / g.d, j = o % g.d;
      const int node = s_node[i];
      float v = 0.f;
      if (node >= 0 && j < g.d_s)
        v = s_mode[i] == 2 ? rs.mem_post[(base + i - pre_rows) * g.ld_s + j]
                           : rs.mem[(int64_t)node * g.ld_s + j];
      X[r4(i, j, g.d)] = v;
    }
    __syncthreads();

    for (int l = 0; l < g.K; ++l) {
      const float* wq = w.wq + (int64_t)l * g.d * w.ld_hd;
      const float* bq = w.bq + (int64_t)l * g.HD;
      const float* wkt = w.wkt + (int64_t)l * g.H * g.d_k * w.ld_kin;
      const float* wv = w.wv + (int64_t)l * g.H * g.k_in * w.ld_dk;
      const float* wo = w.wo + (int64_t)l * g.HD * w.ld_d;
      // q = x W_Q[:d] + phi0 W_Q[d:]
      gemm_staged<A2_MAXI>(X, g.d, 0, T, g.d, wq, w.ld_hd, 0, g.HD, 1, Q, g.HD, 0, 1.f, bq, 0,
                           false, Wsm, wsm_floats);
      // qk_h = W_K[l,h] q_h / sqrt(d_k), all heads in one staged pass
      gemm_staged<A2_MAXI>(Q, g.HD, g.d_k, T, g.d_k, wkt, w.ld_kin, (int64_t)g.d_k * w.ld_kin,
                           g.k_in, g.H, U, UK, g.k_in, g.inv_sqrt_dk, nullptr, 0, false, Wsm,
                           wsm_floats);
      // per-node online softmax over the ring entries, ubar into U
      if constexpr (GEN) {
        float* ub = Wsm + warp * round_up(g.k_in, 4);
        for (int i = warp; i < T; i += A2_WARPS) {
          const int node = s_node[i];
          const int E = s_E[i];
          for (int hh = 0; hh < g.H; ++hh) {
            const int hb = hh * g.k_in;
            for (int a = lane; a < g.k_in; a += 32) ub[a] = 0.f;
            float mx = -INFINITY, zs = 0.f;
            for (int e = 0; e < E; ++e) {
              int slot = s_head[i] + e;
              if (slot >= g.L) slot -= g.L;
              const float* pay = rs.ring_pay + (((int64_t)node * g.K + l) * g.L + slot) * g.ld_d;
              const float* ft = rs.ring_feat + ((int64_t)node * g.L + slot) * g.ld_e;
              const double dt = s_tref[i] - rs.ring_t[(int64_t)node * g.L + slot];
              float part = 0.f;
              for (int a = lane; a < g.k_in; a += 32)
                part = fmaf(U[r4(i, hb + a, UK)], a2_key(g, w, pay, ft, dt, a), part);
              const float logit = warp_sum(part);
              const float nm = fmaxf(mx, logit);
              const float sc = __expf(mx - nm);
              const float p = __expf(logit - nm);
              zs = fmaf(zs, sc, p);
              for (int a = lane; a < g.k_in; a += 32)
                ub[a] = fmaf(p, a2_key(g, w, pay, ft, dt, a), ub[a] * sc);
              mx = nm;
            }
            const float inv = E > 0 ? 1.f / zs : 0.f;
            for (int a = lane; a < g.k_in; a += 32) U[r4(i, hb + a, UK)] = ub[a] * inv;
          }
        }
      } else
      for (int i = warp; i < T; i += A2_WARPS) {
        const int node = s_node[i];
        const int E = s_E[i];
        float qp[MAXH][KP], qf[MAXH][KF > 0 ? KF : 1], qc[MAXH][KT], qs[MAXH][KT];
        float up[MAXH][KP], uf[MAXH][KF > 0 ? KF : 1], uc[MAXH][KT], us[MAXH][KT];
        float mx[MAXH], zs[MAXH];
#pragma unroll
        for (int hh = 0; hh < MAXH; ++hh) {
          const bool hv = hh < g.H;
          const int hb = hh * g.k_in;
          mx[hh] = -INFINITY;
          zs[hh] = 0.f;
#pragma unroll
          for (int j = 0; j < KP; ++j) {
            const int a = lane + 32 * j;
            qp[hh][j] = (hv && a < g.d) ? U[r4(i, hb + a, UK)] : 0.f;
            up[hh][j] = 0.f;
          }
#pragma unroll
          for (int j = 0; j < KF; ++j) {
            const int a = lane + 32 * j;
            qf[hh][j] = (hv && a < g.d_e) ? U[r4(i, hb + g.d + a, UK)] : 0.f;
            uf[hh][j] = 0.f;
          }
#pragma unroll
          for (int j = 0; j < KT; ++j) {
            const int f = lane + 32 * j;
            const bool fv = hv && f < g.half;
            qc[hh][j] = fv ? U[r4(i, hb + g.d + g.d_e + 2 * f, UK)] : 0.f;
            qs[hh][j] = fv ? U[r4(i, hb + g.d + g.d_e + 2 * f + 1, UK)] : 0.f;
            uc[hh][j] = 0.f;
            us[hh][j] = 0.f;
          }
        }
        for (int e = 0; e < E; ++e) {
          int slot = s_head[i] + e;
          if (slot >= g.L) slot -= g.L;
          const float* pay = rs.ring_pay + (((int64_t)node * g.K + l) * g.L + slot) * g.ld_d;
          const float* ft = rs.ring_feat + ((int64_t)node * g.L + slot) * g.ld_e;
          const double dt = s_tref[i] - rs.ring_t[(int64_t)node * g.L + slot];
          float kp[KP], kf[KF > 0 ? KF : 1], kc[KT], ks[KT];
#pragma unroll
          for (int j = 0; j < KP; ++j) {
            const int a = lane + 32 * j;
            kp[j] = a < g.d ? pay[a] : 0.f;
          }
#pragma unroll
          for (int j = 0; j < KF; ++j) {
            const int a = lane + 32 * j;
            kf[j] = a < g.d_e ? ft[a] : 0.f;
          }
#pragma unroll
          for (int j = 0; j < KT; ++j) {
            const int f = lane + 32 * j;
            float sv = 0.f, cv = 0.f;
            if (f < g.half) phase_sincos(w.omega[f], dt, &sv, &cv);
            kc[j] = cv * g.phi_amp;
            ks[j] = sv * g.phi_amp;
          }
#pragma unroll
          for (int hh = 0; hh < MAXH; ++hh) {
            if (hh < g.H) {
              float part = 0.f;
#pragma unroll
              for (int j = 0; j < KP; ++j) part = fmaf(qp[hh][j], kp[j], part);
#pragma unroll
              for (int j = 0; j < KF; ++j) part = fmaf(qf[hh][j], kf[j], part);
#pragma unroll
              for (int j = 0; j < KT; ++j) part = fmaf(qc[hh][j], kc[j], fmaf(qs[hh][j], ks[j], part));
              const float logit = warp_sum(part);
              const float nm = fmaxf(mx[hh], logit);
              const float sc = __expf(mx[hh] - nm);
              const float p = __expf(logit - nm);
              zs[hh] = fmaf(zs[hh], sc, p);
#pragma unroll
              for (int j = 0; j < KP; ++j) up[hh][j] = fmaf(p, kp[j], up[hh][j] * sc);
#pragma unroll
              for (int j = 0; j < KF; ++j) uf[hh][j] = fmaf(p, kf[j], uf[hh][j] * sc);
#pragma unroll
              for (int j = 0; j < KT; ++j) {
                uc[hh][j] = fmaf(p, kc[j], uc[hh][j] * sc);
                us[hh][j] = fmaf(p, ks[j], us[hh][j] * sc);
              }
              mx[hh] = nm;
            }
          }
        }
        __syncwarp();
#pragma unroll
        for (int hh = 0; hh < MAXH; ++hh) {
          if (hh < g.H) {
            const int hb = hh * g.k_in;
            const float inv = E > 0 ? 1.f / zs[hh] : 0.f;
#pragma unroll
            for (int j = 0; j < KP; ++j) {
              const int a = lane + 32 * j;
              if (a < g.d) U[r4(i, hb + a, UK)] = up[hh][j] * inv;
            }
#pragma unroll
            for (int j = 0; j < KF; ++j) {
              const int a = lane + 32 * j;
              if (a < g.d_e) U[r4(i, hb + g.d + a, UK)] = uf[hh][j] * inv;
            }
#pragma unroll
            for (int j = 0; j < KT; ++j) {
              const int f = lane + 32 * j;
              if (f < g.half) {
                U[r4(i, hb + g.d + g.d_e + 2 * f, UK)] = uc[hh][j] * inv;
                U[r4(i, hb + g.d + g.d_e + 2 * f + 1, UK)] = us[hh][j] * inv;
              }
            }
          }
        }
      }
      __syncthreads();
      // c_h = ubar_h W_V[l,h]
      gemm_staged<A2_MAXI>(U, UK, g.k_in, T, g.k_in, wv, w.ld_dk, (int64_t)g.k_in * w.ld_dk,
                           g.d_k, g.H, Cc, g.HD, g.d_k, 1.f, nullptr, 0, false, Wsm, wsm_floats);
      // out_l = c W_O  (next layer's x)
      gemm_staged<A2_MAXI>(Cc, g.HD, 0, T, g.HD, wo, w.ld_d, 0, g.d, 1, X, g.d, 0, 1.f, nullptr,
                           0, false, Wsm, wsm_floats);
      const bool last = (l == g.K - 1);
      for (int o = tid; o < T * g.d; o += A2_THREADS) {
        const int i = o / g.d, j = o % g.d;
        const int node = s_node[i];
        if (node < 0) continue;
        const float v = X[r4(i, j, g.d)];
        const int64_t idx = base + i;
        const int mode = s_mode[i];
        if (mode == 1) {  // direct node, pre-batch memory: prediction embedding only
          if (last) rs.dpred[idx * g.ld_d + j] = v;
        } else if (rs.layers_out) {
          rs.layers_out[(idx * g.K + l) * g.ld_d + j] = v;
        } else if (rs.final_out) {
          if (last) rs.final_out[idx * g.ld_d + j] = v;
        } else {
          rs.h[((int64_t)node * g.K + l) * g.ld_d + j] = v;
        }
      }
      if (last && rs.write_valid && tid < T) {
        const int node = s_node[tid];
        if (node >= 0 && s_mode[tid] != 1) {
          rs.valid[node] = 1;
          rs.valid_at[node] = rs.valid_at_ptr ? rs.valid_at_ptr[0] : rs.valid_at_const;
        }
      }
    }
    __syncthreads();
  }
}
