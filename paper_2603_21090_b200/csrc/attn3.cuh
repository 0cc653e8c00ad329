// Tensor-core (tcgen05) version of the engine recompute kernel.
//
// Same function and row scheduling as attn2_kernel (one wave of row tiles,
// fused pre/post-memory rows), but the four dense GEMMs of every layer run
// on the 5th-generation tensor cores:
//   q = x W_Q + b,  qk_h = W_K,h q_h / sqrt(d_k),  c_h = ubar_h W_V,h,  out = c W_O
// as split-TF32 UMMAs (hi*hi + hi*lo + lo*hi, fp32 accumulate in TMEM).
// Activations are the A operand *in TMEM* (lane = node row of the tile,
// 32-bit column = k), weights the K-major B operand in shared memory,
// pre-packed on the host as [hi block | lo block] per GEMM. Accumulators
// come back with tcgen05.ld (lane = node, column = output feature), so
// epilogues write the next GEMM's A operand straight back into TMEM.
// The per-node online-softmax walk (the only non-GEMM step) is the attn2
// code reading q~ / writing ubar in row-major shared memory.
#pragma once

#include "attn2.cuh"
#include "tc.cuh"

struct TcW {
  const float *wq, *wk, *wv, *wo;  // packed B operands (stgn.h), per layer [hi | lo]
  const float* bq;                 // [K][HD]
  const double* omega;
  int Np_q, Kp_x, Np_k, Kp_qh, Np_v, Kp_u, Np_o, Kp_c;
  int dq, dqt, dv, dO;             // TMEM column offsets of the accumulators
};

static inline int r8(int x) { return (x + 7) & ~7; }
static inline int r16(int x) { return (x + 15) & ~15; }

// TMEM column plan; returns false if it does not fit in 512 columns.
static inline bool tc_plan(const Geo& g, TcW* w) {
  w->Kp_x = r8(g.d);
  w->Np_q = r16(g.HD);
  w->Kp_qh = r8(g.d_k);
  w->Np_k = r16(g.k_in);
  w->Kp_u = r8(g.k_in);
  w->Np_v = r16(g.d_k);
  w->Kp_c = r8(g.HD);
  w->Np_o = r16(g.d);
  auto up32 = [](int x) { return (x + 31) & ~31; };
  const int aq = 2 * g.H * w->Kp_qh;
  w->dq = up32(std::max(2 * w->Kp_x, aq));
  w->dqt = up32(aq);
  w->dv = up32(2 * w->Kp_u);
  w->dO = up32(std::max(2 * w->Kp_c, 2 * w->Kp_x));
  return w->dq + w->Np_q + 16 <= 512 && w->dqt + w->Np_k <= 512 && w->dv + w->Np_v <= 512 &&
         w->dO + w->Np_o <= 512 && w->Np_k <= 256 && w->Np_q <= 256 && w->Np_o <= 256 &&
         g.d <= 128 && g.half <= 64 && g.d_e <= 192;
}

// floats of one packed GEMM block (hi + lo)
__host__ __device__ inline int64_t tc_blk(int Np, int Kp) { return 2ll * Np * Kp; }

#define A3_THREADS 512
#define A3_WARPS 16

// per-row stride of the q~/ubar rows (odd: conflict-free column access by row-lanes)
__host__ __device__ inline int a3_ldu(const Geo& g) { return (g.H * g.k_in) | 1; }
__host__ __device__ inline int a3_ldc(const Geo& g) { return g.HD | 1; }

static inline int64_t attn3_row_floats(const Geo& g) { return a3_ldu(g) + a3_ldc(g); }
static inline int64_t attn3_wbuf_floats(const Geo& g, const TcW& w) {
  int64_t m = tc_blk(w.Np_q, w.Kp_x);
  m = std::max(m, tc_blk(w.Np_k, w.Kp_qh));
  m = std::max(m, tc_blk(w.Np_v, w.Kp_u));
  m = std::max(m, tc_blk(w.Np_o, w.Kp_c));
  return m;
}

// all threads: copy one packed weight block into shared memory
__device__ __forceinline__ void a3_stage(float* Wb, const float* __restrict__ src, int64_t nfl) {
  const uint32_t sb = smem_u32(Wb);
  for (int64_t x = threadIdx.x; x < nfl / 4; x += A3_THREADS)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sb + 16u * (uint32_t)x),
                 "l"(src + 4 * x));
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  fence_async_smem();
}

// one thread: split-TF32 MMAs, A (TMEM hi at a_hi, lo at a_lo) x B (smem block), then commit
__device__ __forceinline__ void a3_mma(uint32_t tmem, int a_hi, int a_lo, const float* Wb, int Np,
                                       int Kp, int dcol, uint64_t* bar) {
  tc_fence_after();
  const uint32_t idesc = umma_idesc_tf32(128, Np) & ~((1u << 15) | (1u << 16));  // K-major
  const uint32_t sbo = (uint32_t)(Kp / 4) * 128u;
  const uint32_t bh = smem_u32(Wb), bl = bh + (uint32_t)Np * Kp * 4u;
  for (int s = 0; s < Kp / 8; ++s) {
    const uint32_t off = (uint32_t)s * 256u;
    const uint64_t dh = umma_desc(bh + off, 128, sbo), dl = umma_desc(bl + off, 128, sbo);
    const uint32_t ah = tmem + (uint32_t)(a_hi + 8 * s), al = tmem + (uint32_t)(a_lo + 8 * s);
    umma_tf32_ts(tmem + (uint32_t)dcol, ah, dh, idesc, s > 0 ? 1u : 0u);
    umma_tf32_ts(tmem + (uint32_t)dcol, ah, dl, idesc, 1u);
    umma_tf32_ts(tmem + (uint32_t)dcol, al, dh, idesc, 1u);
  }
  umma_commit(bar);
}

template <int KF, int MAXH>
__global__ void __launch_bounds__(A3_THREADS, 1)
attn3_kernel(Geo g, TcW w, RingSrc rs, int tmax) {
  constexpr int KP = 4;
  constexpr int KT = 2;
  extern __shared__ float4 smem4[];
  const int LDU = a3_ldu(g), LDC = a3_ldc(g);
  float* Ur = reinterpret_cast<float*>(smem4);  // [tmax][LDU]  q~ then ubar (both heads)
  float* Cr = Ur + (int64_t)tmax * LDU;          // [tmax][LDC]  c = [c_1..c_H]
  float* Wb = Cr + (int64_t)tmax * LDC;          // staged packed weight block
  Wb = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(Wb) + 127) & ~uintptr_t(127));
  __shared__ int s_node[A2_TMAX], s_E[A2_TMAX], s_head[A2_TMAX], s_mode[A2_TMAX];
  __shared__ double s_tref[A2_TMAX];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int quad = warp & 3, cg = warp >> 2;  // TMEM lane quadrant, column group
  const int64_t N = rs.count();
  if (N <= 0) return;
  int T = (int)cdiv(N, gridDim.x);
  if (T > tmax) T = tmax;
  const int64_t ntiles = cdiv(N, T);
  const int64_t pre_rows = rs.fused ? (int64_t)rs.pre_n[0] : N;
  const int64_t d_rows = rs.fused ? (int64_t)rs.post_n[0] : 0;
  const int pay_lines = (g.d * 4 + 127) / 128;
  const int feat_lines = g.d_e ? (g.d_e * 4 + 127) / 128 : 0;

  if (warp == 0) tmem_alloc(&tslot, 512);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  uint32_t phase = 0;
  const uint32_t lane_base = (uint32_t)(32 * quad) << 16;
  const int row = 32 * quad + lane;  // this thread's tile row in TMEM epilogues
  const bool quad_live_base = true;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * T;
    const bool quad_live = quad_live_base && (32 * quad < T);
    if (tid < A2_TMAX) {
      const int i = tid;
      const int64_t idx = base + i;
      int node = -1, E = 0, head = 0, mode = 0;
      double tref = 0.0;
      if (i < T && idx < N) {
        node = rs.node(idx);
        if (rs.fused) mode = idx >= pre_rows ? 2 : (idx < d_rows ? 1 : 0);
        const int cc = rs.ring_ccnt[node];
        E = cc >= 0 ? cc : (rs.use_store ? rs.ring_cnt[node] : 0);
        head = rs.ring_head[node];
        if (E > 0) tref = rs.ring_t[(int64_t)node * g.L + head];
      }
      s_node[i] = node; s_E[i] = E; s_head[i] = head; s_tref[i] = tref; s_mode[i] = mode;
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
    {  // L2 prefetch of the tile's payload / feature rows
      const int per_entry = g.K * pay_lines + feat_lines;
      const int total = T * g.L * per_entry;
      for (int x = tid; x < total; x += A3_THREADS) {
        const int i = x / (g.L * per_entry);
        const int rem = x % (g.L * per_entry);
        const int e = rem / per_entry, q = rem % per_entry;
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
    // x_0 -> TMEM A region (hi at col 0, lo at col Kp_x)
    if (quad_live) {
      const int node = row < T ? s_node[row] : -1;
      for (int c0 = 8 * cg; c0 < w.Kp_x; c0 += 32) {
        float h8[8], l8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int j = c0 + q;
          float v = 0.f;
          if (node >= 0 && j < g.d_s)
            v = s_mode[row] == 2 ? rs.mem_post[(base + row - pre_rows) * g.ld_s + j]
                                 : rs.mem[(int64_t)node * g.ld_s + j];
          h8[q] = v;
          l8[q] = tf32_lo(v);
        }
        tmem_st8(tmem + lane_base + (uint32_t)c0, h8);
        tmem_st8(tmem + lane_base + (uint32_t)(w.Kp_x + c0), l8);
      }
      tmem_st_wait();
    }

    for (int l = 0; l < g.K; ++l) {
      const float* bq = w.bq + (int64_t)l * g.HD;
      // ---- q = x W_Q + b -> per-head A blocks for the q~ GEMMs ----
      a3_stage(Wb, w.wq + (int64_t)l * tc_blk(w.Np_q, w.Kp_x), tc_blk(w.Np_q, w.Kp_x));
      tc_fence_before();
      __syncthreads();
      if (tid == 0) a3_mma(tmem, 0, w.Kp_x, Wb, w.Np_q, w.Kp_x, w.dq, &bar);
      mbar_wait(&bar, phase);
      phase ^= 1;
      tc_fence_after();
      const int aq_lo = g.H * w.Kp_qh;
      if (quad_live) {
        for (int c0 = 8 * cg; c0 < g.H * w.Kp_qh; c0 += 32) {
          // destination columns c0..c0+7 of the Q A-region: head hh, feature b
          float v[8], h8[8], l8[8];
          const int hh = c0 / w.Kp_qh;
          const int b0 = c0 - hh * w.Kp_qh;
          // source feature index hh*d_k + b for b < d_k (padding -> 0)
          const int src0 = hh * g.d_k + b0;
          // the 8 destination columns map to contiguous source features while b < d_k
          tmem_ld8(tmem + lane_base + (uint32_t)(w.dq + (src0 & ~7)), v);
          float v2[8];
          tmem_ld8(tmem + lane_base + (uint32_t)(w.dq + (src0 & ~7) + 8), v2);
          const int sh = src0 & 7;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int b = b0 + q;
            float x = 0.f;
            if (b < g.d_k) {
              const int si = sh + q;
              x = (si < 8 ? v[si] : v2[si - 8]) + bq[hh * g.d_k + b];
            }
            h8[q] = x;
            l8[q] = tf32_lo(x);
          }
          tmem_st8(tmem + lane_base + (uint32_t)c0, h8);
          tmem_st8(tmem + lane_base + (uint32_t)(aq_lo + c0), l8);
        }
        tmem_st_wait();
      }
      // ---- q~_h = W_K,h q_h / sqrt(d_k) -> Ur rows ----
      for (int hh = 0; hh < g.H; ++hh) {
        tc_fence_before();
        __syncthreads();  // previous MMA consumers / A writes done before restaging
        a3_stage(Wb, w.wk + ((int64_t)l * g.H + hh) * tc_blk(w.Np_k, w.Kp_qh),
                 tc_blk(w.Np_k, w.Kp_qh));
        tc_fence_before();
        __syncthreads();
        if (tid == 0)
          a3_mma(tmem, hh * w.Kp_qh, aq_lo + hh * w.Kp_qh, Wb, w.Np_k, w.Kp_qh, w.dqt, &bar);
        mbar_wait(&bar, phase);
        phase ^= 1;
        tc_fence_after();
        if (quad_live) {
          for (int c0 = 8 * cg; c0 < g.k_in; c0 += 32) {
            float v[8];
            tmem_ld8(tmem + lane_base + (uint32_t)(w.dqt + c0), v);
            if (row < T) {
#pragma unroll
              for (int q = 0; q < 8; ++q)
                if (c0 + q < g.k_in) Ur[(int64_t)row * LDU + hh * g.k_in + c0 + q] = v[q] * g.inv_sqrt_dk;
            }
          }
        }
      }
      __syncthreads();
      // ---- per-node online softmax over the ring entries (attn2), ubar in place ----
      for (int i = warp; i < T; i += A3_WARPS) {
        const int node = s_node[i];
        const int E = s_E[i];
        float* Ui = Ur + (int64_t)i * LDU;
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
            qp[hh][j] = (hv && a < g.d) ? Ui[hb + a] : 0.f;
            up[hh][j] = 0.f;
          }
#pragma unroll
          for (int j = 0; j < KF; ++j) {
            const int a = lane + 32 * j;
            qf[hh][j] = (hv && a < g.d_e) ? Ui[hb + g.d + a] : 0.f;
            uf[hh][j] = 0.f;
          }
#pragma unroll
          for (int j = 0; j < KT; ++j) {
            const int f = lane + 32 * j;
            const bool fv = hv && f < g.half;
            qc[hh][j] = fv ? Ui[hb + g.d + g.d_e + 2 * f] : 0.f;
            qs[hh][j] = fv ? Ui[hb + g.d + g.d_e + 2 * f + 1] : 0.f;
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
              if (a < g.d) Ui[hb + a] = up[hh][j] * inv;
            }
#pragma unroll
            for (int j = 0; j < KF; ++j) {
              const int a = lane + 32 * j;
              if (a < g.d_e) Ui[hb + g.d + a] = uf[hh][j] * inv;
            }
#pragma unroll
            for (int j = 0; j < KT; ++j) {
              const int f = lane + 32 * j;
              if (f < g.half) {
                Ui[hb + g.d + g.d_e + 2 * f] = uc[hh][j] * inv;
                Ui[hb + g.d + g.d_e + 2 * f + 1] = us[hh][j] * inv;
              }
            }
          }
        }
      }
      __syncthreads();
      // ---- c_h = ubar_h W_V,h -> Cr rows ----
      for (int hh = 0; hh < g.H; ++hh) {
        if (quad_live) {
          for (int c0 = 8 * cg; c0 < w.Kp_u; c0 += 32) {
            float h8[8], l8[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int a = c0 + q;
              const float x = (row < T && a < g.k_in) ? Ur[(int64_t)row * LDU + hh * g.k_in + a] : 0.f;
              h8[q] = x;
              l8[q] = tf32_lo(x);
            }
            tmem_st8(tmem + lane_base + (uint32_t)c0, h8);
            tmem_st8(tmem + lane_base + (uint32_t)(w.Kp_u + c0), l8);
          }
          tmem_st_wait();
        }
        a3_stage(Wb, w.wv + ((int64_t)l * g.H + hh) * tc_blk(w.Np_v, w.Kp_u), tc_blk(w.Np_v, w.Kp_u));
        tc_fence_before();
        __syncthreads();
        if (tid == 0) a3_mma(tmem, 0, w.Kp_u, Wb, w.Np_v, w.Kp_u, w.dv, &bar);
        mbar_wait(&bar, phase);
        phase ^= 1;
        tc_fence_after();
        if (quad_live) {
          for (int c0 = 8 * cg; c0 < g.d_k; c0 += 32) {
            float v[8];
            tmem_ld8(tmem + lane_base + (uint32_t)(w.dv + c0), v);
            if (row < T) {
#pragma unroll
              for (int q = 0; q < 8; ++q)
                if (c0 + q < g.d_k) Cr[(int64_t)row * LDC + hh * g.d_k + c0 + q] = v[q];
            }
          }
        }
        tc_fence_before();
        __syncthreads();  // A region / weight buffer are reused by the next head
      }
      // ---- out_l = c W_O ----
      if (quad_live) {
        for (int c0 = 8 * cg; c0 < w.Kp_c; c0 += 32) {
          float h8[8], l8[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int a = c0 + q;
            const float x = (row < T && a < g.HD) ? Cr[(int64_t)row * LDC + a] : 0.f;
            h8[q] = x;
            l8[q] = tf32_lo(x);
          }
          tmem_st8(tmem + lane_base + (uint32_t)c0, h8);
          tmem_st8(tmem + lane_base + (uint32_t)(w.Kp_c + c0), l8);
        }
        tmem_st_wait();
      }
      a3_stage(Wb, w.wo + (int64_t)l * tc_blk(w.Np_o, w.Kp_c), tc_blk(w.Np_o, w.Kp_c));
      tc_fence_before();
      __syncthreads();
      if (tid == 0) a3_mma(tmem, 0, w.Kp_c, Wb, w.Np_o, w.Kp_c, w.dO, &bar);
      mbar_wait(&bar, phase);
      phase ^= 1;
      tc_fence_after();
      const bool last = (l == g.K - 1);
      if (quad_live) {
        const int node = row < T ? s_node[row] : -1;
        const int mode = row < T ? s_mode[row] : 0;
        const int64_t idx = base + row;
        for (int c0 = 8 * cg; c0 < w.Kp_x; c0 += 32) {
          float v[8];
          tmem_ld8(tmem + lane_base + (uint32_t)(w.dO + c0), v);
          float h8[8], l8[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int j = c0 + q;
            const float x = (j < g.d) ? v[q] : 0.f;
            h8[q] = x;
            l8[q] = tf32_lo(x);
            if (node >= 0 && j < g.d) {
              if (mode == 1) {
                if (last) rs.dpred[idx * g.ld_d + j] = x;
              } else if (rs.final_out) {
                if (last) rs.final_out[idx * g.ld_d + j] = x;
              } else {
                rs.h[((int64_t)node * g.K + l) * g.ld_d + j] = x;
              }
            }
          }
          if (!last) {  // next layer's query input x_{l+1}
            tmem_st8(tmem + lane_base + (uint32_t)c0, h8);
            tmem_st8(tmem + lane_base + (uint32_t)(w.Kp_x + c0), l8);
          }
        }
        if (!last) tmem_st_wait();
      }
      if (last && rs.write_valid && tid < T) {
        const int node = s_node[tid];
        if (node >= 0 && s_mode[tid] != 1) {
          rs.valid[node] = 1;
          rs.valid_at[node] = rs.valid_at_ptr ? rs.valid_at_ptr[0] : rs.valid_at_const;
        }
      }
      tc_fence_before();
      __syncthreads();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tmem, 512);
}
