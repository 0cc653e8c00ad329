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
// The per-node softmax walk (the only non-GEMM step) reads q~ / writes ubar
// in row-major shared memory, warp per row, lanes across the key features.
//
// Latency structure (v2): weight blocks are staged by one thread with TMA
// bulk copies (cp.async.bulk -> mbarrier complete_tx), issued as soon as the
// MMA that read the previous block commits, so staging overlaps the
// epilogues and the walk; the walk loads its ring entries in chunks of
// A3_EC (all loads of a chunk in flight before any math) and the payload
// rows of the NEXT tile are prefetched into L2 while the current tile runs.
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

#define A3_EC 5  // ring entries loaded per chunk of the walk

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

// Weight block j of layer l in issue order Q, K_0..K_{H-1}, V_0..V_{H-1}, O.
struct A3Blk {
  const float* src;
  int64_t floats;
};
__device__ __forceinline__ A3Blk a3_block(const Geo& g, const TcW& w, int l, int j) {
  if (j == 0) return {w.wq + (int64_t)l * tc_blk(w.Np_q, w.Kp_x), tc_blk(w.Np_q, w.Kp_x)};
  if (j <= g.H) {
    const int hh = j - 1;
    return {w.wk + ((int64_t)l * g.H + hh) * tc_blk(w.Np_k, w.Kp_qh), tc_blk(w.Np_k, w.Kp_qh)};
  }
  if (j <= 2 * g.H) {
    const int hh = j - 1 - g.H;
    return {w.wv + ((int64_t)l * g.H + hh) * tc_blk(w.Np_v, w.Kp_u), tc_blk(w.Np_v, w.Kp_u)};
  }
  return {w.wo + (int64_t)l * tc_blk(w.Np_o, w.Kp_c), tc_blk(w.Np_o, w.Kp_c)};
}
__device__ __forceinline__ void a3_stage_async(float* Wb, const Geo& g, const TcW& w, int l, int j,
                                               uint64_t* wbar) {
  const A3Blk b = a3_block(g, w, l, j);
  bulk_stage(Wb, b.src, (uint32_t)(b.floats * 4), wbar);
}

// L2 prefetch of the ring rows (payload of every layer, features, timestamps)
// of `T` tile rows whose node / entry count / ring head are in the arrays.
__device__ __forceinline__ void a3_prefetch_rows(const Geo& g, const RingSrc& rs, const int* nodes,
                                                 const int* Es, const int* heads, int T) {
  const int pay_b = g.ld_d * 4, feat_b = g.d_e ? g.ld_e * 4 : 0;
  const int per_entry = g.K * 5 + (feat_b ? (feat_b + 127) / 128 + 1 : 0);
  const int per_row = g.L * per_entry + 1;
  for (int x = threadIdx.x; x < T * per_row; x += A3_THREADS) {
    const int i = x / per_row, r = x % per_row;
    const int node = nodes[i];
    if (node < 0) continue;
    if (r == g.L * per_entry) {  // the row's timestamps
      prefetch_l2(rs.ring_t + (int64_t)node * g.L);
      continue;
    }
    const int e = r / per_entry, q = r % per_entry;
    if (e >= Es[i]) continue;
    int slot = heads[i] + e;
    if (slot >= g.L) slot -= g.L;
    const char* base;
    int qq, nb;
    if (q < g.K * 5) {
      const int l = q / 5;
      qq = q % 5;
      nb = pay_b;
      base = reinterpret_cast<const char*>(rs.ring_pay + (((int64_t)node * g.K + l) * g.L + slot) * g.ld_d);
    } else {
      qq = q - g.K * 5;
      nb = feat_b;
      base = reinterpret_cast<const char*>(rs.ring_feat + ((int64_t)node * g.L + slot) * g.ld_e);
    }
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(base);
    const uintptr_t line = (a0 >> 7) + (uintptr_t)qq;
    if (line > ((a0 + (uintptr_t)nb - 1) >> 7)) continue;
    prefetch_l2(reinterpret_cast<const void*>(line << 7));
  }
}

template <int KF, int MAXH>
__global__ void __launch_bounds__(A3_THREADS, 1)
attn3_kernel(Geo g, TcW w, RingSrc rs, int tmax) {
  constexpr int KP = 4;
  constexpr int KT = 2;
  constexpr int EC = (KF > 0 || MAXH > 2) ? 2 : A3_EC;
  extern __shared__ float4 smem4[];
  const int LDU = a3_ldu(g), LDC = a3_ldc(g);
  float* Ur = reinterpret_cast<float*>(smem4);  // [tmax][LDU]  q~ then ubar (both heads)
  float* Cr = Ur + (int64_t)tmax * LDU;          // [tmax][LDC]  c = [c_1..c_H]
  float* Wb = Cr + (int64_t)tmax * LDC;          // staged packed weight block
  Wb += ((128u - (smem_u32(Wb) & 127u)) & 127u) / 4;  // 128-B aligned, still a shared pointer
  __shared__ int s_node[A2_TMAX], s_E[A2_TMAX], s_head[A2_TMAX], s_mode[A2_TMAX];
  __shared__ int s_nnode[A2_TMAX], s_nE[A2_TMAX], s_nhead[A2_TMAX];  // next tile (prefetch)
  __shared__ double s_tref[A2_TMAX];
  __shared__ uint64_t bar, wbar;
  __shared__ uint32_t tslot;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int quad = warp & 3, cg = warp >> 2;  // TMEM lane quadrant, column group
  const int64_t N = rs.count();
  if (N <= 0) return;
  int T = (int)cdiv(N, gridDim.x);
  if (T > tmax) T = tmax;
  const int64_t ntiles = cdiv(N, T);
  if ((int64_t)blockIdx.x >= ntiles) return;
  const int64_t pre_rows = rs.fused ? (int64_t)rs.pre_n[0] : N;
  const int64_t d_rows = rs.fused ? (int64_t)rs.post_n[0] : 0;

  if (warp == 0) tmem_alloc(&tslot, 512);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&wbar, 1);
    mbar_fence_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) a3_stage_async(Wb, g, w, 0, 0, &wbar);  // Q of layer 0, first tile
  const uint32_t tmem = tslot;
  uint32_t phase = 0, wphase = 0;
  const uint32_t lane_base = (uint32_t)(32 * quad) << 16;
  const int row = 32 * quad + lane;  // this thread's tile row in TMEM epilogues
  const int nblk = 2 + 2 * g.H;      // weight blocks per layer

  // one weight block: wait for its staging, MMA, wait for the MMA, then stage
  // the next block into the freed buffer (overlapping the caller's epilogue)
  auto gemm = [&](int l, int j, int a_hi, int a_lo, int Np, int Kp, int dcol, bool more) {
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    mbar_wait(&wbar, wphase);
    wphase ^= 1;
    if (tid == 0) a3_mma(tmem, a_hi, a_lo, Wb, Np, Kp, dcol, &bar);
    mbar_wait(&bar, phase);
    phase ^= 1;
    tc_fence_after();
    if (tid == 0 && more) {
      int nl = l, nj = j + 1;
      if (nj == nblk) { nj = 0; nl = (l + 1) % g.K; }
      a3_stage_async(Wb, g, w, nl, nj, &wbar);
    }
  };

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * T;
    const int64_t nbase = (tile + gridDim.x) * T;
    const bool has_next = tile + gridDim.x < ntiles;
    const bool quad_live = 32 * quad < T;
    if (tid < A2_TMAX) {
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
    } else if (tid >= 256 && tid < 256 + A2_TMAX) {  // next tile's ring meta, for the prefetch
      const int i = tid - 256;
      const int64_t idx = nbase + i;
      int node = -1, E = 0, head = 0;
      if (has_next && i < T && idx < N) {
        node = rs.node(idx);
        const int cc = node >= 0 ? rs.ring_ccnt[node] : 0;
        E = node < 0 ? 0 : (cc >= 0 ? cc : (rs.use_store ? rs.ring_cnt[node] : 0));
        head = node >= 0 ? rs.ring_head[node] : 0;
      }
      s_nnode[i] = node; s_nE[i] = E; s_nhead[i] = head;
    }
    __syncthreads();
    if (tile == blockIdx.x) a3_prefetch_rows(g, rs, s_node, s_E, s_head, T);
    if (has_next) a3_prefetch_rows(g, rs, s_nnode, s_nE, s_nhead, T);
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
      const bool last = (l == g.K - 1);
      const float* bq = w.bq + (int64_t)l * g.HD;
      // ---- q = x W_Q + b -> per-head A blocks for the q~ GEMMs ----
      gemm(l, 0, 0, w.Kp_x, w.Np_q, w.Kp_x, w.dq, true);
      const int aq_lo = g.H * w.Kp_qh;
      if (quad_live) {
        for (int c0 = 8 * cg; c0 < g.H * w.Kp_qh; c0 += 32) {
          // destination columns c0..c0+7 of the Q A-region: head hh, feature b
          float v[8], h8[8], l8[8];
          const int hh = c0 / w.Kp_qh;
          const int b0 = c0 - hh * w.Kp_qh;
          const int src0 = hh * g.d_k + b0;  // source feature hh*d_k + b (b < d_k)
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
        gemm(l, 1 + hh, hh * w.Kp_qh, aq_lo + hh * w.Kp_qh, w.Np_k, w.Kp_qh, w.dqt, true);
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
      // ---- per-node softmax walk over the ring entries, ubar in place ----
      for (int i = warp; i < T; i += A3_WARPS) {
        const int node = s_node[i];
        const int E = s_E[i];
        const int hd = s_head[i];
        const double tref = s_tref[i];
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
        const float* payb = rs.ring_pay + ((int64_t)node * g.K + l) * g.L * g.ld_d;
        const float* ftb = rs.ring_feat + (int64_t)node * g.L * g.ld_e;
        const double* tb = rs.ring_t + (int64_t)node * g.L;
        for (int e0 = 0; e0 < E; e0 += EC) {
          // all loads of the chunk first (independent, in flight together)
          float kp[EC][KP], kf[EC][KF > 0 ? KF : 1];
          double dtv[EC];
#pragma unroll
          for (int u = 0; u < EC; ++u) {
            const bool ev = e0 + u < E;
            int slot = ev ? hd + e0 + u : 0;
            if (slot >= g.L) slot -= g.L;
            const float* pay = payb + (int64_t)slot * g.ld_d;
#pragma unroll
            for (int j = 0; j < KP; ++j) {
              const int a = lane + 32 * j;
              kp[u][j] = (ev && a < g.d) ? __ldg(pay + a) : 0.f;
            }
#pragma unroll
            for (int j = 0; j < KF; ++j) {
              const int a = lane + 32 * j;
              kf[u][j] = (ev && a < g.d_e) ? __ldg(ftb + (int64_t)slot * g.ld_e + a) : 0.f;
            }
            dtv[u] = ev ? tref - __ldg(tb + slot) : 0.0;
          }
          float lg[EC][MAXH];
          float kc[EC][KT], ks[EC][KT];
#pragma unroll
          for (int u = 0; u < EC; ++u) {
#pragma unroll
            for (int j = 0; j < KT; ++j) {
              const int f = lane + 32 * j;
              float sv = 0.f, cv = 0.f;
              if (f < g.half) phase_sincos(w.omega[f], dtv[u], &sv, &cv);
              kc[u][j] = cv * g.phi_amp;
              ks[u][j] = sv * g.phi_amp;
            }
#pragma unroll
            for (int hh = 0; hh < MAXH; ++hh) {
              float part = 0.f;
              if (hh < g.H) {
#pragma unroll
                for (int j = 0; j < KP; ++j) part = fmaf(qp[hh][j], kp[u][j], part);
#pragma unroll
                for (int j = 0; j < KF; ++j) part = fmaf(qf[hh][j], kf[u][j], part);
#pragma unroll
                for (int j = 0; j < KT; ++j)
                  part = fmaf(qc[hh][j], kc[u][j], fmaf(qs[hh][j], ks[u][j], part));
              }
              lg[u][hh] = warp_sum(part);
            }
          }
#pragma unroll
          for (int hh = 0; hh < MAXH; ++hh) {
            if (hh < g.H) {
              float cm = -INFINITY;
#pragma unroll
              for (int u = 0; u < EC; ++u)
                if (e0 + u < E) cm = fmaxf(cm, lg[u][hh]);
              const float nm = fmaxf(mx[hh], cm);
              const float sc = __expf(mx[hh] - nm);
              zs[hh] *= sc;
#pragma unroll
              for (int j = 0; j < KP; ++j) up[hh][j] *= sc;
#pragma unroll
              for (int j = 0; j < KF; ++j) uf[hh][j] *= sc;
#pragma unroll
              for (int j = 0; j < KT; ++j) {
                uc[hh][j] *= sc;
                us[hh][j] *= sc;
              }
#pragma unroll
              for (int u = 0; u < EC; ++u) {
                if (e0 + u < E) {
                  const float p = __expf(lg[u][hh] - nm);
                  zs[hh] += p;
#pragma unroll
                  for (int j = 0; j < KP; ++j) up[hh][j] = fmaf(p, kp[u][j], up[hh][j]);
#pragma unroll
                  for (int j = 0; j < KF; ++j) uf[hh][j] = fmaf(p, kf[u][j], uf[hh][j]);
#pragma unroll
                  for (int j = 0; j < KT; ++j) {
                    uc[hh][j] = fmaf(p, kc[u][j], uc[hh][j]);
                    us[hh][j] = fmaf(p, ks[u][j], us[hh][j]);
                  }
                }
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
        gemm(l, 1 + g.H + hh, 0, w.Kp_u, w.Np_v, w.Kp_u, w.dv, true);
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
      }
      __syncthreads();  // every column group's c rows are in Cr
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
      gemm(l, nblk - 1, 0, w.Kp_c, w.Np_o, w.Kp_c, w.dO, !last || has_next);
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
              } else if (rs.layers_out) {
                rs.layers_out[(idx * g.K + l) * g.ld_d + j] = x;
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
    }
    tc_fence_before();
    __syncthreads();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tmem, 512);
}
