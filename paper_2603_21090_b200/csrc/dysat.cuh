// DySAT streaming inference (paper_2603_21090_b200/dysat.py states the model;
// SURVEY §8f row 4; the reference ships no DySAT code).
//
// Per batch (one snapshot segment):
//   k_dy_predict   link scores from the pre-batch embeddings (warp per edge)
//   k_dy_claim     endpoints -> affected list (node stamps)
//   k_dy_lists     warp per endpoint: prepend its new entries to its
//                  per-snapshot ring (newest first, L most recent)
//   k_dy_struct    warp per node: GAT over [self] + list on the static
//                  projected features P (precomputed head scores ss / sn),
//                  ELU -> compact rows
//   k_dy_temporal  128..256-thread tiles of up to 32 rows: y = z + pos[k];
//                  Q, K, V by staged-weight FFMA GEMMs (gemm.cuh); K, V rows
//                  kept in the node's history slot (k mod W); per-row warp
//                  attention over the window's cached K / V rows; emb = o W_o + y
// A snapshot roll clears the lists and runs struct + temporal over every node.
// Bytes per recomputed node (HBM): list ids 4L + L gathered P rows 4d +
// 2(W-1) history rows 4d read, 2 history rows + 1 embedding row written.
#pragma once

#include "gemm.cuh"
#include "attn4.cuh"

#define DY_TMAX 32
#define DY_THREADS 256

__global__ void k_dy_predict(stgn_dysat s, int B, const int32_t* __restrict__ src,
                             const int32_t* __restrict__ dst, double* preds) {
  const int lane = threadIdx.x & 31;
  const int warps = (int)(gridDim.x * (blockDim.x >> 5));
  for (int i = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < B; i += warps) {
    const float* eu = s.emb + (int64_t)src[i] * s.ld;
    const float* ev = s.emb + (int64_t)dst[i] * s.ld;
    double acc = 0.0;
    for (int c = lane; c < s.d; c += 32) acc += s.wpred[c] * (double)eu[c] + s.wpred[s.d + c] * (double)ev[c];
    acc = warp_sum_d(acc);
    if (lane == 0) preds[i] = 1.0 / (1.0 + exp(-(acc + s.bpred)));
  }
}

__global__ void k_dy_claim(stgn_dysat s, int B, const int32_t* __restrict__ src,
                           const int32_t* __restrict__ dst, uint32_t stamp) {
  int32_t* cnt = s.work + 2 * s.max_batch;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < 2 * B; r += gridDim.x * blockDim.x) {
    const int v = (r & 1) ? dst[r >> 1] : src[r >> 1];
    if (atomicExch(reinterpret_cast<unsigned*>(s.mark) + v, stamp) != stamp) s.work[atomicAdd(cnt, 1)] = v;
  }
}

// Entry m (0-based, batch order) of node v goes to slot head0 - 1 - m; only the
// last L survive, so a first pass counts the node's entries M.
__global__ void k_dy_lists(stgn_dysat s, int B, const int32_t* __restrict__ src,
                           const int32_t* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int warps = (int)(gridDim.x * (blockDim.x >> 5));
  const int nd = s.work[2 * s.max_batch];
  const int L = s.fanout;
  for (int i = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < nd; i += warps) {
    const int v = s.work[i];
    int M = 0;
    for (int e0 = 0; e0 < B; e0 += 32) {
      const int e = e0 + lane;
      M += __popc(__ballot_sync(0xffffffffu, e < B && (src[e] == v || dst[e] == v)));
    }
    const int head0 = s.lst_head[v];
    int m = 0;
    for (int e0 = 0; e0 < B; e0 += 32) {
      const int e = e0 + lane;
      const bool hit = e < B && (src[e] == v || dst[e] == v);
      const unsigned mask = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const int mm = m + __popc(mask & ((1u << lane) - 1u));
        if (mm >= M - L) {
          int slot = (head0 - 1 - mm) % L;
          if (slot < 0) slot += L;
          s.lst_nbr[(int64_t)v * L + slot] = src[e] == v ? dst[e] : src[e];
        }
      }
      m += __popc(mask);
    }
    if (lane == 0) {
      int h = (head0 - M) % L;
      if (h < 0) h += L;
      s.lst_head[v] = h;
      const int c = s.lst_cnt[v] + M;
      s.lst_cnt[v] = c < L ? c : L;
    }
  }
}

// Structural attention of `count` nodes (list[i], or base + i) into rows[i].
__global__ void __launch_bounds__(DY_THREADS)
k_dy_struct(stgn_dysat s, const int32_t* list, const int32_t* count_ptr, int64_t count_const,
            int64_t base) {
  __shared__ float s_alpha[DY_THREADS / 32][32 * 32];  // [head][entry]
  __shared__ int s_u[DY_THREADS / 32][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t N = count_ptr ? (int64_t)*count_ptr : count_const;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int L = s.fanout, Hs = s.heads_s, dh = s.d / s.heads_s;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += warps) {
    const int v = list ? list[i] : (int)(base + i);
    const int E = s.lst_cnt[v];
    const bool live = lane <= E;
    const int u = lane == 0 ? v : (live ? s.lst_nbr[(int64_t)v * L + (s.lst_head[v] + lane - 1) % L] : v);
    s_u[w][lane] = u;
    __syncwarp();
    // lane = head: softmax over [self] + list sequentially in the lane (no shuffles)
    for (int h = lane; h < Hs; h += 32) {
      const float sv = s.ss[(int64_t)v * Hs + h];
      float mx = -INFINITY;
      for (int j = 0; j <= E; ++j) {
        float e = sv + s.sn[(int64_t)s_u[w][j] * Hs + h];
        e = e > 0.f ? e : 0.2f * e;
        s_alpha[w][h * 32 + j] = e;
        mx = fmaxf(mx, e);
      }
      float z = 0.f;
      for (int j = 0; j <= E; ++j) {
        const float p = __expf(s_alpha[w][h * 32 + j] - mx);
        s_alpha[w][h * 32 + j] = p;
        z += p;
      }
      const float inv = 1.f / z;
      for (int j = 0; j <= E; ++j) s_alpha[w][h * 32 + j] *= inv;
    }
    __syncwarp();
    float* out = s.rows + i * s.ld;
    for (int c = lane; c < s.d; c += 32) {
      const float* al = &s_alpha[w][(c / dh) * 32];
      float z = 0.f;
      for (int j = 0; j <= E; ++j) z = fmaf(al[j], s.P[(int64_t)s_u[w][j] * s.ld + c], z);
      out[c] = z > 0.f ? z : expm1f(z);
    }
    __syncwarp();
  }
}

// Tile rows: ~75 KB of shared memory (three CTAs per SM) when the width allows,
// else up to ~220 KB.
static inline int dy_tile_rows(int d, int wsm) {
  for (int kb : {75, 220}) {
    int t = (kb * 1024 / 4 - wsm) / (5 * d) / 4 * 4;
    if (t > DY_TMAX) t = DY_TMAX;
    if (t >= 4) return t;
  }
  return 0;
}

// Temporal attention of `count` nodes whose structural rows are rows[0, count).
__global__ void __launch_bounds__(DY_THREADS)
k_dy_temporal(stgn_dysat s, const int32_t* list, const int32_t* count_ptr, int64_t count_const,
              int64_t base, int T, int wsm_floats) {
  extern __shared__ float4 dsm4[];
  const int d = s.d;
  float* Y = reinterpret_cast<float*>(dsm4);  // R4 [T][d]
  float* Q = Y + T * d;
  float* Kc = Q + T * d;
  float* Vc = Kc + T * d;
  float* O = Vc + T * d;
  float* Wsm = O + T * d;
  __shared__ int s_node[DY_TMAX];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t N = count_ptr ? (int64_t)*count_ptr : count_const;
  const int64_t k = s.snapshot;
  const int W = s.window;
  const int slot = (int)(k % W);
  const int64_t j0 = k - W + 1 > 0 ? k - W + 1 : 0;
  const int np = (int)(k - j0 + 1);
  const int Ht = s.heads_t, dt = d / Ht;
  const float scale = rsqrtf((float)dt);
  for (int64_t tb = (int64_t)blockIdx.x * T; tb < N; tb += (int64_t)gridDim.x * T) {
    if (tid < T) s_node[tid] = tb + tid < N ? (list ? list[tb + tid] : (int)(base + tb + tid)) : -1;
    for (int o = tid; o < T * d; o += blockDim.x) {
      const int i = o / d, c = o % d;
      Y[r4(i, c, d)] = tb + i < N ? s.rows[(tb + i) * s.ld + c] + s.pos[k * s.ld + c] : 0.f;
    }
    __syncthreads();
    gemm_staged<2>(Y, d, 0, T, d, s.wq, s.ld, 0, d, 1, Q, d, 0, 1.f, nullptr, 0, false, Wsm, wsm_floats);
    gemm_staged<2>(Y, d, 0, T, d, s.wk, s.ld, 0, d, 1, Kc, d, 0, 1.f, nullptr, 0, false, Wsm, wsm_floats);
    gemm_staged<2>(Y, d, 0, T, d, s.wv, s.ld, 0, d, 1, Vc, d, 0, 1.f, nullptr, 0, false, Wsm, wsm_floats);
    for (int o = tid; o < T * d; o += blockDim.x) {  // this snapshot's key / value rows
      const int i = o / d, c = o % d;
      const int v = s_node[i];
      if (v < 0) continue;
      const int64_t hr = ((int64_t)v * W + slot) * s.ld + c;
      s.hist_k[hr] = Kc[r4(i, c, d)];
      s.hist_v[hr] = Vc[r4(i, c, d)];
    }
    // fast path: lane owns CH = d / 32 consecutive elements; a head spans
    // dt / CH lanes (a power of two), so a logit is a segmented shuffle sum
    const int CH = d >> 5;
    const int lph = (d % 32 == 0 && CH <= 8 && dt % CH == 0) ? dt / CH : 0;
    const bool fast = lph > 0 && lph <= 32 && (lph & (lph - 1)) == 0;
    if (fast) {
      for (int i = warp; i < T; i += blockDim.x >> 5) {
        const int v = s_node[i];
        if (v < 0) continue;
        const int c0 = lane * CH;
        float q[8], o[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          q[x] = x < CH ? Q[r4(i, c0 + x, d)] * scale : 0.f;
          o[x] = 0.f;
        }
        float mx = -INFINITY, z = 0.f;
        for (int p = 0; p < np; ++p) {  // online softmax over the window
          const int64_t j = j0 + p;
          const float* kr = s.hist_k + ((int64_t)v * W + (int)(j % W)) * s.ld + c0;
          const float* vr = s.hist_v + ((int64_t)v * W + (int)(j % W)) * s.ld + c0;
          float part = 0.f, vv[8];
#pragma unroll
          for (int x = 0; x < 8; ++x) {
            if (x < CH) {
              const float kx = j == k ? Kc[r4(i, c0 + x, d)] : kr[x];
              vv[x] = j == k ? Vc[r4(i, c0 + x, d)] : vr[x];
              part = fmaf(q[x], kx, part);
            }
          }
          for (int m = 1; m < lph; m <<= 1) part += __shfl_xor_sync(0xffffffffu, part, m);
          const float nm = fmaxf(mx, part);
          const float sc = __expf(mx - nm), pe = __expf(part - nm);
          z = fmaf(z, sc, pe);
#pragma unroll
          for (int x = 0; x < 8; ++x) o[x] = fmaf(pe, vv[x], o[x] * sc);
          mx = nm;
        }
        const float inv = 1.f / z;
#pragma unroll
        for (int x = 0; x < 8; ++x)
          if (x < CH) O[r4(i, c0 + x, d)] = o[x] * inv;
      }
    } else
    for (int i = warp; i < T; i += blockDim.x >> 5) {
      const int v = s_node[i];
      if (v < 0) continue;
      for (int g = 0; g < Ht; ++g) {
        float lg[32];
        float mx = -INFINITY;
#pragma unroll
        for (int p = 0; p < 32; ++p) {
          if (p < np) {
            const int64_t j = j0 + p;
            float part = 0.f;
            for (int c = g * dt + lane; c < (g + 1) * dt; c += 32) {
              const float kv = j == k ? Kc[r4(i, c, d)]
                                      : s.hist_k[((int64_t)v * W + (int)(j % W)) * s.ld + c];
              part = fmaf(Q[r4(i, c, d)], kv, part);
            }
            lg[p] = warp_sum(part) * scale;
            mx = fmaxf(mx, lg[p]);
          }
        }
        float z = 0.f;
#pragma unroll
        for (int p = 0; p < 32; ++p)
          if (p < np) {
            lg[p] = __expf(lg[p] - mx);
            z += lg[p];
          }
        const float inv = 1.f / z;
        for (int c = g * dt + lane; c < (g + 1) * dt; c += 32) {
          float o = 0.f;
#pragma unroll
          for (int p = 0; p < 32; ++p) {
            if (p < np) {
              const int64_t j = j0 + p;
              const float vv = j == k ? Vc[r4(i, c, d)]
                                      : s.hist_v[((int64_t)v * W + (int)(j % W)) * s.ld + c];
              o = fmaf(lg[p], vv, o);
            }
          }
          O[r4(i, c, d)] = o * inv;
        }
      }
    }
    __syncthreads();
    gemm_staged<2>(O, d, 0, T, d, s.wo, s.ld, 0, d, 1, Q, d, 0, 1.f, nullptr, 0, false, Wsm, wsm_floats);
    for (int o = tid; o < T * d; o += blockDim.x) {
      const int i = o / d, c = o % d;
      const int v = s_node[i];
      if (v >= 0) s.emb[(int64_t)v * s.ld + c] = Q[r4(i, c, d)] + Y[r4(i, c, d)];
    }
    __syncthreads();
  }
}

// ---- tcgen05 temporal layer (d = 4 CW, CW in {16, 32}; head width DT <= CW) ----
// 128-row tiles, 512 threads = 4 TMEM lane quadrants x 4 column groups; thread
// (quadrant q, group cg, lane) owns row 32q + lane and columns [cg CW, (cg+1) CW),
// so every head lies inside one thread (softmax over the window without shuffles).
// bf16x3 GEMMs (hi*hi + hi*lo + lo*hi, fp32 accumulate) with y / o as the TMEM A
// operand and W^T (K-major bf16 hi | lo blocks, stgn_dysat.wtc) staged by TMA bulk
// copies into two shared buffers, two blocks ahead (blocks Q, K, V, O per tile).
// TMEM: A [0, d)  D_Q [d, 2d)  D_K [2d, 3d)  D_V [3d, 4d); D_E reuses D_Q.
#define DTC_THREADS 512

static inline bool dy_tc_ok(int d, int heads_t) {
  const int dt = d / heads_t;
  return (d == 64 || d == 128) && (dt == 8 || dt == 16 || dt == 32) && dt <= d / 4;
}
static inline size_t dy_tc_smem(int d) { return 1024 + 2 * (size_t)(2 * d * d * 2); }

template <int CW, int DT>
__global__ void __launch_bounds__(DTC_THREADS, 1)
k_dy_temporal_tc(stgn_dysat s, const int32_t* list, const int32_t* count_ptr, int64_t count_const,
                 int64_t base) {
  constexpr int d = 4 * CW;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sbase = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr uint32_t blk_bytes = (uint32_t)(2 * d * d * 2);
  uint16_t* Wb0 = reinterpret_cast<uint16_t*>(sbase);
  uint16_t* Wb1 = reinterpret_cast<uint16_t*>(sbase + blk_bytes);
  __shared__ int s_node[128];
  __shared__ uint64_t mbar, wbar[2];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int quad = warp & 3, cg = warp >> 2;
  const int64_t N = count_ptr ? (int64_t)*count_ptr : count_const;
  const int64_t ntiles = cdiv(N, 128);
  if ((int64_t)blockIdx.x >= ntiles) return;
  const int64_t total_blocks = cdiv(ntiles - blockIdx.x, (int64_t)gridDim.x) * 4;
  if (warp == 0) tmem_alloc(&tslot, 512);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    mbar_init(&wbar[0], 1);
    mbar_init(&wbar[1], 1);
    mbar_fence_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t trow = tmem + ((uint32_t)(32 * quad) << 16);
  const int row = 32 * quad + lane;
  auto stage = [&](int64_t Gi) {  // one thread: weight block Gi % 4 -> buffer Gi & 1
    bulk_stage((Gi & 1) ? (void*)Wb1 : (void*)Wb0, s.wtc + (Gi % 4) * (int64_t)(2 * d * d),
               blk_bytes, &wbar[Gi & 1]);
  };
  if (tid == 0) {
    stage(0);
    if (total_blocks > 1) stage(1);
  }
  int64_t G = 0;
  uint32_t mph = 0;
  auto cta_sync_tc = [&]() {
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  };
  auto issue = [&](int off, int dcol, bool commit) {  // tid 0: block G + off, A = TMEM [0, d)
    const int64_t Gi = G + off;
    mbar_wait(&wbar[Gi & 1], (uint32_t)((Gi >> 1) & 1));
    a4_mma(tmem, 0, (Gi & 1) ? Wb1 : Wb0, d, d, dcol, &mbar, false, commit);
  };
  auto wait_mma = [&](int nb) {  // the one commit covering the next nb blocks; refill
    if (tid == 0) {
      mbar_wait(&mbar, mph & 1u);
      for (int k = 0; k < nb; ++k)
        if (G + k + 2 < total_blocks) stage(G + k + 2);
    }
    ++mph;
    G += nb;
    cta_sync_tc();
  };
  const int64_t k = s.snapshot;
  const int W = s.window;
  const int slot = (int)(k % W);
  const int64_t j0 = k - W + 1 > 0 ? k - W + 1 : 0;
  const int np = (int)(k - j0 + 1);
  const float scale = rsqrtf((float)DT);
  const int c0 = cg * CW;  // this thread's columns [c0, c0 + CW)
  constexpr int DQ = d, DK = 2 * d, DV = 3 * d;
  const float* pr = s.pos + k * s.ld + c0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t tb = tile * 128;
    if (tid < 128) s_node[tid] = tb + tid < N ? (list ? list[tb + tid] : (int)(base + tb + tid)) : -1;
    __syncthreads();
    const int v = s_node[row];
    const float* yr = s.rows + (tb + row) * s.ld + c0;
    // ---- A = y = z + pos (bf16 hi | lo), this thread's CW / 16 blocks of 16 columns ----
#pragma unroll
    for (int b = 0; b < CW / 16; ++b) {
      float x[16];
#pragma unroll
      for (int t = 0; t < 16; t += 4) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        if (v >= 0) {
          const float4 r4v = *reinterpret_cast<const float4*>(yr + 16 * b + t);
          const float4 p4v = __ldg(reinterpret_cast<const float4*>(pr + 16 * b + t));
          a = make_float4(r4v.x + p4v.x, r4v.y + p4v.y, r4v.z + p4v.z, r4v.w + p4v.w);
        }
        x[t] = a.x; x[t + 1] = a.y; x[t + 2] = a.z; x[t + 3] = a.w;
      }
      const int blk = c0 / 16 + b;
      a4_st16(trow + (uint32_t)(8 * blk), trow + (uint32_t)(d / 2 + 8 * blk), x);
    }
    tmem_st_wait();
    cta_sync_tc();
    if (tid == 0) {
      issue(0, DQ, false);
      issue(1, DK, true);
    }
    wait_mma(2);
    if (tid == 0) issue(0, DV, true);
    wait_mma(1);
    // ---- this snapshot's key / value rows -> the node's history slot ----
    float* hk = s.hist_k + ((int64_t)(v >= 0 ? v : 0) * W + slot) * s.ld + c0;
    float* hv = s.hist_v + ((int64_t)(v >= 0 ? v : 0) * W + slot) * s.ld + c0;
#pragma unroll
    for (int x8 = 0; x8 < CW / 8; ++x8) {  // warp-collective TMEM loads; stores guarded
      float a8[8], b8[8];
      tmem_ld8_nw(trow + (uint32_t)(DK + c0 + 8 * x8), a8);
      tmem_ld8_nw(trow + (uint32_t)(DV + c0 + 8 * x8), b8);
      tmem_ld_wait();
      if (v >= 0) {
        reinterpret_cast<float4*>(hk + 8 * x8)[0] = make_float4(a8[0], a8[1], a8[2], a8[3]);
        reinterpret_cast<float4*>(hk + 8 * x8)[1] = make_float4(a8[4], a8[5], a8[6], a8[7]);
        reinterpret_cast<float4*>(hv + 8 * x8)[0] = make_float4(b8[0], b8[1], b8[2], b8[3]);
        reinterpret_cast<float4*>(hv + 8 * x8)[1] = make_float4(b8[4], b8[5], b8[6], b8[7]);
      }
    }
    float q[CW], o[CW];
#pragma unroll
    for (int x8 = 0; x8 < CW / 8; ++x8) {
      float t8[8];
      tmem_ld8_nw(trow + (uint32_t)(DQ + c0 + 8 * x8), t8);
      tmem_ld_wait();
#pragma unroll
      for (int t = 0; t < 8; ++t) q[8 * x8 + t] = t8[t] * scale;
    }
#pragma unroll
    for (int c = 0; c < CW; ++c) o[c] = 0.f;
    if (v >= 0) {
      // online softmax over the window, all of this thread's heads at once; the
      // current snapshot's rows are read back from the slot just written
      float mx[CW / DT], z[CW / DT];
#pragma unroll
      for (int h = 0; h < CW / DT; ++h) {
        mx[h] = -INFINITY;
        z[h] = 0.f;
      }
      for (int p = 0; p < np; ++p) {
        const int64_t j = j0 + p;
        const float* kr = s.hist_k + ((int64_t)v * W + (int)(j % W)) * s.ld + c0;
        const float* vr = s.hist_v + ((int64_t)v * W + (int)(j % W)) * s.ld + c0;
#pragma unroll
        for (int h = 0; h < CW / DT; ++h) {
          float lg = 0.f;
#pragma unroll
          for (int c = 0; c < DT; c += 4) {
            const float4 k4 = *reinterpret_cast<const float4*>(kr + h * DT + c);
            lg = fmaf(q[h * DT + c], k4.x, lg);
            lg = fmaf(q[h * DT + c + 1], k4.y, lg);
            lg = fmaf(q[h * DT + c + 2], k4.z, lg);
            lg = fmaf(q[h * DT + c + 3], k4.w, lg);
          }
          const float nm = fmaxf(mx[h], lg);
          const float sc = __expf(mx[h] - nm), pe = __expf(lg - nm);
          z[h] = fmaf(z[h], sc, pe);
#pragma unroll
          for (int c = 0; c < DT; c += 4) {
            const float4 v4 = *reinterpret_cast<const float4*>(vr + h * DT + c);
            o[h * DT + c] = fmaf(pe, v4.x, o[h * DT + c] * sc);
            o[h * DT + c + 1] = fmaf(pe, v4.y, o[h * DT + c + 1] * sc);
            o[h * DT + c + 2] = fmaf(pe, v4.z, o[h * DT + c + 2] * sc);
            o[h * DT + c + 3] = fmaf(pe, v4.w, o[h * DT + c + 3] * sc);
          }
          mx[h] = nm;
        }
      }
#pragma unroll
      for (int h = 0; h < CW / DT; ++h) {
        const float inv = 1.f / z[h];
#pragma unroll
        for (int c = 0; c < DT; ++c) o[h * DT + c] *= inv;
      }
    }
    // ---- A = o, D_E = o W_O (over D_Q) ----
#pragma unroll
    for (int b = 0; b < CW / 16; ++b) {
      float x[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) x[t] = o[16 * b + t];
      const int blk = c0 / 16 + b;
      a4_st16(trow + (uint32_t)(8 * blk), trow + (uint32_t)(d / 2 + 8 * blk), x);
    }
    tmem_st_wait();
    cta_sync_tc();
    if (tid == 0) issue(0, DQ, true);
    wait_mma(1);
    float* er = s.emb + (int64_t)(v >= 0 ? v : 0) * s.ld + c0;
#pragma unroll
    for (int x8 = 0; x8 < CW / 8; ++x8) {  // warp-collective TMEM loads; stores guarded
      float t8[8];
      tmem_ld8_nw(trow + (uint32_t)(DQ + c0 + 8 * x8), t8);
      tmem_ld_wait();
      if (v >= 0) {  // emb = o W_O + y, y re-read (L2)
        const int cc = 8 * x8;
        const float4 ra = *reinterpret_cast<const float4*>(yr + cc);
        const float4 rb = *reinterpret_cast<const float4*>(yr + cc + 4);
        const float4 pa = __ldg(reinterpret_cast<const float4*>(pr + cc));
        const float4 pb = __ldg(reinterpret_cast<const float4*>(pr + cc + 4));
        reinterpret_cast<float4*>(er + cc)[0] = make_float4(
            t8[0] + (ra.x + pa.x), t8[1] + (ra.y + pa.y), t8[2] + (ra.z + pa.z), t8[3] + (ra.w + pa.w));
        reinterpret_cast<float4*>(er + cc)[1] = make_float4(
            t8[4] + (rb.x + pb.x), t8[5] + (rb.y + pb.y), t8[6] + (rb.z + pb.z), t8[7] + (rb.w + pb.w));
      }
    }
    cta_sync_tc();
  }
  if (warp == 0) tmem_free(tmem, 512);
}
