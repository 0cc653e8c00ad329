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
