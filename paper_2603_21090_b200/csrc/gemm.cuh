// Row-tile GEMM for the node-batched dense steps (SIMT fp32, FFMA).
//
// Activations live in shared memory in an "R4" layout: rows are grouped
// by four and, for every k, the four rows' values are contiguous
//     addr(i, k) = ((i >> 2) * ld + k) * 4 + (i & 3)
// so one 16-byte broadcast load feeds four rows. Weights are read from
// global (L1/L2 resident, shared by every CTA) as float2 pairs of
// adjacent columns; a thread owns a 4-row x 2-column register block.
#pragma once

#include "common.cuh"

__device__ __forceinline__ int r4(int i, int k, int ld) { return (((i >> 2) * ld + k) << 2) + (i & 3); }

enum Act { ACT_NONE = 0, ACT_SIGMOID = 1, ACT_TANH = 2 };

// C[T][N] (=|+=) alpha * A[T][kd] W[kd][N] (+ bias[N])
// A: R4 (lda), C: R4 (ldc), W: global row-major with even row stride ldw
// (padded, zero-filled beyond N). T must be a multiple of 4.
__device__ __forceinline__ void gemm_r4(const float* __restrict__ A, int lda, int T, int kd,
                                        const float* __restrict__ W, int ldw, int N,
                                        float* __restrict__ C, int ldc, float alpha,
                                        const float* __restrict__ bias, bool accumulate,
                                        int tid, int nthreads) {
  constexpr int KB = 8;  // weight rows loaded per batch (kept in flight together)
  const int ncp = (N + 1) >> 1;
  const int items = ncp * (T >> 2);
  const int ws = ldw >> 1;
  for (int o = tid; o < items; o += nthreads) {
    const int cp = o % ncp;
    const int rg = o / ncp;
    const float4* a4 = reinterpret_cast<const float4*>(A) + (int64_t)rg * lda;
    const float2* wp = reinterpret_cast<const float2*>(W + 2 * cp);
    float c00 = 0.f, c01 = 0.f, c10 = 0.f, c11 = 0.f, c20 = 0.f, c21 = 0.f, c30 = 0.f, c31 = 0.f;
    float2 wb[KB];
#pragma unroll
    for (int u = 0; u < KB; ++u) wb[u] = u < kd ? __ldg(wp + u * ws) : make_float2(0.f, 0.f);
    for (int k0 = 0; k0 < kd; k0 += KB) {
      float2 wn[KB];
      const float2* wq = wp + (int64_t)(k0 + KB) * ws;
#pragma unroll
      for (int u = 0; u < KB; ++u)
        wn[u] = (k0 + KB + u < kd) ? __ldg(wq + u * ws) : make_float2(0.f, 0.f);
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        if (k0 + u < kd) {
          const float4 a = a4[k0 + u];
          const float2 w = wb[u];
          c00 = fmaf(a.x, w.x, c00); c01 = fmaf(a.x, w.y, c01);
          c10 = fmaf(a.y, w.x, c10); c11 = fmaf(a.y, w.y, c11);
          c20 = fmaf(a.z, w.x, c20); c21 = fmaf(a.z, w.y, c21);
          c30 = fmaf(a.w, w.x, c30); c31 = fmaf(a.w, w.y, c31);
        }
      }
#pragma unroll
      for (int u = 0; u < KB; ++u) wb[u] = wn[u];
    }
    const int n0 = 2 * cp;
    float b0 = 0.f, b1 = 0.f;
    if (bias) {
      b0 = bias[n0];
      if (n0 + 1 < N) b1 = bias[n0 + 1];
    }
    float4* c4 = reinterpret_cast<float4*>(C) + (int64_t)rg * ldc + n0;
    float4 v0 = make_float4(alpha * c00 + b0, alpha * c10 + b0, alpha * c20 + b0, alpha * c30 + b0);
    float4 v1 = make_float4(alpha * c01 + b1, alpha * c11 + b1, alpha * c21 + b1, alpha * c31 + b1);
    if (accumulate) {
      float4 p0 = c4[0];
      v0.x += p0.x; v0.y += p0.y; v0.z += p0.z; v0.w += p0.w;
    }
    c4[0] = v0;
    if (n0 + 1 < N) {
      if (accumulate) {
        float4 p1 = c4[1];
        v1.x += p1.x; v1.y += p1.y; v1.z += p1.z; v1.w += p1.w;
      }
      c4[1] = v1;
    }
  }
}

// Grouped GEMM with shared-memory-staged weights. G independent GEMMs
// (e.g. attention heads) run concurrently:
//   C_g[T][N] (=|+=) alpha * A_g[T][kd] W_g[kd][N] (+ bias_g)
// A_g = R4 columns [g*a_hoff, g*a_hoff+kd) of A (lda), C_g = R4 columns
// [g*c_hoff, ...) of C (ldc), W_g = W + g*w_hstride (row stride ldw, a
// multiple of 4, zero-padded). Weight rows are copied into Wsm in chunks
// by every thread with 16-byte loads (one L2 round trip per chunk instead
// of one per k step), then each thread accumulates up to MAXI 4x2 blocks
// from shared memory. Must be called by all threads of the block.
template <int MAXI>
__device__ __forceinline__ void gemm_staged(const float* A, int lda, int a_hoff, int T, int kd,
                                            const float* __restrict__ W, int ldw,
                                            int64_t w_hstride, int N, int G, float* C, int ldc,
                                            int c_hoff, float alpha, const float* bias,
                                            int bias_hstride, bool accumulate, float* Wsm,
                                            int wsm_floats) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int ncp = (N + 1) >> 1;
  const int per_g = ncp * (T >> 2);
  const int items = G * per_g;
  const int wc = (N + 3) & ~3;  // staged columns per weight row (row stride in Wsm)
  int KC = wsm_floats / (G * wc);
  if (KC > kd) KC = kd;
  for (int base = 0; base < items; base += MAXI * nt) {
    float acc[MAXI][8];
#pragma unroll
    for (int it = 0; it < MAXI; ++it)
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[it][q] = 0.f;
    for (int k0 = 0; k0 < kd; k0 += KC) {
      const int kc = kd - k0 < KC ? kd - k0 : KC;
      __syncthreads();  // previous chunk fully consumed
      const int row4 = wc >> 2;
      const int per_g4 = kc * row4;
      // cp.async: every thread fires all of its 16-byte copies, then waits once
      const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(Wsm);
      for (int x = tid; x < G * per_g4; x += nt) {
        const int g = x / per_g4, rem = x - g * per_g4;
        const int r = rem / row4, c4 = rem - r * row4;
        const float* src = W + g * w_hstride + (int64_t)(k0 + r) * ldw + 4 * c4;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + 16u * x),
                     "l"(src));
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();
#pragma unroll
      for (int it = 0; it < MAXI; ++it) {
        const int o = base + it * nt + tid;
        if (o < items) {
          const int g = o / per_g, rem = o - g * per_g;
          const int cp = rem % ncp, rg = rem / ncp;
          const float4* a4 = reinterpret_cast<const float4*>(A) + (int64_t)rg * lda + g * a_hoff + k0;
          const float2* w2 = reinterpret_cast<const float2*>(Wsm + g * kc * wc) + cp;
          float c00 = acc[it][0], c01 = acc[it][1], c10 = acc[it][2], c11 = acc[it][3];
          float c20 = acc[it][4], c21 = acc[it][5], c30 = acc[it][6], c31 = acc[it][7];
#pragma unroll 4
          for (int k = 0; k < kc; ++k) {
            const float4 a = a4[k];
            const float2 w = w2[k * (wc >> 1)];
            c00 = fmaf(a.x, w.x, c00); c01 = fmaf(a.x, w.y, c01);
            c10 = fmaf(a.y, w.x, c10); c11 = fmaf(a.y, w.y, c11);
            c20 = fmaf(a.z, w.x, c20); c21 = fmaf(a.z, w.y, c21);
            c30 = fmaf(a.w, w.x, c30); c31 = fmaf(a.w, w.y, c31);
          }
          acc[it][0] = c00; acc[it][1] = c01; acc[it][2] = c10; acc[it][3] = c11;
          acc[it][4] = c20; acc[it][5] = c21; acc[it][6] = c30; acc[it][7] = c31;
        }
      }
    }
#pragma unroll
    for (int it = 0; it < MAXI; ++it) {
      const int o = base + it * nt + tid;
      if (o >= items) continue;
      const int g = o / per_g, rem = o - g * per_g;
      const int cp = rem % ncp, rg = rem / ncp;
      const int n0 = 2 * cp;
      float b0 = 0.f, b1 = 0.f;
      if (bias) {
        b0 = bias[g * bias_hstride + n0];
        if (n0 + 1 < N) b1 = bias[g * bias_hstride + n0 + 1];
      }
      float4* c4 = reinterpret_cast<float4*>(C) + (int64_t)rg * ldc + g * c_hoff + n0;
      float4 v0 = make_float4(alpha * acc[it][0] + b0, alpha * acc[it][2] + b0,
                              alpha * acc[it][4] + b0, alpha * acc[it][6] + b0);
      float4 v1 = make_float4(alpha * acc[it][1] + b1, alpha * acc[it][3] + b1,
                              alpha * acc[it][5] + b1, alpha * acc[it][7] + b1);
      if (accumulate) {
        const float4 p0 = c4[0];
        v0.x += p0.x; v0.y += p0.y; v0.z += p0.z; v0.w += p0.w;
      }
      c4[0] = v0;
      if (n0 + 1 < N) {
        if (accumulate) {
          const float4 p1 = c4[1];
          v1.x += p1.x; v1.y += p1.y; v1.z += p1.z; v1.w += p1.w;
        }
        c4[1] = v1;
      }
    }
  }
  __syncthreads();
}

// sin/cos of omega*dt: angle and its reduction to [-pi, pi] in float64
// (Delta t reaches ~1e7 ticks), then the float32 SFU pair; abs error ~1e-6.
__device__ __forceinline__ void phase_sincos(double omega, double dt, float* s, float* c) {
  const double ang = omega * dt;
  const double k = rint(ang * 0.15915494309189535);  // 1/(2 pi)
  double r = fma(-k, 6.283185307179586, ang);
  r = fma(-k, 2.4492935982947064e-16, r);             // 2 pi - fl(2 pi)
  __sincosf((float)r, s, c);
}
