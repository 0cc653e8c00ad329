// 5th-generation tensor-core helpers (tcgen05 / TMEM / mbarrier), sm_100a.
//
// Orientation used by the engine: D[f][i] = sum_k W[k][f] X[i][k], i.e. the
// weights are the MMA A operand (M = 128 output features per instruction)
// and the node-tile activations are the B operand (N = tile rows), so a
// small row tile costs no padding. Both operands are MN-major, no swizzle,
// in the canonical interleaved layout (16-byte groups of 4 elements along
// MN, 8 K-rows per 128-byte core matrix):
//     A:  W4[(f/4)][k][f%4]      SBO = Kp*16 B (next 4 features), LBO = 128 B
//     B:  R4[(i/4)][k][i%4]      SBO = ld*16 B (next 4 rows),     LBO = 128 B
// which is exactly the R4 activation layout of gemm.cuh. Precision is
// split-TF32 (hi*hi + hi*lo + lo*hi into one fp32 TMEM accumulator), where
// hi is the fp32 value itself (the MMA reads its top 19 bits) and lo is
// x - trunc_tf32(x): ~2^-20 relative per product, fp32-class accuracy.
#pragma once

#include "common.cuh"

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// trunc to tf32 (the bits the tensor core consumes) and the exact remainder
__device__ __forceinline__ float tf32_lo(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// ---- shared-memory matrix descriptor (SWIZZLE_NONE, Blackwell version 1) ----
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // version
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

// ---- instruction descriptor: kind::tf32, fp32 accumulate, A/B MN-major ----
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
  return (1u << 4)                       // c_format F32
         | (2u << 7)                     // a_format TF32
         | (2u << 10)                    // b_format TF32
         | (1u << 15)                    // a_major MN
         | (1u << 16)                    // b_major MN
         | ((uint32_t)(N >> 3) << 17)    // N >> 3
         | ((uint32_t)(M >> 4) << 24);   // M >> 4
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// A operand from TMEM (rows = lanes, K = 32-bit columns), B from smem.
__device__ __forceinline__ void umma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// registers -> TMEM: 32 lanes x 8 consecutive columns per warp
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])));
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

// K-major, no-swizzle operand layout: 8-row x 4-element (16 B) core
// matrices; element (r, k) of a [R][Kp] operand (R a multiple of 8).
__host__ __device__ __forceinline__ int kmaj_idx(int r, int k, int Kp) {
  return ((r >> 3) * (Kp >> 2) + (k >> 2)) * 32 + (r & 7) * 4 + (k & 3);
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(bar))
      : "memory");
}

// ---- TMEM allocation (one warp) ----
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   smem_u32(slot)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}

__device__ __forceinline__ void tmem_free(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols));
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// ---- mbarrier ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// With MBAR_SUSPEND_NS > 0 a waiting thread is suspended by the hardware until
// the phase completes (or the hint elapses) instead of spinning, so waiting
// warps stop taking issue slots from the warps they wait for.
#ifndef MBAR_SUSPEND_NS
#define MBAR_SUSPEND_NS 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
#if MBAR_SUSPEND_NS > 0
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "n"(MBAR_SUSPEND_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
#endif
}

// non-blocking: has the phase with this parity completed? (warp-uniform result)
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// ---- TMA bulk copy (1-D, global -> shared) completing on an mbarrier ----
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// one thread: stage `bytes` (multiple of 16) into dst in <= 32 KB pieces, one tx count
__device__ __forceinline__ void bulk_stage(void* dst, const void* src, uint32_t bytes,
                                           uint64_t* bar) {
  mbar_expect_tx(bar, bytes);
  for (uint32_t o = 0; o < bytes; o += 32768u) {
    const uint32_t n = bytes - o < 32768u ? bytes - o : 32768u;
    bulk_g2s(reinterpret_cast<char*>(dst) + o, reinterpret_cast<const char*>(src) + o, n, bar);
  }
}

// ---- TMEM -> registers: 32 lanes x 8 consecutive 32-bit columns per warp ----
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = __uint_as_float(r[q]);
}

// Self-test kernel (stgn_debug_tc_gemm): D[i][f] = sum_k X[i][k] W[k][f] for
// F <= 128 features, N <= 256 rows, one CTA of 128 threads.
__device__ __forceinline__ void umma_split_tf32(uint32_t tmem_d, uint32_t a_hi, uint32_t a_lo,
                                                uint32_t a_sbo, uint32_t b_hi, uint32_t b_lo,
                                                uint32_t b_sbo, int Kp, uint32_t idesc,
                                                bool accumulate);

__global__ void __launch_bounds__(128) k_tc_gemm_test(int F, int N, int K, const float* W,
                                                      const float* X, float* D, int mode) {
  extern __shared__ float4 smem4[];
  const int Kp = (K + 7) & ~7, Np = (N + 15) & ~15;
  float* Ah = reinterpret_cast<float*>(smem4);
  float* Al = Ah + 128 * Kp;
  float* Bh = Al + 128 * Kp;
  float* Bl = Bh + Np * Kp;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool kmaj = (mode & 8) != 0;  // debug: K-major interleaved operands
  for (int x = tid; x < 128 * Kp; x += 128) {
    const int f = x / Kp, k = x % Kp;
    const float v = (f < F && k < K) ? W[(int64_t)k * F + f] : 0.f;
    const int idx = kmaj ? ((f >> 3) * (Kp / 4) + (k >> 2)) * 32 + (f & 7) * 4 + (k & 3)
                         : ((f >> 2) * Kp + k) * 4 + (f & 3);
    Ah[idx] = v;
    Al[idx] = tf32_lo(v);
  }
  for (int x = tid; x < Np * Kp; x += 128) {
    const int i = x / Kp, k = x % Kp;
    const float v = (i < N && k < K) ? X[(int64_t)i * K + k] : 0.f;
    const int idx = kmaj ? ((i >> 3) * (Kp / 4) + (k >> 2)) * 32 + (i & 7) * 4 + (k & 3)
                         : ((i >> 2) * Kp + k) * 4 + (i & 3);
    Bh[idx] = v;
    Bl[idx] = tf32_lo(v);
  }
  if (warp == 0) tmem_alloc(&tslot, 256);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = tslot;
  if (mode & 1) {  // debug: sentinel store (value = -(lane*1000 + column)) before the MMA
    for (int c0 = 0; c0 < Np; c0 += 8) {
      uint32_t r[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) r[q] = __float_as_uint(-(float)((32 * warp + lane) * 1000 + c0 + q));
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(
              taddr + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (mode & 32) {  // TS test: node rows of X into TMEM (hi at col 256, lo at col 384)
    const int i = 32 * warp + lane;
    for (int c0 = 0; c0 < Kp; c0 += 8) {
      float h[8], lo[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int k = c0 + q;
        const float v = (i < N && k < K) ? X[(int64_t)i * K + k] : 0.f;
        h[q] = v;
        lo[q] = tf32_lo(v);
      }
      tmem_st8(taddr + ((uint32_t)(32 * warp) << 16) + 256u + (uint32_t)c0, h);
      tmem_st8(taddr + ((uint32_t)(32 * warp) << 16) + 384u + (uint32_t)c0, lo);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (tid == 0 && !(mode & 2)) {
    if (mode & 16)
      printf("tc_test: Ah=%u Al=%u Bh=%u Bl=%u taddr=%u Kp=%d Np=%d idesc=%08x desc0=%016llx\n",
             smem_u32(Ah), smem_u32(Al), smem_u32(Bh), smem_u32(Bl), taddr, Kp, Np,
             umma_idesc_tf32(128, Np), (unsigned long long)umma_desc(smem_u32(Ah), 128, Kp * 16));
    if (mode & 32) {
      // TS: A = X rows in TMEM (cols 256.. hi, 384.. lo), B = W^T K-major in smem (Ah/Al)
      const uint32_t idesc = umma_idesc_tf32(128, 128) & ~((1u << 15) | (1u << 16));
      const uint32_t sbo = (uint32_t)(Kp / 4) * 128;
      for (int s = 0; s < Kp / 8; ++s) {
        const uint32_t off = (uint32_t)s * 256u;
        const uint64_t bh = umma_desc(smem_u32(Ah) + off, 128, sbo);
        const uint64_t bl = umma_desc(smem_u32(Al) + off, 128, sbo);
        umma_tf32_ts(taddr, taddr + 256 + 8 * s, bh, idesc, s > 0 ? 1u : 0u);
        umma_tf32_ts(taddr, taddr + 256 + 8 * s, bl, idesc, 1u);
        umma_tf32_ts(taddr, taddr + 384 + 8 * s, bh, idesc, 1u);
      }
    } else if (kmaj) {
      // K-major: (8 rows x 16 B) core matrices; LBO = next 4 k (128 B), SBO = next 8 rows
      const uint32_t idesc = umma_idesc_tf32(128, Np) & ~((1u << 15) | (1u << 16));
      const uint32_t sbo = (uint32_t)(Kp / 4) * 128;
      for (int s = 0; s < Kp / 8; ++s) {
        const uint32_t off = (uint32_t)s * 256u;
        const uint64_t ah = umma_desc(smem_u32(Ah) + off, 128, sbo);
        const uint64_t al = umma_desc(smem_u32(Al) + off, 128, sbo);
        const uint64_t bh = umma_desc(smem_u32(Bh) + off, 128, sbo);
        const uint64_t bl = umma_desc(smem_u32(Bl) + off, 128, sbo);
        umma_tf32(taddr, ah, bh, idesc, ((mode & 4) || s > 0) ? 1u : 0u);
        umma_tf32(taddr, ah, bl, idesc, 1u);
        umma_tf32(taddr, al, bh, idesc, 1u);
      }
    } else {
      umma_split_tf32(taddr, smem_u32(Ah), smem_u32(Al), (uint32_t)Kp * 16, smem_u32(Bh),
                      smem_u32(Bl), (uint32_t)Kp * 16, Kp, umma_idesc_tf32(128, Np),
                      (mode & 4) != 0);
    }
    umma_commit(&bar);
  }
  if (!(mode & 2)) mbar_wait(&bar, 0);
  tc_fence_after();
  if (mode & 32) {  // D: lanes = nodes, columns = features
    const int i = 32 * warp + lane;
    for (int c0 = 0; c0 < 128; c0 += 8) {
      float v[8];
      tmem_ld8(taddr + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0, v);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int f = c0 + q;
        if (f < F && i < N) D[(int64_t)i * F + f] = v[q];
      }
    }
  }
  for (int c0 = 0; c0 < Np && !(mode & 32); c0 += 8) {
    float v[8];
    tmem_ld8(taddr + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0, v);
    const int f = 32 * warp + lane;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int i = c0 + q;
      if (f < F && i < N) D[(int64_t)i * F + f] = v[q];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(taddr, 256);
}

// Issue the split-TF32 MMAs of one GEMM block: D (128 x N, TMEM columns
// starting at tmem_d) = A (128 x Kp) * B (Kp x N), Kp a multiple of 8.
// A_hi/A_lo, B_hi/B_lo are smem byte addresses of the operand bases.
__device__ __forceinline__ void umma_split_tf32(uint32_t tmem_d, uint32_t a_hi, uint32_t a_lo,
                                                uint32_t a_sbo, uint32_t b_hi, uint32_t b_lo,
                                                uint32_t b_sbo, int Kp, uint32_t idesc,
                                                bool accumulate) {
  for (int s = 0; s < Kp / 8; ++s) {
    const uint32_t off = (uint32_t)s * 128u;
    const uint64_t ah = umma_desc(a_hi + off, 128, a_sbo), al = umma_desc(a_lo + off, 128, a_sbo);
    const uint64_t bh = umma_desc(b_hi + off, 128, b_sbo), bl = umma_desc(b_lo + off, 128, b_sbo);
    umma_tf32(tmem_d, ah, bh, idesc, (accumulate || s > 0) ? 1u : 0u);
    umma_tf32(tmem_d, ah, bl, idesc, 1u);
    umma_tf32(tmem_d, al, bh, idesc, 1u);
  }
}
