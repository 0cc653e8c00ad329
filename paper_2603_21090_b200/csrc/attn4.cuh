// Recompute kernel v4: 128-row tiles on tcgen05 with bf16x3 split GEMMs.
//
// Function: the engine recompute of attn2/attn3 (reference
// S/kernels/pipeline_numba.py:15-111 with the key/value projections folded to
// the query side), for H = 2 and k_in <= 224 (the C3/C4 widths).
//
// Why a v4. At the end of a 30M-edge C4 stream one batch recomputes ~109K rows
// with ~10 ring entries each (1 GB of frozen payload). attn3 ran 61-row tiles
// (its q~/ubar rows for a tile live in shared memory) and re-staged ~1 MB of
// split-TF32 weights per tile, and its walk spent ~147 instructions per ring
// entry. v4:
//  * bf16x3 split GEMMs (hi*hi + hi*lo + lo*hi, fp32 accumulate in TMEM;
//    ~1e-5 row-relative, the 1e-4 bar has a 10x margin): A operands and
//    weight blocks are half the size of split-TF32, so q~ for both heads
//    stays in TMEM and a tile is the full 128 lanes; weight blocks (~52 KB)
//    are double-buffered and staged by TMA bulk copies one block ahead.
//  * q~ leaves TMEM one 32-row quadrant at a time through a double-buffered
//    shared-memory row buffer; the walk writes ubar back into the same
//    buffer and the quadrant's warps pack it (bf16 hi/lo) into the TMEM
//    columns q~ occupied, where it is the A operand of the W_V GEMMs.
//  * the walk: one LDG.128 per ring entry and lane, the time encoding's
//    sqrt(1/d_t) folded into W_K / W_V, the logits of a chunk of entries
//    (both heads) reduced with one transposing butterfly, packed f32x2 FMAs.
//  * L2 prefetch one quadrant ahead (the next quadrant's ring rows while the
//    current one is walked), so the walk's loads hit L2.
//
// TMEM columns (fp32 accumulators; bf16 A operands pack two per column):
//   X_A  [0, Kx)           x_l hi|lo                (A of Q)
//   ACCQ [Kx, Kx+Nq)       q, head h at h*Kq         (D of Q)
//   QA   [0, Kq)           q_h hi|lo                 (A of K_h)
//   QT0  [512-Nk, 512)     q~_0  -> ubar_0 hi|lo     (D of K_0, then A of V_0)
//   QT1  [Kq, Kq+Nk)       q~_1  -> ubar_1 hi|lo
//   C0   [0, Nv)  C1 [Kq+max(Nk,Kc), +Nv)            (D of V_h)
//   CA   [Kq, Kq+Kc)       c hi|lo, head h at h*Kq   (A of O)
//   ACCO [Kq+Kc, +No)      out                       (D of O)
// Host-side checks (a4_plan) guarantee every live range is disjoint.
#pragma once

#include <cuda_bf16.h>

#include "attn3.cuh"

#ifndef A4_WARPS
#define A4_WARPS 16
#endif
#define A4_THREADS (A4_WARPS * 32)
// Phase timestamps of CTA 0 (debug builds with -DA4_PROF; read by stgn_debug_a4_prof).
#ifdef A4_PROF
__device__ unsigned long long g_a4_prof[8192];
__device__ int g_a4_prof_n;
// Per CTA: start ns, end ns, summed ring entries of its rows, tiles (all CTAs).
__device__ unsigned long long g_a4_cta[4 * 1024];
__device__ __forceinline__ unsigned long long a4_now() {
  unsigned long long t_;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
  return t_;
}
#define A4_MARK(tag)                                                              \
  do {                                                                           \
    if (blockIdx.x == 0 && threadIdx.x == 0 && g_a4_prof_n < 8190) {             \
      unsigned long long t_;                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                      \
      g_a4_prof[g_a4_prof_n++] = (t_ << 4) | (unsigned long long)(tag);           \
    }                                                                            \
  } while (0)
#else
#define A4_MARK(tag) do {} while (0)
#endif
#define A4_NCG (A4_WARPS / 4)  // warps per TMEM lane quadrant (column groups)
#define A4_TMAX 128
#ifndef A4_PREFETCH
#define A4_PREFETCH 0  // L2 prefetch of ring rows: 0 none, 1 one quadrant ahead, 2 whole tile per layer
#endif
#ifndef A4_NUB
#define A4_NUB 2  // quadrant row buffers (2: the next quadrant's q~ copy overlaps the walk)
#endif
#ifndef A4_CPK
#define A4_CPK 0  // walk 1: compact stages (an entry's segments back to back, kpad/4 float4s,
                  // instead of 32 float4 slots per segment), so four stages fit the buffers
#endif
#ifndef A4_NST
#if A4_CPK
#define A4_NST 4
#else
#define A4_NST 3  // cp.async stages (chunks in flight) per warp in the walk
#endif
#endif
#ifndef A4_STATIC
#define A4_STATIC 0  // static row assignment with one cp.async stream across rows and quadrants
#endif
#if A4_STATIC && A4_WARPS != 16
#error "A4_STATIC assigns two rows of every 32-row quadrant to each of 16 warps"
#endif
#ifndef A4_HINTS
#define A4_HINTS 1  // L2 eviction hints on the walk's loads
#endif
#ifndef A4_EC
#define A4_EC 2  // ring entries per chunk of the walk (2 or 4)
#endif
#ifndef A4_WALK
#define A4_WALK 1  // 1: per-lane cp.async chunks of A4_EC entries; 2: TMA bulk-copied chunks of A4_EC2 entries
#endif
#ifndef A4_EC2
#define A4_EC2 4  // ring entries per bulk-copied chunk (walk 2); two chunk stages per warp
#endif
#ifndef A4_EVQ
#define A4_EVQ 1  // quadrant fill/pack duties as an event loop (see the walk phase)
#endif
#ifndef A4_VOF
#define A4_VOF 0  // out = sum_h ubar_h (W_V,h W_O,h): the V GEMMs, the c pack and the O GEMM fold
                  // into two passes of two MMA blocks over the TMEM ubar operands
#endif
#ifndef A4_ISS
#define A4_ISS 0  // walk 1: every lane copies 16 bytes of every entry from an address that is
                  // always valid (lanes past a segment re-read the row's first 16 bytes, entries
                  // past E the row's last entry; their weights are 0 and their q~ lanes 0), so
                  // the issue has no per-copy size predicates; slot = hd + e with one wrap
#endif
#ifndef A4_GA
#define A4_GA 0  // event-loop walk: dynamic grab-ahead issue stream across the rows of a quadrant
#endif
#if A4_GA && (!A4_EVQ || A4_HW || A4_STATIC || A4_WALK != 1 || A4_CPK || A4_TRIG)
#error "A4_GA is an issue stream of the event-loop walk (walk 1)"
#endif
#ifndef A4_HEADROT
#define A4_HEADROT 0  // walk 1: the row's rotation by w t_ref read from the newest slot's stored basis
#endif
#ifndef A4_LEAN
#define A4_LEAN 0  // walk 1: cp.async issue from 32-bit byte offsets, always 16 valid bytes
#endif
#if A4_LEAN && (A4_ISS || A4_CPK || A4_TRIG || !A4_HINTS || A4_HW)
#error "A4_LEAN is an issue order of a4_walk_row (walk 1)"
#endif
#ifndef A4_SWP
#define A4_SWP 0  // walk 1: software-pipelined chunk loop (logits of c + 1 beside the update of c)
#endif
#if A4_SWP && (A4_NST < 3 || A4_CPK || A4_TRIG || A4_GA || A4_STATIC || A4_HW || A4_WALK != 1)
#error "A4_SWP is a chunk loop of walk 1 with its own issue stream (a4_walk_row, NST >= 3)"
#endif
#ifndef A4_VV
#define A4_VV 0  // V_0 and V_1 GEMMs issued back to back under one commit
#endif
#ifndef A4_EVQW
#define A4_EVQW 0  // event loop: a warp with no pending duty waits for the next quadrant in try_wait
#endif
#ifndef A4_RUNPTR
#define A4_RUNPTR 1  // walk 1: running source pointers for the cp.async issue
#endif
#ifndef A4_NXH
#define A4_NXH 1  // the next tile's row headers loaded during this tile's first walk (warp A4_WARPS-1)
#endif
#ifndef A4_LPT
#define A4_LPT 0  // rows of a tile sorted by descending entry count (see the tile header)
#endif
#ifndef A4_TRIG
#define A4_TRIG 0  // 1: time encoding computed per entry (fp64 phase) instead of read from ring_tb
#endif
#ifndef A4_BPF
#define A4_BPF 0  // 1: TMA bulk L2 prefetch of a tile-layer's payload rows before its Q/K GEMMs;
                  // 2: rolling, A4_PFD rows ahead of the walk (payload and basis)
#endif
#ifndef A4_PFD
#define A4_PFD 32
#endif
#ifndef A4_HW
#define A4_HW 0  // walk 1 with the event loop: two rows per warp, a half-warp per row
#endif
#if A4_ISS && (A4_CPK || A4_HW || A4_STATIC || A4_WALK != 1 || !A4_HINTS || A4_TRIG)
#error "A4_ISS is an issue order of walk 1 (a4_walk_row)"
#endif
#if A4_CPK && (A4_HW || A4_STATIC || A4_WALK != 1 || !A4_RUNPTR || !A4_HINTS || A4_TRIG)
#error "A4_CPK is a layout of walk 1's per-warp stages (a4_walk_row)"
#endif
#if A4_HW && A4_EC != 2
#error "A4_HW reuses the stage size of A4_EC = 2 (one entry of two rows per stage)"
#endif


struct A4W {
  const uint16_t *wq, *wk, *wv, *wo;  // packed bf16 B operands, hi block then lo block
  const uint16_t* wp;                 // folded P_h = W_V,h W_O,h (A4_VOF): [K][Pa_0 Pa_1 Pb_0 Pb_1]
  int Npa, Npb, nbl;                  // out columns of the two P passes; weight blocks per layer
  const float* bq;                    // [K][H*Kq]
  const double* omega;
  int Kx, Kq, Ku, Kc, Nq, Nk, Nv, No;
  int qt0, qt1, c1, ca, acco;         // TMEM columns
  int kfo, kto, kpad;                 // key layout [payload | features | time], each 4-padded
  int ldu;                            // row stride of the quadrant row buffer (floats)
  int wblk_bytes;                     // one staged weight block buffer (bytes)
  int region_bytes;                   // weight buffers / walk stage area (shared)
};

static inline bool a4_plan(const Geo& g, A4W* w) {
  auto r4 = [](int x) { return (x + 3) & ~3; };
  w->kfo = r4(g.d);
  w->kto = w->kfo + r4(g.d_e);
  w->kpad = w->kto + r4(g.d_t);
  if (g.H != 2 || r4(g.d) > 128 || r4(g.d_e) > 128 || r4(g.d_t) > 128) return false;
  w->Kx = r16(g.d);
  w->Kq = r16(g.d_k);
  w->Ku = r16(w->kpad);
  w->Kc = g.H * w->Kq;
  w->Nq = g.H * w->Kq;
  w->Nk = r16(w->kpad);
  w->Nv = r16(g.d_k);
  w->No = r16(g.d);
  w->qt0 = 512 - w->Nk;
  w->qt1 = w->Kq;
  w->c1 = w->Kq + std::max(w->Nk, w->Kc);  // above ubar_1 (read by V_1) and above CA
  w->ca = w->Kq;
  w->acco = w->Kq + w->Kc;
  int ldu = g.H * w->kpad;
  while (ldu % 8 != 4) ++ldu;  // 8 consecutive rows hit distinct 16-byte bank groups
  w->ldu = ldu;
  w->Npa = std::min(w->No, 64);
  w->Npb = w->No - w->Npa;
  w->nbl = A4_VOF ? (w->Npb > 0 ? 7 : 5) : 6;
  int mb = std::max(std::max(w->Nq * w->Kx, w->Nk * w->Kq), std::max(w->Nv * w->Ku, w->No * w->Kc));
  mb = std::max(mb, w->Npa * w->Ku);
  w->wblk_bytes = (mb * 2 * 2 + 1023) & ~1023;
#if A4_WALK == 2
  // two chunk stages per warp: [A4_EC2][ld_d] payload, [A4_EC2][ld_t] basis, [A4_EC2][ld_e] features
  const int stage_bytes = A4_WARPS * 2 * A4_EC2 * (g.ld_d + g.ld_t + (g.d_e > 0 ? g.ld_e : 0)) * 4;
#elif A4_CPK
  const int stage_bytes = A4_WARPS * A4_NST * A4_EC * (w->kpad / 4) * 16;
#else
  const int stage_bytes = A4_WARPS * A4_NST * A4_EC * (g.d_e > 0 ? 3 : 2) * 32 * 16;  // (TRIG: basis segment unused)
#endif
  w->region_bytes = std::max(2 * w->wblk_bytes, (stage_bytes + 1023) & ~1023);
  return w->Nk <= 256 && w->Nq <= 256 && w->No <= 256 && w->Ku <= w->Nk &&
         w->Kx + w->Nq <= w->qt0 &&            // ACCQ alive while K_0 writes QT0
         w->qt1 + w->Nk <= w->qt0 &&           // QT1 / QT0 disjoint
         w->Kq <= w->Kx && w->Nv <= w->Kq &&   // QA inside X_A; C0 below QT1
         w->c1 + w->Nv <= 512 &&               // C1 (may overlap QT0: V_0 is done)
         w->acco + w->No <= 512 &&             // ACCO
         w->Kx <= w->acco;                     // X_A (next layer) below ACCO
}

__host__ __device__ inline int64_t a4_blk_elems(int Np, int Kp) { return 2ll * Np * Kp; }

static inline size_t attn4_smem_bytes(const A4W& w) {
  return 1024 + (size_t)w.region_bytes + A4_NUB * 32 * (size_t)w.ldu * 4;
}

// ---- bf16 helpers ----
__device__ __forceinline__ uint32_t bf16_bits(float x) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(x));
}
// hi/lo bf16 split of (a, b), packed two per 32-bit column (element 2c low)
__device__ __forceinline__ void bf16x2_split(float a, float b, uint32_t& hi, uint32_t& lo) {
  // one packed conversion per pair for each of hi and lo (cvt.rn.bf16x2.f32)
  __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
  hi = *reinterpret_cast<uint32_t*>(&h2);
  const float ra = a - __uint_as_float(hi << 16), rb = b - __uint_as_float(hi & 0xFFFF0000u);
  __nv_bfloat162 l2 = __floats2bfloat162_rn(ra, rb);
  lo = *reinterpret_cast<uint32_t*>(&l2);
}
// 16 consecutive elements -> 8 hi columns at col, 8 lo columns at col + half
__device__ __forceinline__ void a4_st16(uint32_t taddr_hi, uint32_t taddr_lo, const float (&v)[16]) {
  float h[8], l[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint32_t a, b;
    bf16x2_split(v[2 * q], v[2 * q + 1], a, b);
    h[q] = __uint_as_float(a);
    l[q] = __uint_as_float(b);
  }
  tmem_st8(taddr_hi, h);
  tmem_st8(taddr_lo, l);
}
__device__ __forceinline__ void tmem_ld8_nw(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = __uint_as_float(r[q]);
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
  return (1u << 4)                       // c_format F32
         | (1u << 7)                     // a_format BF16
         | (1u << 10)                    // b_format BF16
         | ((uint32_t)(N >> 3) << 17)    // N >> 3 (A and B K-major)
         | ((uint32_t)(M >> 4) << 24);   // M >> 4
}
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// one thread: bf16x3 MMAs of one block, A = TMEM [a, a+Kp) (hi then lo), B = smem
// K-major bf16 [Np][Kp] (8x8 core matrices, hi block then lo block), then commit
__device__ __forceinline__ void a4_mma(uint32_t tmem, int a, const uint16_t* Wb, int Np, int Kp,
                                       int dcol, uint64_t* bar, bool acc0 = false,
                                       bool commit = true) {
  tc_fence_after();
  const uint32_t idesc = umma_idesc_bf16(128, Np);
  const uint32_t sbo = (uint32_t)(Kp / 8) * 128u;
  const uint32_t bh = smem_u32(Wb), bl = bh + (uint32_t)Np * Kp * 2u;
  const uint32_t ah0 = tmem + (uint32_t)a, al0 = ah0 + (uint32_t)(Kp / 2);
  for (int s = 0; s < Kp / 16; ++s) {
    const uint32_t off = (uint32_t)s * 256u;
    const uint64_t dh = umma_desc(bh + off, 128, sbo), dl = umma_desc(bl + off, 128, sbo);
    const uint32_t ah = ah0 + 8u * s, al = al0 + 8u * s;
    umma_bf16_ts(tmem + (uint32_t)dcol, ah, dh, idesc, (acc0 || s > 0) ? 1u : 0u);
    umma_bf16_ts(tmem + (uint32_t)dcol, ah, dl, idesc, 1u);
    umma_bf16_ts(tmem + (uint32_t)dcol, al, dh, idesc, 1u);
  }
  if (commit) umma_commit(bar);
}

// weight block j (Q, K_0, K_1, V_0, V_1, O) of layer l: source and element count
__device__ __forceinline__ const uint16_t* a4_block(const Geo& g, const A4W& w, int l, int j,
                                                    int64_t* elems) {
  if (j == 0) {
    *elems = a4_blk_elems(w.Nq, w.Kx);
    return w.wq + (int64_t)l * *elems;
  }
  if (j <= 2) {
    *elems = a4_blk_elems(w.Nk, w.Kq);
    return w.wk + ((int64_t)l * 2 + (j - 1)) * *elems;
  }
#if A4_VOF
  // layer l: Pa_0, Pa_1 ([Npa][Ku]), then Pb_0, Pb_1 ([Npb][Ku])
  const int64_t ea = a4_blk_elems(w.Npa, w.Ku), eb = a4_blk_elems(w.Npb, w.Ku);
  const uint16_t* base = w.wp + (int64_t)l * 2 * (ea + eb);
  if (j <= 4) {
    *elems = ea;
    return base + (int64_t)(j - 3) * ea;
  }
  *elems = eb;
  return base + 2 * ea + (int64_t)(j - 5) * eb;
#else
  if (j <= 4) {
    *elems = a4_blk_elems(w.Nv, w.Ku);
    return w.wv + ((int64_t)l * 2 + (j - 3)) * *elems;
  }
  *elems = a4_blk_elems(w.No, w.Kc);
  return w.wo + (int64_t)l * *elems;
#endif
}

// L2 prefetch of layer l's ring rows of tile rows [r0, r1): the valid slots
// of the payload block and of the time-basis block (each a contiguous run of
// slots, split in two when the ring wraps). One warp per row, lanes over lines.
__device__ __forceinline__ void a4_prefetch(const Geo& g, const RingSrc& rs, const int* nodes,
                                            const int* Es, const int* heads, int r0, int r1,
                                            int l, int tid) {
  const int lane = tid & 31;
  for (int i = r0 + (tid >> 5); i < r1; i += A4_WARPS) {
    const int node = nodes[i], E = Es[i], hd = heads[i];
    if (node < 0 || E <= 0) continue;
    const int n1 = min(E, g.L - hd), n2 = E - n1;  // slots [hd, hd+n1) and [0, n2)
    const char* pay = reinterpret_cast<const char*>(rs.ring_pay + ((int64_t)node * g.K + l) * g.L * g.ld_d);
    const char* tb = reinterpret_cast<const char*>(rs.ring_tb + (int64_t)node * g.L * g.ld_t);
    const int pb = g.ld_d * 4, tbb = g.ld_t * 4;
#pragma unroll
    for (int part = 0; part < 4; ++part) {
      const char* base = (part < 2 ? pay : tb);
      const int stride = part < 2 ? pb : tbb;
      const int s0 = (part & 1) ? 0 : hd, ns = (part & 1) ? n2 : n1;
      if (ns <= 0) continue;
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(base + (int64_t)s0 * stride);
      const uintptr_t a1 = a0 + (uintptr_t)ns * stride - 1;
      for (uintptr_t line = (a0 >> 7) + lane; line <= (a1 >> 7); line += 32)
        prefetch_l2(reinterpret_cast<const void*>(line << 7));
    }
  }
}

// TMA bulk prefetch of [p, p + bytes) into L2 (16-byte aligned, multiple of 16)
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
// one lane: bulk L2 prefetch of layer l's payload and time-basis runs of a ring row
__device__ __forceinline__ void a4_row_prefetch(const Geo& g, const RingSrc& rs, int node, int E,
                                                int hd, int l) {
  if (node < 0 || E <= 0) return;
  const int n1 = min(E, g.L - hd), n2 = E - n1;
  const float* pay = rs.ring_pay + ((int64_t)node * g.K + l) * g.L * g.ld_d;
  const float* tb = rs.ring_tb + (int64_t)node * g.L * g.ld_t;
  bulk_prefetch_l2(pay + (int64_t)hd * g.ld_d, (uint32_t)(n1 * g.ld_d * 4));
  bulk_prefetch_l2(tb + (int64_t)hd * g.ld_t, (uint32_t)(n1 * g.ld_t * 4));
  if (n2 > 0) {
    bulk_prefetch_l2(pay, (uint32_t)(n2 * g.ld_d * 4));
    bulk_prefetch_l2(tb, (uint32_t)(n2 * g.ld_t * 4));
  }
}
// 16-byte global -> shared async copy (L1 bypass); src_bytes = 0 zero-fills
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async16_pol(void* dst, const void* src, int src_bytes,
                                               uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(src_bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ float ex2f(float x) {  // 2^x on the SFU (ex2(-inf) = 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("mul.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return d;
}

// Per-warp cp.async issue stream over the ring chunks of the warp's rows of a
// tile-layer (static assignment: rows 32q + warp and 32q + warp + 16 of every
// quadrant q, in order). The stream runs A4_NST - 1 chunks ahead of the walk,
// across row and quadrant boundaries (ring rows do not depend on the quadrant
// row buffers), so a row's first chunks are in flight before it starts.
struct A4Iss {
  int k;     // position in the warp's row sequence
  int c;     // next chunk of that row
  int kiss;  // groups committed
  int nseq;  // rows in the sequence (2 per quadrant)
};
template <int KF>
__device__ __forceinline__ void a4_issue_next(const Geo& g, const A4W& w, const RingSrc& rs,
                                              A4Iss& is, const int* s_node, const int* s_E,
                                              const int* s_head, int T, int warp, int l, int lane,
                                              float4* stg) {
  constexpr int EC = A4_EC, NSEG = KF ? 3 : 2, NST = A4_NST;
  int r = -1, nch = 0;
  while (is.k < is.nseq) {
    r = 32 * (is.k >> 1) + warp + 16 * (is.k & 1);
    nch = (r < T && s_node[r] >= 0) ? (s_E[r] + EC - 1) / EC : 0;
    if (is.c < nch) break;
    ++is.k;
    is.c = 0;
  }
  if (is.k < is.nseq) {
    const int node = s_node[r], E = s_E[r], hd = s_head[r];
    const bool lp = lane < w.kfo / 4, lf = KF && lane < (w.kto - w.kfo) / 4,
               lt = lane < (w.kpad - w.kto) / 4;
    const float* payb = rs.ring_pay + ((int64_t)node * g.K + l) * g.L * g.ld_d + 4 * lane;
    const float* ftb = rs.ring_feat + (int64_t)node * g.L * g.ld_e + 4 * lane;
    const float* tbb = rs.ring_tb + (int64_t)node * g.L * g.ld_t + 4 * lane;
    float4* sb = stg + (is.kiss % NST) * (EC * NSEG * 32) + lane;
#pragma unroll
    for (int u = 0; u < EC; ++u) {
      const int e = is.c * EC + u;
      const bool ev = e < E;
      int slot = hd + e;
      if (slot >= g.L) slot -= g.L;
      if (EC > 2 && !ev) slot = 0;  // EC = 2: hd + e < 2L, one wrap keeps it in the ring
      cp_async16(sb + (u * NSEG) * 32, payb + slot * g.ld_d, (ev && lp) ? 16 : 0);
      cp_async16(sb + (u * NSEG + 1) * 32, tbb + slot * g.ld_t, (ev && lt) ? 16 : 0);
      if (KF) cp_async16(sb + (u * NSEG + 2) * 32, ftb + slot * g.ld_e, (ev && lf) ? 16 : 0);
    }
    ++is.c;
  }
  cp_async_commit();
  ++is.kiss;
}

// Dynamic grab-ahead issue stream (A4_GA) over the rows of one quadrant: when the
// row being issued runs out of chunks, the warp takes the next row from the
// quadrant's counter and issues its first chunks while it still reduces the
// current row, so the cp.async pipeline does not drain and refill at every row.
// Rows taken are queued (q_rows, per warp, in shared memory, at most the
// quadrant's 32) and walked in order.
struct A4Dyn {
  int r;      // row (tile index) being issued, -1 if none
  int c;      // its next chunk
  int nch;    // its chunk count
  int kiss;   // groups committed
  int qh, qt; // queue head (next row to walk) / tail (rows taken)
  int done;   // the quadrant's counter is exhausted
};
template <int KF>
__device__ __forceinline__ void a4_issue_dyn(const Geo& g, const A4W& w, const RingSrc& rs,
                                             A4Dyn& d, const int* s_node, const int* s_E,
                                             const int* s_head, int q, int nrows, int* qctr,
                                             int* q_rows, int l, int lane, float4* stg) {
  constexpr int EC = A4_EC, NSEG = KF ? 3 : 2, NST = A4_NST;
  while (d.r < 0 || d.c >= d.nch) {
    if (d.done) {
      d.r = -1;
      break;
    }
    int i = 0;
    if (lane == 0) i = atomicAdd(qctr, 1);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= nrows) {
      d.done = 1;
      d.r = -1;
      break;
    }
    const int r = 32 * q + i;
    if (s_node[r] < 0) continue;  // no row (another rank's node): nothing to write
    d.r = r;
    d.c = 0;
    d.nch = (max(s_E[r], 0) + EC - 1) / EC;  // an empty list is walked too (ubar = 0)
    if (lane == 0) q_rows[d.qt & 31] = r;
    ++d.qt;
  }
  if (d.r >= 0) {
    const int node = s_node[d.r], E = s_E[d.r], hd = s_head[d.r];
    const bool lp = lane < w.kfo / 4, lf = KF && lane < (w.kto - w.kfo) / 4,
               lt = lane < (w.kpad - w.kto) / 4;
    const float* payb = rs.ring_pay + ((int64_t)node * g.K + l) * g.L * g.ld_d + 4 * lane;
    const float* ftb = rs.ring_feat + (int64_t)node * g.L * g.ld_e + 4 * lane;
    const float* tbb = rs.ring_tb + (int64_t)node * g.L * g.ld_t + 4 * lane;
    const uint64_t pol_pay = pol_evict_first();
    const uint64_t pol_tb = l + 1 < g.K ? pol_evict_last() : pol_evict_first();
    float4* sb = stg + (d.kiss % NST) * (EC * NSEG * 32) + lane;
#pragma unroll
    for (int u = 0; u < EC; ++u) {
      const int e = d.c * EC + u;
      const bool ev = e < E;
      int slot = hd + e;
      if (slot >= g.L) slot -= g.L;
      if (EC > 2 && !ev) slot = 0;
      cp_async16_pol(sb + (u * NSEG) * 32, payb + slot * g.ld_d, (ev && lp) ? 16 : 0, pol_pay);
      cp_async16_pol(sb + (u * NSEG + 1) * 32, tbb + slot * g.ld_t, (ev && lt) ? 16 : 0, pol_tb);
      if (KF) cp_async16(sb + (u * NSEG + 2) * 32, ftb + slot * g.ld_e, (ev && lf) ? 16 : 0);
    }
    ++d.c;
  }
  cp_async_commit();
  ++d.kiss;
}

// Walk of one row (warp-per-row): softmax over its ring entries for both
// heads; q~ read from, ubar written to the row buffer U (both heads, kpad each).
// Lane l owns key features [4l, 4l+4) of the payload (l < d/4), of the edge
// features and of the time encoding (frequencies 2l, 2l+1).
//
// Time encoding without per-entry trigonometry: phi(tref - t_e) is the
// rotation by w tref of the slot's stored basis b_e = [cos w t_e, sin w t_e]
// (ring_tb, written at insertion), so
//   q~_phi . phi(tref - t_e) = [P | Q] . b_e,  P = qc cos a + qs sin a,
//                                              Q = qc sin a - qs cos a  (a = w tref)
// and sum_e alpha_e phi(tref - t_e) = R(a) sum_e alpha_e b_e: the row pays two
// sincos per lane, each entry one LDG.128 of basis and plain FMAs.
template <int KF, typename IssueFn>
__device__ __forceinline__ void a4_walk_row(const Geo& g, const A4W& w, const RingSrc& rs,
                                            float* U, int node, int E, int hd, double tref, int l,
                                            int lane, float4* stg, IssueFn&& ext_issue,
                                            int* kcons) {
  constexpr int EC = A4_EC;
  const int kfo = w.kfo, kto = w.kto, kp = w.kpad;
  const bool lp = lane < kfo / 4, lf = KF && lane < (kto - kfo) / 4, lt = lane < (kp - kto) / 4;
  float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
  // rotation of this row's reference time, frequencies 2l and 2l+1
#if A4_TRIG
  // phi(tref - t_e) per entry: lanes 0..E-1 hold t_e, the frequencies 2l, 2l+1 per lane
  double te = 0.0;
  if (lane < E) {
    int s = hd + lane;
    if (s >= g.L) s -= g.L;
    te = rs.ring_t[(int64_t)node * g.L + s];
  }
  const bool f0 = lt && 2 * lane < g.half, f1 = lt && 2 * lane + 1 < g.half;
  const double om0 = f0 ? __ldg(w.omega + 2 * lane) : 0.0;
  const double om1 = f1 ? __ldg(w.omega + 2 * lane + 1) : 0.0;
#else
  float ca0 = 1.f, sa0 = 0.f, ca1 = 1.f, sa1 = 0.f;
#if A4_HEADROT
  // t_ref is the time of the row's newest ring entry (slot hd), whose stored basis is
  // [cos w t_ref, sin w t_ref] from the same phase_sincos: one 16-byte load instead
  // of two float64 phase reductions per lane, bit-identical
  if (E > 0 && lt && 2 * lane < g.half) {
    const float4 b = *reinterpret_cast<const float4*>(rs.ring_tb + ((int64_t)node * g.L + hd) * g.ld_t + 4 * lane);
    ca0 = b.x; sa0 = b.y;
    if (2 * lane + 1 < g.half) { ca1 = b.z; sa1 = b.w; }
  }
#else
  if (lt && 2 * lane < g.half) phase_sincos(__ldg(w.omega + 2 * lane), tref, &sa0, &ca0);
  if (lt && 2 * lane + 1 < g.half) phase_sincos(__ldg(w.omega + 2 * lane + 1), tref, &sa1, &ca1);
#endif
#endif
  float4 qp[2], qf[2], qt[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float* Uh = U + h * kp;
    qp[h] = lp ? *reinterpret_cast<const float4*>(Uh + 4 * lane) : zero4;
    qf[h] = lf ? *reinterpret_cast<const float4*>(Uh + kfo + 4 * lane) : zero4;
    float4 q = lt ? *reinterpret_cast<const float4*>(Uh + kto + 4 * lane) : zero4;
#if A4_TRIG
    qt[h] = q;
#else
    qt[h] = make_float4(q.x * ca0 + q.y * sa0, q.x * sa0 - q.y * ca0,
                        q.z * ca1 + q.w * sa1, q.z * sa1 - q.w * ca1);
#endif
  }
  float2 up[2][2], uf[2][2], ut[2][2];
  float mx[2] = {-INFINITY, -INFINITY}, zs[2] = {0.f, 0.f};
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < 2; ++c) up[h][c] = uf[h][c] = ut[h][c] = make_float2(0.f, 0.f);
  const float* payb = rs.ring_pay + ((int64_t)node * g.K + l) * g.L * g.ld_d + 4 * lane;
  const float* ftb = rs.ring_feat + (int64_t)node * g.L * g.ld_e + 4 * lane;
  const float* tbb = rs.ring_tb + (int64_t)node * g.L * g.ld_t + 4 * lane;
  // ring rows move through a per-warp cp.async pipeline of A4_NST chunks in
  // shared memory (the weight buffers, idle during the walk): the loads of the
  // next A4_NST - 1 chunks are in flight while one chunk is reduced
  constexpr int NSEG = KF ? 3 : 2;
  constexpr int NST = A4_NST;
#if A4_HINTS
  // a layer's payload rows are read once; the time basis again by the next layer
  const uint64_t pol_pay = pol_evict_first();
  const uint64_t pol_tb = l + 1 < g.K ? pol_evict_last() : pol_evict_first();
#endif
  const int nch = (E + EC - 1) / EC;
  int iss_slot = 0, con_slot = 0;  // stage slots of the next issue / the next consumed chunk
#if A4_RUNPTR
  // running per-lane source rows of the next entry to issue (chunks are issued in
  // order): one pointer bump per entry instead of slot arithmetic and 64-bit
  // multiplies per copy; the ring wraps once at most
  int r_slot = hd;
  const float* r_pay = payb + (int64_t)hd * g.ld_d;
  const float* r_tb = tbb + (int64_t)hd * g.ld_t;
  const float* r_ft = ftb + (int64_t)hd * g.ld_e;
#endif
#if A4_LEAN
  // byte offsets of the next entry to issue from the node's slot-0 rows (lanes past a
  // segment read lane 0's 16 bytes: every copy is 16 valid bytes, no size predicate);
  // after the last entry the offsets stop, so a chunk's tail re-reads that entry
  // (its logit is -inf, its weight 0)
  const char* l_pay = reinterpret_cast<const char*>(rs.ring_pay + ((int64_t)node * g.K + l) * g.L * g.ld_d) +
                      (lp ? 16 * lane : 0);
  const char* l_tb = reinterpret_cast<const char*>(rs.ring_tb + (int64_t)node * g.L * g.ld_t) +
                     (lt ? 16 * lane : 0);
  const char* l_ft = reinterpret_cast<const char*>(rs.ring_feat + (int64_t)node * g.L * g.ld_e) +
                     (lf ? 16 * lane : 0);
  const uint32_t sp_pay = 4u * g.ld_d, sp_tb = 4u * g.ld_t, sp_ft = 4u * g.ld_e;
  uint32_t o_pay = (uint32_t)hd * sp_pay, o_tb = (uint32_t)hd * sp_tb, o_ft = (uint32_t)hd * sp_ft;
  int l_slot = hd, l_left = E;
#endif
#if A4_ISS
  const float* i_pay = rs.ring_pay + ((int64_t)node * g.K + l) * g.L * g.ld_d + (lp ? 4 * lane : 0);
  const float* i_tb = rs.ring_tb + (int64_t)node * g.L * g.ld_t + (lt ? 4 * lane : 0);
  const float* i_ft = rs.ring_feat + (int64_t)node * g.L * g.ld_e + (lf ? 4 * lane : 0);
#endif
#if A4_CPK
  // compact stage: entry u of a chunk at float4 u*SE: payload [0, kfo/4), features
  // [kfo/4, kto/4), time basis [kto/4, kpad/4); lanes past a segment copy nothing
  const int SE = kp / 4, o_f = kfo / 4, o_t = kto / 4;
#endif
  auto issue = [&](int c) {
#ifdef A4_XNOLOAD  // timing experiment only (results wrong): no ring-row copies
    if (false) {
#else
    if (c < nch) {
#endif
#if A4_CPK
      float4* sb = stg + iss_slot * (EC * SE) + lane;
#else
      float4* sb = stg + iss_slot * (EC * NSEG * 32) + lane;
#endif
#pragma unroll
      for (int u = 0; u < EC; ++u) {
        const int e = c * EC + u;
        const bool ev = e < E;
#if A4_LEAN
        {
          cp_async16_pol(sb + (u * NSEG) * 32, l_pay + o_pay, 16, pol_pay);
          cp_async16_pol(sb + (u * NSEG + 1) * 32, l_tb + o_tb, 16, pol_tb);
          if (KF) cp_async16(sb + (u * NSEG + 2) * 32, l_ft + o_ft, 16);
          if (--l_left > 0) {
            if (++l_slot == g.L) {
              l_slot = 0;
              o_pay = o_tb = o_ft = 0;
            } else {
              o_pay += sp_pay;
              o_tb += sp_tb;
              if (KF) o_ft += sp_ft;
            }
          }
          (void)ev;
          continue;
        }
#endif
#if A4_ISS
        {
          int slot = hd + (ev ? e : E - 1);
          if (slot >= g.L) slot -= g.L;
          cp_async16_pol(sb + (u * NSEG) * 32, i_pay + slot * g.ld_d, 16, pol_pay);
          cp_async16_pol(sb + (u * NSEG + 1) * 32, i_tb + slot * g.ld_t, 16, pol_tb);
          if (KF) cp_async16(sb + (u * NSEG + 2) * 32, i_ft + slot * g.ld_e, 16);
          continue;
        }
#endif
#if A4_CPK
        {
          const int nb = ev ? 16 : 0;  // entries past E: zero-filled (weight 0, no NaN)
          if (lp) cp_async16_pol(sb + u * SE, r_pay, nb, pol_pay);
          if (lt) cp_async16_pol(sb + u * SE + o_t, r_tb, nb, pol_tb);
          if (KF && lf) cp_async16(sb + u * SE + o_f, r_ft, nb);
          if (++r_slot == g.L) {
            r_slot = 0;
            r_pay = payb;
            r_tb = tbb;
            r_ft = ftb;
          } else {
            r_pay += g.ld_d;
            r_tb += g.ld_t;
            r_ft += g.ld_e;
          }
          continue;
        }
#endif
#if A4_RUNPTR
        const int pay_bytes = (ev && lp) ? 16 : 0, tb_bytes = (ev && lt) ? 16 : 0;
#if A4_HINTS
        cp_async16_pol(sb + (u * NSEG) * 32, r_pay, pay_bytes, pol_pay);
        if (!A4_TRIG) cp_async16_pol(sb + (u * NSEG + 1) * 32, r_tb, tb_bytes, pol_tb);
#else
        cp_async16(sb + (u * NSEG) * 32, r_pay, pay_bytes);
        if (!A4_TRIG) cp_async16(sb + (u * NSEG + 1) * 32, r_tb, tb_bytes);
#endif
        if (KF) cp_async16(sb + (u * NSEG + 2) * 32, r_ft, (ev && lf) ? 16 : 0);
        if (++r_slot == g.L) {
          r_slot = 0;
          r_pay = payb;
          r_tb = tbb;
          r_ft = ftb;
        } else {
          r_pay += g.ld_d;
          r_tb += g.ld_t;
          r_ft += g.ld_e;
        }
        continue;
#endif
        int slot = hd + e;
        if (slot >= g.L) slot -= g.L;
        if (EC > 2 && !ev) slot = 0;  // EC = 2: hd + e < 2L, one wrap keeps it in the ring
#if A4_HINTS
        cp_async16_pol(sb + (u * NSEG) * 32, payb + slot * g.ld_d, (ev && lp) ? 16 : 0, pol_pay);
        if (!A4_TRIG) cp_async16_pol(sb + (u * NSEG + 1) * 32, tbb + slot * g.ld_t, (ev && lt) ? 16 : 0, pol_tb);
#else
        cp_async16(sb + (u * NSEG) * 32, payb + slot * g.ld_d, (ev && lp) ? 16 : 0);
        cp_async16(sb + (u * NSEG + 1) * 32, tbb + slot * g.ld_t, (ev && lt) ? 16 : 0);
#endif
        if (KF) cp_async16(sb + (u * NSEG + 2) * 32, ftb + slot * g.ld_e, (ev && lf) ? 16 : 0);
      }
    }
    cp_async_commit();  // (possibly empty) group per chunk index keeps the counting uniform
    if (++iss_slot == NST) iss_slot = 0;
  };
  if (!kcons) {
#pragma unroll
    for (int c = 0; c < NST - 1; ++c) issue(c);
  }
#if A4_SWP
  // Software-pipelined chunk loop: the logits of chunk c + 1 (dot products and the
  // transposing butterfly) are formed while chunk c's softmax update and accumulation
  // run, two independent dependency chains; chunk c + 2 is in flight meanwhile.
  auto load_k = [&](int slot, float4 (&kp)[EC], float4 (&kt)[EC], float4 (&kf)[EC]) {
    const float4* sb = stg + slot * (EC * NSEG * 32) + lane;
#pragma unroll
    for (int u = 0; u < EC; ++u) {
      kp[u] = sb[(u * NSEG) * 32];
      kt[u] = sb[(u * NSEG + 1) * 32];
      kf[u] = KF ? sb[(u * NSEG + 2) * 32] : zero4;
    }
  };
  auto logits = [&](const float4 (&kp)[EC], const float4 (&kt)[EC], const float4 (&kf)[EC],
                    int e0, float (&lg)[2 * EC]) {
    // per-lane partial logits, value index v = 2u + h
    float part[2 * EC];
#pragma unroll
    for (int u = 0; u < EC; ++u) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float2 a = fmul2(make_float2(qp[h].x, qp[h].y), make_float2(kp[u].x, kp[u].y));
        a = ffma2(make_float2(qp[h].z, qp[h].w), make_float2(kp[u].z, kp[u].w), a);
        a = ffma2(make_float2(qt[h].x, qt[h].y), make_float2(kt[u].x, kt[u].y), a);
        a = ffma2(make_float2(qt[h].z, qt[h].w), make_float2(kt[u].z, kt[u].w), a);
        if (KF) {
          a = ffma2(make_float2(qf[h].x, qf[h].y), make_float2(kf[u].x, kf[u].y), a);
          a = ffma2(make_float2(qf[h].z, qf[h].w), make_float2(kf[u].z, kf[u].w), a);
        }
        part[2 * u + h] = a.x + a.y;
      }
    }
    // transposing butterfly: 2*EC values; value v ends on lanes v*(32/(2*EC)) ..
    {
      const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
      for (int j = 0; j < EC; ++j) {
        const float send = b4 ? part[j] : part[j + EC];
        const float keep = b4 ? part[j + EC] : part[j];
        part[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      }
      if constexpr (EC >= 2) {
#pragma unroll
        for (int j = 0; j < EC / 2; ++j) {
          const float send = b3 ? part[j] : part[j + EC / 2];
          const float keep = b3 ? part[j + EC / 2] : part[j];
          part[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
      }
      if constexpr (EC >= 4) {
        const float send = b2 ? part[0] : part[1];
        const float keep = b2 ? part[1] : part[0];
        part[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
      } else {
        part[0] += __shfl_xor_sync(0xffffffffu, part[0], 4);
      }
      part[0] += __shfl_xor_sync(0xffffffffu, part[0], 2);
      part[0] += __shfl_xor_sync(0xffffffffu, part[0], 1);
      constexpr int stride = 32 / (2 * EC);
#pragma unroll
      for (int v = 0; v < 2 * EC; ++v) lg[v] = __shfl_sync(0xffffffffu, part[0], stride * v);
    }
    // entries past E (zero-filled stages) get logit -inf: out of the max, weight 0
#pragma unroll
    for (int u = 1; u < EC; ++u)
      if (e0 + u >= E) lg[2 * u] = lg[2 * u + 1] = -INFINITY;
  };
  auto soft_acc = [&](const float4 (&kp)[EC], const float4 (&kt)[EC], const float4 (&kf)[EC],
                      const float (&lg)[2 * EC]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float cm = lg[h];
#pragma unroll
      for (int u = 1; u < EC; ++u) cm = fmaxf(cm, lg[2 * u + h]);
      const float nm = fmaxf(mx[h], cm);
      const float sc = ex2f(mx[h] - nm);  // logits are in log2 units (W_K carries log2 e)
      const float2 sc2 = make_float2(sc, sc);
      zs[h] *= sc;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        up[h][c] = fmul2(up[h][c], sc2);
        ut[h][c] = fmul2(ut[h][c], sc2);
        if (KF) uf[h][c] = fmul2(uf[h][c], sc2);
      }
#pragma unroll
      for (int u = 0; u < EC; ++u) {
        const float p = ex2f(lg[2 * u + h] - nm);
        const float2 p2 = make_float2(p, p);
        zs[h] += p;
        up[h][0] = ffma2(p2, make_float2(kp[u].x, kp[u].y), up[h][0]);
        up[h][1] = ffma2(p2, make_float2(kp[u].z, kp[u].w), up[h][1]);
        ut[h][0] = ffma2(p2, make_float2(kt[u].x, kt[u].y), ut[h][0]);
        ut[h][1] = ffma2(p2, make_float2(kt[u].z, kt[u].w), ut[h][1]);
        if (KF) {
          uf[h][0] = ffma2(p2, make_float2(kf[u].x, kf[u].y), uf[h][0]);
          uf[h][1] = ffma2(p2, make_float2(kf[u].z, kf[u].w), uf[h][1]);
        }
      }
      mx[h] = nm;
    }
  };
  float lg_c[2 * EC];
  if (nch > 0) {
    cp_async_wait<NST - 2>();  // chunk 0 has landed
    float4 kp0[EC], kt0[EC], kf0[EC];
    load_k(0, kp0, kt0, kf0);
    logits(kp0, kt0, kf0, 0, lg_c);
  }
  int slot_s = 0;
  for (int c = 0; c < nch; ++c) {
    issue(c + NST - 1);  // into the slot chunk c - 1 used
    cp_async_wait<NST - 2>();  // chunk c + 1 has landed
    const int slot_n = slot_s + 1 == NST ? 0 : slot_s + 1;
    float lg_n[2 * EC];
    if (c + 1 < nch) {
      float4 kpn[EC], ktn[EC], kfn[EC];
      load_k(slot_n, kpn, ktn, kfn);
      logits(kpn, ktn, kfn, (c + 1) * EC, lg_n);
    }
    {
      float4 kpc[EC], ktc[EC], kfc[EC];
      load_k(slot_s, kpc, ktc, kfc);
      soft_acc(kpc, ktc, kfc, lg_c);
    }
#pragma unroll
    for (int v = 0; v < 2 * EC; ++v) lg_c[v] = lg_n[v];
    slot_s = slot_n;
  }
#else
  for (int c = 0; c < nch; ++c) {
    const int e0 = c * EC;
    int slot_c = con_slot;
    if (++con_slot == NST) con_slot = 0;
    if (kcons) {  // the warp-wide stream issues (and runs ahead of) this row's chunks
      ext_issue();
      slot_c = (*kcons)++ % NST;
    } else {
      issue(c + NST - 1);
    }
    cp_async_wait<NST - 1>();  // chunk c has landed (this lane's own copies)
    float4 kp[EC], kf[EC], kt[EC];
#if A4_CPK
    {
      const float4* sb = stg + slot_c * (EC * SE) + lane;
#pragma unroll
      for (int u = 0; u < EC; ++u) {
        kp[u] = lp ? sb[u * SE] : zero4;
        kt[u] = lt ? sb[u * SE + o_t] : zero4;
        kf[u] = (KF && lf) ? sb[u * SE + o_f] : zero4;
      }
    }
    if (false)
#endif
    {
      const float4* sb = stg + slot_c * (EC * NSEG * 32) + lane;
#pragma unroll
      for (int u = 0; u < EC; ++u) {
        kp[u] = sb[(u * NSEG) * 32];
#if A4_TRIG
        const double tu = __shfl_sync(0xffffffffu, te, (e0 + u) & 31);
        const double dt = tref - tu;
        float s0 = 0.f, c0 = 0.f, s1 = 0.f, c1 = 0.f;
        if (f0) phase_sincos(om0, dt, &s0, &c0);
        if (f1) phase_sincos(om1, dt, &s1, &c1);
        kt[u] = make_float4(c0, s0, c1, s1);
#else
        kt[u] = sb[(u * NSEG + 1) * 32];
#endif
        kf[u] = KF ? sb[(u * NSEG + 2) * 32] : zero4;
      }
    }
#ifdef A4_XNOMATH  // timing experiment only (results wrong): loads and waits, no softmax math
#pragma unroll
    for (int u = 0; u < EC; ++u) {
      up[0][0] = ffma2(make_float2(1.f, 1.f), make_float2(kp[u].x, kp[u].y), up[0][0]);
      ut[0][0] = ffma2(make_float2(1.f, 1.f), make_float2(kt[u].x, kt[u].y), ut[0][0]);
    }
    zs[0] = zs[1] = 1.f;
    continue;
#endif
    // per-lane partial logits, value index v = 2u + h
    float part[2 * EC];
#pragma unroll
    for (int u = 0; u < EC; ++u) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float2 a = fmul2(make_float2(qp[h].x, qp[h].y), make_float2(kp[u].x, kp[u].y));
        a = ffma2(make_float2(qp[h].z, qp[h].w), make_float2(kp[u].z, kp[u].w), a);
        a = ffma2(make_float2(qt[h].x, qt[h].y), make_float2(kt[u].x, kt[u].y), a);
        a = ffma2(make_float2(qt[h].z, qt[h].w), make_float2(kt[u].z, kt[u].w), a);
        if (KF) {
          a = ffma2(make_float2(qf[h].x, qf[h].y), make_float2(kf[u].x, kf[u].y), a);
          a = ffma2(make_float2(qf[h].z, qf[h].w), make_float2(kf[u].z, kf[u].w), a);
        }
        part[2 * u + h] = a.x + a.y;
      }
    }
    // transposing butterfly: 2*EC values; value v ends on lanes v*(32/(2*EC)) ..
    float lg[2 * EC];
    {
      const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
      for (int j = 0; j < EC; ++j) {
        const float send = b4 ? part[j] : part[j + EC];
        const float keep = b4 ? part[j + EC] : part[j];
        part[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      }
      if constexpr (EC >= 2) {
#pragma unroll
        for (int j = 0; j < EC / 2; ++j) {
          const float send = b3 ? part[j] : part[j + EC / 2];
          const float keep = b3 ? part[j + EC / 2] : part[j];
          part[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
      }
      if constexpr (EC >= 4) {
        const float send = b2 ? part[0] : part[1];
        const float keep = b2 ? part[1] : part[0];
        part[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
      } else {
        part[0] += __shfl_xor_sync(0xffffffffu, part[0], 4);
      }
      part[0] += __shfl_xor_sync(0xffffffffu, part[0], 2);
      part[0] += __shfl_xor_sync(0xffffffffu, part[0], 1);
      constexpr int stride = 32 / (2 * EC);
#pragma unroll
      for (int v = 0; v < 2 * EC; ++v) lg[v] = __shfl_sync(0xffffffffu, part[0], stride * v);
    }
    // entries past E (zero-filled stages) get logit -inf: out of the max, weight 0
#pragma unroll
    for (int u = 1; u < EC; ++u)
      if (e0 + u >= E) lg[2 * u] = lg[2 * u + 1] = -INFINITY;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float cm = lg[h];
#pragma unroll
      for (int u = 1; u < EC; ++u) cm = fmaxf(cm, lg[2 * u + h]);
      const float nm = fmaxf(mx[h], cm);
      const float sc = ex2f(mx[h] - nm);  // logits are in log2 units (W_K carries log2 e)
      const float2 sc2 = make_float2(sc, sc);
      zs[h] *= sc;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        up[h][c] = fmul2(up[h][c], sc2);
        ut[h][c] = fmul2(ut[h][c], sc2);
        if (KF) uf[h][c] = fmul2(uf[h][c], sc2);
      }
#pragma unroll
      for (int u = 0; u < EC; ++u) {
        const float p = ex2f(lg[2 * u + h] - nm);
        const float2 p2 = make_float2(p, p);
        zs[h] += p;
        up[h][0] = ffma2(p2, make_float2(kp[u].x, kp[u].y), up[h][0]);
        up[h][1] = ffma2(p2, make_float2(kp[u].z, kp[u].w), up[h][1]);
        ut[h][0] = ffma2(p2, make_float2(kt[u].x, kt[u].y), ut[h][0]);
        ut[h][1] = ffma2(p2, make_float2(kt[u].z, kt[u].w), ut[h][1]);
        if (KF) {
          uf[h][0] = ffma2(p2, make_float2(kf[u].x, kf[u].y), uf[h][0]);
          uf[h][1] = ffma2(p2, make_float2(kf[u].z, kf[u].w), uf[h][1]);
        }
      }
      mx[h] = nm;
    }
  }
#endif
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float* Uh = U + h * kp;
    const float inv = E > 0 ? 1.f / zs[h] : 0.f;
    if (lp)
      *reinterpret_cast<float4*>(Uh + 4 * lane) =
          make_float4(up[h][0].x * inv, up[h][0].y * inv, up[h][1].x * inv, up[h][1].y * inv);
    if (lf)
      *reinterpret_cast<float4*>(Uh + kfo + 4 * lane) =
          make_float4(uf[h][0].x * inv, uf[h][0].y * inv, uf[h][1].x * inv, uf[h][1].y * inv);
    if (lt) {
      const float uc0 = ut[h][0].x * inv, us0 = ut[h][0].y * inv;
      const float uc1 = ut[h][1].x * inv, us1 = ut[h][1].y * inv;
#if A4_TRIG
      *reinterpret_cast<float4*>(Uh + kto + 4 * lane) = make_float4(uc0, us0, uc1, us1);
#else  // rotate the accumulated basis back by w tref
      *reinterpret_cast<float4*>(Uh + kto + 4 * lane) =
          make_float4(ca0 * uc0 + sa0 * us0, sa0 * uc0 - ca0 * us0, ca1 * uc1 + sa1 * us1,
                      sa1 * uc1 - ca1 * us1);
#endif
    }
  }
}

// Walk of two rows per warp (A4_HW): lanes 0-15 walk this warp's first row,
// lanes 16-31 its second (node < 0 / E = 0 for an idle half). Math as
// a4_walk_row with 16 lanes per row: lane hl of a half owns key features
// [8 hl, 8 hl + 8) of the payload, of the edge features and of the time
// encoding (frequencies 4 hl .. 4 hl + 3). One entry of each row per stage
// (the stage of two A4_EC = 2 chunks); the loop runs to the longer row, the
// other half's extra entries are zero-filled with logit -inf. Per entry one
// 16-lane transposing reduction serves both heads of both rows.
template <int KF>
__device__ __forceinline__ void a4_walk_half(const Geo& g, const A4W& w, const RingSrc& rs,
                                             float* U, int node, int E, int hd, double tref,
                                             int l, int lane, float4* stg) {
  constexpr int NSEG = KF ? 3 : 2;
  constexpr int NST = A4_NST;
  const int hl = lane & 15, hf = lane >> 4;
  const int kfo = w.kfo, kto = w.kto, kp = w.kpad;
  const bool valid = node >= 0;  // a row with no entries still gets ubar = 0 written
  if (!valid) {
    node = 0;
    E = 0;
  }
  const int nf4p = kfo / 4, nf4f = (kto - kfo) / 4, nf4t = (kp - kto) / 4;
  const bool lp0 = 2 * hl < nf4p, lp1 = 2 * hl + 1 < nf4p;
  const bool lf0 = KF && 2 * hl < nf4f, lf1 = KF && 2 * hl + 1 < nf4f;
  const bool lt0 = 2 * hl < nf4t, lt1 = 2 * hl + 1 < nf4t;
  const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
  // rotation by w tref, frequencies 4 hl + i
  float ca[4], sa[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    ca[i] = 1.f;
    sa[i] = 0.f;
    const int f = 4 * hl + i;
    if (E > 0 && f < g.half) phase_sincos(__ldg(w.omega + f), tref, &sa[i], &ca[i]);
  }
  float4 qp[2][2], qf[2][2], qt[2][2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float* Uh = U + h * kp;
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const bool vp = x ? lp1 : lp0, vf = x ? lf1 : lf0, vt = x ? lt1 : lt0;
      qp[h][x] = vp ? *reinterpret_cast<const float4*>(Uh + 8 * hl + 4 * x) : zero4;
      qf[h][x] = vf ? *reinterpret_cast<const float4*>(Uh + kfo + 8 * hl + 4 * x) : zero4;
      const float4 q = vt ? *reinterpret_cast<const float4*>(Uh + kto + 8 * hl + 4 * x) : zero4;
      const float c0 = ca[2 * x], s0 = sa[2 * x], c1 = ca[2 * x + 1], s1 = sa[2 * x + 1];
      qt[h][x] = make_float4(q.x * c0 + q.y * s0, q.x * s0 - q.y * c0, q.z * c1 + q.w * s1,
                             q.z * s1 - q.w * c1);
    }
  }
  float2 up[2][4], uf[2][4], ut[2][4];
  float mx[2] = {-INFINITY, -INFINITY}, zs[2] = {0.f, 0.f};
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < 4; ++c) up[h][c] = uf[h][c] = ut[h][c] = make_float2(0.f, 0.f);
  const float* payb = rs.ring_pay + ((int64_t)node * g.K + l) * g.L * g.ld_d + 8 * hl;
  const float* ftb = rs.ring_feat + (int64_t)node * g.L * g.ld_e + 8 * hl;
  const float* tbb = rs.ring_tb + (int64_t)node * g.L * g.ld_t + 8 * hl;
#if A4_HINTS
  const uint64_t pol_pay = pol_evict_first();
  const uint64_t pol_tb = l + 1 < g.K ? pol_evict_last() : pol_evict_first();
#endif
  const int nent = max(E, __shfl_xor_sync(0xffffffffu, E, 16));  // warp-uniform trip count
  int iss_slot = 0, con_slot = 0;
  int r_slot = hd;
  const float* r_pay = payb + (int64_t)hd * g.ld_d;
  const float* r_tb = tbb + (int64_t)hd * g.ld_t;
  const float* r_ft = ftb + (int64_t)hd * g.ld_e;
  auto issue = [&](int e) {
    if (e < nent) {
      float4* sb = stg + iss_slot * (NSEG * 64) + hf * 32 + 2 * hl;
      const bool ev = e < E;
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int pb = (ev && (x ? lp1 : lp0)) ? 16 : 0, tb = (ev && (x ? lt1 : lt0)) ? 16 : 0;
#if A4_HINTS
        cp_async16_pol(sb + x, r_pay + 4 * x, pb, pol_pay);
        cp_async16_pol(sb + 64 + x, r_tb + 4 * x, tb, pol_tb);
#else
        cp_async16(sb + x, r_pay + 4 * x, pb);
        cp_async16(sb + 64 + x, r_tb + 4 * x, tb);
#endif
        if (KF) cp_async16(sb + 128 + x, r_ft + 4 * x, (ev && (x ? lf1 : lf0)) ? 16 : 0);
      }
      if (++r_slot == g.L) {
        r_slot = 0;
        r_pay = payb;
        r_tb = tbb;
        r_ft = ftb;
      } else {
        r_pay += g.ld_d;
        r_tb += g.ld_t;
        r_ft += g.ld_e;
      }
    }
    cp_async_commit();
    if (++iss_slot == NST) iss_slot = 0;
  };
#pragma unroll
  for (int c = 0; c < NST - 1; ++c) issue(c);
  for (int e = 0; e < nent; ++e) {
    const int slot_c = con_slot;
    if (++con_slot == NST) con_slot = 0;
    issue(e + NST - 1);
    cp_async_wait<NST - 1>();
    const float4* sb = stg + slot_c * (NSEG * 64) + hf * 32 + 2 * hl;
    float4 kpv[2], ktv[2], kfv[2];
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      kpv[x] = sb[x];
      ktv[x] = sb[64 + x];
      kfv[x] = KF ? sb[128 + x] : zero4;
    }
    float part[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float2 a = fmul2(make_float2(qp[h][0].x, qp[h][0].y), make_float2(kpv[0].x, kpv[0].y));
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        if (x) a = ffma2(make_float2(qp[h][1].x, qp[h][1].y), make_float2(kpv[1].x, kpv[1].y), a);
        a = ffma2(make_float2(qp[h][x].z, qp[h][x].w), make_float2(kpv[x].z, kpv[x].w), a);
        a = ffma2(make_float2(qt[h][x].x, qt[h][x].y), make_float2(ktv[x].x, ktv[x].y), a);
        a = ffma2(make_float2(qt[h][x].z, qt[h][x].w), make_float2(ktv[x].z, ktv[x].w), a);
        if (KF) {
          a = ffma2(make_float2(qf[h][x].x, qf[h][x].y), make_float2(kfv[x].x, kfv[x].y), a);
          a = ffma2(make_float2(qf[h][x].z, qf[h][x].w), make_float2(kfv[x].z, kfv[x].w), a);
        }
      }
      part[h] = a.x + a.y;
    }
    // 16-lane transposing reduction: head 0 ends on lanes hl < 8, head 1 on hl >= 8
    const bool b3 = hl & 8;
    float v = (b3 ? part[1] : part[0]) + __shfl_xor_sync(0xffffffffu, b3 ? part[0] : part[1], 8);
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    float lg[2];
    lg[0] = __shfl_sync(0xffffffffu, v, hf * 16);
    lg[1] = __shfl_sync(0xffffffffu, v, hf * 16 + 8);
    if (e >= E) lg[0] = lg[1] = -INFINITY;  // this half's row has no entry e: weight 0
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float nm = fmaxf(mx[h], lg[h]);
      // an idle half keeps nm = -inf: the exponents below are then NaN-free by the selects
      const float sc = nm == -INFINITY ? 1.f : ex2f(mx[h] - nm);
      const float p = nm == -INFINITY ? 0.f : ex2f(lg[h] - nm);
      const float2 sc2 = make_float2(sc, sc), p2 = make_float2(p, p);
      zs[h] = fmaf(zs[h], sc, p);
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        up[h][2 * x] = ffma2(p2, make_float2(kpv[x].x, kpv[x].y), fmul2(up[h][2 * x], sc2));
        up[h][2 * x + 1] = ffma2(p2, make_float2(kpv[x].z, kpv[x].w), fmul2(up[h][2 * x + 1], sc2));
        ut[h][2 * x] = ffma2(p2, make_float2(ktv[x].x, ktv[x].y), fmul2(ut[h][2 * x], sc2));
        ut[h][2 * x + 1] = ffma2(p2, make_float2(ktv[x].z, ktv[x].w), fmul2(ut[h][2 * x + 1], sc2));
        if (KF) {
          uf[h][2 * x] = ffma2(p2, make_float2(kfv[x].x, kfv[x].y), fmul2(uf[h][2 * x], sc2));
          uf[h][2 * x + 1] = ffma2(p2, make_float2(kfv[x].z, kfv[x].w), fmul2(uf[h][2 * x + 1], sc2));
        }
      }
      mx[h] = nm;
    }
  }
  __syncwarp();
  if (!valid) return;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float* Uh = U + h * kp;
    const float inv = E > 0 ? 1.f / zs[h] : 0.f;
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      if (x ? lp1 : lp0)
        *reinterpret_cast<float4*>(Uh + 8 * hl + 4 * x) =
            make_float4(up[h][2 * x].x * inv, up[h][2 * x].y * inv, up[h][2 * x + 1].x * inv,
                        up[h][2 * x + 1].y * inv);
      if (x ? lf1 : lf0)
        *reinterpret_cast<float4*>(Uh + kfo + 8 * hl + 4 * x) =
            make_float4(uf[h][2 * x].x * inv, uf[h][2 * x].y * inv, uf[h][2 * x + 1].x * inv,
                        uf[h][2 * x + 1].y * inv);
      if (x ? lt1 : lt0) {
        const float uc0 = ut[h][2 * x].x * inv, us0 = ut[h][2 * x].y * inv;
        const float uc1 = ut[h][2 * x + 1].x * inv, us1 = ut[h][2 * x + 1].y * inv;
        const float c0 = ca[2 * x], s0 = sa[2 * x], c1 = ca[2 * x + 1], s1 = sa[2 * x + 1];
        *reinterpret_cast<float4*>(Uh + kto + 8 * hl + 4 * x) =
            make_float4(c0 * uc0 + s0 * us0, s0 * uc0 - c0 * us0, c1 * uc1 + s1 * us1,
                        s1 * uc1 - c1 * us1);
      }
    }
  }
}

// Walk 2: the rows of one 32-row quadrant, warp per row, taken from a shared
// counter. Ring rows reach shared memory as TMA bulk copies: one lane issues
// a chunk of A4_EC2 entries (payload, time basis and features of consecutive
// ring slots: at most two contiguous runs each, as the ring may wrap) into one
// of the warp's two stages, completing on the stage's mbarrier; the next
// chunk (of this row or of the next row, taken one ahead) is always in flight
// while one is reduced. No per-lane copy issue, no address arithmetic per lane.
// Per chunk: logits of both heads (packed FMAs, one transposing butterfly),
// online softmax update, ubar accumulation. Math as a4_walk_row.
struct A4Stg {
  float* base;     // this warp's two stages
  uint64_t* bar;   // this warp's two stage mbarriers
  int stg_floats;  // floats per stage
  uint32_t n_iss, n_con;  // chunks issued / consumed by this warp (stage = n & 1, parity = (n >> 1) & 1)
};

template <int KF>
__device__ __forceinline__ void a4_issue2(const Geo& g, const RingSrc& rs, A4Stg& S, int node,
                                          int E, int hd, int c, int l, int lane) {
  constexpr int EC = A4_EC2;
  const int st = (int)(S.n_iss & 1u);
  ++S.n_iss;
  if (lane == 0) {
    const int e0 = c * EC;
    const int n = min(EC, E - e0);
    int s0 = hd + e0;
    if (s0 >= g.L) s0 -= g.L;
    const int n1 = min(n, g.L - s0), n2 = n - n1;
    uint64_t* bar = S.bar + st;
    const uint32_t per = (uint32_t)(g.ld_d + g.ld_t + (KF ? g.ld_e : 0)) * 4u;
    mbar_expect_tx(bar, (uint32_t)n * per);
    float* dst = S.base + st * S.stg_floats;
    const float* pay = rs.ring_pay + ((int64_t)node * g.K + l) * g.L * g.ld_d;
    const float* tb = rs.ring_tb + (int64_t)node * g.L * g.ld_t;
    bulk_g2s(dst, pay + (int64_t)s0 * g.ld_d, (uint32_t)(n1 * g.ld_d * 4), bar);
    if (n2 > 0) bulk_g2s(dst + n1 * g.ld_d, pay, (uint32_t)(n2 * g.ld_d * 4), bar);
    float* dtb = dst + EC * g.ld_d;
    bulk_g2s(dtb, tb + (int64_t)s0 * g.ld_t, (uint32_t)(n1 * g.ld_t * 4), bar);
    if (n2 > 0) bulk_g2s(dtb + n1 * g.ld_t, tb, (uint32_t)(n2 * g.ld_t * 4), bar);
    if (KF) {
      const float* ft = rs.ring_feat + (int64_t)node * g.L * g.ld_e;
      float* dft = dtb + EC * g.ld_t;
      bulk_g2s(dft, ft + (int64_t)s0 * g.ld_e, (uint32_t)(n1 * g.ld_e * 4), bar);
      if (n2 > 0) bulk_g2s(dft + n1 * g.ld_e, ft, (uint32_t)(n2 * g.ld_e * 4), bar);
    }
  }
}

template <int KF>
__device__ __forceinline__ void a4_walk2_quadrant(const Geo& g, const A4W& w, const RingSrc& rs,
                                                  float* Ub, int q, int nrows, int* ctr,
                                                  const int* s_node, const int* s_E,
                                                  const int* s_head, const double* s_tref, int l,
                                                  int lane, A4Stg& S, int T) {
  constexpr int EC = A4_EC2;
  const int kfo = w.kfo, kto = w.kto, kp = w.kpad;
  const bool lp = lane < kfo / 4, lf = KF && lane < (kto - kfo) / 4, lt = lane < (kp - kto) / 4;
  const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
  auto grab = [&]() {
    int i = 0;
    for (;;) {
      if (lane == 0) i = atomicAdd(ctr, 1);
      i = __shfl_sync(0xffffffffu, i, 0);
#if A4_BPF == 2
      if (lane == 0 && i < nrows && 32 * q + i + A4_PFD < T) {
        const int rp = 32 * q + i + A4_PFD;
        a4_row_prefetch(g, rs, s_node[rp], s_E[rp], s_head[rp], l);
      }
#endif
      if (i >= nrows || s_node[32 * q + i] >= 0) return i;
    }
  };
  int i = grab();
  if (i < nrows && s_E[32 * q + i] > 0)
    a4_issue2<KF>(g, rs, S, s_node[32 * q + i], s_E[32 * q + i], s_head[32 * q + i], 0, l, lane);
  while (i < nrows) {
    const int r = 32 * q + i;
    const int nx = grab();  // next row, one ahead: its first chunk is issued during this row's last
    const int rn = 32 * q + nx;
    const bool nx_issue = nx < nrows && s_E[rn] > 0;
    const int node = s_node[r], E = s_E[r], hd = s_head[r];
    const double tref = s_tref[r];
    float* U = Ub + i * w.ldu;
    if (E == 0 && nx_issue) a4_issue2<KF>(g, rs, S, s_node[rn], s_E[rn], s_head[rn], 0, l, lane);
    float ca0 = 1.f, sa0 = 0.f, ca1 = 1.f, sa1 = 0.f;
    if (lt && 2 * lane < g.half) phase_sincos(__ldg(w.omega + 2 * lane), tref, &sa0, &ca0);
    if (lt && 2 * lane + 1 < g.half) phase_sincos(__ldg(w.omega + 2 * lane + 1), tref, &sa1, &ca1);
    float4 qp[2], qf[2], qt[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float* Uh = U + h * kp;
      qp[h] = lp ? *reinterpret_cast<const float4*>(Uh + 4 * lane) : zero4;
      qf[h] = lf ? *reinterpret_cast<const float4*>(Uh + kfo + 4 * lane) : zero4;
      const float4 qq = lt ? *reinterpret_cast<const float4*>(Uh + kto + 4 * lane) : zero4;
      qt[h] = make_float4(qq.x * ca0 + qq.y * sa0, qq.x * sa0 - qq.y * ca0,
                          qq.z * ca1 + qq.w * sa1, qq.z * sa1 - qq.w * ca1);
    }
    float2 up[2][2], uf[2][2], ut[2][2];
    float mx[2] = {-INFINITY, -INFINITY}, zs[2] = {0.f, 0.f};
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int c = 0; c < 2; ++c) up[h][c] = uf[h][c] = ut[h][c] = make_float2(0.f, 0.f);
    const int nch = (E + EC - 1) / EC;
    for (int c = 0; c < nch; ++c) {
      if (c + 1 < nch) a4_issue2<KF>(g, rs, S, node, E, hd, c + 1, l, lane);
      else if (nx_issue) a4_issue2<KF>(g, rs, S, s_node[rn], s_E[rn], s_head[rn], 0, l, lane);
      const int st = (int)(S.n_con & 1u);
      mbar_wait(S.bar + st, (S.n_con >> 1) & 1u);
      ++S.n_con;
      const int e0 = c * EC;
      const float* sp = S.base + st * S.stg_floats;
      const float* stb = sp + EC * g.ld_d;
      const float* sft = stb + EC * g.ld_t;
      float4 kpv[EC], ktv[EC], kfv[EC];
#pragma unroll
      for (int u = 0; u < EC; ++u) {
        const bool ev = e0 + u < E;  // warp-uniform; slots past E hold stale bytes: zero them
        kpv[u] = (ev && lp) ? *reinterpret_cast<const float4*>(sp + u * g.ld_d + 4 * lane) : zero4;
        ktv[u] = (ev && lt) ? *reinterpret_cast<const float4*>(stb + u * g.ld_t + 4 * lane) : zero4;
        kfv[u] = (KF && ev && lf) ? *reinterpret_cast<const float4*>(sft + u * g.ld_e + 4 * lane) : zero4;
      }
      __syncwarp();  // every lane has its chunk in registers: the stage may be refilled
      float part[2 * EC];
#pragma unroll
      for (int u = 0; u < EC; ++u) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float2 a = fmul2(make_float2(qp[h].x, qp[h].y), make_float2(kpv[u].x, kpv[u].y));
          a = ffma2(make_float2(qp[h].z, qp[h].w), make_float2(kpv[u].z, kpv[u].w), a);
          a = ffma2(make_float2(qt[h].x, qt[h].y), make_float2(ktv[u].x, ktv[u].y), a);
          a = ffma2(make_float2(qt[h].z, qt[h].w), make_float2(ktv[u].z, ktv[u].w), a);
          if (KF) {
            a = ffma2(make_float2(qf[h].x, qf[h].y), make_float2(kfv[u].x, kfv[u].y), a);
            a = ffma2(make_float2(qf[h].z, qf[h].w), make_float2(kfv[u].z, kfv[u].w), a);
          }
          part[2 * u + h] = a.x + a.y;
        }
      }
      // transposing butterfly over the 2*EC values; value v ends on lanes [v*32/(2EC), ...)
      float lg[2 * EC];
      {
        constexpr int V = 2 * EC;
#pragma unroll
        for (int m = 16, nv = V; m >= 1; m >>= 1) {
          if (nv > 1) {
            const bool hi = lane & m;
#pragma unroll
            for (int j = 0; j < nv / 2; ++j) {
              const float send = hi ? part[j] : part[j + nv / 2];
              const float keep = hi ? part[j + nv / 2] : part[j];
              part[j] = keep + __shfl_xor_sync(0xffffffffu, send, m);
            }
            nv >>= 1;
          } else {
            part[0] += __shfl_xor_sync(0xffffffffu, part[0], m);
          }
        }
        constexpr int stride = 32 / V;
#pragma unroll
        for (int v = 0; v < V; ++v) lg[v] = __shfl_sync(0xffffffffu, part[0], stride * v);
      }
#pragma unroll
      for (int u = 1; u < EC; ++u)
        if (e0 + u >= E) lg[2 * u] = lg[2 * u + 1] = -INFINITY;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float cm = lg[h];
#pragma unroll
        for (int u = 1; u < EC; ++u) cm = fmaxf(cm, lg[2 * u + h]);
        const float nm = fmaxf(mx[h], cm);
        const float sc = ex2f(mx[h] - nm);
        const float2 sc2 = make_float2(sc, sc);
        zs[h] *= sc;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          up[h][cc] = fmul2(up[h][cc], sc2);
          ut[h][cc] = fmul2(ut[h][cc], sc2);
          if (KF) uf[h][cc] = fmul2(uf[h][cc], sc2);
        }
#pragma unroll
        for (int u = 0; u < EC; ++u) {
          const float pr = ex2f(lg[2 * u + h] - nm);
          const float2 p2 = make_float2(pr, pr);
          zs[h] += pr;
          up[h][0] = ffma2(p2, make_float2(kpv[u].x, kpv[u].y), up[h][0]);
          up[h][1] = ffma2(p2, make_float2(kpv[u].z, kpv[u].w), up[h][1]);
          ut[h][0] = ffma2(p2, make_float2(ktv[u].x, ktv[u].y), ut[h][0]);
          ut[h][1] = ffma2(p2, make_float2(ktv[u].z, ktv[u].w), ut[h][1]);
          if (KF) {
            uf[h][0] = ffma2(p2, make_float2(kfv[u].x, kfv[u].y), uf[h][0]);
            uf[h][1] = ffma2(p2, make_float2(kfv[u].z, kfv[u].w), uf[h][1]);
          }
        }
        mx[h] = nm;
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float* Uh = U + h * kp;
      const float inv = E > 0 ? 1.f / zs[h] : 0.f;
      if (lp)
        *reinterpret_cast<float4*>(Uh + 4 * lane) =
            make_float4(up[h][0].x * inv, up[h][0].y * inv, up[h][1].x * inv, up[h][1].y * inv);
      if (lf)
        *reinterpret_cast<float4*>(Uh + kfo + 4 * lane) =
            make_float4(uf[h][0].x * inv, uf[h][0].y * inv, uf[h][1].x * inv, uf[h][1].y * inv);
      if (lt) {  // rotate the accumulated basis back by w tref
        const float uc0 = ut[h][0].x * inv, us0 = ut[h][0].y * inv;
        const float uc1 = ut[h][1].x * inv, us1 = ut[h][1].y * inv;
        *reinterpret_cast<float4*>(Uh + kto + 4 * lane) =
            make_float4(ca0 * uc0 + sa0 * us0, sa0 * uc0 - ca0 * us0, ca1 * uc1 + sa1 * us1,
                        sa1 * uc1 - ca1 * us1);
      }
    }
    i = nx;
  }
}

template <int KF>
__global__ void __launch_bounds__(A4_THREADS, 1)
attn4_kernel(Geo g, A4W w, RingSrc rs) {
  PDL_WAIT();
#ifdef STGN_SKIP_RECOMPUTE  // timing experiments only: results are wrong
  return;
#endif
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align by indexing the shared array (not by integer arithmetic on its
  // address), so the compiler keeps the shared address space: LDS/STS instead
  // of generic LD/ST on the row buffers and the cp.async stages
  unsigned char* sbase = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint16_t* Wb0 = reinterpret_cast<uint16_t*>(sbase);
  uint16_t* Wb1 = reinterpret_cast<uint16_t*>(sbase + w.wblk_bytes);
  float* Ub0 = reinterpret_cast<float*>(sbase + (size_t)w.region_bytes);
  float* Ub1 = A4_NUB > 1 ? Ub0 + 32 * w.ldu : Ub0;
  __shared__ int s_node[A4_TMAX], s_E[A4_TMAX], s_head[A4_TMAX], s_mode[A4_TMAX];
#if A4_NXH
  __shared__ int nx_node[A4_TMAX], nx_E[A4_TMAX], nx_head[A4_TMAX], nx_mode[A4_TMAX];
  __shared__ double nx_tref[A4_TMAX];
#endif
#if A4_LPT
  __shared__ int s_idx[A4_TMAX], t_node[A4_TMAX], t_E[A4_TMAX], t_head[A4_TMAX], t_mode[A4_TMAX];
  __shared__ double t_tref[A4_TMAX];
#endif
  __shared__ double s_tref[A4_TMAX];
  __shared__ uint64_t mbar, wbar[2];
  __shared__ uint64_t qbar_full[2], qbar_done[2], qbar_packed[2];
#if A4_WALK == 2
  __shared__ uint64_t sbar2[2 * A4_WARPS];
#endif
  __shared__ int qctr[2];
  __shared__ uint32_t tslot;
#if A4_GA
  __shared__ int s_wq[32 * A4_WARPS];  // per warp: rows taken by the issue stream, in order
#endif

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int quad = warp & 3, cg = warp >> 2;
  const int64_t N = rs.count();
  if (N <= 0) return;
  const int64_t grid = gridDim.x;
  const int64_t waves = cdiv(N, grid * A4_TMAX);
  const int T = (int)cdiv(N, grid * waves);  // balanced tile rows (<= 128)
  const int64_t ntiles = cdiv(N, T);
  if ((int64_t)blockIdx.x >= ntiles) return;
  const int64_t my_tiles = cdiv(ntiles - blockIdx.x, grid);
  const int64_t total_blocks = my_tiles * g.K * w.nbl;
  const int64_t pre_rows = rs.fused ? (int64_t)rs.pre_n[0] : N;
  const int64_t d_rows = rs.fused ? (int64_t)rs.post_n[0] : 0;

#ifdef A4_PROF
  if (tid == 0 && blockIdx.x < 1024) g_a4_cta[4 * blockIdx.x] = a4_now();
  unsigned long long prof_e = 0;
#endif
  if (warp == 0) tmem_alloc(&tslot, 512);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    mbar_init(&wbar[0], 1);
    mbar_init(&wbar[1], 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&qbar_full[b], 32 * A4_NCG);
      mbar_init(&qbar_done[b], A4_THREADS);
      mbar_init(&qbar_packed[b], 32 * A4_NCG);
    }
#if A4_WALK == 2
    for (int b = 0; b < 2 * A4_WARPS; ++b) mbar_init(&sbar2[b], 1);
#endif
    mbar_fence_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t lane_base = (uint32_t)(32 * quad) << 16;
  const int row = 32 * quad + lane;
  auto stage = [&](int64_t G) {  // one thread
    int64_t el;
    const uint16_t* src = a4_block(g, w, (int)((G / w.nbl) % g.K), (int)(G % w.nbl), &el);
    bulk_stage((G & 1) ? (void*)Wb1 : (void*)Wb0, src, (uint32_t)(el * 2), &wbar[G & 1]);
  };
  if (tid == 0) {
    stage(0);
    if (total_blocks > 1) stage(1);
  }
  // the walk's per-warp cp.async stages live in the two weight buffers: V_0 and
  // V_1 (blocks 3, 4 of a layer) are staged after the walk instead of during it
#if A4_CPK
  float4* stg_warp = reinterpret_cast<float4*>(sbase) + (size_t)warp * A4_NST * A4_EC * (w.kpad / 4);
#else
  float4* stg_warp = reinterpret_cast<float4*>(sbase) + (size_t)warp * A4_NST * A4_EC * (KF ? 3 : 2) * 32;
#endif
#if A4_WALK == 2
  A4Stg S2;
  S2.stg_floats = A4_EC2 * (g.ld_d + g.ld_t + (KF ? g.ld_e : 0));
  S2.base = reinterpret_cast<float*>(sbase) + (size_t)warp * 2 * S2.stg_floats;
  S2.bar = sbar2 + 2 * warp;
  S2.n_iss = S2.n_con = 0;
#endif
  auto deferred = [&](int64_t Gb) { const int j = (int)(Gb % w.nbl); return j == 3 || j == 4; };
  int64_t G = 0;  // weight blocks consumed by this CTA
  int ub_use[2] = {0, 0};  // uses of each quadrant row buffer so far (mbarrier phases)
  // one GEMM: wait for its weights, MMA, wait for the MMA, refill the buffer.
  // Callers put a CTA barrier before every gemm: mbarrier waits are by phase
  // parity, so no thread may fall two commit phases behind.
  uint32_t mph = 0;  // commits of the MMA barrier so far (its phase parity)
  auto gemm = [&](int a, int Np, int Kp, int dcol) {
    if (tid == 0) {  // only the issuing thread waits for the weights
      mbar_wait(&wbar[G & 1], (uint32_t)((G >> 1) & 1));
      a4_mma(tmem, a, (G & 1) ? Wb1 : Wb0, Np, Kp, dcol, &mbar);
    }
    mbar_wait(&mbar, mph & 1u);
    ++mph;
    tc_fence_after();
    if (tid == 0 && G + 2 < total_blocks && !deferred(G + 2)) stage(G + 2);
    ++G;
  };
  // two blocks (both weight buffers) accumulated into one D, one commit
  auto gemm_pair = [&](int a0, int a1, int Np, int Kp, int dcol) {
    if (tid == 0) {
      mbar_wait(&wbar[G & 1], (uint32_t)((G >> 1) & 1));
      a4_mma(tmem, a0, (G & 1) ? Wb1 : Wb0, Np, Kp, dcol, &mbar, false, false);
      mbar_wait(&wbar[(G + 1) & 1], (uint32_t)(((G + 1) >> 1) & 1));
      a4_mma(tmem, a1, ((G + 1) & 1) ? Wb1 : Wb0, Np, Kp, dcol, &mbar, true, true);
    }
    mbar_wait(&mbar, mph & 1u);
    ++mph;
    tc_fence_after();
    if (tid == 0) {
      if (G + 2 < total_blocks && !deferred(G + 2)) stage(G + 2);
      if (G + 3 < total_blocks && !deferred(G + 3)) stage(G + 3);
    }
    G += 2;
  };
  auto cta_sync_tc = [&]() {
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  };

  // row i of tile `tl`: node (-1 if none / another rank's), ring entry count, head, t_ref, mode
  auto row_header = [&](int64_t tl, int i, int& node, int& E, int& head, int& mode, double& tref) {
    const int64_t idx = tl * T + i;
    node = -1; E = 0; head = 0; mode = 0; tref = 0.0;
    if (i < T && idx < N) {
      node = rs.node(idx);
      if (rs.fused) mode = idx >= pre_rows ? 2 : (idx < d_rows ? 1 : 0);
      const int cc = node >= 0 ? rs.ring_ccnt[node] : 0;
      E = node < 0 ? 0 : (cc >= 0 ? cc : (rs.use_store ? rs.ring_cnt[node] : 0));
      head = node >= 0 ? rs.ring_head[node] : 0;
      if (E > 0) tref = rs.ring_t[(int64_t)node * g.L + head];
    }
  };
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += grid) {
    const int64_t base = tile * T;
    if (tid < A4_TMAX) {
      const int i = tid;
      int node, E, head, mode;
      double tref;
#if A4_NXH
      if (tile != blockIdx.x) {  // loaded during the previous tile's first walk
        node = nx_node[i]; E = nx_E[i]; head = nx_head[i]; mode = nx_mode[i]; tref = nx_tref[i];
      } else {
        row_header(tile, i, node, E, head, mode, tref);
      }
#else
      row_header(tile, i, node, E, head, mode, tref);
#endif
#if A4_LPT
      t_node[i] = node; t_E[i] = E; t_head[i] = head; t_tref[i] = tref; t_mode[i] = mode;
#else
      s_node[i] = node; s_E[i] = E; s_head[i] = head; s_tref[i] = tref; s_mode[i] = mode;
#endif
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
#if A4_LPT
    // rows by descending entry count (longest first, stable): the walk takes
    // rows in this order, so the last rows of a tile-layer are the short ones
    // and the tail before the V GEMMs shrinks; s_idx maps back to the row index
    if (tid < A4_TMAX) {
      const int i = tid;
      if (i < T) {
        const int Ei = t_E[i];
        int rank = 0;
        for (int j = 0; j < T; ++j) {
          const int Ej = t_E[j];
          rank += (Ej > Ei) || (Ej == Ei && j < i);
        }
        s_node[rank] = t_node[i]; s_E[rank] = Ei; s_head[rank] = t_head[i];
        s_tref[rank] = t_tref[i]; s_mode[rank] = t_mode[i]; s_idx[rank] = i;
      } else {
        s_node[i] = -1; s_E[i] = 0; s_head[i] = 0; s_tref[i] = 0.0; s_mode[i] = 0; s_idx[i] = i;
      }
    }
    __syncthreads();
#define A4_ROWIDX(r) (base + s_idx[r])
#else
#define A4_ROWIDX(r) (base + (r))
#endif
    const int nq = (T + 31) / 32;
    const bool quad_live = quad < nq;
    // x_0 -> X_A (bf16 hi|lo)
    if (quad_live) {
      const int node = row < T ? s_node[row] : -1;
      const float* src = nullptr;
      if (node >= 0)
        src = s_mode[row] == 2 ? rs.mem_post + (A4_ROWIDX(row) - pre_rows) * g.ld_s
                               : rs.mem + (int64_t)node * g.ld_s;
      for (int j = cg; j < w.Kx / 16; j += A4_NCG) {
        float v[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = 16 * j + 4 * q;
          float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
          if (src && c < g.d_s) x = __ldg(reinterpret_cast<const float4*>(src + c));
          v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
        }
        a4_st16(tmem + lane_base + (uint32_t)(8 * j), tmem + lane_base + (uint32_t)(w.Kx / 2 + 8 * j), v);
      }
      tmem_st_wait();
    }

    for (int l = 0; l < g.K; ++l) {
      const bool last = (l == g.K - 1);
#if A4_BPF == 2
      if (tid < min(A4_PFD, T)) a4_row_prefetch(g, rs, s_node[tid], s_E[tid], s_head[tid], l);
#elif A4_BPF
      if (tid < T) {  // this tile-layer's payload rows -> L2, one bulk prefetch per contiguous run
        const int node = s_node[tid], E = s_E[tid], hd = s_head[tid];
        if (node >= 0 && E > 0) {
          const int n1 = min(E, g.L - hd), n2 = E - n1;
          const float* pay = rs.ring_pay + ((int64_t)node * g.K + l) * g.L * g.ld_d;
          bulk_prefetch_l2(pay + (int64_t)hd * g.ld_d, (uint32_t)(n1 * g.ld_d * 4));
          if (n2 > 0) bulk_prefetch_l2(pay, (uint32_t)(n2 * g.ld_d * 4));
        }
      }
#endif
#if A4_PREFETCH == 2
      a4_prefetch(g, rs, s_node, s_E, s_head, 0, T, l, tid);  // this layer's ring rows
#elif A4_PREFETCH == 1
      a4_prefetch(g, rs, s_node, s_E, s_head, 0, min(32, T), l, tid);  // first quadrant
#endif
      // ---- q = x W_Q + b ----
      A4_MARK(0);
      cta_sync_tc();
      gemm(0, w.Nq, w.Kx, w.Kx);
      for (int h = 0; h < 2; ++h) {
        // q_h (+ bias) -> QA as bf16 hi|lo
        if (quad_live) {
          const float* bq = w.bq + ((int64_t)l * 2 + h) * w.Kq;
          for (int j = cg; j < w.Kq / 16; j += A4_NCG) {
            float a[8], b[8], v[16];
            tmem_ld8_nw(tmem + lane_base + (uint32_t)(w.Kx + h * w.Kq + 16 * j), a);
            tmem_ld8_nw(tmem + lane_base + (uint32_t)(w.Kx + h * w.Kq + 16 * j + 8), b);
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              v[q] = a[q] + __ldg(bq + 16 * j + q);
              v[8 + q] = b[q] + __ldg(bq + 16 * j + 8 + q);
            }
            a4_st16(tmem + lane_base + (uint32_t)(8 * j), tmem + lane_base + (uint32_t)(w.Kq / 2 + 8 * j), v);
          }
          tmem_st_wait();
        }
        A4_MARK(1);
        cta_sync_tc();
        // ---- q~_h = (W_K,h / sqrt(d_k)) q_h -> QT_h ----
        gemm(0, w.Nk, w.Kq, h == 0 ? w.qt0 : w.qt1);
      }
#if A4_NXH
      // the next tile's row headers (dependent global loads) and an L2 prefetch of its
      // query rows, by the last warp before it joins this tile's first walk
      if (l == 0 && warp == A4_WARPS - 1 && tile + grid < ntiles) {
        for (int i = lane; i < A4_TMAX; i += 32) {
          int node, E, head, mode;
          double tref;
          row_header(tile + grid, i, node, E, head, mode, tref);
          nx_node[i] = node; nx_E[i] = E; nx_head[i] = head; nx_mode[i] = mode; nx_tref[i] = tref;
          if (node >= 0) {
            const float* xr = mode == 2 ? rs.mem_post + ((tile + grid) * T + i - pre_rows) * g.ld_s
                                        : rs.mem + (int64_t)node * g.ld_s;
            bulk_prefetch_l2(xr, (uint32_t)(g.ld_s * 4));
          }
        }
      }
#endif
      // ---- walk, one 32-row quadrant at a time ----
      A4_MARK(2);
      fence_async_smem();
#if A4_STATIC
      A4Iss iss{0, 0, 0, 2 * nq};
      int kcons = 0;
      auto issue_next = [&]() {
        a4_issue_next<KF>(g, w, rs, iss, s_node, s_E, s_head, T, warp, l, lane, stg_warp);
      };
#pragma unroll
      for (int p0 = 0; p0 < A4_NST - 1; ++p0) issue_next();
#endif
#if A4_EVQ && A4_WALK == 1 && !A4_STATIC
      // Quadrant pipeline as an event loop: the copy-out of quadrant q's q~
      // (fill) and the pack of its ubar (pack) are duties of the quadrant's
      // own four warps (TMEM lane access), done as soon as their mbarrier
      // condition holds (fill of q >= 2: quadrant q - 2 packed; pack: every
      // warp done with q), polled between walked rows and while waiting for
      // the next quadrant, so no warp blocks on a duty another warp has not
      // reached yet. Quadrant q uses row buffer q & 1.
      {
        const int ub0 = ub_use[0], ub1 = ub_use[1];
        auto uphase = [&](int qq) { return (uint32_t)((((qq & 1) ? ub1 : ub0) + (qq >> 1)) & 1); };
        bool fill_done = quad >= nq, pack_done = quad >= nq;
        auto duties = [&]() {
          const int b = quad & 1;
          float* Ubq = b ? Ub1 : Ub0;
          if (!fill_done && (quad < 2 || mbar_test(&qbar_packed[b], uphase(quad - 2)))) {
            const int nch = (w.kpad + 7) / 8;  // q~ rows of this quadrant -> Ub
            for (int c = cg; c < 2 * nch; c += A4_NCG) {
              const int h = c / nch, j = c % nch;
              float v[8];
              tmem_ld8_nw(tmem + lane_base + (uint32_t)((h == 0 ? w.qt0 : w.qt1) + 8 * j), v);
              tmem_ld_wait();
              float* dst = Ubq + lane * w.ldu + h * w.kpad + 8 * j;
              *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
              if (8 * j + 8 <= w.kpad)
                *reinterpret_cast<float4*>(dst + 4) = make_float4(v[4], v[5], v[6], v[7]);
            }
            if (cg == 0 && lane == 0) qctr[b] = 0;
            mbar_arrive(&qbar_full[b]);
            fill_done = true;
          }
          if (fill_done && !pack_done && mbar_test(&qbar_done[b], uphase(quad))) {
            const int nch = w.Ku / 16;  // ubar rows -> TMEM (bf16 hi|lo) where q~ was
            for (int c = cg; c < 2 * nch; c += A4_NCG) {
              const int h = c / nch, j = c % nch;
              const float* srow = Ubq + lane * w.ldu + h * w.kpad;
              float v[16];
#pragma unroll
              for (int k4 = 0; k4 < 4; ++k4) {
                const int k = 16 * j + 4 * k4;
                float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
                if (k < w.kpad) x = *reinterpret_cast<const float4*>(srow + k);
                v[4 * k4] = x.x; v[4 * k4 + 1] = x.y; v[4 * k4 + 2] = x.z; v[4 * k4 + 3] = x.w;
              }
              const int base_col = h == 0 ? w.qt0 : w.qt1;
              a4_st16(tmem + lane_base + (uint32_t)(base_col + 8 * j),
                      tmem + lane_base + (uint32_t)(base_col + w.Ku / 2 + 8 * j), v);
            }
            tmem_st_wait();
            mbar_arrive(&qbar_packed[b]);
            pack_done = true;
          }
        };
        for (int q = 0; q < nq; ++q) {
          const int b = q & 1;
          float* Ub = b ? Ub1 : Ub0;
          const int nrows = min(32, T - 32 * q);
#if A4_EVQW
          // with no duty of its own left the warp blocks in try_wait (hardware
          // suspend) instead of spinning on test_wait and taking issue slots
          // from the walking warps
          while (!mbar_test(&qbar_full[b], uphase(q))) {
            if (fill_done && pack_done) {
              mbar_wait(&qbar_full[b], uphase(q));
              break;
            }
            duties();
          }
#else
          while (!mbar_test(&qbar_full[b], uphase(q))) duties();
#endif
#if A4_GA
          // this quadrant's issue stream: the first NST - 1 chunks (rows taken as needed)
          A4Dyn dy{-1, 0, 0, 0, 0, 0, 0};
          int kcons_dyn = 0;
          int* q_rows = s_wq + 32 * warp;
          auto issue_dyn = [&]() {
            a4_issue_dyn<KF>(g, w, rs, dy, s_node, s_E, s_head, q, nrows, &qctr[b], q_rows, l,
                             lane, stg_warp);
          };
#pragma unroll
          for (int p0 = 0; p0 < A4_NST - 1; ++p0) issue_dyn();
#endif
          for (;;) {
            int i = 0;
#if A4_HW
            if (lane == 0) i = atomicAdd(&qctr[b], 2);  // two rows, a half-warp each
            i = __shfl_sync(0xffffffffu, i, 0);
            if (i >= nrows) break;
            {
              const int ih = i + (lane >> 4);
              const int r = 32 * q + ih;
              const bool ok = ih < nrows;
              a4_walk_half<KF>(g, w, rs, Ub + (ok ? ih : i) * w.ldu, ok ? s_node[r] : -1,
                               ok ? s_E[r] : 0, ok ? s_head[r] : 0, ok ? s_tref[r] : 0.0, l, lane,
                               stg_warp);
            }
#else
#if A4_GA
            if (dy.qh == dy.qt) break;  // every row taken has been walked
            __syncwarp();
            i = q_rows[dy.qh & 31] - 32 * q;
            ++dy.qh;
            {
              const int r = 32 * q + i;
              a4_walk_row<KF>(g, w, rs, Ub + i * w.ldu, s_node[r], s_E[r], s_head[r], s_tref[r],
                              l, lane, stg_warp, issue_dyn, &kcons_dyn);
            }
#else
            if (lane == 0) i = atomicAdd(&qctr[b], 1);
            i = __shfl_sync(0xffffffffu, i, 0);
            if (i >= nrows) break;
            const int r = 32 * q + i;
            if (s_node[r] >= 0)
              a4_walk_row<KF>(g, w, rs, Ub + i * w.ldu, s_node[r], s_E[r], s_head[r], s_tref[r],
                              l, lane, stg_warp, [] {}, nullptr);
#endif
#endif
            duties();
          }
          mbar_arrive(&qbar_done[b]);
        }
        while (!fill_done || !pack_done) duties();
        ub_use[0] += (nq + 1) / 2;
        ub_use[1] += nq / 2;
      }
#else
      // Quadrant pipeline over two row buffers, ordered by mbarriers instead of
      // CTA barriers: the quadrant's own warps copy q~ out of TMEM (full), every
      // warp takes rows of the buffer from a shared counter and walks them
      // (done), the quadrant's warps pack ubar back into TMEM (packed), which
      // frees the buffer for quadrant q + 2. A warp that finishes early moves
      // on to the next quadrant's rows.
      for (int q = 0; q < nq; ++q) {
        const int b = A4_NUB > 1 ? (q & 1) : 0;
        float* Ub = b ? Ub1 : Ub0;
        const int nrows = min(32, T - 32 * q);
#if A4_PREFETCH == 1
        if (q + 1 < nq) a4_prefetch(g, rs, s_node, s_E, s_head, 32 * (q + 1), min(32 * (q + 2), T), l, tid);
#endif
        if (quad == q) {  // q~ rows of this quadrant -> Ub
          if (ub_use[b] > 0) mbar_wait(&qbar_packed[b], (uint32_t)((ub_use[b] - 1) & 1));
          const int nch = (w.kpad + 7) / 8;
          for (int c = cg; c < 2 * nch; c += A4_NCG) {
            const int h = c / nch, j = c % nch;
            float v[8];
            tmem_ld8_nw(tmem + lane_base + (uint32_t)((h == 0 ? w.qt0 : w.qt1) + 8 * j), v);
            tmem_ld_wait();
            float* dst = Ub + lane * w.ldu + h * w.kpad + 8 * j;
            *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
            if (8 * j + 8 <= w.kpad)
              *reinterpret_cast<float4*>(dst + 4) = make_float4(v[4], v[5], v[6], v[7]);
          }
          if (tid == 32 * q) qctr[b] = 0;  // warp (quad q, cg 0), lane 0
          mbar_arrive(&qbar_full[b]);
        }
        mbar_wait(&qbar_full[b], (uint32_t)(ub_use[b] & 1));
#if A4_STATIC
        for (int hh = 0; hh < 2; ++hh) {  // this warp's rows of the quadrant
          const int i = warp + 16 * hh;
          const int r = 32 * q + i;
          if (i >= nrows || s_node[r] < 0) continue;
          a4_walk_row<KF>(g, w, rs, Ub + i * w.ldu, s_node[r], s_E[r], s_head[r], s_tref[r], l,
                          lane, stg_warp, issue_next, &kcons);
        }
#elif A4_WALK == 2
        a4_walk2_quadrant<KF>(g, w, rs, Ub, q, nrows, &qctr[b], s_node, s_E, s_head, s_tref, l,
                              lane, S2, T);
#else
        for (;;) {
          int i = 0;
          if (lane == 0) i = atomicAdd(&qctr[b], 1);
          i = __shfl_sync(0xffffffffu, i, 0);
          if (i >= nrows) break;
          const int r = 32 * q + i;
#if A4_BPF == 2
          if (lane == 0 && r + A4_PFD < T)
            a4_row_prefetch(g, rs, s_node[r + A4_PFD], s_E[r + A4_PFD], s_head[r + A4_PFD], l);
#endif
          if (s_node[r] < 0) continue;
          a4_walk_row<KF>(g, w, rs, Ub + i * w.ldu, s_node[r], s_E[r], s_head[r], s_tref[r], l,
                          lane, stg_warp, [] {}, nullptr);
        }
#endif
        mbar_arrive(&qbar_done[b]);
        if (quad == q) {  // ubar rows -> TMEM (bf16 hi|lo) where q~ was
          mbar_wait(&qbar_done[b], (uint32_t)(ub_use[b] & 1));
          const int nch = w.Ku / 16;
          for (int c = cg; c < 2 * nch; c += A4_NCG) {
            const int h = c / nch, j = c % nch;
            const float* srow = Ub + lane * w.ldu + h * w.kpad;
            float v[16];
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4) {
              const int k = 16 * j + 4 * k4;
              float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
              if (k < w.kpad) x = *reinterpret_cast<const float4*>(srow + k);
              v[4 * k4] = x.x; v[4 * k4 + 1] = x.y; v[4 * k4 + 2] = x.z; v[4 * k4 + 3] = x.w;
            }
            const int base_col = h == 0 ? w.qt0 : w.qt1;
            a4_st16(tmem + lane_base + (uint32_t)(base_col + 8 * j),
                    tmem + lane_base + (uint32_t)(base_col + w.Ku / 2 + 8 * j), v);
          }
          tmem_st_wait();
          mbar_arrive(&qbar_packed[b]);
        }
        ++ub_use[b];
      }
#endif
      A4_MARK(3);
      cta_sync_tc();
      A4_MARK(6);
      if (tid == 0) {  // the walk is done with the weight buffers: stage V_0, V_1
        fence_async_smem();
        stage(G);
        stage(G + 1);
      }
#if A4_VOF
      // ---- out_l = sum_h ubar_h P_h (P_h = W_V,h W_O,h), columns [0, Npa) then [Npa, No),
      //      accumulated in TMEM [0, 64) (free: QA is dead, ubar_1 starts at Kq) ----
      float va[16], vb[16];
      int64_t o_idx = 0;
      float* dst = nullptr;
      if (quad_live) {
        const int node = row < T ? s_node[row] : -1;
        const int mode = row < T ? s_mode[row] : 0;
        o_idx = A4_ROWIDX(row);
        if (node >= 0) {
          if (mode == 1) dst = last ? rs.dpred + o_idx * g.ld_d : nullptr;
          else if (rs.layers_out) dst = rs.layers_out + (o_idx * g.K + l) * g.ld_d;
          else if (rs.final_out) dst = last ? rs.final_out + o_idx * g.ld_d : nullptr;
          else dst = rs.h + ((int64_t)node * g.K + l) * g.ld_d;
        }
      }
      auto out_block = [&](int jj, float (&v)[16]) {  // TMEM [16*i, +16) -> output columns 16*jj..
        float a[8], b[8];
        const int col = 16 * (jj - (jj >= w.Npa / 16 ? w.Npa / 16 : 0));
        tmem_ld8_nw(tmem + lane_base + (uint32_t)col, a);
        tmem_ld8_nw(tmem + lane_base + (uint32_t)(col + 8), b);
        tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          v[k] = (16 * jj + k < g.d) ? a[k] : 0.f;
          v[8 + k] = (16 * jj + 8 + k < g.d) ? b[k] : 0.f;
        }
        if (dst) {
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const int c = 16 * jj + 4 * k4;
            if (c < g.d)
              *reinterpret_cast<float4*>(dst + c) =
                  make_float4(v[4 * k4], v[4 * k4 + 1], v[4 * k4 + 2], v[4 * k4 + 3]);
          }
        }
      };
      gemm_pair(w.qt0, w.qt1, w.Npa, w.Ku, 0);
      A4_MARK(7);
      const int ja = cg, jb = w.Npa / 16 + cg;
      // part a's x_{l+1} block waits in the (idle) row buffers, not in registers
      float4* stash = reinterpret_cast<float4*>(Ub0) + (size_t)tid * 4;
      if (quad_live && ja < w.Npa / 16) {
        out_block(ja, va);
        if (!last)
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            stash[q4] = make_float4(va[4 * q4], va[4 * q4 + 1], va[4 * q4 + 2], va[4 * q4 + 3]);
      }
      if (w.Npb > 0) {
        cta_sync_tc();  // every part-a read is done before part b overwrites the columns
        gemm_pair(w.qt0, w.qt1, w.Npb, w.Ku, 0);
        if (quad_live && jb < w.No / 16) out_block(jb, vb);
      }
      A4_MARK(4);
      if (!last) {  // x_{l+1} -> X_A (bf16 hi|lo); X_A overlaps the part-b columns and ubar_1
        cta_sync_tc();
        if (quad_live) {
          if (ja < w.Npa / 16) {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const float4 f = stash[q4];
              va[4 * q4] = f.x; va[4 * q4 + 1] = f.y; va[4 * q4 + 2] = f.z; va[4 * q4 + 3] = f.w;
            }
            a4_st16(tmem + lane_base + (uint32_t)(8 * ja), tmem + lane_base + (uint32_t)(w.Kx / 2 + 8 * ja), va);
          }
          if (w.Npb > 0 && jb < w.No / 16)
            a4_st16(tmem + lane_base + (uint32_t)(8 * jb), tmem + lane_base + (uint32_t)(w.Kx / 2 + 8 * jb), vb);
          tmem_st_wait();
        }
      }
#else
      // ---- c_h = ubar_h W_V,h ----
#if A4_VV
      // V_0 and V_1 back to back under one commit (one MMA round trip): the MMAs of one
      // thread run in issue order, so V_1's C1 columns over QT0 are written after V_0
      // has read them
      if (tid == 0) {
        mbar_wait(&wbar[G & 1], (uint32_t)((G >> 1) & 1));
        a4_mma(tmem, w.qt0, (G & 1) ? Wb1 : Wb0, w.Nv, w.Ku, 0, &mbar, false, false);
        mbar_wait(&wbar[(G + 1) & 1], (uint32_t)(((G + 1) >> 1) & 1));
        a4_mma(tmem, w.qt1, ((G + 1) & 1) ? Wb1 : Wb0, w.Nv, w.Ku, w.c1, &mbar, false, true);
      }
      mbar_wait(&mbar, mph & 1u);
      ++mph;
      tc_fence_after();
      if (tid == 0) {
        if (G + 2 < total_blocks && !deferred(G + 2)) stage(G + 2);
        if (G + 3 < total_blocks && !deferred(G + 3)) stage(G + 3);
      }
      G += 2;
      A4_MARK(7);
#else
      gemm(w.qt0, w.Nv, w.Ku, 0);
      A4_MARK(7);
      // every thread must observe the V_0 commit phase before V_1 can complete the
      // next one (a parity wait cannot tell phase G from phase G + 2)
      cta_sync_tc();
      gemm(w.qt1, w.Nv, w.Ku, w.c1);
#endif
      if (quad_live) {  // c -> CA (bf16 hi|lo), head h at element h*Kq
        const int nch = w.Kq / 16;
        for (int c = cg; c < 2 * nch; c += A4_NCG) {
          const int h = c / nch, j = c % nch;
          float a[8], b[8], v[16];
          const int src = (h == 0 ? 0 : w.c1) + 16 * j;
          tmem_ld8_nw(tmem + lane_base + (uint32_t)src, a);
          tmem_ld8_nw(tmem + lane_base + (uint32_t)(src + 8), b);
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            v[k] = a[k];
            v[8 + k] = b[k];
          }
          const int e0 = h * w.Kq + 16 * j;  // element index in the c operand
          a4_st16(tmem + lane_base + (uint32_t)(w.ca + e0 / 2),
                  tmem + lane_base + (uint32_t)(w.ca + w.Kc / 2 + e0 / 2), v);
        }
        tmem_st_wait();
      }
      A4_MARK(4);
      cta_sync_tc();
      // ---- out_l = c W_O ----
      gemm(w.ca, w.No, w.Kc, w.acco);
      if (quad_live) {
        const int node = row < T ? s_node[row] : -1;
        const int mode = row < T ? s_mode[row] : 0;
        const int64_t idx = A4_ROWIDX(row);
        float* dst = nullptr;
        if (node >= 0) {
          if (mode == 1) dst = last ? rs.dpred + idx * g.ld_d : nullptr;
          else if (rs.layers_out) dst = rs.layers_out + (idx * g.K + l) * g.ld_d;
          else if (rs.final_out) dst = last ? rs.final_out + idx * g.ld_d : nullptr;
          else dst = rs.h + ((int64_t)node * g.K + l) * g.ld_d;
        }
        for (int j = cg; j < w.Kx / 16; j += A4_NCG) {
          float a[8], b[8], v[16];
          tmem_ld8_nw(tmem + lane_base + (uint32_t)(w.acco + 16 * j), a);
          tmem_ld8_nw(tmem + lane_base + (uint32_t)(w.acco + 16 * j + 8), b);
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            v[k] = (16 * j + k < g.d) ? a[k] : 0.f;
            v[8 + k] = (16 * j + 8 + k < g.d) ? b[k] : 0.f;
          }
          if (dst) {
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4) {
              const int c = 16 * j + 4 * k4;
              if (c < g.d)
                *reinterpret_cast<float4*>(dst + c) =
                    make_float4(v[4 * k4], v[4 * k4 + 1], v[4 * k4 + 2], v[4 * k4 + 3]);
            }
          }
          if (!last)
            a4_st16(tmem + lane_base + (uint32_t)(8 * j), tmem + lane_base + (uint32_t)(w.Kx / 2 + 8 * j), v);
        }
        if (!last) tmem_st_wait();
      }
#endif
      A4_MARK(5);
      if (last && rs.write_valid && tid < T) {
        const int node = s_node[tid];
        if (node >= 0 && s_mode[tid] != 1) {
          rs.valid[node] = 1;
          rs.valid_at[node] = rs.valid_at_ptr ? rs.valid_at_ptr[0] : rs.valid_at_const;
        }
      }
    }
    cta_sync_tc();
#ifdef A4_PROF
    if (tid < T) prof_e += (unsigned long long)s_E[tid];
#endif
  }
#ifdef A4_PROF
  if (blockIdx.x < 1024) {
    if (prof_e) atomicAdd(&g_a4_cta[4 * blockIdx.x + 2], prof_e);
    if (tid == 0) {
      g_a4_cta[4 * blockIdx.x + 1] = a4_now();
      unsigned smid_;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));
      g_a4_cta[4 * blockIdx.x + 3] = (unsigned long long)my_tiles | ((unsigned long long)smid_ << 16);
    }
  }
#endif
  if (warp == 0) tmem_free(tmem, 512);
}
