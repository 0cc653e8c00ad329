// Memory update v4: messages, per-node aggregation and the GRU of the batch's
// direct nodes on tcgen05 (bf16x3: hi*hi + hi*lo + lo*hi, fp32 accumulate in
// TMEM), 128 rows of D per tile.
//
// Function (reference S/engine_base.py:193-247, S/kernels/reference.py:32-90):
//   x_q   = [s_owner || s_other || feat || phi(t - last[owner])]   (pre-batch)
//   msg_q = x_q W_src^T + b_src (even rows) | x_q W_dst^T + b_dst (odd rows)
//   m_v   = last / mean / sum of msg_q over v's records (message order)
//   z = sig(W_z m + U_z s + b_z), r = sig(W_r m + U_r s + b_r)
//   s' = (1 - z) tanh(W_h m + U_h (r * s) + b_h) + z s
// Messages are linear in x, so with the last aggregator (one record per node)
// m_v = x_last W_side^T + b_side, and with sum / mean
// m_v = X_src W_src^T + X_dst W_dst^T + n_src b_src + n_dst b_dst [/ cnt],
// X_side = the sum of the node's side-`side` x rows.
//
// Per tile (one CTA, 1024 threads = 4 TMEM lane quadrants x 8 column groups;
// thread (quadrant, cg) owns row 32*quadrant + lane and 16-column block cg):
//   1. x in K-chunks of 128 columns, bf16 hi|lo into one of two TMEM A
//      buffers while the previous chunk's MMAs run: D_SRC += x_j W_src,j,
//      D_DST += x_j W_dst,j (both sides; the row's side is picked after).
//      sum / mean: X_src,j and X_dst,j in A0 / A1, one chunk at a time.
//   2. A2 = [Ag + bias (/cnt) || s] (bf16 hi|lo); D_ZR = A2 [W_z W_r; U_z U_r].
//   3. z kept in registers, A3 = r * s written over A2's s half;
//      D_H = Ag W_h + A3 U_h (into D_ZR's z columns).
//   4. s' = (1 - z) tanh(D_H + b_h) + z s -> mem_new (committed after the recompute).
// Weight blocks (K-major bf16 hi block then lo block, stgn.h t4mem) are staged
// by TMA bulk copies into two shared buffers, two blocks ahead.
//
// TMEM columns (Nm = r16(d_m), Ks = Ns = r16(d_s), half = (Nm + Ks) / 2):
//   A0 [0,128) A1 [128,256)   x chunks (hi [.,+64) lo [+64,+128))
//   D_SRC [256, 256+Nm)  D_DST [256+Nm, 256+2Nm)
//   A2: Ag hi [0,Nm/2) s hi [Nm/2,half) | Ag lo [half,half+Nm/2) s lo [.., 2 half)
//   D_ZR [2 half, 2 half + 2 Ns)  (z at +0, r at +Ns); D_H reuses z's columns
//   A3 = r * s in A2's s columns
#pragma once

#include "attn4.cuh"

#ifndef M4_L2PF
#define M4_L2PF 0  // L2 prefetch of the weight blocks after the first two at kernel start
#endif

#ifndef M4_THREADS
#define M4_THREADS 1024  // 4 TMEM lane quadrants x M4_NCG column groups
#endif
#define M4_NCG (M4_THREADS / 128)
#define M4_KC 128
#define M4_MAXBLK 24

struct M4W {
  const uint16_t* wblk;     // packed blocks (stgn.h t4mem)
  int64_t off[M4_MAXBLK];   // element offset of block j
  int np[M4_MAXBLK], kp[M4_MAXBLK];
  int nblk, nmsg;           // blocks per tile; message chunks among them (first)
  int Nm, Ks, Ns;
  int wbuf_bytes;           // one shared weight buffer
};

// host: block table for the given dims; false if the TMEM/smem plan does not fit
static inline bool m4_plan(const Geo& g, M4W* w) {
  w->Nm = r16(g.d_m);
  w->Ks = r16(g.d_s);
  w->Ns = w->Ks;
  if (w->Nm > 16 * M4_NCG || w->Ks > 16 * M4_NCG) return false;  // one 16-column block per thread
  w->nmsg = (int)cdiv(g.msg_in, M4_KC);  // K-chunks of x; two weight blocks (src, dst) each
  w->nblk = 2 * w->nmsg + 4;
  if (w->nblk > M4_MAXBLK) return false;
  int64_t off = 0;
  int maxb = 0;
  auto add = [&](int j, int np, int kp) {
    w->off[j] = off;
    w->np[j] = np;
    w->kp[j] = kp;
    off += 2ll * np * kp;
    maxb = std::max(maxb, 2 * np * kp * 2);
  };
  for (int j = 0; j < 2 * w->nmsg; ++j) add(j, w->Nm, M4_KC);  // W_src chunk j, W_dst chunk j
  const int z0 = 2 * w->nmsg;
  add(z0, 2 * w->Ns, w->Nm);      // [W_z; W_r]
  add(z0 + 1, 2 * w->Ns, w->Ks);  // [U_z; U_r]
  add(z0 + 2, w->Ns, w->Nm);      // W_h
  add(z0 + 3, w->Ns, w->Ks);      // U_h
  w->wbuf_bytes = (maxb + 1023) & ~1023;
  const int half = (w->Nm + w->Ks) / 2;
  return 2 * w->Ns <= 256 && 2 * half + 2 * w->Ns <= 512 && 256 + 2 * w->Nm <= 512 &&
         2 * w->wbuf_bytes + 1024 <= 220 * 1024;
}
static inline int64_t m4_total_elems(const M4W& w) {
  return w.off[w.nblk - 1] + 2ll * w.np[w.nblk - 1] * w.kp[w.nblk - 1];
}
static inline size_t mem4_smem_bytes(const M4W& w) { return 1024 + 2 * (size_t)w.wbuf_bytes; }

// one thread: bf16x3 MMAs of one weight block; A = TMEM hi columns [a_hi, +Kp/2)
// and lo columns [a_lo, +Kp/2); B = smem [Np][Kp] K-major (hi block, lo block)
__device__ __forceinline__ void m4_mma(uint32_t tmem, int a_hi, int a_lo, const uint16_t* Wb,
                                       int Np, int Kp, int dcol, bool acc, uint64_t* bar,
                                       bool commit = true) {
  tc_fence_after();
  const uint32_t idesc = umma_idesc_bf16(128, Np);
  const uint32_t sbo = (uint32_t)(Kp / 8) * 128u;
  const uint32_t bh = smem_u32(Wb), bl = bh + (uint32_t)Np * Kp * 2u;
  for (int s = 0; s < Kp / 16; ++s) {
    const uint32_t off = (uint32_t)s * 256u;
    const uint64_t dh = umma_desc(bh + off, 128, sbo), dl = umma_desc(bl + off, 128, sbo);
    const uint32_t ah = tmem + (uint32_t)(a_hi + 8 * s), al = tmem + (uint32_t)(a_lo + 8 * s);
    umma_bf16_ts(tmem + (uint32_t)dcol, ah, dh, idesc, (acc || s > 0) ? 1u : 0u);
    umma_bf16_ts(tmem + (uint32_t)dcol, ah, dl, idesc, 1u);
    umma_bf16_ts(tmem + (uint32_t)dcol, al, dh, idesc, 1u);
  }
  if (commit) umma_commit(bar);
}

__device__ __forceinline__ float m4_sig(float x) { return 1.f / (1.f + __expf(-x)); }

__global__ void __launch_bounds__(M4_THREADS, 1)
mem4_kernel(Geo g, StateView st, Scratch s, M4W w, const float* __restrict__ bmsg,
            const double* __restrict__ omega, const float* __restrict__ bgru, int aggregator) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sbase = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint16_t* Wb0 = reinterpret_cast<uint16_t*>(sbase);
  uint16_t* Wb1 = reinterpret_cast<uint16_t*>(sbase + w.wbuf_bytes);
  __shared__ int s_node[128], s_lo[128], s_hi[128], s_n0[128], s_n1[128];
  __shared__ int s_le[128], s_lside[128], s_loth[128];  // last record: edge, side, other end
  __shared__ double s_ldt[128];                         // its t - last[owner]
  __shared__ uint64_t mbar, wbar[2];
  __shared__ uint32_t tslot;
  __shared__ float s_bmsg[2 * 16 * M4_NCG], s_bgru[3 * 16 * M4_NCG];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int quad = warp & 3, cg = warp >> 2;
  const int nD = s.res->nD;
  for (int i = tid; i < 2 * g.d_m; i += M4_THREADS) s_bmsg[i] = bmsg[i];
  for (int i = tid; i < 3 * g.d_s; i += M4_THREADS) s_bgru[i] = bgru[i];
  const int64_t ntiles = cdiv(nD, 128);
  if ((int64_t)blockIdx.x >= ntiles) return;
  const int64_t my_tiles = cdiv(ntiles - blockIdx.x, (int64_t)gridDim.x);
  const int64_t total_blocks = my_tiles * w.nblk;

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
  const uint32_t lane_base = (uint32_t)(32 * quad) << 16;
  const uint32_t trow = tmem + lane_base;
  const int row = 32 * quad + lane;
  auto stage = [&](int64_t Gi) {  // one thread
    const int j = (int)(Gi % w.nblk);
    bulk_stage((Gi & 1) ? (void*)Wb1 : (void*)Wb0, w.wblk + w.off[j],
               (uint32_t)(2 * w.np[j] * w.kp[j] * 2), &wbar[Gi & 1]);
  };
  if (tid == 0) {
    stage(0);
    if (total_blocks > 1) stage(1);
  }
#if M4_L2PF
  // the later weight blocks -> L2 now, spread over the live CTAs: their TMA stages then
  // read L2 instead of HBM (the recompute streams GBs through L2 between two batches)
  if (tid == 32) {
    const int live = (int)std::min<int64_t>(ntiles, (int64_t)gridDim.x);
    for (int j = 2 + (int)blockIdx.x; j < w.nblk; j += live)
      bulk_prefetch_l2(w.wblk + w.off[j], (uint32_t)(2 * w.np[j] * w.kp[j] * 2));
  }
#endif
  int64_t G = 0;
  auto issue = [&](int a_hi, int a_lo, int dcol, bool acc, int off = 0,
                   bool commit = true) {  // tid 0: block G + off
    const int64_t Gi = G + off;
    const int j = (int)(Gi % w.nblk);
    mbar_wait(&wbar[Gi & 1], (uint32_t)((Gi >> 1) & 1));
    m4_mma(tmem, a_hi, a_lo, (Gi & 1) ? Wb1 : Wb0, w.np[j], w.kp[j], dcol, acc, &mbar, commit);
  };
  auto cta_sync_tc = [&]() {
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  };
  // The MMAs of the next n blocks are done (their buffers refilled two blocks ahead),
  // then a CTA barrier. tid 0 is the only waiter on the commit barrier, in phase
  // order, so no waiter can fall two parity phases behind the commits.
  uint32_t mph = 0;  // commits of the MMA barrier so far (its phase parity)
  // wait for the one commit covering the next nb blocks' MMAs, refill their buffers
  auto wait_mma = [&](int nb) {
    if (tid == 0) {
      mbar_wait(&mbar, mph & 1u);
      for (int k = 0; k < nb; ++k)
        if (G + k + 2 < total_blocks) stage(G + k + 2);
    }
    ++mph;
    G += nb;
    cta_sync_tc();
  };
  const bool last_agg = aggregator == STGN_AGG_LAST;
  const int phi0 = 2 * g.d_s + g.d_e;
  const int half = (w.Nm + w.Ks) / 2;
  const int dz = 2 * half;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int d0 = (int)(tile * 128);
    if (tid < 128) {
      const int d = d0 + tid;
      int v = -1, lo = 0, hi = 0, n0 = 0, n1 = 0, le = 0, lside = 0, loth = 0;
      double ldt = 0.0;
      if (d < nD) {
        v = s.alist[d];
        lo = s.doff[d];
        hi = s.doff[d + 1];
        if (!last_agg)
          for (int q = lo; q < hi; ++q) {
            if (s.rec_s[q] & 1) ++n1; else ++n0;
          }
        const int r = s.rec_s[hi - 1];
        le = r >> 1;
        lside = r & 1;
        loth = lside ? s.in_src[le] : s.in_dst[le];
        ldt = s.in_t[le] - st.last[v];
      }
      s_node[tid] = v; s_lo[tid] = lo; s_hi[tid] = hi; s_n0[tid] = n0; s_n1[tid] = n1;
      s_le[tid] = le; s_lside[tid] = lside; s_loth[tid] = loth; s_ldt[tid] = ldt;
    }
    __syncthreads();
    A4_MARK(8);
    const int v = s_node[row];
    // x_q[cc] of one record (owner v)
    auto xval = [&](int cc, int e, int oth, double dt) -> float {
      if (cc < g.d_s) return st.mem[(int64_t)v * g.ld_s + cc];
      if (cc < 2 * g.d_s) return st.mem[(int64_t)oth * g.ld_s + cc - g.d_s];
      if (cc < phi0) return s.in_feat[(int64_t)e * g.ld_e + (cc - 2 * g.d_s)];
      const int p = cc - phi0;
      float sv, cv;
      phase_sincos(omega[p >> 1], dt, &sv, &cv);
      return ((p & 1) ? sv : cv) * g.phi_amp;
    };
    // chunk j (x columns [128 j, 128 j + 128)) of this thread's row -> A buffer `buf`:
    // side < 0: the last record's x (last aggregator); side 0 / 1: the sum of that
    // side's x over the row's records (sum / mean)
    auto build = [&](int j, int buf, int side_sel) {
      const int abase = buf ? 128 : 0;
      for (int b = cg; b < M4_KC / 16; b += M4_NCG) {
        float x[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) x[t] = 0.f;
        if (v >= 0 && side_sel < 0) {
          // one record: 16 independent loads, then the time-encoding columns
          // (no load in flight waits for another)
          const float* pv = st.mem + (int64_t)v * g.ld_s;
          const float* po = st.mem + (int64_t)s_loth[row] * g.ld_s;
          const float* pf = s.in_feat + (int64_t)s_le[row] * g.ld_e;
          const int c0 = j * M4_KC + 16 * b;  // x column of t = 0
          // a block inside one row segment at a 4-aligned offset: four 16-byte loads
          const float* seg = nullptr;
          if (c0 + 16 <= g.d_s) seg = pv + c0;
          else if (c0 >= g.d_s && c0 + 16 <= 2 * g.d_s && ((c0 - g.d_s) & 3) == 0) seg = po + (c0 - g.d_s);
          else if (c0 >= 2 * g.d_s && c0 + 16 <= phi0 && ((c0 - 2 * g.d_s) & 3) == 0)
            seg = pf + (c0 - 2 * g.d_s);
          if (seg) {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const float4 f = __ldg(reinterpret_cast<const float4*>(seg) + q4);
              x[4 * q4] = f.x; x[4 * q4 + 1] = f.y; x[4 * q4 + 2] = f.z; x[4 * q4 + 3] = f.w;
            }
          } else if (c0 < phi0) {
#pragma unroll
            for (int t = 0; t < 16; ++t) {
              const int cs = c0 + t;
              if (cs < phi0) {
                const float* p = cs < g.d_s ? pv + cs : (cs < 2 * g.d_s ? po + (cs - g.d_s)
                                                                        : pf + (cs - 2 * g.d_s));
                x[t] = __ldg(p);
              }
            }
          }
          if (c0 + 16 > phi0 && c0 < g.msg_in) {  // time encoding: one sincos per frequency
            const double dt = s_ldt[row];
#pragma unroll
            for (int t = 0; t < 16; ++t) {
              const int cs = c0 + t;
              const int p = cs - phi0;
              if (p >= 0 && cs < g.msg_in && (t == 0 || !(p & 1))) {
                float sv, cv;
                phase_sincos(omega[p >> 1], dt, &sv, &cv);
                if (p & 1) {
                  x[t] = sv * g.phi_amp;
                } else {
                  x[t] = cv * g.phi_amp;
                  if (t + 1 < 16 && cs + 1 < g.msg_in) x[t + 1] = sv * g.phi_amp;
                }
              }
            }
          }
        } else if (v >= 0) {
          for (int t = 0; t < 16; ++t) {
            const int cc = j * M4_KC + 16 * b + t;
            if (cc >= g.msg_in) break;
            const int side = side_sel;
            {
              float acc = 0.f;
              for (int q = s_lo[row]; q < s_hi[row]; ++q) {
                const int r = s.rec_s[q];
                if ((r & 1) != side) continue;
                const int e = r >> 1;
                const int oth = side ? s.in_src[e] : s.in_dst[e];
                acc += xval(cc, e, oth, s.in_t[e] - st.last[v]);
              }
              x[t] = acc;
            }
          }
        }
        a4_st16(trow + (uint32_t)(abase + 8 * b), trow + (uint32_t)(abase + 64 + 8 * b), x);
      }
      tmem_st_wait();
    };

    // ---- 1. D_SRC = X_src W_src^T, D_DST = X_dst W_dst^T (TMEM 256 / 256 + Nm) ----
    const int dsrc = 256, ddst = 256 + w.Nm;
    if (last_agg) {  // one x per row, both weight sides; the epilogue keeps the row's side
      build(0, 0, -1);
      cta_sync_tc();
      A4_MARK(9);
      for (int j = 0; j < w.nmsg; ++j) {
        const int ab = (j & 1) ? 128 : 0;
        if (tid == 0) {  // both weight sides, one commit
          issue(ab, ab + 64, dsrc, j > 0, 0, false);
          issue(ab, ab + 64, ddst, j > 0, 1, true);
        }
        if (j + 1 < w.nmsg) build(j + 1, (j + 1) & 1, -1);  // the other buffer, beside the MMAs
        wait_mma(2);
      }
    } else {  // per-side sums: A0 = src side, A1 = dst side
      A4_MARK(9);
      for (int j = 0; j < w.nmsg; ++j) {
        build(j, 0, 0);
        build(j, 1, 1);
        cta_sync_tc();
        if (tid == 0) {
          issue(0, 64, dsrc, j > 0, 0, false);
          issue(128, 128 + 64, ddst, j > 0, 1, true);
        }
        wait_mma(2);
      }
    }
    A4_MARK(10);
    // ---- 2. A2 = [Ag + bias || s] ----
    // the row's pre-batch memory, this thread's 16 columns (float4 loads; padding is 0)
    float sv[16];
    {
      const int c0 = 16 * cg;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        float4 x4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (v >= 0 && c0 + 4 * q4 + 4 <= g.ld_s)
          x4 = __ldg(reinterpret_cast<const float4*>(st.mem + (int64_t)v * g.ld_s + c0 + 4 * q4));
        sv[4 * q4] = x4.x; sv[4 * q4 + 1] = x4.y; sv[4 * q4 + 2] = x4.z; sv[4 * q4 + 3] = x4.w;
      }
#pragma unroll
      for (int t = 0; t < 16; ++t)
        if (c0 + t >= g.d_s) sv[t] = 0.f;
    }
    if (cg < w.Nm / 16) {
      const int j = cg;
      float a[8], b[8], x[16];
      if (last_agg) {
        const int dcol = s_lside[row] ? ddst : dsrc;  // per-lane column: the row's side
        tmem_ld8_nw(trow + (uint32_t)(dsrc + 16 * j), a);
        tmem_ld8_nw(trow + (uint32_t)(dsrc + 16 * j + 8), b);
        float a2[8], b2[8];
        tmem_ld8_nw(trow + (uint32_t)(ddst + 16 * j), a2);
        tmem_ld8_nw(trow + (uint32_t)(ddst + 16 * j + 8), b2);
        tmem_ld_wait();
        if (dcol == ddst) {
#pragma unroll
          for (int t = 0; t < 8; ++t) { a[t] = a2[t]; b[t] = b2[t]; }
        }
      } else {
        float a2[8], b2[8];
        tmem_ld8_nw(trow + (uint32_t)(dsrc + 16 * j), a);
        tmem_ld8_nw(trow + (uint32_t)(dsrc + 16 * j + 8), b);
        tmem_ld8_nw(trow + (uint32_t)(ddst + 16 * j), a2);
        tmem_ld8_nw(trow + (uint32_t)(ddst + 16 * j + 8), b2);
        tmem_ld_wait();
#pragma unroll
        for (int t = 0; t < 8; ++t) { a[t] += a2[t]; b[t] += b2[t]; }
      }
      const float n0 = (float)s_n0[row], n1 = (float)s_n1[row];
      const float* bl = s_bmsg + (last_agg ? s_lside[row] * g.d_m : 0);
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int c = 16 * j + t;
        float y = t < 8 ? a[t] : b[t - 8];
        if (v < 0 || c >= g.d_m) {
          y = 0.f;
        } else if (last_agg) {
          y += bl[c];
        } else {
          y += n0 * s_bmsg[c] + n1 * s_bmsg[g.d_m + c];
          if (aggregator == STGN_AGG_MEAN) y /= (n0 + n1);
        }
        x[t] = y;
      }
      a4_st16(trow + (uint32_t)(8 * j), trow + (uint32_t)(half + 8 * j), x);
    }
    if (cg < w.Ks / 16)
      a4_st16(trow + (uint32_t)(w.Nm / 2 + 8 * cg), trow + (uint32_t)(half + w.Nm / 2 + 8 * cg), sv);
    tmem_st_wait();
    cta_sync_tc();
    A4_MARK(11);
    // ---- D_ZR = Ag [W_z W_r] + s [U_z U_r] ----
    if (tid == 0) {
      issue(0, half, dz, false, 0, false);
      issue(w.Nm / 2, half + w.Nm / 2, dz, true, 1, true);
    }
    wait_mma(2);
    A4_MARK(12);
    // ---- z (registers), A3 = r * s over A2's s half ----
    float zk[16];
    const bool mine = cg < w.Ns / 16;
    if (mine) {
      const int j = cg;
      float az[8], bz[8], ar[8], br[8], x[16];
      tmem_ld8_nw(trow + (uint32_t)(dz + 16 * j), az);
      tmem_ld8_nw(trow + (uint32_t)(dz + 16 * j + 8), bz);
      tmem_ld8_nw(trow + (uint32_t)(dz + w.Ns + 16 * j), ar);
      tmem_ld8_nw(trow + (uint32_t)(dz + w.Ns + 16 * j + 8), br);
      tmem_ld_wait();
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int c = 16 * j + t;
        const bool ok = v >= 0 && c < g.d_s;
        const float zp = (t < 8 ? az[t] : bz[t - 8]) + (ok ? s_bgru[c] : 0.f);
        const float rp = (t < 8 ? ar[t] : br[t - 8]) + (ok ? s_bgru[g.d_s + c] : 0.f);
        zk[t] = m4_sig(zp);
        x[t] = m4_sig(rp) * sv[t];
      }
      a4_st16(trow + (uint32_t)(w.Nm / 2 + 8 * j), trow + (uint32_t)(half + w.Nm / 2 + 8 * j), x);
    }
    tmem_st_wait();
    cta_sync_tc();
    A4_MARK(13);
    // ---- D_H = Ag W_h + (r * s) U_h ----
    if (tid == 0) {
      issue(0, half, dz, false, 0, false);
      issue(w.Nm / 2, half + w.Nm / 2, dz, true, 1, true);
    }
    wait_mma(2);
    if (mine) {
      const int j = cg;
      float a[8], b[8];
      tmem_ld8_nw(trow + (uint32_t)(dz + 16 * j), a);
      tmem_ld8_nw(trow + (uint32_t)(dz + 16 * j + 8), b);
      tmem_ld_wait();
      if (v >= 0) {
        float out[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int c = 16 * j + t;
          const float cand = tanhf((t < 8 ? a[t] : b[t - 8]) + (c < g.d_s ? s_bgru[2 * g.d_s + c] : 0.f));
          out[t] = (1.f - zk[t]) * cand + zk[t] * sv[t];
        }
        float* dst = s.mem_new + (int64_t)(d0 + row) * g.ld_s + 16 * j;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          if (16 * j + 4 * q4 + 4 <= g.ld_s)
            *reinterpret_cast<float4*>(dst + 4 * q4) =
                make_float4(out[4 * q4], out[4 * q4 + 1], out[4 * q4 + 2], out[4 * q4 + 3]);
      }
    }
    A4_MARK(14);
    cta_sync_tc();
    A4_MARK(15);
  }
  if (warp == 0) tmem_free(tmem, 512);
}
