// Per-batch kernels of the incremental path (everything except the
// attention recompute). All sizes are read from the device header/results
// so the whole sequence can be captured once in a CUDA graph.
//
// Reference anchors (S/ = /root/reference/pkg/src/streamtgn):
//   k_claim / k_scan / k_place / k_rank   grouping  S/engine.py:170-180
//   k_ring / k_dupdate                    neighbour cache insert + store append
//                                         S/engine.py:216-243, S/graph_store.py:126-152,
//                                         payload freeze S/engine_base.py:88-106
//   k_hop                                 affected set S/engine.py:182-212
//   k_records                             change records S/engine.py:216-243
//   k_predict                             S/kernels/reference.py:183-186
//   k_memory (messages+aggregate+GRU)     S/engine_base.py:193-247
//   k_predict_commit                      S/engine.py:425-426, S/engine_base.py:241-244
//   k_drift_record / k_drift_decide       S/drift.py:52-78, S/engine.py:366-372, 440-453
#pragma once

#include "attn2.cuh"

struct StateView {
  float* mem;
  double* last;
  int64_t* version;
  float* h;
  uint8_t* valid;
  double* valid_at;
  int32_t *ring_cnt, *ring_head, *ring_ccnt, *ring_nbr;
  int64_t* ring_eid;
  double* ring_t;
  float *ring_pay, *ring_feat, *ring_tb;
  uint32_t *amark, *dmark;
  int32_t *nodecnt, *nodeadj, *nodefill, *nodeoff;
  double* drift_acc;
  int64_t* drift_touched;
  uint32_t* cum_mark;
  int32_t* cum_list;
  int32_t* cum_pos;
  int64_t* attn_ver;
  double* attn_tref;
  double* attn_logz;  // [n][4] delta mode K = 1: log Z per head of the node's attention state
  int32_t *ev_node, *ev_dpos, *ev_dn, *ev_nv;
  double *ev_bound, *ev_maxv, *ev_zdev;
  int64_t ev_cap;
  float* e_pay;       // nullable: [2 cap_edges][K][ld_d] frozen payload of every store entry
  int32_t *e_src, *e_dst;
  double* e_t;
  float* e_feat;
  int64_t *e_prev, *adj_head, *adj_deg;
  const double* gpow;
  int64_t gpow_len;
  stgn_ctl* ctl;
};

__device__ __forceinline__ int rec_node(const Scratch& s, int r) {
  return (r & 1) ? s.in_dst[r >> 1] : s.in_src[r >> 1];
}
__device__ __forceinline__ int rec_other(const Scratch& s, int r) {
  return (r & 1) ? s.in_src[r >> 1] : s.in_dst[r >> 1];
}
// A self-loop produces two messages but one adjacency entry (the src side),
// S/graph_store.py:147-148, S/engine.py:177-179, S/engine_base.py:209-215.
__device__ __forceinline__ bool rec_is_adj(const Scratch& s, int r) {
  return !(r & 1) || (s.in_src[r >> 1] != s.in_dst[r >> 1]);
}

#ifndef STGN_REC_HASH
#define STGN_REC_HASH 0  // k_records_w32: the direct set as a shared-memory hash table
#endif
#ifndef STGN_HOP_TICKET
#define STGN_HOP_TICKET 0  // k_hop's last block writes hop_off[hop + 1]: no k_hop_fin launch
#endif

#define GRID_STRIDE(i, n) \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// Reset per-batch results; derive t_batch (the last edge's timestamp,
// S/engine.py:415) and the window cutoff on the device.
__device__ __forceinline__ void begin_body(const Scratch& s, double window) {
  {
    BatchHdr* hd = s.hdr;
    hd->t_batch = s.in_t[hd->B - 1];
    hd->cutoff = isfinite(window) ? hd->t_batch - window : -INFINITY;
    BatchRes* r = s.res;
    r->nD = 0;
    r->nA = 0;
    for (int k = 0; k < STGN_MAX_LAYERS + 2; ++k) r->hop_off[k] = 0;
    r->n_drifted = 0;
    r->nbr_hit = r->nbr_miss = r->E_A = r->E_D = r->E_R = r->changed = 0;
    r->rebuild_kind = 0;
    r->rebuild_nodes = 0;
    r->global_drift = 0.0;
    r->rb_partial_n = 0;
    r->rb_full_n = 0;
    r->ticket = 0;
    r->hop_ticket = 0;
    r->nC = r->n_skip = r->n_hit = r->n_miss = 0;
    r->E_miss = 0;
  }
}
__global__ void k_begin(Scratch s, double window) {
  PDL_WAIT();
  if (threadIdx.x == 0 && blockIdx.x == 0) begin_body(s, window);
}

// Records r = 2i + side (side 0: owner src, side 1: owner dst). First
// toucher of a node claims its direct-set slot; counts per node; the
// side-0 record also appends the edge to the temporal store.
__device__ __forceinline__ void claim_body(const Geo& g, const StateView& st, const Scratch& s,
                                           int64_t i0, int64_t stride) {
  const BatchHdr* hd = s.hdr;
  const int64_t B = hd->B;
  const uint32_t stamp = hd->stamp;
  for (int64_t r = i0; r < 2 * B; r += stride) {
    const int rr = (int)r;
    const int node = rec_node(s, rr);
    if (atomicExch(&st.dmark[node], stamp) != stamp) {
      const int di = atomicAdd(&s.res->nD, 1);
      s.alist[di] = node;
      s.dmap[node] = di;
      st.amark[node] = stamp;
    }
    atomicAdd(&st.nodecnt[node], 1);
    if (rec_is_adj(s, rr)) atomicAdd(&st.nodeadj[node], 1);
    if (!(rr & 1)) {
      const int64_t i = r >> 1;
      const int64_t eid = hd->m0 + i;
      st.e_src[eid] = s.in_src[i];
      st.e_dst[eid] = s.in_dst[i];
      st.e_t[eid] = s.in_t[i];
      for (int j = 0; j < g.d_e; ++j) st.e_feat[eid * g.ld_e + j] = s.in_feat[i * g.ld_e + j];
    }
  }
}
__global__ void k_claim(Geo g, StateView st, Scratch s) {
  PDL_WAIT();
  claim_body(g, st, s, (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}

// One block: exclusive scan of per-direct-node record counts; per-node
// offsets; remembers each direct node's pre-batch cache state.
__device__ __forceinline__ void scan_body(const Geo& g, const StateView& st, const Scratch& s) {
  __shared__ int32_t warp_tot[32];
  __shared__ int32_t carry;
  const int nD = s.res->nD;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nD; base += blockDim.x) {
    const int d = base + threadIdx.x;
    int c = 0;
    if (d < nD) {
      const int v = s.alist[d];
      c = st.nodecnt[v];
      const int cc = st.ring_ccnt[v];
      s.d_wascached[d] = cc >= 0;
      s.d_baselen[d] = cc >= 0 ? cc : st.ring_cnt[v];
    }
    // block inclusive scan
    int x = c;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;
    }
    __syncthreads();
    const int excl = carry + x - c + (wid > 0 ? warp_tot[wid - 1] : 0);
    if (d < nD) {
      s.doff[d] = excl;
      st.nodeoff[s.alist[d]] = excl;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + c;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    s.doff[nD] = carry;
    s.res->nA = nD;
    s.res->hop_off[0] = 0;
    s.res->hop_off[1] = nD;
  }
}
__global__ void k_scan(Geo g, StateView st, Scratch s) {
  PDL_WAIT();
  scan_body(g, st, s);
}

__device__ __forceinline__ void place_body(const StateView& st, const Scratch& s, int64_t i0,
                                           int64_t stride) {
  const int64_t B = s.hdr->B;
  for (int64_t r = i0; r < 2 * B; r += stride) {
    const int node = rec_node(s, (int)r);
    const int slot = atomicAdd(&st.nodefill[node], 1);
    s.rec_u[st.nodeoff[node] + slot] = (int)r;
  }
}
__global__ void k_place(StateView st, Scratch s) {
  PDL_WAIT();
  place_body(st, s, (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}

// Rank each record inside its node's segment (segments are small: one
// entry per incident batch edge), giving message order (ascending r) and
// the newest-first adjacency rank.
__device__ __forceinline__ void rank_body(const StateView& st, const Scratch& s, int64_t i0,
                                          int64_t stride) {
  const int64_t B = s.hdr->B;
  for (int64_t r64 = i0; r64 < 2 * B; r64 += stride) {
    const int r = (int)r64;
    const int node = rec_node(s, r);
    const int off = st.nodeoff[node];
    const int k = st.nodecnt[node];
    const bool adj = rec_is_adj(s, r);
    int rank = 0, arank = 0, prev = -1;
    for (int q = off; q < off + k; ++q) {
      const int o = s.rec_u[q];
      if (o < r) {
        ++rank;
        if (rec_is_adj(s, o) && o > prev) prev = o;
      } else if (o > r && rec_is_adj(s, o)) {
        ++arank;
      }
    }
    s.rec_s[off + rank] = r;
    s.rec_adjrank[r] = adj ? arank : -1;
    s.rec_prev[r] = prev;
  }
}
__global__ void k_rank(StateView st, Scratch s) {
  PDL_WAIT();
  rank_body(st, s, (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}

// The five ingest steps above in one block, for batches of at most INGEST1_MAX_B
// edges: the kernel boundaries between them (each a few microseconds of launch
// and drain for ~1K records) become block barriers. Same bodies, same results.
#define INGEST1_MAX_B 2048
__global__ void __launch_bounds__(1024) k_ingest1(Geo g, StateView st, Scratch s, double window) {
  PDL_WAIT();
  if (threadIdx.x == 0) begin_body(s, window);
  __syncthreads();
  claim_body(g, st, s, threadIdx.x, blockDim.x);
  __syncthreads();
  scan_body(g, st, s);
  __syncthreads();
  place_body(st, s, threadIdx.x, blockDim.x);
  __syncthreads();
  rank_body(st, s, threadIdx.x, blockDim.x);
}

__device__ __forceinline__ int64_t entry_index(int64_t m0, int r) {
  return 2 * (m0 + (r >> 1)) + (r & 1);
}

// Write the new adjacency entries into the node rings (newest at rank 0),
// freezing the opposite endpoint's pre-batch stack [s || 0, h_0..h_{K-2}]
// as the payload; link the append-only store's per-node chains. One warp
// per record.
__global__ void k_ring(Geo g, StateView st, Scratch s, const double* __restrict__ omega) {
  PDL_WAIT();
  const BatchHdr* hd = s.hdr;
  const int64_t R = 2 * hd->B;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r64 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r64 < R; r64 += warps) {
    const int r = (int)r64;
    if (!rec_is_adj(s, r)) continue;
    const int v = rec_node(s, r);
    const int u = rec_other(s, r);
    const int64_t i = r >> 1;
    const int a = s.rec_adjrank[r];
    if (lane == 0) {
      const int p = s.rec_prev[r];
      st.e_prev[entry_index(hd->m0, r)] = p >= 0 ? entry_index(hd->m0, p) : st.adj_head[v];
    }
    if (!geo_owns(g, v)) {  // sharded engine: another rank keeps this node's payload rows
      if (lane == 0) {
        const int kadj = st.nodeadj[v];
        const int kk = kadj < g.L ? kadj : g.L;
        if (a < kk) {
          int slot = (st.ring_head[v] - kk + a) % g.L;
          if (slot < 0) slot += g.L;
          const int64_t rs = (int64_t)v * g.L + slot;
          st.ring_nbr[rs] = u;
          st.ring_eid[rs] = hd->m0 + i;
          st.ring_t[rs] = s.in_t[i];
        }
      }
      continue;
    }
    if (st.e_pay) {  // the payload log of every store entry (historical snapshots)
      float* ep = st.e_pay + entry_index(hd->m0, r) * g.K * g.ld_d;
      for (int l = 0; l < g.K; ++l) {
        const float* src = l == 0 ? st.mem + (int64_t)u * g.ld_s
                                  : st.h + ((int64_t)u * g.K + (l - 1)) * g.ld_d;
        for (int j = lane; j < g.d; j += 32) ep[l * g.ld_d + j] = (l > 0 || j < g.d_s) ? src[j] : 0.f;
      }
    }
    const int kadj = st.nodeadj[v];
    const int kk = kadj < g.L ? kadj : g.L;
    if (a >= kk) continue;  // evicted within the batch
    int slot = (st.ring_head[v] - kk + a) % g.L;
    if (slot < 0) slot += g.L;
    const int64_t rs = (int64_t)v * g.L + slot;
    if (lane == 0) {
      st.ring_nbr[rs] = u;
      st.ring_eid[rs] = hd->m0 + i;
      st.ring_t[rs] = s.in_t[i];
    }
    for (int j = lane; j < g.d_e; j += 32) st.ring_feat[rs * g.ld_e + j] = s.in_feat[i * g.ld_e + j];
    // time basis of the entry's timestamp: phi(tref - t) = rotation of [cos w t, sin w t] by
    // w tref, so the recompute needs no per-entry trigonometry (attn4.cuh)
    for (int f = lane; f < g.half; f += 32) {
      float sv, cv;
      phase_sincos(omega[f], s.in_t[i], &sv, &cv);
      st.ring_tb[rs * g.ld_t + 2 * f] = cv;
      st.ring_tb[rs * g.ld_t + 2 * f + 1] = sv;
    }
    for (int l = 0; l < g.K; ++l) {
      float* dstp = st.ring_pay + (((int64_t)v * g.K + l) * g.L + slot) * g.ld_d;
      if (l == 0) {
        const float* m = st.mem + (int64_t)u * g.ld_s;
        for (int j = lane; j < g.d; j += 32) dstp[j] = j < g.d_s ? m[j] : 0.f;
      } else {
        const float* hp = st.h + ((int64_t)u * g.K + (l - 1)) * g.ld_d;
        for (int j = lane; j < g.d; j += 32) dstp[j] = hp[j];
      }
    }
  }
}

// Per direct node: advance ring head/count, set the post-insertion cache
// length, and move the store chain head.
__global__ void k_dupdate(Geo g, StateView st, Scratch s) {
  PDL_WAIT();
  const int nD = s.res->nD;
  const int64_t m0 = s.hdr->m0;
  GRID_STRIDE(d64, nD) {
    const int d = (int)d64;
    const int v = s.alist[d];
    const int kadj = st.nodeadj[v];
    const int kk = kadj < g.L ? kadj : g.L;
    int head = (st.ring_head[v] - kk) % g.L;
    if (head < 0) head += g.L;
    st.ring_head[v] = head;
    const int c = st.ring_cnt[v] + kadj;
    st.ring_cnt[v] = c < g.L ? c : g.L;
    const int cc = kadj + s.d_baselen[d];
    st.ring_ccnt[v] = cc < g.L ? cc : g.L;
    // newest adjacency record = last adj record in ascending segment order
    int newest = -1;
    for (int q = s.doff[d + 1] - 1; q >= s.doff[d]; --q) {
      const int r = s.rec_s[q];
      if (rec_is_adj(s, r)) { newest = r; break; }
    }
    st.adj_head[v] = entry_index(m0, newest);
    st.adj_deg[v] += kadj;
  }
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// One BFS hop: every (frontier node, list position) pair marks its
// neighbour; first markers append with warp-ballot compaction.
__global__ void k_hop(Geo g, StateView st, Scratch s, int hop) {
  PDL_WAIT();
  const uint32_t stamp = s.hdr->stamp;
  const int f0 = s.res->hop_off[hop - 1], f1 = s.res->hop_off[hop];
  const int64_t total = (int64_t)(f1 - f0) * g.L;
  const int64_t total_r = cdiv(total, 32) * 32;
  const int lane = threadIdx.x & 31;
  GRID_STRIDE(x, total_r) {
    bool fresh = false;
    int u = -1;
    if (x < total) {
      const int w = s.alist[f0 + (int)(x / g.L)];
      const int j = (int)(x % g.L);
      const int cc = st.ring_ccnt[w];
      const int len = cc >= 0 ? cc : st.ring_cnt[w];
      if (j < len) {
        int slot = st.ring_head[w] + j;
        if (slot >= g.L) slot -= g.L;
        u = st.ring_nbr[(int64_t)w * g.L + slot];
        fresh = atomicExch(&st.amark[u], stamp) != stamp;
      }
    }
    const unsigned mask = __ballot_sync(0xffffffffu, fresh);
    if (mask) {
      int basepos = 0;
      const int leader = __ffs(mask) - 1;
      if (lane == leader) basepos = atomicAdd(&s.res->nA, __popc(mask));
      basepos = __shfl_sync(0xffffffffu, basepos, leader);
      if (fresh) s.alist[basepos + __popc(mask & lanemask_lt())] = u;
    }
  }
#if STGN_HOP_TICKET
  // the last block to finish publishes the hop boundary (k_hop_fin's job)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&s.res->hop_ticket, 1u) == gridDim.x - 1) {
      __threadfence();
      s.res->hop_off[hop + 1] = atomicAdd(&s.res->nA, 0);
      s.res->hop_ticket = 0;
    }
  }
#endif
}

__global__ void k_hop_fin(Scratch s, int hop) {
  PDL_WAIT();
  if (threadIdx.x == 0 && blockIdx.x == 0) s.res->hop_off[hop + 1] = s.res->nA;
}

// Change records for every affected node (sizes only) + the window filter
// + cache bookkeeping; S/engine.py:216-243.
__global__ void k_records(Geo g, StateView st, Scratch s, int finite_window) {
  PDL_WAIT();
  const int nA = s.res->nA, nD = s.res->nD;
  const uint32_t stamp = s.hdr->stamp;
  const double cutoff = s.hdr->cutoff;
  unsigned long long hit = 0, miss = 0, changed = 0;
  GRID_STRIDE(a64, nA) {
    const int a = (int)a64;
    const int v = s.alist[a];
    int added = 0, expired = 0, len, was_cached;
    if (a < nD) {
      const int kadj = st.nodeadj[v];
      was_cached = s.d_wascached[a];
      const int merged = kadj + s.d_baselen[a];
      len = merged < g.L ? merged : g.L;
      expired = was_cached ? (merged > g.L ? merged - g.L : 0) : 0;
      added = kadj;
    } else {
      const int cc = st.ring_ccnt[v];
      was_cached = cc >= 0;
      len = was_cached ? cc : st.ring_cnt[v];
    }
    int n_new = added < len ? added : len;
    const int head = st.ring_head[v];
    const int64_t rb = (int64_t)v * g.L;
    if (finite_window) {
      int keep = 0;
      while (keep < len) {
        int slot = head + keep;
        if (slot >= g.L) slot -= g.L;
        if (st.ring_t[rb + slot] < cutoff) break;
        ++keep;
      }
      expired += len - keep;
      len = keep;
      if (n_new > len) n_new = len;
    }
    // distinct direct neighbours among the kept old entries
    int upd = 0;
    for (int j = n_new; j < len; ++j) {
      int slot = head + j;
      if (slot >= g.L) slot -= g.L;
      const int u = st.ring_nbr[rb + slot];
      if (st.dmark[u] != stamp) continue;
      bool dup = false;
      for (int q = n_new; q < j; ++q) {
        int s2 = head + q;
        if (s2 >= g.L) s2 -= g.L;
        if (st.ring_nbr[rb + s2] == u) { dup = true; break; }
      }
      if (!dup) ++upd;
    }
    const int size = added + expired + upd;
    s.a_size[a] = size;
    s.a_len[a] = len;
    st.ring_ccnt[v] = len;
    if (was_cached) ++hit; else ++miss;
    if (size > 0 && len > 0) ++changed;
  }
  // block-aggregate the counters
  for (int o = 16; o > 0; o >>= 1) {
    hit += __shfl_xor_sync(0xffffffffu, hit, o);
    miss += __shfl_xor_sync(0xffffffffu, miss, o);
    changed += __shfl_xor_sync(0xffffffffu, changed, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (hit) atomicAdd(&s.res->nbr_hit, hit);
    if (miss) atomicAdd(&s.res->nbr_miss, miss);
    if (changed) atomicAdd(&s.res->changed, changed);
  }
}

// Same records with one warp per node and one lane per list position
// (L <= 32): the window prefix is a ballot, the distinct direct
// neighbours a __match_any_sync, so a node costs a few parallel loads.
__global__ void k_records_warp(Geo g, StateView st, Scratch s, int finite_window) {
  PDL_WAIT();
  // floor(32 / L) affected nodes per warp, one L-lane segment each
  const int nA = s.res->nA, nD = s.res->nD;
  const uint32_t stamp = s.hdr->stamp;
  const double cutoff = s.hdr->cutoff;
  const int lane = threadIdx.x & 31;
  const int S = 32 / g.L;
  const int seg = lane / g.L, sl = lane - seg * g.L;  // segment, lane within it
  const bool seg_live = seg < S;
  const unsigned seg_mask = seg_live ? (((1u << g.L) - 1u) << (seg * g.L)) : 0u;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  unsigned long long hit = 0, miss = 0, changed = 0;
  for (int64_t a0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * S; a0 < nA;
       a0 += warps * S) {
    const int a = (int)a0 + seg;
    const bool live = seg_live && a < nA;
    int v = 0, added = 0, expired = 0, len = 0, was_cached = 0;
    if (live) {
      v = s.alist[a];
      if (a < nD) {
        const int kadj = st.nodeadj[v];
        was_cached = s.d_wascached[a];
        const int merged = kadj + s.d_baselen[a];
        len = merged < g.L ? merged : g.L;
        expired = was_cached ? (merged > g.L ? merged - g.L : 0) : 0;
        added = kadj;
      } else {
        const int cc = st.ring_ccnt[v];
        was_cached = cc >= 0;
        len = was_cached ? cc : st.ring_cnt[v];
      }
    }
    int n_new = added < len ? added : len;
    int slot = live ? st.ring_head[v] + sl : 0;
    if (slot >= g.L) slot -= g.L;
    const int64_t rs = (int64_t)v * g.L + slot;
    const bool in_list = live && sl < len;
    if (finite_window) {
      const unsigned old = (__ballot_sync(0xffffffffu, in_list && st.ring_t[rs] < cutoff) & seg_mask) >>
                           (seg_live ? seg * g.L : 0);
      const int keep = old ? __ffs(old) - 1 : len;
      expired += len - keep;
      len = keep;
      if (n_new > len) n_new = len;
    }
    const bool cand = live && sl >= n_new && sl < len;
    const int u = cand ? st.ring_nbr[rs] : -1;
    const bool dir = cand && st.dmark[u] == stamp;
    // ids are compared within the segment only: key = (node id, segment); lanes
    // that hold no candidate get a key no other lane has
    const unsigned long long key = cand ? (((unsigned long long)(unsigned)u << 8) | (unsigned)seg)
                                        : (0xFFFFFFFF00000000ull | (unsigned)lane);
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const bool first = (__ffs(peers) - 1) == lane;  // lowest position holding this id
    const int upd = __popc(__ballot_sync(0xffffffffu, dir && first) & seg_mask);
    if (live && sl == 0) {
      const int size = added + expired + upd;
      s.a_size[a] = size;
      s.a_len[a] = len;
      st.ring_ccnt[v] = len;
      if (was_cached) ++hit; else ++miss;
      if (size > 0 && len > 0) ++changed;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    hit += __shfl_xor_sync(0xffffffffu, hit, o);
    miss += __shfl_xor_sync(0xffffffffu, miss, o);
    changed += __shfl_xor_sync(0xffffffffu, changed, o);
  }
  if (lane == 0) {
    if (hit) atomicAdd(&s.res->nbr_hit, hit);
    if (miss) atomicAdd(&s.res->nbr_miss, miss);
    if (changed) atomicAdd(&s.res->changed, changed);
  }
}

// k_records_warp with 32 nodes per warp: lane k loads node k's header (one
// coalesced alist load, independent per-lane header loads), then floor(32/L)
// nodes per round in L-lane segments take their list entries; the rounds only
// load (ring ids, direct marks) and shuffle, so unrolled rounds overlap their
// loads, and each lane writes its own node's record once at the end.
// The direct set (nD <= REC_HASH_SLOTS / 2 nodes) is looked up in a shared-memory
// hash table built by every block, instead of st.dmark: the marks of random
// neighbours are scattered 4-byte reads of a |V|-sized table (DRAM sectors).
#define REC_HASH_SLOTS 8192
__device__ __forceinline__ uint32_t rec_hash(int u) { return ((uint32_t)u * 2654435761u) >> 19; }
__global__ void k_records_w32(Geo g, StateView st, Scratch s, int finite_window) {
  PDL_WAIT();
  const int nA = s.res->nA, nD = s.res->nD;
  const uint32_t stamp = s.hdr->stamp;
  __shared__ int dset[REC_HASH_SLOTS];
  const bool use_hash = STGN_REC_HASH && nD <= REC_HASH_SLOTS / 2;
  if (use_hash) {
    for (int i = threadIdx.x; i < REC_HASH_SLOTS; i += blockDim.x) dset[i] = -1;
    __syncthreads();
    for (int i = threadIdx.x; i < nD; i += blockDim.x) {
      const int key = s.alist[i];
      uint32_t h = rec_hash(key);
      while (atomicCAS(&dset[h], -1, key) != -1) h = (h + 1) & (REC_HASH_SLOTS - 1);
    }
    __syncthreads();
  }
  auto is_direct = [&](int u) {
    if (!use_hash) return st.dmark[u] == stamp;
    uint32_t h = rec_hash(u);
    for (;;) {
      const int k = dset[h];
      if (k == u) return true;
      if (k < 0) return false;
      h = (h + 1) & (REC_HASH_SLOTS - 1);
    }
  };
  const double cutoff = s.hdr->cutoff;
  const int lane = threadIdx.x & 31;
  const int S = 32 / g.L;
  const int seg = lane / g.L, sl = lane - seg * g.L;
  const bool seg_live = seg < S;
  const unsigned seg_mask = seg_live ? (((1u << g.L) - 1u) << (seg * g.L)) : 0u;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int rounds = (32 + S - 1) / S;
  unsigned long long hit = 0, miss = 0, changed = 0;
  for (int64_t b0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; b0 < nA;
       b0 += warps * 32) {
    // this lane's node: header
    const int a_l = (int)b0 + lane;
    const bool live_l = a_l < nA;
    int v_l = 0, added_l = 0, expired_l = 0, len_l = 0, wc_l = 0, head_l = 0;
    if (live_l) {
      v_l = s.alist[a_l];
      if (a_l < nD) {
        const int kadj = st.nodeadj[v_l];
        wc_l = s.d_wascached[a_l];
        const int merged = kadj + s.d_baselen[a_l];
        len_l = merged < g.L ? merged : g.L;
        expired_l = wc_l ? (merged > g.L ? merged - g.L : 0) : 0;
        added_l = kadj;
      } else {
        const int cc = st.ring_ccnt[v_l];
        wc_l = cc >= 0;
        len_l = wc_l ? cc : st.ring_cnt[v_l];
      }
      head_l = st.ring_head[v_l];
    }
    int out_upd = 0, out_len = len_l;  // this lane's node: results gathered from its segment
#pragma unroll 4
    for (int rr = 0; rr < rounds; ++rr) {
      const int k = rr * S + seg;  // node (lane index) of this segment in this round
      const int ks = (seg_live && k < 32) ? k : 0;
      const int v = __shfl_sync(0xffffffffu, v_l, ks);
      int len = __shfl_sync(0xffffffffu, len_l, ks);
      const int added = __shfl_sync(0xffffffffu, added_l, ks);
      const int head = __shfl_sync(0xffffffffu, head_l, ks);
      const bool live = seg_live && k < 32 && (int)b0 + k < nA;
      int n_new = added < len ? added : len;
      int slot = live ? head + sl : 0;
      if (slot >= g.L) slot -= g.L;
      const int64_t rs = (int64_t)v * g.L + slot;
      const bool in_list = live && sl < len;
      if (finite_window) {
        const unsigned old = (__ballot_sync(0xffffffffu, in_list && st.ring_t[rs] < cutoff) & seg_mask) >>
                             (seg_live ? seg * g.L : 0);
        const int keep = old ? __ffs(old) - 1 : len;
        len = keep;
        if (n_new > len) n_new = len;
      }
      const bool cand = live && sl >= n_new && sl < len;
      const int u = cand ? st.ring_nbr[rs] : -1;
      const bool dir = cand && is_direct(u);
      const unsigned long long key = cand ? (((unsigned long long)(unsigned)u << 8) | (unsigned)seg)
                                          : (0xFFFFFFFF00000000ull | (unsigned)lane);
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const bool first = (__ffs(peers) - 1) == lane;
      const int upd = __popc(__ballot_sync(0xffffffffu, dir && first) & seg_mask);
      // node k = rr*S + j was handled by segment j (lane j*L): its owner lane takes the values
      const int j = lane - rr * S;
      const int src = (j >= 0 && j < S) ? j * g.L : 0;
      const int upd_k = __shfl_sync(0xffffffffu, upd, src);
      const int len_k = __shfl_sync(0xffffffffu, len, src);
      if (j >= 0 && j < S) {
        out_upd = upd_k;
        out_len = len_k;
      }
    }
    if (live_l) {
      const int expired = expired_l + (finite_window ? len_l - out_len : 0);
      const int size = added_l + expired + out_upd;
      s.a_size[a_l] = size;
      s.a_len[a_l] = out_len;
      st.ring_ccnt[v_l] = out_len;
      if (wc_l) ++hit; else ++miss;
      if (size > 0 && out_len > 0) ++changed;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    hit += __shfl_xor_sync(0xffffffffu, hit, o);
    miss += __shfl_xor_sync(0xffffffffu, miss, o);
    changed += __shfl_xor_sync(0xffffffffu, changed, o);
  }
  if (lane == 0) {
    if (hit) atomicAdd(&s.res->nbr_hit, hit);
    if (miss) atomicAdd(&s.res->nbr_miss, miss);
    if (changed) atomicAdd(&s.res->changed, changed);
  }
}

// Delta mode (S/engine.py:287-313): classify every node of A after its change
// record is known. A \ D nodes with an empty record and a valid cache row are
// skipped (embed_skip); every other node is an attn_hit when the node has an
// attention state built on its current memory version and the newest entry of
// its post-batch list still carries the state's t_ref (single-layer models
// only, :302-305), else an attn_miss. Hits and misses are recomputed: a hit's
// delta update (delta_embed, :43-118) is the same softmax over the same
// entries (the key rows are frozen payloads), so the recompute gives the
// delta result up to rounding. State stamps follow the reference's
// _build_attn_state calls: misses of A \ D get (version, t_ref) now; D gets
// the post-commit stamp (version = batch index, S/state.py:25) because the
// commit recomputes it with keep_states (:357-364).
__global__ void k_delta_classify(Geo g, StateView st, Scratch s) {
  PDL_WAIT();
  const int nA = s.res->nA, nD = s.res->nD;
  const int64_t bidx = s.hdr->batch_index;
  const int lane = threadIdx.x & 31;
  int skip = 0, hit = 0, miss = 0;
  unsigned long long e_miss = 0;
  int info = 0;
  const int64_t n_it = ((int64_t)nA + 31) & ~31ll;  // whole warps for the ballot
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < n_it;
       a += (int64_t)gridDim.x * blockDim.x) {
    bool keep = false;
    int v = 0;
    if (a < nA) {
      v = s.alist[a];
      const int len = s.a_len[a];
      const bool direct = a < nD;
      const bool valid = st.valid[v] != 0;
      if (!direct && s.a_size[a] == 0 && valid) {
        ++skip;
      } else {
        const double tref = len > 0 ? st.ring_t[(int64_t)v * g.L + st.ring_head[v]] : 0.0;
        const bool is_hit = g.K == 1 && valid && st.attn_ver[v] == st.version[v] &&
                            st.attn_tref[v] == tref;
        info = (s.a_size[a] << 1) | (is_hit ? 1 : 0);
        if (is_hit) {
          ++hit;
        } else {
          ++miss;
          e_miss += (unsigned long long)len;
        }
        if (direct) {
          s.clist[a] = v;
          s.c_info[a] = (s.a_size[a] << 1) | (is_hit ? 1 : 0);
          st.attn_ver[v] = bidx;
          st.attn_tref[v] = tref;
        } else {
          keep = true;
          if (!is_hit) {
            st.attn_ver[v] = st.version[v];
            st.attn_tref[v] = tref;
          }
        }
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (m) {
      int base = 0;
      const int leader = __ffs(m) - 1;
      if (lane == leader) base = atomicAdd(&s.res->nC, __popc(m));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (keep) {
        const int pos = nD + base + __popc(m & ((1u << lane) - 1u));
        s.clist[pos] = v;
        s.c_info[pos] = info;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    skip += __shfl_xor_sync(0xffffffffu, skip, o);
    hit += __shfl_xor_sync(0xffffffffu, hit, o);
    miss += __shfl_xor_sync(0xffffffffu, miss, o);
    e_miss += __shfl_xor_sync(0xffffffffu, e_miss, o);
  }
  if (lane == 0) {
    if (skip) atomicAdd(&s.res->n_skip, skip);
    if (hit) atomicAdd(&s.res->n_hit, hit);
    if (miss) atomicAdd(&s.res->n_miss, miss);
    if (e_miss) atomicAdd(&s.res->E_miss, e_miss);
  }
}

// nC := nD + (non-skipped nodes of A \ D), the pre-batch recompute's row count.
__global__ void k_delta_fin(Scratch s) {
  PDL_WAIT();
  if (threadIdx.x == 0 && blockIdx.x == 0) s.res->nC += s.res->nD;
}

// valid / valid_at for A \ D when only V_direct is recomputed.
__global__ void k_mark_valid(StateView st, Scratch s) {
  PDL_WAIT();
  const int nA = s.res->nA, nD = s.res->nD;
  const double t = s.hdr->t_batch;
  GRID_STRIDE(a, nA) {
    if (a < nD) continue;
    const int v = s.alist[a];
    st.valid[v] = 1;
    st.valid_at[v] = t;
  }
}

// sigma(w_p . [h_src || h_dst] + b_p) in float64 on the pre-batch-memory
// embeddings of the endpoints (S/engine.py:425-426), one warp per edge;
// then commit the post-batch memory of V_direct (S/engine_base.py:241-244).
__global__ void k_predict_commit(Geo g, StateView st, Scratch s, const double* wpred,
                                 double bpred) {
  PDL_WAIT();
  const int64_t B = s.hdr->B;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t i = gw; i < B; i += warps) {
    const float* hu = s.dpred + (int64_t)s.dmap[s.in_src[i]] * g.ld_d;
    const float* hv = s.dpred + (int64_t)s.dmap[s.in_dst[i]] * g.ld_d;
    double acc = 0.0;
    for (int j = lane; j < g.d; j += 32) acc += wpred[j] * (double)hu[j] + wpred[g.d + j] * (double)hv[j];
    acc = warp_sum_d(acc);
    if (lane == 0) s.preds[i] = 1.0 / (1.0 + exp(-(acc + bpred)));
  }
  const int nD = s.res->nD;
  GRID_STRIDE(x, (int64_t)nD * g.d_s) {
    const int d = (int)(x / g.d_s), c = (int)(x % g.d_s);
    const int v = s.alist[d];
    st.mem[(int64_t)v * g.ld_s + c] = s.mem_new[(int64_t)d * g.ld_s + c];
    if (c == 0) {
      st.version[v] = s.hdr->batch_index;
      st.last[v] = s.in_t[s.rec_s[s.doff[d + 1] - 1] >> 1];  // latest message (t non-decreasing)
    }
  }
}

// Memory update of V_direct, fused: messages (S/kernels/reference.py:32-53),
// per-node aggregation (:56-74) and one GRU step (:81-90). Messages are
// linear in their input row, so the aggregate is formed on the inputs:
//   agg = ([sum_src x || sum_dst x] [W_src; W_dst] + n_src b_src + n_dst b_dst) / (n if mean)
// with x = [s_v || s_other || feat || phi(t - last_v)]; for `last` only the
// node's last message (its own side) enters. The new memory goes to
// mem_new (committed after the recompute, which still reads pre-batch memory).
#define MG_THREADS 512
#ifndef GRU_T
#define GRU_T 16
#endif
#define MEM_SREC 256  // records staged per pass
__global__ void __launch_bounds__(MG_THREADS)
k_memory(Geo g, StateView st, Scratch s, const float* wmsg2, const float* bmsg,
         const double* omega, const float* wgru, const float* ugru, const float* bgru,
         int aggregator, int ld_dm, int ld_ds, int wsm) {
#ifdef STGN_SKIP_MEMORY  // timing experiments only: results are wrong
  return;
#endif
  extern __shared__ float4 smem4[];
  const int T = GRU_T;
  const int MI2 = 2 * g.msg_in;
  float* X2 = reinterpret_cast<float*>(smem4);  // R4 [T][2 msg_in]
  float* Ag = X2 + T * MI2;                      // R4 [T][ld_dm]
  float* Sp = Ag + T * ld_dm;                    // R4 [T][d_s]
  float* G = Sp + T * g.d_s;                     // R4 [T][3 ld_ds]  agg x [Wz|Wr|Wh]
  float* P = G + T * 3 * ld_ds;                  // R4 [T][2 ld_ds]  s x [Uz|Ur]
  float* Rs = P + T * 2 * ld_ds;                 // R4 [T][d_s]      r * s
  float* Hh = Rs + T * g.d_s;                    // R4 [T][ld_ds]    (r * s) x Uh
  float* Wsm = Hh + T * ld_ds;                   // staged weight rows
  __shared__ int s_node[GRU_T], s_lo[GRU_T], s_hi[GRU_T], s_last[GRU_T], s_n0[GRU_T], s_n1[GRU_T];
  __shared__ int s_re[MEM_SREC], s_rside[MEM_SREC], s_roth[MEM_SREC];
  __shared__ double s_rdt[MEM_SREC];
  const int nD = s.res->nD;
  const int64_t ntiles = cdiv(nD, T);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int L3 = 3 * ld_ds;
  const int phi0 = 2 * g.d_s + g.d_e;
  const bool last_agg = aggregator == STGN_AGG_LAST;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int d0 = (int)(tile * T);
    if (tid < T) {
      const int d = d0 + tid;
      int v = -1, lo = 0, hi = 0, lr = -1, n0 = 0, n1 = 0;
      if (d < nD) {
        v = s.alist[d];
        lo = s.doff[d];
        hi = s.doff[d + 1];
        lr = s.rec_s[hi - 1];
        for (int q = lo; q < hi; ++q) {
          if (s.rec_s[q] & 1) ++n1; else ++n0;
        }
      }
      s_node[tid] = v; s_lo[tid] = lo; s_hi[tid] = hi; s_last[tid] = lr;
      s_n0[tid] = n0; s_n1[tid] = n1;
    }
    __syncthreads();
    // aggregated message inputs [sum_src x || sum_dst x]; the tile's records
    // are one contiguous range of rec_s, staged (edge, other end, dt) in smem
    // so the column sweep issues independent loads only
    for (int o = tid; o < T * MI2; o += nt) X2[o] = 0.f;
    const int rlo = s.doff[d0], rhi = s.doff[d0 + T < nD ? d0 + T : nD];
    for (int rc0 = rlo; rc0 < rhi; rc0 += MEM_SREC) {
      const int rcn = rhi - rc0 < MEM_SREC ? rhi - rc0 : MEM_SREC;
      __syncthreads();
      for (int q = tid; q < rcn; q += nt) {
        const int r = s.rec_s[rc0 + q];
        const int64_t e = r >> 1;
        const int own = (r & 1) ? s.in_dst[e] : s.in_src[e];
        s_re[q] = (int)e;
        s_rside[q] = r & 1;
        s_roth[q] = (r & 1) ? s.in_src[e] : s.in_dst[e];
        s_rdt[q] = s.in_t[e] - st.last[own];
      }
      __syncthreads();
      for (int o = tid; o < T * MI2; o += nt) {
        const int i = o / MI2, c = o - i * MI2;
        const int v = s_node[i];
        if (v < 0) continue;
        const int side = c >= g.msg_in;
        const int cc = c - side * g.msg_in;
        int qa = (last_agg ? s_hi[i] - 1 : s_lo[i]) - rc0, qb = s_hi[i] - rc0;
        if (qa < 0) qa = 0;
        if (qb > rcn) qb = rcn;
        float acc = 0.f;
        for (int q = qa; q < qb; ++q) {
          if (s_rside[q] != side) continue;
          float x;
          if (cc < g.d_s) x = st.mem[(int64_t)v * g.ld_s + cc];
          else if (cc < 2 * g.d_s) x = st.mem[(int64_t)s_roth[q] * g.ld_s + cc - g.d_s];
          else if (cc < phi0) x = s.in_feat[(int64_t)s_re[q] * g.ld_e + (cc - 2 * g.d_s)];
          else {
            const int p = cc - phi0;
            float sv, cv;
            phase_sincos(omega[p >> 1], s_rdt[q], &sv, &cv);
            x = ((p & 1) ? sv : cv) * g.phi_amp;
          }
          acc += x;
        }
        X2[r4(i, c, MI2)] += acc;
      }
    }
    for (int o = tid; o < T * g.d_s; o += nt) {
      const int i = o / g.d_s, c = o % g.d_s;
      Sp[r4(i, c, g.d_s)] = s_node[i] >= 0 ? st.mem[(int64_t)s_node[i] * g.ld_s + c] : 0.f;
    }
    __syncthreads();
    gemm_staged<2>(X2, MI2, 0, T, MI2, wmsg2, ld_dm, 0, g.d_m, 1, Ag, ld_dm, 0, 1.f, nullptr, 0,
                   false, Wsm, wsm);
    for (int o = tid; o < T * g.d_m; o += nt) {  // biases and the mean
      const int i = o / g.d_m, c = o % g.d_m;
      if (s_node[i] < 0) continue;
      float& a = Ag[r4(i, c, ld_dm)];
      if (last_agg) {
        a += bmsg[(s_last[i] & 1) * g.d_m + c];
      } else {
        a += (float)s_n0[i] * bmsg[c] + (float)s_n1[i] * bmsg[g.d_m + c];
        if (aggregator == STGN_AGG_MEAN) a /= (float)(s_n0[i] + s_n1[i]);
      }
    }
    __syncthreads();
    gemm_staged<2>(Ag, ld_dm, 0, T, g.d_m, wgru, L3, 0, L3, 1, G, L3, 0, 1.f, nullptr, 0, false,
                   Wsm, wsm);
    gemm_staged<2>(Sp, g.d_s, 0, T, g.d_s, ugru, L3, 0, 2 * ld_ds, 1, P, 2 * ld_ds, 0, 1.f,
                   nullptr, 0, false, Wsm, wsm);
    for (int o = tid; o < T * g.d_s; o += nt) {
      const int i = o / g.d_s, c = o % g.d_s;
      const float z = sigmoidf_(G[r4(i, c, L3)] + P[r4(i, c, 2 * ld_ds)] + bgru[c]);
      const float r = sigmoidf_(G[r4(i, ld_ds + c, L3)] + P[r4(i, ld_ds + c, 2 * ld_ds)] +
                                bgru[g.d_s + c]);
      G[r4(i, c, L3)] = z;
      Rs[r4(i, c, g.d_s)] = r * Sp[r4(i, c, g.d_s)];
    }
    __syncthreads();
    gemm_staged<2>(Rs, g.d_s, 0, T, g.d_s, ugru + 2 * ld_ds, L3, 0, g.d_s, 1, Hh, ld_ds, 0, 1.f,
                   nullptr, 0, false, Wsm, wsm);
    for (int o = tid; o < T * g.d_s; o += nt) {
      const int i = o / g.d_s, c = o % g.d_s;
      if (s_node[i] < 0) continue;
      const float cand = tanhf(G[r4(i, 2 * ld_ds + c, L3)] + Hh[r4(i, c, ld_ds)] + bgru[2 * g.d_s + c]);
      const float z = G[r4(i, c, L3)];
      s.mem_new[(int64_t)(d0 + i) * g.ld_s + c] = (1.f - z) * cand + z * Sp[r4(i, c, g.d_s)];
    }
    __syncthreads();
  }
}

// Drift estimators: acc_v <- gamma^(tau - touched_v) acc_v + |dN_v| / |N_v|
// for nodes with a non-empty change record; cumulative affected set.
// Estimators live at the node's position in the cumulative set (a nonzero
// estimator implies membership), so the per-batch global mean streams
// contiguous arrays and a reset only forgets the set.
__global__ void k_drift_record(StateView st, Scratch s) {
  const int nA = s.res->nA;
  const int64_t tau = st.ctl->tau + 1;
  const uint32_t gen = st.ctl->cum_gen + 1;  // cum_mark starts at 0 = "never"
  GRID_STRIDE(a64, nA) {
    const int a = (int)a64;
    const int v = s.alist[a];
    const int sz = s.a_size[a], len = s.a_len[a];
    int pos;
    bool fresh = false;
    if (st.cum_mark[v] != gen) {
      st.cum_mark[v] = gen;
      pos = (int)atomicAdd((unsigned long long*)&st.ctl->cum_count, 1ull);
      st.cum_list[pos] = v;
      st.cum_pos[v] = pos;
      fresh = true;
    } else {
      pos = st.cum_pos[v];
    }
    if (sz > 0 && len > 0) {
      const double acc = fresh ? 0.0 : st.drift_acc[pos];
      const double dec = acc == 0.0 ? 0.0 : acc * st.gpow[tau - st.drift_touched[pos]];
      st.drift_acc[pos] = dec + (double)sz / (double)len;
      st.drift_touched[pos] = tau;
    } else if (fresh) {
      st.drift_acc[pos] = 0.0;
      st.drift_touched[pos] = 0;
    }
  }
}

// Global drift = mean decayed estimator over the cumulative affected set;
// the policy decision (S/drift.py:16-23, 72-78; S/engine.py:440-453) is
// made by the last block to finish. rebuild: 0 never, 1 fixed, 2 adaptive.
__global__ void k_drift_decide(StateView st, Scratch s, int rebuild, int64_t interval,
                               double delta_max, double alpha, cudaGraphConditionalHandle cond) {
  __shared__ double red[32];
  __shared__ bool is_last;
  const int64_t tau = st.ctl->tau + 1;
  const int64_t n = st.ctl->cum_count;
  double part = 0.0;
  if (rebuild == STGN_REBUILD_ADAPTIVE) {
    // fixed per-block partition -> deterministic sum
    const int64_t per = cdiv(n, gridDim.x);
    const int64_t lo = blockIdx.x * per, hi = lo + per < n ? lo + per : n;
    const int64_t bd = blockDim.x;
    // four independent positions per step (memory-level parallelism), fixed order
    for (int64_t q0 = lo + threadIdx.x; q0 < hi; q0 += 4 * bd) {
      double acc[4];
      int64_t tch[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t q = q0 + u * bd;
        acc[u] = q < hi ? st.drift_acc[q] : 0.0;
        tch[u] = q < hi ? st.drift_touched[q] : tau;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double dec = acc[u] == 0.0 ? 0.0 : acc[u] * st.gpow[tau - tch[u]];
        part += dec;
        if (dec > delta_max) {
          const int pos = atomicAdd(&s.res->n_drifted, 1);
          s.drifted[pos] = st.cum_list[q0 + u * bd];
        }
      }
    }
  }
  part = warp_sum_d(part);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += red[w];
    s.partials[blockIdx.x] = b;
    __threadfence();
    const unsigned t = atomicAdd(&s.res->ticket, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  {  // the last block sums the block partials in a fixed order (deterministic)
    double t = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) t += s.partials[b];
    t = warp_sum_d(t);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int kind = 0;
    double gdrift = 0.0;
    if (rebuild == STGN_REBUILD_ADAPTIVE) {
      double tot = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
      gdrift = n > 0 ? tot / (double)n : 0.0;
      if (gdrift > delta_max) {
        const double nn = (double)s.hdr->node_count;
        kind = ((double)s.res->n_drifted < alpha * nn) ? 1 : 2;
      }
    } else if (rebuild == STGN_REBUILD_FIXED) {
      if (interval >= 1 && s.hdr->batch_index % interval == 0) kind = 2;
    }
    s.res->global_drift = gdrift;
    s.res->rebuild_kind = kind;
    s.res->rb_partial_n = kind == 1 ? s.res->n_drifted : 0;
    s.res->rb_full_n = kind == 2 ? (int32_t)s.hdr->node_count : 0;
    s.res->rebuild_nodes = kind == 1 ? s.res->n_drifted : (kind == 2 ? s.hdr->node_count : 0);
    st.ctl->tau = tau;
    if (cond) cudaGraphSetConditional(cond, kind != 0 ? 1u : 0u);
  }
}

// Rebuild prologue: uncached nodes get their cache filled from the store
// (S/engine.py:390-392).
// In delta mode on single-layer models the rebuilt nodes get attention-state
// stamps, as the rebuild's _compute_exact keeps states (:393-395).
__global__ void k_rb_fill(Geo g, StateView st, const int32_t* list, const int32_t* count_ptr,
                          int64_t count_const, int stamp) {
  const int64_t n = count_ptr ? (int64_t)count_ptr[0] : count_const;
  GRID_STRIDE(q, n) {
    const int v = list ? list[q] : (int)q;
    int cc = st.ring_ccnt[v];
    if (cc < 0) st.ring_ccnt[v] = cc = st.ring_cnt[v];
    if (stamp) {
      st.attn_ver[v] = st.version[v];
      st.attn_tref[v] = cc > 0 ? st.ring_t[(int64_t)v * g.L + st.ring_head[v]] : 0.0;
    }
  }
}

// Scheduler reset after an executed rebuild (S/drift.py:92-96): forgetting
// the cumulative set clears every estimator (they are indexed by position).
__global__ void k_drift_reset_fin(StateView st, Scratch s) {
  if (threadIdx.x || blockIdx.x) return;
  if (s.res->rebuild_kind == 0) return;
  st.ctl->cum_count = 0;
  st.ctl->cum_gen += 1;
  st.ctl->tau = 0;
}

// Clear per-node batch scratch of the direct nodes.
__global__ void k_cleanup(StateView st, Scratch s) {
  PDL_WAIT();
  const int nD = s.res->nD;
  GRID_STRIDE(d, nD) {
    const int v = s.alist[d];
    st.nodecnt[v] = 0;
    st.nodeadj[v] = 0;
    st.nodefill[v] = 0;
  }
}
