// Stage-level surface of the incremental engine: the reference's unit entry
// points that process_batch runs fused (batch.cuh).
//
//   k_stage_affected    IncrementalEngine.detect_affected(pending)   S/engine.py:196-212
//                       (_group_batch S/engine.py:170-180, _sampled_ids :182-194)
//   k_stage_nbr_update  IncrementalEngine.update_neighbor_cache      S/engine.py:216-243
//   k_stage_commit      EngineCore.commit_pending                    S/engine_base.py:108-117
//
// A staged batch lives in small device arrays (src, dst, t, eid; pending
// payload stacks uploaded by the host from stage_batch's frozen copies); none
// of these kernels sits on the streaming path, so they favour a direct
// statement of the reference semantics over throughput (one CTA for the BFS,
// one warp per node for the list update, one thread for the store chains).
#pragma once

#include "batch.cuh"

// j-th newest new entry of node w in a staged batch (reverse batch order; a
// self-loop contributes one entry, its src side). Returns the neighbour or -1.
__device__ __forceinline__ int stage_new_nbr(const int32_t* src, const int32_t* dst, int P, int w,
                                             int j) {
  for (int i = P - 1; i >= 0; --i) {
    const int s = src[i], d = dst[i];
    if (s == w || d == w) {
      if (j == 0) return s == w ? d : s;
      --j;
    }
  }
  return -1;
}

__device__ __forceinline__ int stage_new_count(const int32_t* src, const int32_t* dst, int P,
                                               int w) {
  int k = 0;
  for (int i = 0; i < P; ++i) k += (src[i] == w || dst[i] == w);
  return k;
}

// Direct endpoints, then K hops over the post-insertion truncated lists: the
// staged new entries of w followed by its cached list (or the store's top-L
// when uncached), first L. One CTA; marks are the engine's node stamps.
// out[0 .. hop_off[K+1]) holds the set in discovery order.
__global__ void k_stage_affected(Geo g, StateView st, const int32_t* __restrict__ src,
                                 const int32_t* __restrict__ dst, int P, uint32_t stamp,
                                 int32_t* out, int64_t cap, int32_t* hop_off) {
  __shared__ int nA;
  if (threadIdx.x == 0) nA = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < 2 * P; r += blockDim.x) {
    const int v = (r & 1) ? dst[r >> 1] : src[r >> 1];
    if (atomicExch(&st.amark[v], stamp) != stamp) {
      const int p = atomicAdd(&nA, 1);
      if (p < cap) out[p] = v;
    }
  }
  __syncthreads();
  int f0 = 0, f1 = nA;
  if (threadIdx.x == 0) {
    hop_off[0] = 0;
    hop_off[1] = f1;
  }
  if (f1 > cap) f1 = (int)cap;
  for (int hop = 1; hop <= g.K; ++hop) {
    const int64_t total = (int64_t)(f1 - f0) * g.L;
    for (int64_t x = threadIdx.x; x < total; x += blockDim.x) {
      const int w = out[f0 + (int)(x / g.L)];
      const int j = (int)(x % g.L);
      const int kn = stage_new_count(src, dst, P, w);
      int u = -1;
      if (j < kn) {
        u = stage_new_nbr(src, dst, P, w, j);
      } else {
        const int cc = st.ring_ccnt[w];
        const int len = cc >= 0 ? cc : st.ring_cnt[w];
        const int jj = j - kn;
        if (jj < len) u = st.ring_nbr[(int64_t)w * g.L + (st.ring_head[w] + jj) % g.L];
      }
      if (u >= 0 && atomicExch(&st.amark[u], stamp) != stamp) {
        const int p = atomicAdd(&nA, 1);
        if (p < cap) out[p] = u;
      }
    }
    __syncthreads();
    f0 = f1;
    f1 = nA;
    if (threadIdx.x == 0) hop_off[hop + 1] = f1;  // > cap: the host reports STGN_ERR_CAPACITY
    if (f1 > cap) f1 = (int)cap;                  // never read past the list
    if (f0 > f1) f0 = f1;
    __syncthreads();
  }
}

// New entries of a list of nodes (CSR by node, newest first per node) and the
// per-node record outputs: stgn_stage_entries / stgn_stage_records (stgn.h).
typedef stgn_stage_entries StageEntries;
typedef stgn_stage_records StageRecords;

__device__ __forceinline__ bool stage_in_sorted(const int32_t* a, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo < n && a[lo] == x;
}

// Prepend each node's new entries, evict beyond L, expire outside the window,
// and report the record (added is the caller's list; expired; updated = the
// kept older entries whose neighbour is direct). One warp per node.
__global__ void k_stage_nbr_update(Geo g, StateView st, StageEntries en, int nn,
                                   const int32_t* __restrict__ direct, int nd, double cutoff,
                                   const double* __restrict__ omega, StageRecords rec) {
  const int lane = threadIdx.x & 31;
  const int warps = (int)(gridDim.x * (blockDim.x >> 5));
  for (int i = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < nn; i += warps) {
    const int v = en.nodes[i];
    const int o = en.off[i], kn = en.off[i + 1] - o;
    const int head = st.ring_head[v], cnt = st.ring_cnt[v], cc = st.ring_ccnt[v];
    const bool hit = cc >= 0, put = en.put[i] != 0;
    const int blen = hit ? cc : cnt;
    const int total = kn + blen, keep = total < g.L ? total : g.L;
    __syncwarp();  // every lane has read the node's list header
    if (lane == 0 && put) {
      auto e_nbr = [&](int q) { return q < kn ? en.nbr[o + q] : st.ring_nbr[(int64_t)v * g.L + (head + q - kn) % g.L]; };
      auto e_t = [&](int q) { return q < kn ? en.t[o + q] : st.ring_t[(int64_t)v * g.L + (head + q - kn) % g.L]; };
      auto e_eid = [&](int q) { return q < kn ? en.eid[o + q] : st.ring_eid[(int64_t)v * g.L + (head + q - kn) % g.L]; };
      const int xo = o + i * g.L;
      int ne = 0;
      auto expire = [&](int q) {
        rec.exp_nbr[xo + ne] = e_nbr(q);
        rec.exp_t[xo + ne] = e_t(q);
        rec.exp_eid[xo + ne] = e_eid(q);
        ++ne;
      };
      if (hit)  // a miss evicts nothing: nothing was cached (S/engine.py:226-231)
        for (int q = keep; q < total; ++q) expire(q);
      int kept = keep, nnew = kn < keep ? kn : keep;
      // the window: lists are newest first, so what falls outside is a suffix
      int kf = 0;
      while (kf < keep && !(e_t(kf) < cutoff)) ++kf;
      for (int q = kf; q < keep; ++q) expire(q);
      kept = kf;
      nnew = nnew < kf ? nnew : kf;
      int nu = 0;
      for (int q = nnew; q < kept; ++q) {
        const int u = e_nbr(q);
        if (!stage_in_sorted(direct, nd, u)) continue;
        bool dup = false;
        for (int z = 0; z < nu; ++z) dup |= rec.upd_nbr[i * g.L + z] == u;
        if (!dup) rec.upd_nbr[i * g.L + nu++] = u;
      }
      rec.hit[i] = hit;
      rec.exp_n[i] = ne;
      rec.upd_n[i] = nu;
      st.ring_ccnt[v] = kept;
    }
    __syncwarp();
    // the list reads above are done: write the kept new entries before the head
    const int kk = kn < g.L ? kn : g.L;
    int nh = (head - kk) % g.L;
    if (nh < 0) nh += g.L;
    for (int j = 0; j < kk; ++j) {
      const int slot = (nh + j) % g.L;
      const int64_t rs = (int64_t)v * g.L + slot;
      if (lane == 0) {
        st.ring_nbr[rs] = en.nbr[o + j];
        st.ring_eid[rs] = en.eid[o + j];
        st.ring_t[rs] = en.t[o + j];
      }
      for (int c = lane; c < g.d_e; c += 32) st.ring_feat[rs * g.ld_e + c] = en.feat[(int64_t)(o + j) * g.ld_e + c];
      for (int f = lane; f < g.half; f += 32) {
        float sv, cv;
        phase_sincos(omega[f], en.t[o + j], &sv, &cv);
        st.ring_tb[rs * g.ld_t + 2 * f] = cv;
        st.ring_tb[rs * g.ld_t + 2 * f + 1] = sv;
      }
      for (int l = 0; l < g.K; ++l) {
        const float* sp = en.pay + ((int64_t)(o + j) * g.K + l) * g.ld_d;
        float* dp = st.ring_pay + (((int64_t)v * g.K + l) * g.L + slot) * g.ld_d;
        for (int c = lane; c < g.d; c += 32) dp[c] = sp[c];
      }
    }
    if (lane == 0) {
      st.ring_head[v] = nh;
      st.ring_cnt[v] = cnt + kn < g.L ? cnt + kn : g.L;
    }
  }
}

// Insert the staged edges into the append-only store in id order: the edge log,
// each endpoint's newest-first chain (a self-loop once) and, when the engine
// keeps it, the payload log (pay: [P][2][K][ld_d], side 0 = the src entry's
// payload, i.e. the dst stack). S/graph_store.py:130-156, S/engine_base.py:108-117.
__global__ void k_stage_commit(Geo g, StateView st, const int32_t* __restrict__ src,
                               const int32_t* __restrict__ dst, const double* __restrict__ t,
                               const float* __restrict__ feat, const float* __restrict__ pay,
                               int P, int64_t m0) {
  for (int x = threadIdx.x; x < P * g.d_e; x += blockDim.x) {
    const int i = x / g.d_e, c = x % g.d_e;
    st.e_feat[(m0 + i) * g.ld_e + c] = feat[(int64_t)i * g.ld_e + c];
  }
  if (st.e_pay) {
    const int64_t row = (int64_t)g.K * g.ld_d;
    for (int64_t x = threadIdx.x; x < (int64_t)P * 2 * row; x += blockDim.x) {
      const int64_t r = x / row;  // 2 i + side
      st.e_pay[(2 * m0 + r) * row + x % row] = pay[x];
    }
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < P; ++i) {
      const int64_t eid = m0 + i;
      const int s = src[i], d = dst[i];
      st.e_src[eid] = s;
      st.e_dst[eid] = d;
      st.e_t[eid] = t[i];
      for (int side = 0; side < (s == d ? 1 : 2); ++side) {
        const int v = side ? d : s;
        const int64_t ent = 2 * eid + side;
        st.e_prev[ent] = st.adj_head[v];
        st.adj_head[v] = ent;
        st.adj_deg[v] += 1;
      }
    }
  }
}
