// Historical neighbour lists for OracleEngine.full_recompute(t_now)
// (reference S/oracle.py:40-65: a node's entries are the L newest store entries
// with t <= t_now, get_temporal_neighbors(v, -inf, t_now)[:L],
// S/graph_store.py:158-173; memory is the current one; nothing is mutated).
//
// The append-only store keeps every entry in a per-node chain (adj_head, then
// e_prev, newest first) and, when the engine keeps the payload log (e_pay), the
// frozen payload stack of every entry. One warp per node walks its chain,
// skipping entries newer than t_now, and writes the first L it keeps into
// temporary ring tables laid out like the live rings (head 0, count = cached
// count), which the recompute kernels then read in place of the live rings.
#pragma once

#include "batch.cuh"

struct HistRings {
  int32_t *cnt, *head, *nbr;  // [n], [n], [n][L]
  int64_t* eid;               // [n][L]
  double* t;                  // [n][L]
  float *pay, *feat, *tb;     // [n][K][L][ld_d], [n][L][ld_e], [n][L][ld_t]
};

static inline size_t hist_rings_bytes(const Geo& g, int64_t n) {
  const int64_t L = g.L;
  return (size_t)n * (4 + 4 + 4 * L + 8 * L + 8 * L +
                      4 * (L * (int64_t)g.K * g.ld_d + L * g.ld_e + L * g.ld_t)) +
         8 * 256;
}

static inline HistRings hist_rings_carve(const Geo& g, int64_t n, uint8_t* base) {
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    uint8_t* p = base + off;
    off += round_up(bytes, 256);
    return p;
  };
  const int64_t L = g.L;
  HistRings h;
  h.cnt = (int32_t*)take(4 * n);
  h.head = (int32_t*)take(4 * n);
  h.nbr = (int32_t*)take(4 * n * L);
  h.eid = (int64_t*)take(8 * n * L);
  h.t = (double*)take(8 * n * L);
  h.pay = (float*)take(4 * n * L * g.K * g.ld_d);
  h.feat = (float*)take(4 * n * L * g.ld_e);
  h.tb = (float*)take(4 * n * L * g.ld_t);
  return h;
}

__global__ void k_hist_rings(Geo g, StateView st, HistRings hr, int64_t n, double t_now,
                             const double* __restrict__ omega) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
    int64_t ent = st.adj_head[v];
    int k = 0;
    while (ent >= 0 && k < g.L) {
      const int64_t eid = ent >> 1;
      const double te = st.e_t[eid];
      if (te <= t_now) {
        const int64_t rs = v * g.L + k;
        if (lane == 0) {
          hr.nbr[rs] = (ent & 1) ? st.e_src[eid] : st.e_dst[eid];
          hr.eid[rs] = eid;
          hr.t[rs] = te;
        }
        const float* ep = st.e_pay + ent * g.K * g.ld_d;
        for (int l = 0; l < g.K; ++l)
          for (int j = lane; j < g.ld_d; j += 32)
            hr.pay[((v * g.K + l) * g.L + k) * g.ld_d + j] = ep[l * g.ld_d + j];
        for (int j = lane; j < g.ld_e; j += 32)
          hr.feat[rs * g.ld_e + j] = st.e_feat[eid * g.ld_e + j];
        for (int f = lane; f < g.half; f += 32) {  // time basis of the entry (attn4)
          float sv, cv;
          phase_sincos(omega[f], te, &sv, &cv);
          hr.tb[rs * g.ld_t + 2 * f] = cv;
          hr.tb[rs * g.ld_t + 2 * f + 1] = sv;
        }
        ++k;
      }
      ent = st.e_prev[ent];
    }
    if (lane == 0) {
      hr.cnt[v] = k;
      hr.head[v] = 0;
    }
  }
}
