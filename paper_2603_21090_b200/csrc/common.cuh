// Internal definitions shared by the kernels and the engine driver.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/stgn.h"

#define STGN_MAX_LAYERS 8
#define STGN_WARPS 8
#define STGN_THREADS (STGN_WARPS * 32)

static inline __host__ __device__ int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
static inline __host__ __device__ int64_t cdiv(int64_t x, int64_t m) { return (x + m - 1) / m; }

// Derived widths, passed by value to every kernel.
struct Geo {
  int d_s, d_e, d_t, d_x, d_m, d_k, H, K, L;
  int d, q_in, k_in, msg_in, HD;
  int ld_s, ld_d, ld_e, ld_m, ld_t;
  int half;             // d_t / 2
  float inv_sqrt_dk;
  float phi_amp;        // sqrt(1/d_t)
  int own_lo, own_hi;   // node-id shard of this engine (own_hi <= own_lo: every node);
                        // frozen payload rows are kept and recomputed for owned nodes only
};
__host__ __device__ inline bool geo_owns(const Geo& g, int v) {
  return g.own_hi <= g.own_lo || (v >= g.own_lo && v < g.own_hi);
}

static inline Geo make_geo(const stgn_dims& dm, int L) {
  Geo g;
  g.d_s = dm.d_s; g.d_e = dm.d_e; g.d_t = dm.d_t; g.d_x = dm.d_x; g.d_m = dm.d_m;
  g.d_k = dm.d_k; g.H = dm.heads; g.K = dm.layers; g.L = L;
  g.d = dm.d_s + dm.d_x;
  g.q_in = g.d + dm.d_t;
  g.k_in = g.d + dm.d_e + dm.d_t;
  g.msg_in = 2 * dm.d_s + dm.d_e + dm.d_t;
  g.HD = dm.heads * dm.d_k;
  g.ld_s = (int)round_up(dm.d_s, 4);
  g.ld_d = (int)round_up(g.d, 4);
  g.ld_e = (int)round_up(dm.d_e > 0 ? dm.d_e : 1, 4);
  g.ld_m = (int)round_up(dm.d_m, 4);
  g.ld_t = (int)round_up(dm.d_t, 4);
  g.half = dm.d_t / 2;
  g.inv_sqrt_dk = (float)(1.0 / sqrt((double)dm.d_k));
  g.phi_amp = (float)sqrt(1.0 / (double)dm.d_t);
  g.own_lo = g.own_hi = 0;
  return g;
}

// Per-batch header, written to the device once per batch (H2D) so the
// captured graph can be replayed with new values.
struct BatchHdr {
  int64_t B, m0, batch_index, node_count;
  double t_batch, cutoff;   // cutoff = t_batch - window (or -inf)
  uint32_t stamp;           // batch stamp for amark/dmark
  int32_t pad;
  double gpow_tau;          // unused placeholder
};

// Per-batch results/counters (device, reset at the start of each batch).
struct BatchRes {
  int32_t nD, nA;
  int32_t hop_off[STGN_MAX_LAYERS + 2];
  int32_t n_drifted;
  int32_t pad;
  unsigned long long nbr_hit, nbr_miss, E_A, E_D, E_R, changed;
  int64_t rebuild_kind, rebuild_nodes;
  double global_drift;
  int32_t rb_partial_n, rb_full_n;   // rebuild work sizes (0 unless that kind fired)
  int32_t nAD;                       // rows of the fused recompute (A pre + D post)
  uint32_t hop_ticket;               // last-block-done counter of k_hop (STGN_HOP_TICKET)
  uint32_t ticket;                   // last-block-done counter of k_drift_decide
  int32_t nC;                        // delta mode: rows of the pre-batch recompute (clist)
  int32_t n_skip, n_hit, n_miss;     // delta mode classification
  int32_t pad4;
  unsigned long long E_miss;         // delta mode: entries over attn_miss nodes
};

// Scratch carving (all offsets 256-B aligned).
struct Scratch {
  BatchHdr* hdr;
  BatchRes* res;
  int32_t *in_src, *in_dst;
  double* in_t;
  float* in_feat;           // [Bmax][ld_e]
  int32_t* alist;           // [cap_nodes]  D first (0..nD), then BFS hops
  int32_t* doff;            // [2Bmax+1]
  int32_t *rec_u, *rec_s;   // [2Bmax]
  int32_t* rec_adjrank;     // [2Bmax]  by record id
  int32_t* rec_prev;        // [2Bmax]  by record id: previous (older) adj record of same node, -1
  int32_t *d_wascached, *d_baselen;  // [2Bmax] by D index
  int32_t* a_size;          // [cap_nodes] change-record size by A index
  int32_t* a_len;           // [cap_nodes] cache length after the batch, by A index
  int32_t* clist;           // [cap_nodes] delta mode: D, then the non-skipped nodes of A \ D
  int32_t* c_info;          // [cap_nodes] delta mode, by clist row: change-record size << 1 | attn_hit
  float* msgs;              // [2Bmax][ld_m]
  double* preds;            // [Bmax]
  float* dpred;             // [2Bmax][ld_d]
  int32_t* drifted;         // [cap_nodes]
  double* partials;         // [1024]
  int32_t* rb_ids;          // [cap_nodes] host-provided rebuild list
  int32_t* dmap;            // [cap_nodes] node -> direct index (valid for this batch's D)
  float* mem_new;           // [2Bmax][ld_s] post-batch memory of D (committed after recompute)
};

static inline int64_t carve(int64_t& off, int64_t bytes) {
  int64_t o = off;
  off += round_up(bytes, 256);
  return o;
}

static inline int64_t scratch_layout(const Geo& g, int64_t Bmax, int64_t cap_nodes, Scratch* s,
                                     uint8_t* base) {
  int64_t off = 0;
  int64_t R = 2 * Bmax;
  int64_t o_hdr = carve(off, sizeof(BatchHdr));
  int64_t o_res = carve(off, sizeof(BatchRes));
  int64_t o_src = carve(off, Bmax * 4), o_dst = carve(off, Bmax * 4);
  int64_t o_t = carve(off, Bmax * 8), o_feat = carve(off, Bmax * g.ld_e * 4);
  int64_t o_alist = carve(off, cap_nodes * 4);
  int64_t o_doff = carve(off, (R + 1) * 4);
  int64_t o_ru = carve(off, R * 4), o_rs = carve(off, R * 4);
  int64_t o_rank = carve(off, R * 4), o_prev = carve(off, R * 4);
  int64_t o_wc = carve(off, R * 4), o_bl = carve(off, R * 4);
  int64_t o_asz = carve(off, cap_nodes * 4), o_alen = carve(off, cap_nodes * 4);
  int64_t o_clist = carve(off, cap_nodes * 4);
  int64_t o_cinfo = carve(off, cap_nodes * 4);
  int64_t o_msg = carve(off, R * g.ld_m * 4);
  int64_t o_pred = carve(off, Bmax * 8);
  int64_t o_dpred = carve(off, R * g.ld_d * 4);
  int64_t o_drift = carve(off, cap_nodes * 4);
  int64_t o_part = carve(off, 1024 * 8);
  int64_t o_rb = carve(off, cap_nodes * 4);
  int64_t o_dmap = carve(off, cap_nodes * 4);
  int64_t o_mnew = carve(off, R * g.ld_s * 4);
  if (s && base) {
    s->hdr = (BatchHdr*)(base + o_hdr);
    s->res = (BatchRes*)(base + o_res);
    s->in_src = (int32_t*)(base + o_src);
    s->in_dst = (int32_t*)(base + o_dst);
    s->in_t = (double*)(base + o_t);
    s->in_feat = (float*)(base + o_feat);
    s->alist = (int32_t*)(base + o_alist);
    s->doff = (int32_t*)(base + o_doff);
    s->rec_u = (int32_t*)(base + o_ru);
    s->rec_s = (int32_t*)(base + o_rs);
    s->rec_adjrank = (int32_t*)(base + o_rank);
    s->rec_prev = (int32_t*)(base + o_prev);
    s->d_wascached = (int32_t*)(base + o_wc);
    s->d_baselen = (int32_t*)(base + o_bl);
    s->a_size = (int32_t*)(base + o_asz);
    s->a_len = (int32_t*)(base + o_alen);
    s->clist = (int32_t*)(base + o_clist);
    s->c_info = (int32_t*)(base + o_cinfo);
    s->msgs = (float*)(base + o_msg);
    s->preds = (double*)(base + o_pred);
    s->dpred = (float*)(base + o_dpred);
    s->drifted = (int32_t*)(base + o_drift);
    s->partials = (double*)(base + o_part);
    s->rb_ids = (int32_t*)(base + o_rb);
    s->dmap = (int32_t*)(base + o_dmap);
    s->mem_new = (float*)(base + o_mnew);
  }
  return off;
}

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// phi component p of phi(dt): amp * (p even ? cos : sin)(omega[p/2] * dt).
// Angle and its trig are evaluated in float64 (Delta t reaches ~1e7 ticks,
// where a float32 angle loses the phase), then rounded to float32.
__device__ __forceinline__ float phi_component(const double* __restrict__ omega, int p, double dt,
                                               float amp) {
  double ang = omega[p >> 1] * dt;
  double v = (p & 1) ? sin(ang) : cos(ang);
  return (float)v * amp;
}

__device__ __forceinline__ float sigmoidf_(float x) { return 1.0f / (1.0f + expf(-x)); }

// Programmatic dependent launch (STGN_PDL builds): the kernels of the batch
// chain are launched with programmatic stream serialization, so a kernel's
// launch overlaps its predecessor's tail; it must wait here before touching
// anything the predecessor writes. A no-op for ordinary launches.
#ifdef STGN_PDL
#define PDL_WAIT() asm volatile("griddepcontrol.wait;\n" ::: "memory")
#else
#define PDL_WAIT() do {} while (0)
#endif

// Last CUDA failure (file:line + message), readable through stgn_last_error().
void stgn_set_error(const char* file, int line, cudaError_t e);

#define CUDA_TRY(expr)                                        \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) {                                  \
      stgn_set_error(__FILE__, __LINE__, _e);                 \
      return STGN_ERR_CUDA;                                   \
    }                                                         \
  } while (0)
