/*
 * stgn.h — C ABI of the B200-native StreamTGN incremental inference path.
 *
 * Two plug-in points, matching the two places the reference dispatches
 * this path (reference = /root/reference/pkg/src/streamtgn, "S/"):
 *
 *  1. Engine level — replaces IncrementalEngine (S/engine.py:155-453):
 *       stgn_engine_create / _destroy       <- IncrementalEngine.__init__ (S/engine.py:156-166,
 *                                               S/engine_base.py:62-74)
 *       stgn_engine_bind                    <- the state tables of S/state.py:23-127 and
 *                                               S/graph_store.py:102-152, held on the device
 *       stgn_engine_process_batch           <- IncrementalEngine.process_batch (S/engine.py:400-438)
 *       stgn_engine_process_batch_dev       <- same, inputs already resident on the device
 *       stgn_engine_rebuild                 <- IncrementalEngine.rebuild_nodes (S/engine.py:385-396)
 *       stgn_engine_full_reference          <- IncrementalEngine.full_reference (S/engine.py:374-381)
 *       stgn_engine_affected                <- IncrementalEngine.last_affected (S/engine.py:417-418)
 *  2. Operator level — replaces kernels.pipeline_many (S/kernels/__init__.py:42-44):
 *       stgn_pipeline_many
 *
 * Conventions: plain pointers and sizes; every device buffer is allocated
 * by the caller (the Python shim uses PyTorch) and only borrowed here; the
 * engine handle owns nothing but a few pinned host staging buffers and its
 * CUDA graphs. `stream` is a cudaStream_t passed as void*. Functions
 * return STGN_OK or an error code; the Python shim maps codes onto the
 * reference's exception classes.
 */
#ifndef STGN_H
#define STGN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STGN_OK            0
#define STGN_ERR_INVALID   1  /* bad dims/config/argument   -> ConfigError / KernelInputError */
#define STGN_ERR_BOUNDS    2  /* node id / edge id range    -> InputError                     */
#define STGN_ERR_CUDA      3  /* CUDA runtime failure       -> RuntimeError                   */
#define STGN_ERR_CAPACITY  4  /* bound tables too small     -> host grows + rebinds           */
#define STGN_ERR_ORDER     5  /* timestamps decrease        -> MonotonicityError              */

#define STGN_AGG_MEAN 0
#define STGN_AGG_LAST 1
#define STGN_AGG_SUM  2

#define STGN_REBUILD_NEVER    0
#define STGN_REBUILD_FIXED    1
#define STGN_REBUILD_ADAPTIVE 2

#define STGN_SCOPE_AFFECTED 0  /* recompute every node of A (the reference's literal exact mode) */
#define STGN_SCOPE_DIRECT   1  /* recompute V_direct only; value-identical when window = inf     */
#define STGN_SCOPE_DELTA    2  /* the reference's delta mode (S/engine.py:276-331): untouched
                                  affected nodes keep their cached row (embed_skip), the rest are
                                  classified attn_hit / attn_miss against per-node attention-state
                                  stamps and recomputed                                         */

/* Model widths; same meaning as the reference Dims (S/config.py:11-55). */
typedef struct {
  int32_t d_s, d_e, d_t, d_x, d_m, d_k, heads, layers;
} stgn_dims;

/* Run options; same meaning as RunConfig (S/config.py:61-103). */
typedef struct {
  int32_t fanout;            /* L */
  int32_t aggregator;        /* STGN_AGG_* */
  int32_t rebuild;           /* STGN_REBUILD_* */
  int32_t rebuild_interval;
  double  gamma, delta_max, alpha;
  double  window;            /* +inf = no temporal window */
  int32_t scope;             /* STGN_SCOPE_* */
  int32_t max_batch;         /* capacity of the per-batch scratch (edges) */
} stgn_config;

/*
 * Device-resident weights, float32, packed by the host shim (row-major;
 * every row stride is the column count rounded up to a multiple of 4,
 * "ld(x)", zero-filled):
 *   wq    [K][d][ld(H*d_k)]      rows 0..d-1 of w_q (K,H,q_in,d_k) per layer
 *   bq    [K][H*d_k]             phi(0) . w_q[l, :, d:, :] (the constant query half)
 *   wkt   [K][H][d_k][ld(k_in)]  w_k (K,H,k_in,d_k) transposed per head
 *   wv    [K][H][k_in][ld(d_k)]  w_v
 *   wo    [K][H*d_k][ld(d)]      w_o
 *   wmsg  [2*msg_in][ld(d_m)]    [w_msg_src^T ; w_msg_dst^T] (row blocks)
 *   bmsg  [2][d_m]
 *   wgru  [d_m][3*ld(d_s)]       [w_z^T | w_r^T | w_h^T]
 *   ugru  [d_s][3*ld(d_s)]       [u_z^T | u_r^T | u_h^T]
 *   bgru  [3][d_s]
 *   wpred [2*d] double, bpred (host double)
 *   omega [d_t/2] double;  phi0 [d_t] float
 */
typedef struct {
  const float *wq, *bq, *wkt, *wv, *wo;
  const float *wmsg, *bmsg, *wgru, *ugru, *bgru;
  const double *wpred;
  const double *omega;
  const float *phi0;
  double bpred;
  /* Tensor-core operands (optional; NULL = FFMA path). Each GEMM is a
   * K-major B operand [Np][Kp] in 8x4 core matrices (element (n,k) at
   * ((n/8)*(Kp/4) + k/4)*32 + (n%8)*4 + k%4), hi block then lo block
   * (lo = value - trunc_tf32(value)); Np = round_up(N,16), Kp = round_up(K,8):
   *   tcq [K]    N = H*d_k, K = d      (w_q rows 0..d-1)
   *   tck [K][H] N = k_in,  K = d_k    (w_k[l,h] as is)
   *   tcv [K][H] N = d_k,   K = k_in   (w_v[l,h] transposed)
   *   tco [K]    N = d,     K = H*d_k  (w_o[l] transposed) */
  const float *tcq, *tck, *tcv, *tco;
  /* bf16x3 tensor-core operands of the 128-row recompute kernel (optional;
   * used when H = 2 and the TMEM plan fits, else the split-TF32 ones): K-major
   * bf16 B operands [Np][Kp] in 8x8 core matrices (element (n,k) at
   * ((n/8)*(Kp/8) + k/8)*64 + (n%8)*8 + k%8), hi block then lo block
   * (lo = bf16(w - hi)); Kp = round_up(K,16), Np = round_up(N,16), Kq = round_up(d_k,16):
   *   t4q [K]    N = H*Kq (head h at rows h*Kq), K = d            (w_q rows 0..d-1)
   *   t4k [K][H] N = k_in, K = d_k   w_k * log2(e) / sqrt(d_k), time-encoding rows * sqrt(1/d_t)
   *   t4v [K][H] N = d_k,  K = k_in  w_v^T, time-encoding columns * sqrt(1/d_t)
   *   t4o [K]    N = d,    K = H*Kq (head h at h*Kq)               w_o^T
   *   t4bq [K][H][Kq] float   phi(0) . w_q[l, h, d:, :] (zero padded) */
  const uint16_t *t4q, *t4k, *t4v, *t4o;
  const float *t4bq;
  /* bf16x3 tensor-core operands of the memory update (optional; the FFMA
   * k_memory is used when NULL or when the plan does not fit): the same
   * K-major bf16 hi/lo block layout, blocks concatenated in this order
   * (Nm = round_up(d_m,16), Ns = round_up(d_s,16)):
   *   for j < ceil(msg_in/128):  N = Nm,   K = 128   w_msg_src columns [128j, 128j+128),
   *                              N = Nm,   K = 128   then w_msg_dst columns [128j, 128j+128)
   *   1 block                    N = 2*Ns, K = Nm    [w_z ; w_r] (r at row Ns)
   *   1 block                    N = 2*Ns, K = Ns    [u_z ; u_r]
   *   1 block                    N = Ns,   K = Nm    w_h
   *   1 block                    N = Ns,   K = Ns    u_h */
  const uint16_t *t4mem;
  /* folded output operands of the bf16x3 recompute kernel, per layer:
   *   P_h = w_v[l,h] (time rows * sqrt(1/d_t)) @ w_o[l, h*d_k:(h+1)*d_k, :]   (k_in x d)
   * as B operands [n = output column][k = key feature, 4-padded layout of t4k], split at
   * output column Na = min(round_up(d,16), 64): Pa_0, Pa_1 (N = Na), Pb_0, Pb_1
   * (N = round_up(d,16) - Na, absent when 0), K = round_up(k_in padded, 16) */
  const uint16_t *t4p;
} stgn_weights;

/* Persistent control block (device). */
typedef struct {
  int64_t tau;               /* drift scheduler clock (S/drift.py:30) */
  int64_t cum_count;         /* |cumulative affected set| */
  uint32_t cum_gen;          /* generation stamp of cum_mark */
  uint32_t pad0;
  int64_t reserved[6];
} stgn_ctl;

/*
 * Device state tables (all caller-allocated). Row strides:
 *   ld_s = round_up(d_s,4), ld_d = round_up(d,4), ld_e = round_up(max(d_e,1),4).
 * The ring holds, per node, the L newest adjacency entries (newest at
 * ring_head, walking forward mod L); ring_ccnt is the neighbour-cache
 * prefix length (-1 = node not cached, S/state.py:154-171). Frozen
 * payload stacks live in the ring slot: ring_pay[node][layer][slot][ld_d].
 */
typedef struct {
  int64_t cap_nodes, cap_edges, gpow_len;
  float    *mem;        /* [cap_nodes][ld_s]       S/state.py:23-48 */
  double   *last;       /* [cap_nodes]                                */
  int64_t  *version;    /* [cap_nodes]                                */
  float    *h;          /* [cap_nodes][K][ld_d]    S/state.py:91-127  */
  uint8_t  *valid;      /* [cap_nodes]                                */
  double   *valid_at;   /* [cap_nodes]                                */
  int32_t  *ring_cnt, *ring_head, *ring_ccnt;   /* [cap_nodes] */
  int32_t  *ring_nbr;   /* [cap_nodes][L] */
  int64_t  *ring_eid;   /* [cap_nodes][L] */
  double   *ring_t;     /* [cap_nodes][L] */
  float    *ring_pay;   /* [cap_nodes][K][L][ld_d] */
  float    *ring_feat;  /* [cap_nodes][L][ld_e] */
  float    *ring_tb;    /* [cap_nodes][L][ld_t] time basis [cos w_f t, sin w_f t] of the slot's
                           timestamp (ld_t = round_up(d_t,4)), written at insertion */
  uint32_t *amark, *dmark;                      /* [cap_nodes] batch stamps */
  int32_t  *nodecnt, *nodeadj, *nodefill, *nodeoff;  /* [cap_nodes] scratch */
  double   *drift_acc;  /* [cap_nodes] estimator, indexed by cumulative-set position */
  int64_t  *drift_touched; /* [cap_nodes] tau of last touch, same indexing */
  uint32_t *cum_mark;   /* [cap_nodes] node is in the cumulative affected set (generation stamp) */
  int32_t  *cum_list;   /* [cap_nodes] position -> node */
  int32_t  *cum_pos;    /* [cap_nodes] node -> position */
  int64_t  *attn_ver;   /* [cap_nodes] delta mode: memory version the node's attention state was
                           built on, -1 = no state (AttnState.mem_version, S/state.py:175-190) */
  double   *attn_tref;  /* [cap_nodes] delta mode: the state's t_ref (AttnState.t_ref) */
  int32_t  *e_src, *e_dst;  /* [cap_edges]   append-only temporal store */
  double   *e_t;            /* [cap_edges] */
  float    *e_feat;         /* [cap_edges][ld_e] */
  int64_t  *e_prev;         /* [2*cap_edges] previous entry of the same node, -1 none */
  int64_t  *adj_head;       /* [cap_nodes] newest entry (2*eid+side), -1 none */
  int64_t  *adj_deg;        /* [cap_nodes] */
  double   *gpow;           /* [gpow_len] gamma^k, k = 0..gpow_len-1 (host-computed) */
  stgn_ctl *ctl;
  uint8_t  *scratch;        /* stgn_scratch_bytes(...) bytes */
  /* delta mode, K = 1 (S/engine.py:247-274, 333-353): log Z per head of each node's
   * attention state, and the per-batch error-bound records of its attn_hit updates
   * (ctl->reserved[0] = record count, ctl->reserved[1] = max_value_norm_seen as
   * float64 bits). Unused (may be NULL, ev_cap 0) otherwise. */
  double   *attn_logz;      /* [cap_nodes][4] */
  int32_t  *ev_node, *ev_dpos, *ev_dn, *ev_nv;  /* [ev_cap] node, direct index or -1, |dN|, |N| */
  double   *ev_bound, *ev_maxv, *ev_zdev;        /* [ev_cap] */
  int64_t  ev_cap;
  /* optional payload log for historical snapshots (OracleEngine.full_recompute(t_now),
   * S/oracle.py:40-65): the frozen payload stack of every store entry, indexed like
   * e_prev (2*eid + side); NULL = not kept */
  float    *e_pay;          /* [2*cap_edges][K][ld_d] */
} stgn_state;

/* Per-batch report written by process_batch (host memory). Counter
 * names follow S/runner.py:73-77 and S/engine.py:432-433. */
typedef struct {
  int64_t direct, affected;
  int64_t nbr_hit, nbr_miss;
  int64_t entries_affected, entries_direct;   /* sum of list lengths (MAC tallies) */
  int64_t rebuild_kind;                       /* 0 none, 1 partial, 2 full */
  int64_t rebuild_nodes;
  int64_t entries_rebuild;
  int64_t tau, cum_count;
  int64_t changed;                            /* nodes with a non-empty change record */
  double  global_drift;
  /* delta mode (STGN_SCOPE_DELTA) classification, S/engine.py:287-313 */
  int64_t embed_skip, attn_hit, attn_miss;
  int64_t entries_miss;                       /* sum of list lengths over attn_miss nodes */
  int64_t reserved[3];
} stgn_report;

typedef struct stgn_engine stgn_engine;

/* Bytes of scratch the engine needs for these capacities. */
int64_t stgn_scratch_bytes(const stgn_dims* dims, const stgn_config* cfg, int64_t cap_nodes);

int stgn_engine_create(const stgn_dims* dims, const stgn_config* cfg, stgn_engine** out);
int stgn_engine_destroy(stgn_engine* eng);
int stgn_engine_set_weights(stgn_engine* eng, const stgn_weights* w);
/* (Re)bind state tables after allocation or growth; drops cached graphs. */
int stgn_engine_bind(stgn_engine* eng, const stgn_state* st);

/*
 * One batch, host buffers in, host buffers out (the end-to-end path).
 * src/dst: int32 node ids; t: float64 non-decreasing and >= t_now;
 * feat: float32 [B][d_e] (row stride d_e). m0 = committed edge count,
 * batch_index = 1-based index of this batch, node_count = max(n seen, hint)
 * after this batch. preds_out: float64 [B]. Blocks until done.
 */
int stgn_engine_process_batch(stgn_engine* eng, int32_t B, const int32_t* src,
                              const int32_t* dst, const double* t, const float* feat,
                              int64_t m0, int64_t batch_index, int64_t node_count,
                              double* preds_out, stgn_report* rep, void* stream);

/* Same, inputs already on the device (src/dst int32, t f64, feat f32 [B][d_e], or NULL for zero features);
 * preds_dev f64 [B] stays on the device; the report is copied to rep (host)
 * only if rep != NULL (that forces a stream sync). */
int stgn_engine_process_batch_dev(stgn_engine* eng, int32_t B, const int32_t* src_dev,
                                  const int32_t* dst_dev, const double* t_dev,
                                  const float* feat_dev, int64_t m0, int64_t batch_index,
                                  int64_t node_count, double* preds_dev, stgn_report* rep,
                                  void* stream);

/* Exact recompute of `ids` (host int32 list, or NULL = all of 0..node_count-1)
 * with current memory; fills missing neighbour caches from the store first.
 * valid_at_value is written to valid_at. Returns the count in *count. */
int stgn_engine_rebuild(stgn_engine* eng, const int32_t* ids, int64_t n_ids,
                        int64_t node_count, double valid_at_value, int64_t* count,
                        void* stream);

/* Read-only full recompute; final-layer rows into out_dev f32 [node_count][ld_d]. */
int stgn_engine_full_reference(stgn_engine* eng, int64_t node_count, float* out_dev,
                               void* stream);

/* Copy the last batch's direct / affected node lists (unordered) to host
 * buffers of capacity cap; *n_direct / *n_affected receive the sizes. */
int stgn_engine_affected(stgn_engine* eng, int32_t* direct, int32_t* affected, int64_t cap,
                         int64_t* n_direct, int64_t* n_affected, int32_t* change_sizes,
                         void* stream);

/* Copy the last batch's prediction-time final-layer embeddings of the
 * direct nodes (same order as stgn_engine_affected's direct list):
 * host float32 [n_direct][d]. */
int stgn_engine_pred_embeddings(stgn_engine* eng, float* out, int64_t n_direct, void* stream);

/*
 * Operator level: the reference's pipeline_many on flat inputs, float32
 * device buffers in the reference layouts (row-major):
 *   qbase (N,d) offsets (N+1,int64) payload (E,K,d) feat (E,d_e) dt (E,f64)
 *   omega (d_t/2,f64) phi0 (d_t) wq (K,H,q_in,d_k) wk/wv (K,H,k_in,d_k) wo (K,H*d_k,d)
 * Outputs (caller-allocated): out (N,K,d) scores (E,K,H) values (E,K,H,d_k)
 *   maxlog/zsum (N,K,H) qvecs (N,K,H,d_k). scores are in the max-scaled
 * frame; rows with no entries give out = 0, maxlog = -inf, zsum = 0.
 */
int stgn_pipeline_many(const stgn_dims* dims, int64_t N, int64_t E, const float* qbase,
                       const int64_t* offsets, const float* payload, const float* feat,
                       const double* dt, const double* omega, const float* phi0,
                       const float* wq, const float* wk, const float* wv, const float* wo,
                       float* out, float* scores, float* values, float* maxlog, float* zsum,
                       float* qvecs, void* stream);

/* Recompute scope for the following batches (STGN_SCOPE_*); DIRECT needs an
 * infinite window (else STGN_ERR_INVALID). */
int stgn_engine_set_scope(stgn_engine* eng, int scope);

/* State-only fast-forward (test harness, no reference counterpart in the
 * product API; mirrors the oracle's process_batch(compute=False)): while on,
 * batches advance topology, rings, memory and drift but launch no attention
 * recompute, so the layer cache keeps its values. */
int stgn_engine_set_skip_recompute(stgn_engine* eng, int on);

/* Per-stage device timing (CUDA events; disables graph replay while on).
 * stage_times writes up to cap stage durations (ms) of the last batch and
 * returns how many; *launches = kernel launches per batch. */
int stgn_engine_set_profiling(stgn_engine* eng, int on);
int stgn_engine_stage_times(stgn_engine* eng, float* ms, int cap, int64_t* launches);
const char* stgn_stage_name(int i);

/* Engine facts, up to n of: [graph replay active, rebuild block is a
 * device-side conditional graph node, kernel launches per batch, attention
 * tile rows, staged-weight floats, SM count, attention smem bytes,
 * memory-update smem bytes, split-TF32 tensor-core kernel active, its tile
 * rows, bf16x3 128-row kernel active, its smem bytes]. */
int stgn_engine_info(stgn_engine* eng, int64_t* info, int n);

/* Pure full recompute (OracleEngine.full_recompute, S/oracle.py:47-65): every
 * node's K layers into layers_out_dev [node_count][K][ld_d] (device memory); no
 * state is touched. t_now = +inf: the current lists (the store's top-L, cached
 * or not); a finite t_now: each node's L newest store entries with t <= t_now,
 * rebuilt from the store chains and the payload log (needs stgn_state.e_pay). */
int stgn_engine_snapshot(stgn_engine* eng, int64_t node_count, double t_now,
                         float* layers_out_dev, void* stream);

/* Stage-level surface (the reference's unit entry points that process_batch runs
 * fused; csrc/stage.cuh). All pointers are device memory; each call completes
 * before returning.
 *
 * stage_affected replaces IncrementalEngine.detect_affected(pending)
 * (S/engine.py:196-212): the direct endpoints of the P staged edges (src_dev,
 * dst_dev, int32, batch order) and their K-hop closure over the post-insertion
 * truncated lists (staged entries newest first, then the cached list or the
 * store's top-L; S/engine.py:170-194). Writes the set to out_dev[0 ..
 * hop_off[K+1]) in discovery order, hop_off_dev[K+2] (int32) the hop
 * boundaries. stamp: a node-mark value no batch uses (the host takes them
 * above 2^31). Nothing but the marks is written. STGN_ERR_CAPACITY when the
 * set exceeds cap. */
int stgn_engine_stage_affected(stgn_engine* eng, int32_t P, const int32_t* src_dev,
                               const int32_t* dst_dev, uint32_t stamp, int32_t* out_dev,
                               int64_t cap, int32_t* hop_off_dev, void* stream);

/* New neighbour entries of nn distinct nodes, CSR by node, newest first. */
typedef struct {
  const int32_t* nodes;  /* [nn] */
  const int32_t* off;    /* [nn + 1] */
  const int32_t* nbr;    /* [ne] */
  const double* t;       /* [ne] */
  const int64_t* eid;    /* [ne] */
  const float* pay;      /* [ne][K][ld_d] frozen stack of the opposite endpoint */
  const float* feat;     /* [ne][ld_e] */
  const int32_t* put;    /* [nn] 1: cache put with a record; 0: store-list refresh only */
} stgn_stage_entries;

/* Per-node records; node i's expired entries start at off[i] + i * L. */
typedef struct {
  int32_t* hit;      /* [nn] 1 when the node was cached */
  int32_t* exp_n;    /* [nn] */
  int32_t* exp_nbr;  /* [ne + nn L] */
  double* exp_t;
  int64_t* exp_eid;
  int32_t* upd_n;    /* [nn] */
  int32_t* upd_nbr;  /* [nn L] */
} stgn_stage_records;

/* update_neighbor_cache (S/engine.py:216-243) for nn nodes: prepend the new
 * entries, evict beyond L, expire entries older than t_now - window; with put,
 * the node's cache becomes the kept list and its record is written (expired;
 * updated = kept older entries whose neighbour is in direct_dev, sorted, nd).
 * put = 0 moves only the store's top-L list (commit of an uncached node). */
int stgn_engine_stage_nbr_update(stgn_engine* eng, int32_t nn, const stgn_stage_entries* entries,
                                 const int32_t* direct_dev, int32_t nd, double t_now,
                                 const stgn_stage_records* records, void* stream);

/* commit_pending (S/engine_base.py:108-117): the P staged edges enter the
 * append-only store as edge ids m0 .. m0+P-1 (edge log, per-node chains, and
 * the payload log when bound: pay_dev [P][2][K][ld_d], side 0 the src entry's
 * payload = the dst stack). feat_dev [P][ld_e]. Lists are not touched. */
int stgn_engine_stage_commit(stgn_engine* eng, int32_t P, const int32_t* src_dev,
                             const int32_t* dst_dev, const double* t_dev, const float* feat_dev,
                             const float* pay_dev, int64_t m0, void* stream);

/* DySAT streaming inference (paper_2603_21090_b200/dysat.py states the model;
 * the reference reports DySAT results only, and ships no
 * code). All pointers are device memory bound by the caller; row widths padded
 * to ld (a multiple of 4). */
typedef struct {
  int32_t d_in, d, heads_s, heads_t, window, fanout, ld, max_batch;
  int64_t n, snapshot, pos_len, chunk;
  const float* P;        /* [n][ld]  X W_s */
  const float* ss;       /* [n][heads_s]  a_self,h . P_v,h */
  const float* sn;       /* [n][heads_s]  a_nbr,h . P_v,h */
  int32_t* lst_nbr;      /* [n][fanout]  current-snapshot lists (rings, newest at head) */
  int32_t* lst_head;     /* [n] */
  int32_t* lst_cnt;      /* [n] */
  float* hist_k;         /* [n][window][ld]  temporal key rows by snapshot mod window */
  float* hist_v;         /* [n][window][ld] */
  float* emb;            /* [n][ld]  current embeddings */
  int32_t* mark;         /* [n] node stamps */
  int32_t* work;         /* [2 max_batch + 8]: affected list, count at [2 max_batch] */
  float* rows;           /* [max(chunk, 2 max_batch)][ld] structural rows */
  const float* pos;      /* [pos_len][ld] */
  const float *wq, *wk, *wv, *wo;  /* [d][ld] */
  const double* wpred;   /* [2 d] */
  double bpred;
  const uint16_t* wtc;   /* nullable: [4][2 d d] W_q^T, W_k^T, W_v^T, W_o^T as K-major bf16
                            hi | lo blocks (tcgen05 B operands; d = 64 or 128) */
  int64_t tc_min_rows;   /* launches of at least this many rows use the tcgen05 kernel */
} stgn_dysat;

/* One snapshot segment of B edges (device int32 ids, all of snapshot
 * s->snapshot): scores from the pre-batch embeddings into preds_dev, then the
 * endpoints' lists, structural and temporal rows. *n_affected (host, nullable:
 * no synchronisation) = the endpoints' count; the list is s->work[0 .. n). */
int stgn_dysat_batch(const stgn_dysat* s, int32_t B, const int32_t* src_dev,
                     const int32_t* dst_dev, uint32_t stamp, double* preds_dev,
                     int32_t* n_affected, void* stream);
/* Every node at the current snapshot (the full-recompute baseline). */
int stgn_dysat_recompute_all(const stgn_dysat* s, void* stream);
/* Snapshot boundary (the caller has advanced s->snapshot): clear the lists,
 * recompute every node. */
int stgn_dysat_roll(const stgn_dysat* s, void* stream);

/* Node-id-range sharding (multi-GPU, paper_2603_21090_b200/shard.py). The engine
 * keeps and recomputes the frozen payload rows of nodes [lo, hi) only (hi <= lo:
 * every node; ring_pay / ring_tb / ring_feat may then be bound with a base
 * offset so that only rows lo..hi-1 are backed); the topology is replicated.
 * A sharded batch runs in two phases: phase 1 (inputs staged, everything up to
 * the recompute), the exchange of the direct nodes' prediction rows
 * (stgn_engine_dpred_export on every rank, stgn_engine_dpred_import of the
 * others' rows), then phase 2 (scores, memory commit, drift, rebuild). */
int stgn_engine_set_ownership(stgn_engine* eng, int32_t lo, int32_t hi);
int stgn_engine_batch_phase(stgn_engine* eng, int32_t phase, int32_t B, const int32_t* src_dev,
                            const int32_t* dst_dev, const double* t_dev, const float* feat_dev,
                            int64_t m0, int64_t batch_index, int64_t node_count,
                            double* preds_dev, stgn_report* rep, void* stream);
int stgn_engine_dpred_export(stgn_engine* eng, int32_t* nodes_dev, float* rows_dev,
                             int64_t* count, void* stream);
int stgn_engine_dpred_import(stgn_engine* eng, const int32_t* nodes_dev, const float* rows_dev,
                             int64_t n, void* stream);

/* Per-batch result block (counters of the last enqueued batch), for pipelined
 * callers that do not block on a report: stgn_engine_result_copy copies it
 * (stream-ordered) to device memory (to_device != 0) or pinned host memory;
 * stgn_report_from_result turns a host copy into a stgn_report. */
int64_t stgn_batch_result_bytes(void);
int stgn_engine_result_copy(stgn_engine* eng, void* dst, int32_t to_device, void* stream);
int stgn_report_from_result(const void* res, stgn_report* rep);

/* Delta mode, K = 1: the last batch's error-bound records (DeltaEvent,
 * S/engine.py:20-29, 333-353), copied to host arrays of capacity max (sorted
 * by node id); emb receives each record's embedding (d floats per record).
 * *mvn = max_value_norm_seen. Returns the record count (>= 0) or an error. */
int stgn_engine_delta_events(stgn_engine* eng, int64_t max, int32_t* node, double* bound,
                             int32_t* dn, int32_t* nv, double* max_v, double* z_dev, float* emb,
                             double* mvn);

/* Tensor-core self-test: D[N][F] = X[N][K] W[K][F] (device f32 buffers)
 * through the split-TF32 tcgen05 path (F <= 128, N <= 256). mode 0 = the
 * GEMM; bits: 1 pre-fill TMEM with a sentinel, 2 skip the MMA, 4 accumulate. */
int stgn_debug_tc_gemm(int F, int N, int K, const float* W, const float* X, float* D, int mode,
                       void* stream);

/*
 * Native synthetic stream generator: the reference's generate_stream
 * (S/streamio.py:86-145) for d_e = 0, edge for edge. rng_state[6] is the
 * numpy PCG64 bit-generator state of default_rng(seed) as
 * {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger}; the state after
 * the last draw goes to rng_state_out (may be NULL). Host buffers src, dst
 * (int64) and t (float64) of length m.
 */
int stgn_generate_stream(const uint64_t* rng_state, int64_t n, int64_t m, int32_t preferential,
                         double burstiness, int64_t* src, int64_t* dst, double* t,
                         uint64_t* rng_state_out);

/* Debug: phase timestamps of CTA 0 of the bf16x3 recompute kernel, returns the
 * count copied (0 unless the library was built with -DA4_PROF); resets. */
int stgn_debug_a4_prof(uint64_t* out, int cap);
/* Per-CTA start/end ns, ring entries, tiles of the recompute launches since the
   last read (-DA4_PROF builds only; 0 otherwise). Debug, no reference analogue. */
int stgn_debug_a4_cta(uint64_t* out, int cap);

/*
 * Native reader of the edge-stream CSV format (S/streamio.py:15-79). Returns
 * the edge count in *m_out and d_e in *d_e_out; with cap >= *m_out and
 * buffers (src, dst int64; t float64; feat float64 [m][d_e]) it also fills
 * them, stably re-sorted by t when sort != 0. Any line it cannot parse as
 * plain decimal fields, a negative id, or a decreasing timestamp without sort
 * returns STGN_ERR_INVALID (*bad_line = the line, or -1): the Python shim then
 * re-reads the file with the reference's parser for the exact error.
 */
int stgn_read_stream(const char* path, int32_t sort, int64_t cap, int64_t* m_out, int64_t* d_e_out,
                     int64_t* src, int64_t* dst, double* t, double* feat, int64_t* bad_line);

/* Library version string and the sm architecture it was built for. */
const char* stgn_version(void);

/* Description of the last CUDA failure in this thread (file:line: message). */
const char* stgn_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* STGN_H */
