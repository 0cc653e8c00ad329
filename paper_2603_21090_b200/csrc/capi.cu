// C ABI driver: engine handle, per-batch launch sequence (captured once
// as a CUDA graph), rebuild / full_reference entry points and the
// operator-level pipeline_many. See include/stgn.h for the contract.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>

#include <algorithm>
#include <utility>
#include <mutex>
#include <vector>

#include "batch.cuh"
#include "attn3.cuh"
#include "attn4.cuh"
#include "mem4.cuh"
#include "delta.cuh"
#include "snapshot.cuh"
#include "stage.cuh"
#include "dysat.cuh"

#ifndef STGN_DRIFT_FORK
#define STGN_DRIFT_FORK 1  // drift estimators + decision on a branch beside the recompute
#endif
#ifndef STGN_REC32
#define STGN_REC32 0  // change records: k_records_w32 (32 nodes per warp) instead of k_records_warp
#endif
#ifndef STGN_INGEST1
#define STGN_INGEST1 0  // batches of <= INGEST1_MAX_B edges: the five ingest kernels as one block
#endif
#ifndef STGN_LATE_RECORDS
#define STGN_LATE_RECORDS 0
#endif

#ifndef STGN_VERSION
#define STGN_VERSION "stgn 0.1.0 sm_100a"
#endif

// ---------------------------------------------------------------------------
// attention launch (template dispatch on the per-lane register widths)
// ---------------------------------------------------------------------------
typedef void (*attn_fn_t)(Geo, AttnWeights, RingSrc, FlatSrc, int);
typedef void (*attn2_fn_t)(Geo, EngW, RingSrc, int, int);
typedef void (*attn3_fn_t)(Geo, TcW, RingSrc, int);
typedef void (*attn4_fn_t)(Geo, A4W, RingSrc);

template <bool FLAT>
static attn_fn_t pick_attn(const Geo& g) {
  const int a = (int)cdiv(g.k_in, 32);
  const bool h4 = g.H > 2;
#define PICK(MA)                                                             \
  if (a <= MA) return h4 ? (attn_fn_t)attn_kernel<MA, 4, FLAT> : (attn_fn_t)attn_kernel<MA, 2, FLAT>;
  PICK(2)
  PICK(4)
  PICK(8)
  PICK(12)
  PICK(16)
#undef PICK
  return nullptr;
}

struct AttnLaunch {
  attn_fn_t fn = nullptr;
  int T = 0;
  size_t smem = 0;
  int grid = 0;
};

static int plan_attn(const Geo& g, bool flat, int num_sms, AttnLaunch* out) {
  attn_fn_t fn = flat ? pick_attn<true>(g) : pick_attn<false>(g);
  if (!fn) return STGN_ERR_INVALID;
  int T = 0;
  size_t smem = 0;
  for (int cand : {32, 16, 8, 4}) {
    size_t b = (size_t)attn_smem_floats(g, cand, flat) * sizeof(float);
    if (b <= 200 * 1024) {
      T = cand;
      smem = b;
      break;
    }
  }
  if (!T) return STGN_ERR_INVALID;
  CUDA_TRY(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, STGN_THREADS, smem));
  if (per_sm < 1) per_sm = 1;
  out->fn = fn;
  out->T = T;
  out->smem = smem;
  out->grid = per_sm * num_sms;
  return STGN_OK;
}

// ---------------------------------------------------------------------------
// engine handle
// ---------------------------------------------------------------------------
struct stgn_engine {
  stgn_dims dims;
  stgn_config cfg;
  Geo g;
  AttnWeights aw;
  stgn_weights w;
  bool have_w = false;
  stgn_state st;
  bool bound = false;
  StateView sv;
  Scratch sc;
  int num_sms = 148;
  AttnLaunch attn;            // attn_kernel (reserved for the flat operator path)
  attn2_fn_t attn2 = nullptr; // engine recompute kernel
  size_t attn2_smem = 0;
  int attn2_tmax = 0, attn2_wsm = 0;
  attn3_fn_t attn3 = nullptr;  // tcgen05 recompute kernel (when the TMEM plan fits)
  size_t attn3_smem = 0;
  int attn3_tmax = 0;
  TcW tcw;
  bool tc_ok = false, use_tc = false;
  attn4_fn_t attn4 = nullptr;  // bf16x3 tcgen05 recompute kernel, 128-row tiles (H = 2)
  size_t attn4_smem = 0;
  A4W a4w;
  bool a4_ok = false, use_a4 = false;
  M4W m4w;                      // bf16x3 tcgen05 memory update (when the plan fits)
  size_t mem4_smem = 0;
  bool m4_ok = false, use_m4 = false;
  bool ds_ok = false;           // k_delta_state's shared-memory plan fits (delta mode)
  bool skip_recompute = false;  // state-only fast-forward (tests): no attention launches
  EngW ew;
  size_t mem_smem = 0;
  int mem_wsm = 0;
  // pinned staging mirror of [hdr .. in_feat] and the result area
  uint8_t* h_in = nullptr;
  int64_t in_bytes = 0;
  BatchRes* h_res = nullptr;
  double* h_preds = nullptr;
  uint32_t stamp = 0;
  cudaGraphExec_t graph = nullptr;
  bool graph_ok = true;   // capture allowed
  bool profiling = false;
  bool fork_always = true;    // graph branches also when no conditional node is captured
  cudaEvent_t ev[16] = {};
  int64_t launches = 0;
  cudaStream_t aux = nullptr;   // captures the conditional rebuild body
  bool capture_failed = false;
  bool cond_used = false;       // rebuild block is a device-side conditional graph node
  cudaStream_t work = nullptr;  // the batch sequence / graph runs here
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  // graph branches: the memory update runs beside the BFS/records, the drift
  // policy beside the recompute (captured fork/join, graph mode only)
  cudaStream_t side[2] = {nullptr, nullptr};
  cudaEvent_t ev_fork[2] = {nullptr, nullptr}, ev_join[2] = {nullptr, nullptr};
};

static void drop_graph(stgn_engine* e) {
  if (e->graph) {
    cudaGraphExecDestroy(e->graph);
    e->graph = nullptr;
  }
}

// operator = true: the flat pipeline_many kernel's register budget (attn.cuh:
// H <= 4, k_in <= 512). The engine takes any widths its shared-memory plans fit
// (the width-generic attn2 walk covers what the register-resident walks do not).
static int validate_dims(const stgn_dims* d, const stgn_config* c, bool op = false) {
  if (!d || !c) return STGN_ERR_INVALID;
  if (d->d_s <= 0 || d->d_t <= 0 || d->d_m <= 0 || d->d_k <= 0 || d->heads <= 0 ||
      d->layers <= 0 || d->d_e < 0 || d->d_x < 0 || (d->d_t & 1))
    return STGN_ERR_INVALID;
  if (d->layers > STGN_MAX_LAYERS || d->heads > (op ? 4 : 64)) return STGN_ERR_INVALID;
  if (c->fanout < 1 || c->max_batch < 1) return STGN_ERR_INVALID;
  const int k_in = d->d_s + d->d_x + d->d_e + d->d_t;
  if (k_in > (op ? 16 * 32 : 8192)) return STGN_ERR_INVALID;
  return STGN_OK;
}

static thread_local char g_err[512] = "";

void stgn_set_error(const char* file, int line, cudaError_t e) {
  snprintf(g_err, sizeof(g_err), "%s:%d: %s (%s)", file, line, cudaGetErrorString(e),
           cudaGetErrorName(e));
}

extern "C" {

const char* stgn_version(void) { return STGN_VERSION; }

const char* stgn_last_error(void) { return g_err; }

int64_t stgn_scratch_bytes(const stgn_dims* dims, const stgn_config* cfg, int64_t cap_nodes) {
  if (validate_dims(dims, cfg) != STGN_OK) return -1;
  Geo g = make_geo(*dims, cfg->fanout);
  return scratch_layout(g, cfg->max_batch, cap_nodes, nullptr, nullptr);
}

int stgn_engine_create(const stgn_dims* dims, const stgn_config* cfg, stgn_engine** out) {
  if (!out) return STGN_ERR_INVALID;
  int rc = validate_dims(dims, cfg);
  if (rc) return rc;
  stgn_engine* e = new (std::nothrow) stgn_engine();
  if (!e) return STGN_ERR_INVALID;
  e->dims = *dims;
  e->cfg = *cfg;
  if (std::isfinite(cfg->window) && cfg->scope == STGN_SCOPE_DIRECT)
    e->cfg.scope = STGN_SCOPE_AFFECTED;  // A\D can change
  e->g = make_geo(*dims, cfg->fanout);
  int dev = 0;
  cudaError_t ce = cudaGetDevice(&dev);
  if (ce == cudaSuccess) ce = cudaDeviceGetAttribute(&e->num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (ce != cudaSuccess) {
    stgn_set_error(__FILE__, __LINE__, ce);
    delete e;
    return STGN_ERR_CUDA;
  }
  // register-resident walk within its budget, else the width-generic walk
  const bool a2_gen = e->g.d > 128 || e->g.d_e > 192 || e->g.half > 64 || e->g.H > 4;
  e->attn2 = a2_gen ? attn2_kernel<0, 1, 1>
                    : e->g.d_e > 0 ? (e->g.H > 2 ? attn2_kernel<6, 4> : attn2_kernel<6, 2>)
                                   : (e->g.H > 2 ? attn2_kernel<0, 4> : attn2_kernel<0, 2>);
  {  // tile rows vs staged-weight space within ~220 KB of shared memory
    const int64_t budget = 220 * 1024 / 4;
    // the generic walk keeps one k_in row per warp in the weight stage
    const int64_t gen_ws = a2_gen ? A2_WARPS * round_up(e->g.k_in, 4) : 0;
    const int64_t row = attn2_row_floats(e->g),
                  full = std::max<int64_t>(attn2_wsm_full(e->g), gen_ws);
    int64_t tmax = (budget - full) / row / 4 * 4;
    int64_t wsm;
    if (tmax >= 8) {
      if (tmax > A2_TMAX) tmax = A2_TMAX;
      wsm = budget - tmax * row;
    } else {  // stage weights in chunks
      wsm = std::max<int64_t>(16 * 1024, gen_ws);
      tmax = (budget - wsm) / row / 4 * 4;
      if (tmax > A2_TMAX) tmax = A2_TMAX;
      wsm = budget - tmax * row;
    }
    const int64_t ldmax = round_up(e->g.k_in > e->g.HD ? e->g.k_in : e->g.HD, 4);
    const int64_t need = std::max<int64_t>((int64_t)e->g.H * ldmax, gen_ws);
    if (tmax < 4 || wsm < need) {
      delete e;
      return STGN_ERR_INVALID;
    }
    e->attn2_tmax = (int)tmax;
    e->attn2_wsm = (int)(wsm / 4 * 4);
    e->attn2_smem = (size_t)(tmax * row + e->attn2_wsm) * sizeof(float);
  }
  memset(&e->tcw, 0, sizeof(e->tcw));
  if (tc_plan(e->g, &e->tcw)) {  // tcgen05 path: q~/ubar rows + c rows + one staged block
    const int64_t budget = 220 * 1024 / 4;
    const int64_t wbuf = attn3_wbuf_floats(e->g, e->tcw) + 32;
    int64_t tmax = (budget - wbuf) / attn3_row_floats(e->g);
    if (tmax > A2_TMAX) tmax = A2_TMAX;
    if (tmax >= 8) {
      e->attn3_tmax = (int)tmax;
      e->attn3_smem = (size_t)(tmax * attn3_row_floats(e->g) + wbuf) * sizeof(float);
      e->attn3 = e->g.d_e > 0 ? (e->g.H > 2 ? attn3_kernel<6, 4> : attn3_kernel<6, 2>)
                              : (e->g.H > 2 ? attn3_kernel<0, 4> : attn3_kernel<0, 2>);
      e->tc_ok = cudaFuncSetAttribute((const void*)e->attn3,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)e->attn3_smem) == cudaSuccess;
      cudaGetLastError();
    }
  }
  memset(&e->a4w, 0, sizeof(e->a4w));
  if (a4_plan(e->g, &e->a4w)) {
    e->attn4_smem = attn4_smem_bytes(e->a4w);
    e->attn4 = e->g.d_e > 0 ? attn4_kernel<1> : attn4_kernel<0>;
    e->a4_ok = e->attn4_smem <= 227 * 1024 &&
               cudaFuncSetAttribute((const void*)e->attn4,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)e->attn4_smem) == cudaSuccess;
    cudaGetLastError();
  }
  memset(&e->m4w, 0, sizeof(e->m4w));
  if (m4_plan(e->g, &e->m4w)) {
    e->mem4_smem = mem4_smem_bytes(e->m4w);
    e->m4_ok = cudaFuncSetAttribute((const void*)mem4_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)e->mem4_smem) == cudaSuccess;
    cudaGetLastError();
  }
  ce = cudaFuncSetAttribute((const void*)e->attn2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)e->attn2_smem);
  if (ce != cudaSuccess) {
    stgn_set_error(__FILE__, __LINE__, ce);
    delete e;
    return STGN_ERR_CUDA;
  }
  {  // k_memory: activations + staged weights within ~200 KB
    const int64_t budget = 200 * 1024 / 4;
    const int64_t ld_dm = round_up(e->g.d_m, 4), ld_ds = round_up(e->g.d_s, 4);
    const int64_t act = GRU_T * (2 * e->g.msg_in + ld_dm + 2 * e->g.d_s + 6 * ld_ds);
    e->mem_wsm = (int)((budget - act) / 4 * 4);
    if (e->mem_wsm < 3 * ld_ds || e->mem_wsm < ld_dm) {
      delete e;
      return STGN_ERR_INVALID;
    }
    e->mem_smem = (size_t)(act + e->mem_wsm) * sizeof(float);
  }
  e->ds_ok = delta_state_smem(e->g) <= 227 * 1024 &&
             cudaFuncSetAttribute((const void*)k_delta_state,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)delta_state_smem(e->g)) == cudaSuccess;
  cudaGetLastError();
  if (e->cfg.scope == STGN_SCOPE_DELTA && e->g.K == 1 && (e->g.H > 4 || !e->ds_ok)) {
    delete e;
    return STGN_ERR_INVALID;
  }
  ce = cudaFuncSetAttribute((const void*)k_memory, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)e->mem_smem);
  if (ce != cudaSuccess) {
    stgn_set_error(__FILE__, __LINE__, ce);
    delete e;
    return STGN_ERR_CUDA;
  }
  Scratch tmp;
  uint8_t* fake = reinterpret_cast<uint8_t*>((uintptr_t)4096);  // offsets only
  scratch_layout(e->g, cfg->max_batch, 1, &tmp, fake);
  e->in_bytes = (int64_t)((uint8_t*)(tmp.in_feat + (int64_t)cfg->max_batch * e->g.ld_e) - fake);
  ce = cudaMallocHost((void**)&e->h_in, e->in_bytes);
  if (ce == cudaSuccess) ce = cudaMallocHost((void**)&e->h_res, sizeof(BatchRes));
  if (ce == cudaSuccess) ce = cudaMallocHost((void**)&e->h_preds, sizeof(double) * cfg->max_batch);
  if (ce != cudaSuccess) {
    stgn_set_error(__FILE__, __LINE__, ce);
    stgn_engine_destroy(e);
    return STGN_ERR_CUDA;
  }
  memset(e->h_in, 0, e->in_bytes);
  ce = cudaStreamCreateWithFlags(&e->aux, cudaStreamNonBlocking);
  if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&e->work, cudaStreamNonBlocking);
  if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&e->ev_in, cudaEventDisableTiming);
  if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&e->ev_out, cudaEventDisableTiming);
  for (int i = 0; i < 2 && ce == cudaSuccess; ++i) {
    ce = cudaStreamCreateWithFlags(&e->side[i], cudaStreamNonBlocking);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&e->ev_fork[i], cudaEventDisableTiming);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&e->ev_join[i], cudaEventDisableTiming);
  }
  if (ce != cudaSuccess) {
    stgn_set_error(__FILE__, __LINE__, ce);
    stgn_engine_destroy(e);
    return STGN_ERR_CUDA;
  }
  *out = e;
  return STGN_OK;
}

int stgn_engine_destroy(stgn_engine* e) {
  if (!e) return STGN_OK;
  drop_graph(e);
  if (e->aux) cudaStreamDestroy(e->aux);
  if (e->work) cudaStreamDestroy(e->work);
  if (e->ev_in) cudaEventDestroy(e->ev_in);
  if (e->ev_out) cudaEventDestroy(e->ev_out);
  for (int i = 0; i < 2; ++i) {
    if (e->side[i]) cudaStreamDestroy(e->side[i]);
    if (e->ev_fork[i]) cudaEventDestroy(e->ev_fork[i]);
    if (e->ev_join[i]) cudaEventDestroy(e->ev_join[i]);
  }
  for (auto& ev : e->ev)
    if (ev) cudaEventDestroy(ev);
  if (e->h_in) cudaFreeHost(e->h_in);
  if (e->h_res) cudaFreeHost(e->h_res);
  if (e->h_preds) cudaFreeHost(e->h_preds);
  delete e;
  return STGN_OK;
}

int stgn_engine_set_weights(stgn_engine* e, const stgn_weights* w) {
  if (!e || !w) return STGN_ERR_INVALID;
  e->w = *w;
  e->ew.wq = w->wq;
  e->ew.bq = w->bq;
  e->ew.wkt = w->wkt;
  e->ew.wv = w->wv;
  e->ew.wo = w->wo;
  e->ew.omega = w->omega;
  e->ew.ld_hd = (int)round_up(e->g.HD, 4);
  e->ew.ld_kin = (int)round_up(e->g.k_in, 4);
  e->ew.ld_dk = (int)round_up(e->g.d_k, 4);
  e->ew.ld_d = (int)round_up(e->g.d, 4);
  e->use_tc = e->tc_ok && w->tcq && w->tck && w->tcv && w->tco;
  if (e->use_tc) {
    e->tcw.wq = w->tcq;
    e->tcw.wk = w->tck;
    e->tcw.wv = w->tcv;
    e->tcw.wo = w->tco;
    e->tcw.bq = w->bq;
    e->tcw.omega = w->omega;
  }
  e->use_a4 = e->a4_ok && w->t4q && w->t4k && w->t4v && w->t4o && w->t4bq && (!A4_VOF || w->t4p);
  if (e->use_a4) {
    e->a4w.wq = w->t4q;
    e->a4w.wk = w->t4k;
    e->a4w.wv = w->t4v;
    e->a4w.wo = w->t4o;
    e->a4w.bq = w->t4bq;
    e->a4w.wp = w->t4p;
    e->a4w.omega = w->omega;
  }
#ifdef STGN_NO_MEM4  // experiments: the FFMA memory update
  e->use_m4 = false;
#else
  {
    const char* env = getenv("STGN_MEM4");  // "0": the FFMA memory update
    e->use_m4 = e->m4_ok && w->t4mem && !(env && env[0] == '0');
  }
#endif
  if (e->use_m4) e->m4w.wblk = w->t4mem;
  e->aw.wq = w->wq;
  e->aw.wkt = w->wkt;
  e->aw.wv = w->wv;
  e->aw.wo = w->wo;
  e->aw.omega = w->omega;
  e->aw.phi0 = w->phi0;
  e->have_w = true;
  drop_graph(e);
  return STGN_OK;
}

int stgn_engine_bind(stgn_engine* e, const stgn_state* s) {
  if (!e || !s || !s->scratch || !s->ctl) return STGN_ERR_INVALID;
  e->st = *s;
  StateView& v = e->sv;
  v.mem = s->mem; v.last = s->last; v.version = s->version; v.h = s->h; v.valid = s->valid;
  v.valid_at = s->valid_at; v.ring_cnt = s->ring_cnt; v.ring_head = s->ring_head;
  v.ring_ccnt = s->ring_ccnt; v.ring_nbr = s->ring_nbr; v.ring_eid = s->ring_eid;
  v.ring_t = s->ring_t; v.ring_pay = s->ring_pay; v.ring_feat = s->ring_feat;
  v.ring_tb = s->ring_tb;
  v.amark = s->amark; v.dmark = s->dmark; v.nodecnt = s->nodecnt; v.nodeadj = s->nodeadj;
  v.nodefill = s->nodefill; v.nodeoff = s->nodeoff; v.drift_acc = s->drift_acc;
  v.drift_touched = s->drift_touched; v.cum_mark = s->cum_mark; v.cum_list = s->cum_list;
  v.cum_pos = s->cum_pos; v.attn_ver = s->attn_ver; v.attn_tref = s->attn_tref;
  v.attn_logz = s->attn_logz; v.ev_node = s->ev_node; v.ev_dpos = s->ev_dpos; v.ev_dn = s->ev_dn;
  v.ev_nv = s->ev_nv; v.ev_bound = s->ev_bound; v.ev_maxv = s->ev_maxv; v.ev_zdev = s->ev_zdev;
  v.ev_cap = s->attn_logz ? s->ev_cap : 0;
  v.e_pay = s->e_pay;
  v.e_src = s->e_src; v.e_dst = s->e_dst; v.e_t = s->e_t; v.e_feat = s->e_feat;
  v.e_prev = s->e_prev; v.adj_head = s->adj_head; v.adj_deg = s->adj_deg;
  v.gpow = s->gpow; v.gpow_len = s->gpow_len; v.ctl = s->ctl;
  scratch_layout(e->g, e->cfg.max_batch, s->cap_nodes, &e->sc, s->scratch);
  e->bound = true;
  drop_graph(e);
  return STGN_OK;
}

}  // extern "C"

// Launch on the batch chain: with STGN_PDL, programmatic stream serialization
// (the kernel waits for its predecessor in PDL_WAIT instead of at launch).
template <typename... KArgs, typename... Args>
static void chain_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                         cudaStream_t st, Args&&... args) {
#ifdef STGN_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
#else
  kern<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
#endif
}

static RingSrc ring_src(const stgn_engine* e) {
  RingSrc r;
  memset(&r, 0, sizeof(r));
  const StateView& v = e->sv;
  r.mem = v.mem; r.h = v.h; r.valid = v.valid; r.valid_at = v.valid_at;
  r.ring_cnt = v.ring_cnt; r.ring_head = v.ring_head; r.ring_ccnt = v.ring_ccnt;
  r.ring_t = v.ring_t; r.ring_pay = v.ring_pay; r.ring_feat = v.ring_feat;
  r.ring_tb = v.ring_tb;
  r.own_lo = e->g.own_lo;  // sharded engine: rows of other ranks' nodes are skipped
  r.own_hi = e->g.own_hi;
  return r;
}

static void launch_attn(const stgn_engine* e, const RingSrc& rs, cudaStream_t st,
                        bool chain = false) {
  if (e->skip_recompute) return;
  if (e->use_a4 && chain)
    chain_launch(e->attn4, e->num_sms, A4_THREADS, e->attn4_smem, st, e->g, e->a4w, rs);
  else if (e->use_a4)
    e->attn4<<<e->num_sms, A4_THREADS, e->attn4_smem, st>>>(e->g, e->a4w, rs);
  else if (e->use_tc)
    e->attn3<<<e->num_sms, A3_THREADS, e->attn3_smem, st>>>(e->g, e->tcw, rs, e->attn3_tmax);
  else
    e->attn2<<<e->num_sms, A2_THREADS, e->attn2_smem, st>>>(e->g, e->ew, rs, e->attn2_tmax,
                                                            e->attn2_wsm);
}

static const char* kStageNames[] = {"group+ring", "affected_bfs", "change_records",
                                    "memory_update", "recompute", "predict+commit", "drift",
                                    "rebuild", "cleanup"};
#define NSTAGES 9


static void launch_memory(const stgn_engine* e, cudaStream_t st) {
  const Geo& g = e->g;
  const int64_t R = 2 * (int64_t)e->cfg.max_batch;
  if (e->use_m4) {
    mem4_kernel<<<(int)std::min<int64_t>(cdiv(R, 128), e->num_sms), M4_THREADS, e->mem4_smem, st>>>(
        g, e->sv, e->sc, e->m4w, e->w.bmsg, e->w.omega, e->w.bgru, e->cfg.aggregator);
    return;
  }
  k_memory<<<(int)std::min<int64_t>(cdiv(R, GRU_T), e->num_sms), MG_THREADS, e->mem_smem, st>>>(
      g, e->sv, e->sc, e->w.wmsg, e->w.bmsg, e->w.omega, e->w.wgru, e->w.ugru, e->w.bgru,
      e->cfg.aggregator, (int)round_up(g.d_m, 4), (int)round_up(g.d_s, 4), e->mem_wsm);
}

static void launch_drift(const stgn_engine* e, cudaStream_t st, cudaGraphConditionalHandle cond) {
  k_drift_record<<<4 * e->num_sms, 256, 0, st>>>(e->sv, e->sc);
  k_drift_decide<<<4 * e->num_sms, 256, 0, st>>>(e->sv, e->sc, e->cfg.rebuild,
                                                 e->cfg.rebuild_interval, e->cfg.delta_max,
                                                 e->cfg.alpha, cond);
}

// The whole per-batch sequence; every size is read on the device. With
// profiling on, an event is recorded after every stage (no graph).
// part 0: the whole batch. Sharded engines (shard.py) run it eagerly in two
// parts around the exchange of the direct nodes' prediction rows: part 1 up to
// and including the recompute, part 2 from the scores on (no graph, no fork).
static void enqueue_batch(stgn_engine* e, cudaStream_t st, cudaGraphConditionalHandle cond,
                          int part = 0) {
  const Geo& g = e->g;
  const StateView& v = e->sv;
  const Scratch& s = e->sc;
  const int64_t R = 2 * (int64_t)e->cfg.max_batch;
  const int T = 256;
  const int g_rec = (int)std::min<int64_t>(cdiv(R, T), 4 * e->num_sms);
  const int g_wide = 4 * e->num_sms;
  const int g_warp = (int)std::min<int64_t>(cdiv(R * 32, T), 8 * e->num_sms);
  int n = 0;  // kernel launches
  int stage = 0;
  auto mark = [&]() {
    if (e->profiling && part == 0) cudaEventRecord(e->ev[stage], st);
    ++stage;
  };
  mark();
  cudaStream_t dst_ = st;  // drift branch (graph mode)
  // Change records: with an infinite window and exact scope the recompute does not
  // need them (every list is the store's top-L: k_dupdate sets the direct nodes'
  // cached length and the recompute reads ring_cnt for uncached nodes), so they move
  // to the drift branch, whose estimators are their only consumer.
  const bool late_records = STGN_LATE_RECORDS && !std::isfinite(e->cfg.window) &&
                            e->cfg.scope != STGN_SCOPE_DELTA;
  auto launch_records = [&](cudaStream_t rst, bool chain) {
    if (STGN_REC32 && g.L <= 32) {
      const int gw = 8 * e->num_sms;
      if (chain)
        chain_launch(k_records_w32, gw, T, 0, rst, g, v, s, std::isfinite(e->cfg.window) ? 1 : 0);
      else
        k_records_w32<<<gw, T, 0, rst>>>(g, v, s, std::isfinite(e->cfg.window) ? 1 : 0);
    } else if (g.L <= 32) {
      if (chain)
        chain_launch(k_records_warp, 8 * e->num_sms, T, 0, rst, g, v, s, std::isfinite(e->cfg.window) ? 1 : 0);
      else
        k_records_warp<<<8 * e->num_sms, T, 0, rst>>>(g, v, s, std::isfinite(e->cfg.window) ? 1 : 0);
    } else {
      k_records<<<g_wide, T, 0, rst>>>(g, v, s, std::isfinite(e->cfg.window) ? 1 : 0);
    }
    n += 1;
  };
  if (part != 2) {
  if (e->cfg.scope == STGN_SCOPE_DELTA && g.K == 1 && v.attn_logz)
    cudaMemsetAsync(&v.ctl->reserved[0], 0, sizeof(int64_t), st);  // this batch's bound records
  // ingest: direct set, per-node record order, ring insert with payload freeze, store append
  if (STGN_INGEST1 && e->cfg.max_batch <= INGEST1_MAX_B) {
    chain_launch(k_ingest1, 1, 1024, 0, st, g, v, s, e->cfg.window);
    n -= 4;
  } else {
    chain_launch(k_begin, 1, 32, 0, st, s, e->cfg.window);
    chain_launch(k_claim, g_rec, T, 0, st, g, v, s);
    chain_launch(k_scan, 1, 1024, 0, st, g, v, s);
    chain_launch(k_place, g_rec, T, 0, st, v, s);
    chain_launch(k_rank, g_rec, T, 0, st, v, s);
  }
  // Branch 0 (graph mode): the memory update needs only the grouped records
  // (rec_s, doff) and pre-batch memory and writes scratch only, so it runs
  // beside the ring insertion, the BFS and the change records.
  const bool fork = cond != 0 || e->fork_always;
  cudaStream_t mst = st;
  if (fork && !e->profiling) {
    cudaEventRecord(e->ev_fork[0], st);
    cudaStreamWaitEvent(e->side[0], e->ev_fork[0], 0);
    mst = e->side[0];
    launch_memory(e, mst);
    n += 1;
    cudaEventRecord(e->ev_join[0], mst);
  }
  chain_launch(k_ring, g_warp, T, 0, st, g, v, s, e->w.omega);
  chain_launch(k_dupdate, g_rec, T, 0, st, g, v, s);
  n += 7;
  mark();
  for (int hop = 1; hop <= g.K; ++hop) {
    chain_launch(k_hop, g_wide, T, 0, st, g, v, s, hop);
    if (STGN_HOP_TICKET) {
      n += 1;
    } else {
      chain_launch(k_hop_fin, 1, 32, 0, st, s, hop);
      n += 2;
    }
  }
  mark();
  if (!late_records) launch_records(st, true);
  if (e->cfg.scope == STGN_SCOPE_DELTA) {
    chain_launch(k_delta_classify, g_rec, T, 0, st, g, v, s);
    chain_launch(k_delta_fin, 1, 32, 0, st, s);
    n += 2;
  }
  mark();
  // stage 5 (memory update of V_direct) into mem_new; commits after the recompute
  if (mst == st) {
    launch_memory(e, st);
    n += 1;
  } else {
    cudaStreamWaitEvent(st, e->ev_join[0], 0);
  }
  mark();
  // stages 2-4 and the post-commit refresh in one launch: rows = A (or V_direct)
  // with pre-batch memory, then V_direct with post-batch memory
  // Branch 1 (graph mode): the drift estimators and the rebuild decision read
  // the change records only, so they overlap the recompute; joined before the
  // (conditional) rebuild block.
  if (fork && !e->profiling && STGN_DRIFT_FORK) {
    cudaEventRecord(e->ev_fork[1], st);
    cudaStreamWaitEvent(e->side[1], e->ev_fork[1], 0);
    dst_ = e->side[1];
    if (late_records) launch_records(dst_, false);
    launch_drift(e, dst_, cond);
    n += 2;
    cudaEventRecord(e->ev_join[1], dst_);
  }
  RingSrc rs = ring_src(e);
  rs.list = s.alist;
  rs.fused = 1;
  if (e->cfg.scope == STGN_SCOPE_DELTA) {
    rs.list = s.clist;
    rs.pre_n = &s.res->nC;
  } else {
    rs.pre_n = e->cfg.scope == STGN_SCOPE_DIRECT ? &s.res->nD : &s.res->nA;
  }
  rs.post_n = &s.res->nD;
  if (late_records) rs.use_store = 1;  // uncached lists are the store's top-L (records run later)
  rs.mem_post = s.mem_new;
  rs.valid_at_ptr = &s.hdr->t_batch;
  rs.write_valid = 1;
  rs.dpred = s.dpred;
  rs.e_count = &s.res->E_A;
  rs.e_count_post = &s.res->E_D;
  launch_attn(e, rs, st, true);
  n += 1;
  const bool dstate = e->cfg.scope == STGN_SCOPE_DELTA && g.K == 1 && v.attn_logz;
  if (dstate) {  // attention-state statistics + bound records, before the memory commit
    k_delta_state<<<4 * e->num_sms, DS_THREADS, delta_state_smem(g), st>>>(g, v, s, e->ew, nullptr,
                                                                          nullptr, 0, 0);
    n += 1;
  }
  if (e->cfg.scope == STGN_SCOPE_DIRECT) {
    k_mark_valid<<<g_wide, T, 0, st>>>(v, s);
    n += 1;
  }
  mark();
  }  // part 1
  if (part == 1) {
    e->launches = n;
    return;
  }
  chain_launch(k_predict_commit, g_warp, T, 0, st, g, v, s, e->w.wpred, e->w.bpred);
  n += 1;
  mark();
  // drift + rebuild policy
  if (dst_ == st) {
    if (late_records) launch_records(st, false);
    launch_drift(e, st, cond);
    n += 2;
  } else {
    cudaStreamWaitEvent(st, e->ev_join[1], 0);
  }
  mark();
  if (e->cfg.rebuild != STGN_REBUILD_NEVER) {
    const int stamp = e->cfg.scope == STGN_SCOPE_DELTA && g.K == 1;
    // Inside a captured graph the rebuild block is the body of a conditional
    // IF node whose flag k_drift_decide sets on the device; eager launches
    // (profiling) run it unconditionally (each kernel is a no-op unless chosen).
    cudaStream_t rs = st;
    bool body = false;
    if (cond) {
      cudaStreamCaptureStatus cs;
      cudaGraph_t gcap = nullptr;
      const cudaGraphNode_t* deps = nullptr;
      size_t ndeps = 0;
      if (cudaStreamGetCaptureInfo(st, &cs, nullptr, &gcap, &deps, &ndeps) == cudaSuccess &&
          cs == cudaStreamCaptureStatusActive) {
        alignas(cudaGraphNodeParams) unsigned char cp_buf[sizeof(cudaGraphNodeParams)] = {};
        cudaGraphNodeParams& cp = *reinterpret_cast<cudaGraphNodeParams*>(cp_buf);
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = cond;
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        if (cudaGraphAddNode(&cnode, gcap, deps, ndeps, &cp) == cudaSuccess &&
            cudaStreamUpdateCaptureDependencies(st, &cnode, 1,
                                                cudaStreamSetCaptureDependencies) == cudaSuccess &&
            cudaStreamBeginCaptureToGraph(e->aux, cp.conditional.phGraph_out[0], nullptr, nullptr,
                                          0, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
          rs = e->aux;
          body = true;
          e->cond_used = true;
        } else {
          e->capture_failed = true;
        }
      }
    }
    // partial: the drifted list; full: all node ids
    k_rb_fill<<<g_wide, T, 0, rs>>>(g, v, s.drifted, &s.res->rb_partial_n, 0, stamp);
    k_rb_fill<<<g_wide, T, 0, rs>>>(g, v, nullptr, &s.res->rb_full_n, 0, stamp);
    RingSrc rp = ring_src(e);
    rp.list = s.drifted;
    rp.count_ptr = &s.res->rb_partial_n;
    rp.valid_at_ptr = &s.hdr->t_batch;
    rp.write_valid = 1;
    rp.e_count = &s.res->E_R;
    launch_attn(e, rp, rs);
    if (stamp && v.attn_logz)
      k_delta_state<<<4 * e->num_sms, DS_THREADS, delta_state_smem(g), rs>>>(
          g, v, s, e->ew, s.drifted, &s.res->rb_partial_n, 0, 1);
    RingSrc rf = rp;
    rf.list = nullptr;
    rf.count_ptr = &s.res->rb_full_n;
    launch_attn(e, rf, rs);
    if (stamp && v.attn_logz)
      k_delta_state<<<4 * e->num_sms, DS_THREADS, delta_state_smem(g), rs>>>(
          g, v, s, e->ew, nullptr, &s.res->rb_full_n, 0, 1);
    k_drift_reset_fin<<<1, 32, 0, rs>>>(v, s);
    n += 5;
    if (body) {
      cudaGraph_t bg = nullptr;
      if (cudaStreamEndCapture(e->aux, &bg) != cudaSuccess) e->capture_failed = true;
    }
  }
  mark();
  chain_launch(k_cleanup, g_rec, T, 0, st, v, s);
  n += 1;
  mark();
  e->launches = n;
}

// The sequence runs on the engine's own stream (graph capture is illegal on
// the legacy default stream callers often use), ordered after and before
// the caller's stream by events.
static int run_on_work(stgn_engine* e, cudaStream_t st);

static int run_sequence(stgn_engine* e, cudaStream_t caller) {
  CUDA_TRY(cudaEventRecord(e->ev_in, caller));
  CUDA_TRY(cudaStreamWaitEvent(e->work, e->ev_in, 0));
  int rc = run_on_work(e, e->work);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(e->ev_out, e->work));
  CUDA_TRY(cudaStreamWaitEvent(caller, e->ev_out, 0));
  return STGN_OK;
}

static int run_on_work(stgn_engine* e, cudaStream_t st) {
  if (e->profiling) {
    enqueue_batch(e, st, 0);
    CUDA_TRY(cudaGetLastError());
    return STGN_OK;
  }
  if (e->graph_ok && !e->graph) {
    cudaGraph_t gr = nullptr;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      cudaGraphConditionalHandle cond = 0;
      cudaStreamCaptureStatus cs;
      cudaGraph_t gcap = nullptr;
      if (e->cfg.rebuild != STGN_REBUILD_NEVER &&
          cudaStreamGetCaptureInfo(st, &cs, nullptr, &gcap, nullptr, nullptr) == cudaSuccess) {
        if (cudaGraphConditionalHandleCreate(&cond, gcap, 0, cudaGraphCondAssignDefault) !=
            cudaSuccess)
          cond = 0;
      }
      e->capture_failed = false;
      enqueue_batch(e, st, cond);
      if (cudaStreamEndCapture(st, &gr) == cudaSuccess && gr && !e->capture_failed) {
        if (cudaGraphInstantiate(&e->graph, gr, 0) != cudaSuccess) e->graph = nullptr;
        cudaGraphDestroy(gr);
      }
    }
    cudaGetLastError();
    if (!e->graph) e->graph_ok = false;  // fall back to direct launches
  }
  if (e->graph) {
    CUDA_TRY(cudaGraphLaunch(e->graph, st));
  } else {
    enqueue_batch(e, st, 0);
  }
  CUDA_TRY(cudaGetLastError());
  return STGN_OK;
}

extern "C" int stgn_engine_set_profiling(stgn_engine* e, int on) {
  if (!e) return STGN_ERR_INVALID;
  if (on && !e->ev[0]) {
    for (int i = 0; i <= NSTAGES; ++i) CUDA_TRY(cudaEventCreate(&e->ev[i]));
  }
  e->profiling = on != 0;
  return STGN_OK;
}

extern "C" int stgn_engine_stage_times(stgn_engine* e, float* ms, int cap, int64_t* launches) {
  if (!e) return -1;
  if (launches) *launches = e->launches;
  if (!e->profiling || !e->ev[0]) return 0;
  const int n = cap < NSTAGES ? cap : NSTAGES;
  for (int i = 0; i < n; ++i) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, e->ev[i], e->ev[i + 1]) != cudaSuccess) t = -1.f;
    ms[i] = t;
  }
  return n;
}

extern "C" const char* stgn_stage_name(int i) {
  return (i >= 0 && i < NSTAGES) ? kStageNames[i] : "";
}

static void fill_report(const BatchRes& r, const stgn_ctl* /*unused*/, stgn_report* rep) {
  memset(rep, 0, sizeof(*rep));
  rep->direct = r.nD;
  rep->affected = r.nA;
  rep->nbr_hit = (int64_t)r.nbr_hit;
  rep->nbr_miss = (int64_t)r.nbr_miss;
  rep->entries_affected = (int64_t)r.E_A;
  rep->entries_direct = (int64_t)r.E_D;
  rep->rebuild_kind = r.rebuild_kind;
  rep->rebuild_nodes = r.rebuild_nodes;
  rep->entries_rebuild = (int64_t)r.E_R;
  rep->changed = (int64_t)r.changed;
  rep->embed_skip = r.n_skip;
  rep->attn_hit = r.n_hit;
  rep->attn_miss = r.n_miss;
  rep->entries_miss = (int64_t)r.E_miss;
  rep->global_drift = r.global_drift;
}

extern "C" int64_t stgn_batch_result_bytes(void) { return (int64_t)sizeof(BatchRes); }

// Copy the last enqueued batch's device result block (stream-ordered after its
// sequence) to dst: device memory (to_device != 0, e.g. a per-slot buffer on the
// engine stream, before the next batch reuses the scratch) or pinned host memory.
extern "C" int stgn_engine_result_copy(stgn_engine* e, void* dst, int32_t to_device,
                                       void* stream) {
  if (!e || !e->bound || !dst) return STGN_ERR_INVALID;
  CUDA_TRY(cudaMemcpyAsync(dst, e->sc.res, sizeof(BatchRes),
                           to_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                           (cudaStream_t)stream));
  return STGN_OK;
}

// Host: the report of a result block copied by stgn_engine_result_copy.
extern "C" int stgn_report_from_result(const void* res, stgn_report* rep) {
  if (!res || !rep) return STGN_ERR_INVALID;
  fill_report(*reinterpret_cast<const BatchRes*>(res), nullptr, rep);
  return STGN_OK;
}

static int check_batch(stgn_engine* e, int32_t B, int64_t m0, int64_t batch_index,
                       int64_t node_count) {
  if (!e->bound || !e->have_w) return STGN_ERR_INVALID;
  if (B < 1 || B > e->cfg.max_batch) return STGN_ERR_CAPACITY;
  if (m0 + B > e->st.cap_edges || node_count > e->st.cap_nodes) return STGN_ERR_CAPACITY;
  if (batch_index + 1 >= e->st.gpow_len) return STGN_ERR_CAPACITY;
  return STGN_OK;
}

static void fill_hdr(stgn_engine* e, BatchHdr* h, int32_t B, double t_batch, int64_t m0,
                     int64_t batch_index, int64_t node_count) {
  memset(h, 0, sizeof(*h));
  h->B = B;
  h->m0 = m0;
  h->batch_index = batch_index;
  h->node_count = node_count;
  h->t_batch = t_batch;
  h->cutoff = std::isfinite(e->cfg.window) ? t_batch - e->cfg.window : -INFINITY;
  // The amark/dmark stamp is the engine's batch index (>= 1), which the host
  // keeps across handle rebuilds: a stamp restarting at 1 in a new handle would
  // alias the stamps an earlier handle left in the (preserved) node tables.
  uint32_t stamp = (uint32_t)(batch_index & 0xffffffffll);
  if (stamp == 0) stamp = 1;
  e->stamp = stamp;
  h->stamp = stamp;
}

extern "C" int stgn_engine_process_batch(stgn_engine* e, int32_t B, const int32_t* src,
                                         const int32_t* dst, const double* t, const float* feat,
                                         int64_t m0, int64_t batch_index, int64_t node_count,
                                         double* preds_out, stgn_report* rep, void* stream) {
  if (!e) return STGN_ERR_INVALID;
  int rc = check_batch(e, B, m0, batch_index, node_count);
  if (rc) return rc;
  for (int32_t i = 0; i < B; ++i) {
    if (src[i] < 0 || dst[i] < 0 || src[i] >= node_count || dst[i] >= node_count)
      return STGN_ERR_BOUNDS;
    if (i && t[i] < t[i - 1]) return STGN_ERR_ORDER;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const Scratch& s = e->sc;
  uint8_t* base = e->h_in;
  const uint8_t* dbase = (const uint8_t*)s.hdr;
  fill_hdr(e, (BatchHdr*)base, B, t[B - 1], m0, batch_index, node_count);
  memcpy(base + ((uint8_t*)s.in_src - dbase), src, sizeof(int32_t) * B);
  memcpy(base + ((uint8_t*)s.in_dst - dbase), dst, sizeof(int32_t) * B);
  memcpy(base + ((uint8_t*)s.in_t - dbase), t, sizeof(double) * B);
  if (e->g.d_e > 0) {
    float* fdst = (float*)(base + ((uint8_t*)s.in_feat - dbase));
    for (int32_t i = 0; i < B; ++i)
      memcpy(fdst + (int64_t)i * e->g.ld_e, feat + (int64_t)i * e->g.d_e, sizeof(float) * e->g.d_e);
  }
  const int64_t bytes = ((uint8_t*)(s.in_feat + (int64_t)B * e->g.ld_e)) - dbase;
  CUDA_TRY(cudaMemcpyAsync((void*)s.hdr, base, bytes, cudaMemcpyHostToDevice, st));
  rc = run_sequence(e, st);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(e->h_preds, s.preds, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(e->h_res, s.res, sizeof(BatchRes), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  memcpy(preds_out, e->h_preds, sizeof(double) * B);
  if (rep) fill_report(*e->h_res, nullptr, rep);
  return STGN_OK;
}

__global__ void k_set_hdr(BatchHdr* dst, BatchHdr h) { *dst = h; }

__global__ void k_pack_feat(const float* src, float* dst, int64_t B, int d_e, int ld_e) {
  GRID_STRIDE(x, B * d_e) {
    const int64_t i = x / d_e, j = x % d_e;
    dst[i * ld_e + j] = src[x];
  }
}

extern "C" int stgn_engine_process_batch_dev(stgn_engine* e, int32_t B, const int32_t* src_dev,
                                             const int32_t* dst_dev, const double* t_dev,
                                             const float* feat_dev, int64_t m0,
                                             int64_t batch_index, int64_t node_count,
                                             double* preds_dev, stgn_report* rep, void* stream) {
  if (!e) return STGN_ERR_INVALID;
  int rc = check_batch(e, B, m0, batch_index, node_count);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const Scratch& s = e->sc;
  BatchHdr hdr;  // passed by value: nothing on the host is reused before the copy lands
  fill_hdr(e, &hdr, B, 0.0, m0, batch_index, node_count);  // t_batch is set on the device
  k_set_hdr<<<1, 1, 0, st>>>(s.hdr, hdr);
  CUDA_TRY(cudaMemcpyAsync(s.in_src, src_dev, sizeof(int32_t) * B, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(s.in_dst, dst_dev, sizeof(int32_t) * B, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(s.in_t, t_dev, sizeof(double) * B, cudaMemcpyDeviceToDevice, st));
  if (e->g.d_e > 0 && feat_dev)
    k_pack_feat<<<(int)std::min<int64_t>(cdiv((int64_t)B * e->g.d_e, 256), 1024), 256, 0, st>>>(
        feat_dev, s.in_feat, B, e->g.d_e, e->g.ld_e);
  else if (e->g.d_e > 0)  // no features given: zero rows, as the host-buffer path does
    CUDA_TRY(cudaMemsetAsync(s.in_feat, 0, sizeof(float) * (size_t)B * e->g.ld_e, st));
  rc = run_sequence(e, st);
  if (rc) return rc;
  if (preds_dev)
    CUDA_TRY(cudaMemcpyAsync(preds_dev, s.preds, sizeof(double) * B, cudaMemcpyDeviceToDevice, st));
  if (rep) {
    CUDA_TRY(cudaMemcpyAsync(e->h_res, s.res, sizeof(BatchRes), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    fill_report(*e->h_res, nullptr, rep);
  }
  return STGN_OK;
}

// ---- node-id-range sharding (paper_2603_21090_b200/shard.py) ----
extern "C" int stgn_engine_set_ownership(stgn_engine* e, int32_t lo, int32_t hi) {
  if (!e || lo < 0 || (hi > 0 && hi < lo)) return STGN_ERR_INVALID;
  e->g.own_lo = lo;
  e->g.own_hi = hi;
  drop_graph(e);
  return STGN_OK;
}

// One batch in two eager parts around the prediction-row exchange: phase 1
// stages the inputs and runs everything through the recompute; phase 2 the
// scores, the memory commit, drift and rebuild (and returns the report).
extern "C" int stgn_engine_batch_phase(stgn_engine* e, int32_t phase, int32_t B,
                                       const int32_t* src_dev, const int32_t* dst_dev,
                                       const double* t_dev, const float* feat_dev, int64_t m0,
                                       int64_t batch_index, int64_t node_count, double* preds_dev,
                                       stgn_report* rep, void* stream) {
  if (!e || (phase != 1 && phase != 2)) return STGN_ERR_INVALID;
  int rc = check_batch(e, B, m0, batch_index, node_count);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const Scratch& s = e->sc;
  if (phase == 1) {
    BatchHdr hdr;
    fill_hdr(e, &hdr, B, 0.0, m0, batch_index, node_count);
    k_set_hdr<<<1, 1, 0, st>>>(s.hdr, hdr);
    CUDA_TRY(cudaMemcpyAsync(s.in_src, src_dev, sizeof(int32_t) * B, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(s.in_dst, dst_dev, sizeof(int32_t) * B, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(s.in_t, t_dev, sizeof(double) * B, cudaMemcpyDeviceToDevice, st));
    if (e->g.d_e > 0 && feat_dev)
      k_pack_feat<<<(int)std::min<int64_t>(cdiv((int64_t)B * e->g.d_e, 256), 1024), 256, 0, st>>>(
          feat_dev, s.in_feat, B, e->g.d_e, e->g.ld_e);
    else if (e->g.d_e > 0)
      CUDA_TRY(cudaMemsetAsync(s.in_feat, 0, sizeof(float) * (size_t)B * e->g.ld_e, st));
    enqueue_batch(e, st, 0, 1);
    CUDA_TRY(cudaGetLastError());
    return STGN_OK;
  }
  enqueue_batch(e, st, 0, 2);
  CUDA_TRY(cudaGetLastError());
  if (preds_dev)
    CUDA_TRY(cudaMemcpyAsync(preds_dev, s.preds, sizeof(double) * B, cudaMemcpyDeviceToDevice, st));
  if (rep) {
    CUDA_TRY(cudaMemcpyAsync(e->h_res, s.res, sizeof(BatchRes), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    fill_report(*e->h_res, nullptr, rep);
  }
  return STGN_OK;
}

__global__ void k_dpred_export(Geo g, Scratch s, int32_t* nodes, float* rows, int* count) {
  const int nD = s.res->nD;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t d = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; d < nD; d += warps) {
    const int v = s.alist[d];
    if (!geo_owns(g, v)) continue;
    int pos = 0;
    if (lane == 0) pos = atomicAdd(count, 1);
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (lane == 0) nodes[pos] = v;
    for (int j = lane; j < g.ld_d; j += 32) rows[(int64_t)pos * g.ld_d + j] = s.dpred[d * g.ld_d + j];
  }
}

__global__ void k_dpred_import(Geo g, Scratch s, const int32_t* nodes, const float* rows, int n) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const int v = nodes[i];
    if (geo_owns(g, v)) continue;  // computed here
    const int64_t d = s.dmap[v];
    for (int j = lane; j < g.ld_d; j += 32) s.dpred[d * g.ld_d + j] = rows[i * g.ld_d + j];
  }
}

// The batch's prediction rows (final layer, pre-batch memory) of the direct
// nodes this engine owns: node ids and [ld_d] rows into caller device buffers
// of capacity 2*max_batch; *count on the host (synchronises the stream).
extern "C" int stgn_engine_dpred_export(stgn_engine* e, int32_t* nodes_dev, float* rows_dev,
                                        int64_t* count, void* stream) {
  if (!e || !e->bound || !nodes_dev || !rows_dev || !count) return STGN_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  int* dcount = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&dcount, sizeof(int), st));
  CUDA_TRY(cudaMemsetAsync(dcount, 0, sizeof(int), st));
  k_dpred_export<<<4 * e->num_sms, 256, 0, st>>>(e->g, e->sc, nodes_dev, rows_dev, dcount);
  int h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, dcount, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaFreeAsync(dcount, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *count = h;
  return STGN_OK;
}

// The other owners' rows (node ids + [ld_d] rows, device) into this batch's
// prediction rows, before phase 2.
extern "C" int stgn_engine_dpred_import(stgn_engine* e, const int32_t* nodes_dev,
                                        const float* rows_dev, int64_t n, void* stream) {
  if (!e || !e->bound) return STGN_ERR_INVALID;
  if (n <= 0) return STGN_OK;
  k_dpred_import<<<4 * e->num_sms, 256, 0, (cudaStream_t)stream>>>(e->g, e->sc, nodes_dev,
                                                                     rows_dev, (int)n);
  CUDA_TRY(cudaGetLastError());
  return STGN_OK;
}

extern "C" int stgn_engine_rebuild(stgn_engine* e, const int32_t* ids, int64_t n_ids,
                                   int64_t node_count, double valid_at_value, int64_t* count,
                                   void* stream) {
  if (!e || !e->bound || !e->have_w) return STGN_ERR_INVALID;
  if (node_count > e->st.cap_nodes) return STGN_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  const Scratch& s = e->sc;
  const int32_t* list = nullptr;
  int64_t n = node_count;
  if (ids) {
    if (n_ids > e->st.cap_nodes) return STGN_ERR_CAPACITY;
    for (int64_t i = 0; i < n_ids; ++i)
      if (ids[i] < 0 || ids[i] >= node_count) return STGN_ERR_BOUNDS;
    if (n_ids) CUDA_TRY(cudaMemcpyAsync(s.rb_ids, ids, sizeof(int32_t) * n_ids, cudaMemcpyHostToDevice, st));
    list = s.rb_ids;
    n = n_ids;
  }
  if (count) *count = n;
  if (n == 0) return STGN_OK;
  k_rb_fill<<<4 * e->num_sms, 256, 0, st>>>(e->g, e->sv, list, nullptr, n,
                                             e->cfg.scope == STGN_SCOPE_DELTA && e->g.K == 1);
  RingSrc r = ring_src(e);
  r.list = list;
  r.count_const = n;
  r.valid_at_const = valid_at_value;
  r.write_valid = 1;
  launch_attn(e, r, st);
  if (e->cfg.scope == STGN_SCOPE_DELTA && e->g.K == 1 && e->sv.attn_logz)
    k_delta_state<<<4 * e->num_sms, DS_THREADS, delta_state_smem(e->g), st>>>(
        e->g, e->sv, s, e->ew, list, nullptr, (int)n, 1);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
  return STGN_OK;
}

extern "C" int stgn_engine_delta_events(stgn_engine* e, int64_t max, int32_t* node, double* bound,
                                        int32_t* dn, int32_t* nv, double* max_v, double* z_dev,
                                        float* emb, double* mvn) {
  if (!e || !e->bound) return STGN_ERR_INVALID;
  const StateView& v = e->sv;
  int64_t ctl_r[2] = {0, 0};
  CUDA_TRY(cudaMemcpy(ctl_r, &v.ctl->reserved[0], sizeof(ctl_r), cudaMemcpyDeviceToHost));
  if (mvn) memcpy(mvn, &ctl_r[1], sizeof(double));
  if (!v.attn_logz || v.ev_cap == 0) return 0;
  const int64_t n = std::min<int64_t>(ctl_r[0], v.ev_cap);
  if (n > max) return STGN_ERR_CAPACITY;
  if (n == 0) return 0;
  std::vector<int32_t> hn(n), hp(n), hdn(n), hnv(n);
  std::vector<double> hb(n), hm(n), hz(n);
  CUDA_TRY(cudaMemcpy(hn.data(), v.ev_node, 4 * n, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(hp.data(), v.ev_dpos, 4 * n, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(hdn.data(), v.ev_dn, 4 * n, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(hnv.data(), v.ev_nv, 4 * n, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(hb.data(), v.ev_bound, 8 * n, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(hm.data(), v.ev_maxv, 8 * n, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(hz.data(), v.ev_zdev, 8 * n, cudaMemcpyDeviceToHost));
  std::vector<float> he((size_t)n * e->g.d);
  if (emb) {
    float* dout = nullptr;
    CUDA_TRY(cudaMalloc(&dout, sizeof(float) * n * e->g.d));
    k_delta_ev_gather<<<4 * e->num_sms, 256>>>(e->g, v, e->sc, v.ev_node, v.ev_dpos, (int)n, dout);
    cudaError_t ce = cudaMemcpy(he.data(), dout, sizeof(float) * n * e->g.d, cudaMemcpyDeviceToHost);
    cudaFree(dout);
    CUDA_TRY(ce);
  }
  std::vector<int64_t> ord(n);
  for (int64_t i = 0; i < n; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return hn[a] < hn[b]; });
  for (int64_t k = 0; k < n; ++k) {
    const int64_t i = ord[k];
    node[k] = hn[i]; bound[k] = hb[i]; dn[k] = hdn[i]; nv[k] = hnv[i];
    max_v[k] = hm[i]; z_dev[k] = hz[i];
    if (emb) memcpy(emb + k * e->g.d, he.data() + i * e->g.d, sizeof(float) * e->g.d);
  }
  return (int)n;
}

extern "C" int stgn_engine_snapshot(stgn_engine* e, int64_t node_count, double t_now,
                                    float* layers_out_dev, void* stream) {
  if (!e || !e->bound || !e->have_w || !layers_out_dev) return STGN_ERR_INVALID;
  if (node_count > e->st.cap_nodes) return STGN_ERR_CAPACITY;
  if (node_count <= 0) return STGN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  RingSrc r = ring_src(e);
  r.list = nullptr;
  r.count_const = node_count;
  r.use_store = 1;
  r.ring_ccnt = e->sv.ring_cnt;  // the store's top-L lists (S/oracle.py:40-45), not the window's
  r.layers_out = layers_out_dev;
  uint8_t* tmp = nullptr;
  if (std::isfinite(t_now)) {  // historical lists from the store chains + payload log
    if (!e->sv.e_pay) return STGN_ERR_INVALID;
    const size_t bytes = hist_rings_bytes(e->g, node_count);
    CUDA_TRY(cudaMallocAsync((void**)&tmp, bytes, st));
    CUDA_TRY(cudaMemsetAsync(tmp, 0, bytes, st));
    HistRings hr = hist_rings_carve(e->g, node_count, tmp);
    k_hist_rings<<<8 * e->num_sms, 256, 0, st>>>(e->g, e->sv, hr, node_count, t_now, e->w.omega);
    r.ring_cnt = hr.cnt;
    r.ring_ccnt = hr.cnt;
    r.ring_head = hr.head;
    r.ring_t = hr.t;
    r.ring_pay = hr.pay;
    r.ring_feat = hr.feat;
    r.ring_tb = hr.tb;
  }
  launch_attn(e, r, st);
  cudaError_t ce = cudaGetLastError();
  if (tmp) cudaFreeAsync(tmp, st);
  if (ce != cudaSuccess) {
    stgn_set_error(__FILE__, __LINE__, ce);
    return STGN_ERR_CUDA;
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  return STGN_OK;
}

extern "C" int stgn_engine_stage_affected(stgn_engine* e, int32_t P, const int32_t* src_dev,
                                          const int32_t* dst_dev, uint32_t stamp, int32_t* out_dev,
                                          int64_t cap, int32_t* hop_off_dev, void* stream) {
  if (!e || !e->bound || P < 0 || !out_dev || !hop_off_dev || (P > 0 && (!src_dev || !dst_dev)))
    return STGN_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  k_stage_affected<<<1, 1024, 0, st>>>(e->g, e->sv, src_dev, dst_dev, P, stamp, out_dev, cap,
                                       hop_off_dev);
  CUDA_TRY(cudaGetLastError());
  int32_t n = 0;
  CUDA_TRY(cudaMemcpyAsync(&n, hop_off_dev + e->g.K + 1, sizeof(n), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return n > cap ? STGN_ERR_CAPACITY : STGN_OK;
}

extern "C" int stgn_engine_stage_nbr_update(stgn_engine* e, int32_t nn,
                                            const stgn_stage_entries* entries,
                                            const int32_t* direct_dev, int32_t nd, double t_now,
                                            const stgn_stage_records* records, void* stream) {
  if (!e || !e->bound || !e->have_w || nn < 0 || !entries || !records || nd < 0 ||
      (nd > 0 && !direct_dev))
    return STGN_ERR_INVALID;
  if (nn == 0) return STGN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const double cutoff = std::isfinite(e->cfg.window) ? t_now - e->cfg.window : -INFINITY;
  const int blocks = (int)std::min<int64_t>(cdiv(nn, 8), 4 * e->num_sms);
  k_stage_nbr_update<<<blocks, 256, 0, st>>>(e->g, e->sv, *entries, nn, direct_dev, nd, cutoff,
                                             e->w.omega, *records);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
  return STGN_OK;
}

extern "C" int stgn_engine_stage_commit(stgn_engine* e, int32_t P, const int32_t* src_dev,
                                        const int32_t* dst_dev, const double* t_dev,
                                        const float* feat_dev, const float* pay_dev, int64_t m0,
                                        void* stream) {
  if (!e || !e->bound || P < 0) return STGN_ERR_INVALID;
  if (P == 0) return STGN_OK;
  if (!src_dev || !dst_dev || !t_dev || !feat_dev || (e->sv.e_pay && !pay_dev))
    return STGN_ERR_INVALID;
  if (m0 < 0 || m0 + P > e->st.cap_edges) return STGN_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  k_stage_commit<<<1, 512, 0, st>>>(e->g, e->sv, src_dev, dst_dev, t_dev, feat_dev, pay_dev, P, m0);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
  return STGN_OK;
}

// ---- DySAT (csrc/dysat.cuh) -------------------------------------------------
static bool dy_valid(const stgn_dysat* s) {
  return s && s->n > 0 && s->d > 0 && s->heads_s > 0 && s->heads_s <= 32 && s->heads_t > 0 &&
         s->d % s->heads_s == 0 && s->d % s->heads_t == 0 && s->window >= 1 && s->window <= 32 &&
         s->fanout >= 1 && s->fanout <= 31 && s->ld >= s->d && s->ld % 4 == 0 &&
         s->snapshot >= 0 && s->snapshot < s->pos_len && s->chunk > 0 && s->max_batch > 0 &&
         s->P && s->ss && s->sn && s->lst_nbr && s->lst_head && s->lst_cnt && s->hist_k &&
         s->hist_v && s->emb && s->mark && s->work && s->rows && s->pos && s->wq && s->wk &&
         s->wv && s->wo && s->wpred;
}

static int dy_temporal(const stgn_dysat* s, const int32_t* list, const int32_t* count_ptr,
                       int64_t count_const, int64_t base, int64_t max_rows, cudaStream_t st) {
  // tcgen05 bf16x3 GEMMs for large row counts (snapshot rolls, full recomputes); a
  // batch's ~2B rows fill only a few 128-row tiles, where the 16-row FFMA tiles
  // spread over more SMs and finish sooner
  if (s->wtc && dy_tc_ok(s->d, s->heads_t) && s->ld == s->d && max_rows >= s->tc_min_rows) {
    const int dt = s->d / s->heads_t;
    using KFn = void (*)(stgn_dysat, const int32_t*, const int32_t*, int64_t, int64_t);
    KFn fn = s->d == 128 ? (dt == 8 ? k_dy_temporal_tc<32, 8> : dt == 16 ? k_dy_temporal_tc<32, 16>
                                                                          : k_dy_temporal_tc<32, 32>)
                         : (dt == 8 ? k_dy_temporal_tc<16, 8> : k_dy_temporal_tc<16, 16>);
    const size_t smem = dy_tc_smem(s->d);
    CUDA_TRY(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    int dev = 0, sms = 148;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(cdiv(max_rows, 128), sms));
    fn<<<(int)grid, DTC_THREADS, smem, st>>>(*s, list, count_ptr, count_const, base);
    CUDA_TRY(cudaGetLastError());
    return STGN_OK;
  }
  const int wsm = 8192;
  const int T = dy_tile_rows(s->d, wsm);
  if (T < 4) return STGN_ERR_INVALID;
  const size_t smem = (size_t)(5 * T * s->d + wsm) * sizeof(float);
  CUDA_TRY(cudaFuncSetAttribute((const void*)k_dy_temporal,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(cdiv(max_rows, T), 4 * sms));
  k_dy_temporal<<<(int)grid, DY_THREADS, smem, st>>>(*s, list, count_ptr, count_const, base, T, wsm);
  CUDA_TRY(cudaGetLastError());
  return STGN_OK;
}

extern "C" int stgn_dysat_batch(const stgn_dysat* s, int32_t B, const int32_t* src_dev,
                                const int32_t* dst_dev, uint32_t stamp, double* preds_dev,
                                int32_t* n_affected, void* stream) {
  if (!dy_valid(s) || B < 0 || (B > 0 && (!src_dev || !dst_dev || !preds_dev)))
    return STGN_ERR_INVALID;
  if (B > s->max_batch) return STGN_ERR_CAPACITY;
  if (n_affected) *n_affected = 0;
  if (B == 0) return STGN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* cnt = s->work + 2 * s->max_batch;
  k_dy_predict<<<(int)cdiv(B, 8), 256, 0, st>>>(*s, B, src_dev, dst_dev, preds_dev);
  CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int32_t), st));
  k_dy_claim<<<(int)cdiv(2 * B, 256), 256, 0, st>>>(*s, B, src_dev, dst_dev, stamp);
  k_dy_lists<<<(int)cdiv(2 * B, 8), 256, 0, st>>>(*s, B, src_dev, dst_dev);
  k_dy_struct<<<(int)cdiv(2 * B, DY_THREADS / 32), DY_THREADS, 0, st>>>(*s, s->work, cnt, 0, 0);
  CUDA_TRY(cudaGetLastError());
  int rc = dy_temporal(s, s->work, cnt, 0, 0, 2 * (int64_t)B, st);
  if (rc) return rc;
  if (n_affected) {
    CUDA_TRY(cudaMemcpyAsync(n_affected, cnt, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  return STGN_OK;
}

extern "C" int stgn_dysat_recompute_all(const stgn_dysat* s, void* stream) {
  if (!dy_valid(s)) return STGN_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  for (int64_t lo = 0; lo < s->n; lo += s->chunk) {
    const int64_t c = std::min<int64_t>(s->chunk, s->n - lo);
    k_dy_struct<<<(int)cdiv(c, DY_THREADS / 32), DY_THREADS, 0, st>>>(*s, nullptr, nullptr, c, lo);
    CUDA_TRY(cudaGetLastError());
    int rc = dy_temporal(s, nullptr, nullptr, c, lo, c, st);
    if (rc) return rc;
  }
  return STGN_OK;
}

extern "C" int stgn_dysat_roll(const stgn_dysat* s, void* stream) {
  if (!dy_valid(s)) return STGN_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(s->lst_cnt, 0, sizeof(int32_t) * s->n, st));
  CUDA_TRY(cudaMemsetAsync(s->lst_head, 0, sizeof(int32_t) * s->n, st));
  return stgn_dysat_recompute_all(s, stream);
}

extern "C" int stgn_engine_full_reference(stgn_engine* e, int64_t node_count, float* out_dev,
                                          void* stream) {
  if (!e || !e->bound || !e->have_w || !out_dev) return STGN_ERR_INVALID;
  if (node_count > e->st.cap_nodes) return STGN_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  RingSrc r = ring_src(e);
  r.list = nullptr;
  r.count_const = node_count;
  r.use_store = 1;
  r.final_out = out_dev;
  launch_attn(e, r, st);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
  return STGN_OK;
}

extern "C" int stgn_engine_affected(stgn_engine* e, int32_t* direct, int32_t* affected,
                                    int64_t cap, int64_t* n_direct, int64_t* n_affected,
                                    int32_t* change_sizes, void* stream) {
  if (!e || !e->bound) return STGN_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const Scratch& s = e->sc;
  CUDA_TRY(cudaMemcpyAsync(e->h_res, s.res, sizeof(BatchRes), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  const int64_t nD = e->h_res->nD, nA = e->h_res->nA;
  if (n_direct) *n_direct = nD;
  if (n_affected) *n_affected = nA;
  if (nA > cap) return STGN_ERR_CAPACITY;
  if (direct && nD) CUDA_TRY(cudaMemcpyAsync(direct, s.alist, 4 * nD, cudaMemcpyDeviceToHost, st));
  if (affected && nA) CUDA_TRY(cudaMemcpyAsync(affected, s.alist, 4 * nA, cudaMemcpyDeviceToHost, st));
  if (change_sizes && nA)
    CUDA_TRY(cudaMemcpyAsync(change_sizes, s.a_size, 4 * nA, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return STGN_OK;
}

extern "C" int stgn_engine_pred_embeddings(stgn_engine* e, float* out, int64_t n_direct,
                                           void* stream) {
  if (!e || !e->bound || !out) return STGN_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  if (n_direct <= 0) return STGN_OK;
  CUDA_TRY(cudaMemcpy2DAsync(out, sizeof(float) * e->g.d, e->sc.dpred, sizeof(float) * e->g.ld_d,
                             sizeof(float) * e->g.d, n_direct, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return STGN_OK;
}

// ---------------------------------------------------------------------------
// operator level
// ---------------------------------------------------------------------------
// reference layouts -> packed layouts of stgn.h
__global__ void k_pack_attn(Geo g, const float* wq, const float* wk, const float* wv,
                            float* pq, float* pkt, float* pv) {
  const int64_t nq = (int64_t)g.K * g.H * g.q_in * g.d_k;
  const int64_t nk = (int64_t)g.K * g.H * g.k_in * g.d_k;
  GRID_STRIDE(x, nq) {  // (l,h,a,b) -> pq[l][a][h*d_k+b]
    const int b = (int)(x % g.d_k);
    int64_t y = x / g.d_k;
    const int a = (int)(y % g.q_in);
    y /= g.q_in;
    const int hh = (int)(y % g.H);
    const int l = (int)(y / g.H);
    pq[((int64_t)l * g.q_in + a) * g.HD + hh * g.d_k + b] = wq[x];
  }
  GRID_STRIDE(x, nk) {  // (l,h,a,b) -> pkt[l][h][b][a], pv[l][h][a][b]
    const int b = (int)(x % g.d_k);
    int64_t y = x / g.d_k;
    const int a = (int)(y % g.k_in);
    y /= g.k_in;
    const int hh = (int)(y % g.H);
    const int l = (int)(y / g.H);
    pkt[(((int64_t)l * g.H + hh) * g.d_k + b) * g.k_in + a] = wk[x];
    pv[x] = wv[x];
  }
}

extern "C" int stgn_pipeline_many(const stgn_dims* dims, int64_t N, int64_t E, const float* qbase,
                                  const int64_t* offsets, const float* payload, const float* feat,
                                  const double* dt, const double* omega, const float* phi0,
                                  const float* wq, const float* wk, const float* wv,
                                  const float* wo, float* out, float* scores, float* values,
                                  float* maxlog, float* zsum, float* qvecs, void* stream) {
  if (!dims) return STGN_ERR_INVALID;
  stgn_config c;
  memset(&c, 0, sizeof(c));
  c.fanout = 1;
  c.max_batch = 1;
  int rc = validate_dims(dims, &c, true);
  if (rc) return rc;
  if (N < 0 || E < 0) return STGN_ERR_INVALID;
  if (N == 0) return STGN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Geo g = make_geo(*dims, 1);
  int dev = 0, sms = 148;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  AttnLaunch al;
  rc = plan_attn(g, true, sms, &al);
  if (rc) return rc;
  const int64_t nq = (int64_t)g.K * g.H * g.q_in * g.d_k;
  const int64_t nk = (int64_t)g.K * g.H * g.k_in * g.d_k;
  // packed weights in a grow-only per-device buffer: no allocation per call (an
  // allocation per call made the call time depend on the memory pool's state)
  static std::mutex pack_mu;
  static float* pack_buf[64] = {};
  static size_t pack_cap[64] = {};
  std::lock_guard<std::mutex> lock(pack_mu);
  const size_t need = sizeof(float) * (size_t)(nq + 2 * nk);
  if (dev < 0 || dev >= 64) return STGN_ERR_INVALID;
  if (need > pack_cap[dev]) {
    CUDA_TRY(cudaStreamSynchronize(st));
    if (pack_buf[dev]) CUDA_TRY(cudaFree(pack_buf[dev]));
    pack_buf[dev] = nullptr;
    pack_cap[dev] = 0;
    CUDA_TRY(cudaMalloc((void**)&pack_buf[dev], need));
    pack_cap[dev] = need;
  }
  float* packed = pack_buf[dev];
  k_pack_attn<<<256, 256, 0, st>>>(g, wq, wk, wv, packed, packed + nq, packed + nq + nk);
  AttnWeights aw;
  aw.wq = packed;
  aw.wkt = packed + nq;
  aw.wv = packed + nq + nk;
  aw.wo = wo;
  aw.omega = omega;
  aw.phi0 = phi0;
  RingSrc rs;
  memset(&rs, 0, sizeof(rs));
  FlatSrc fs;
  fs.N = N;
  fs.offsets = offsets;
  fs.qbase = qbase;
  fs.payload = payload;
  fs.feat = feat;
  fs.dt = dt;
  fs.out = out;
  fs.scores = scores;
  fs.values = values;
  fs.maxlog = maxlog;
  fs.zsum = zsum;
  fs.qvecs = qvecs;
  const int grid = (int)std::min<int64_t>(cdiv(N, al.T), al.grid);
  al.fn<<<grid, STGN_THREADS, al.smem, st>>>(g, aw, rs, fs, al.T);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));  // the shared packed buffer is reused by the next call
  return STGN_OK;
}

extern "C" int stgn_engine_info(stgn_engine* e, int64_t* info, int n) {
  if (!e || !info) return STGN_ERR_INVALID;
  const int64_t v[14] = {e->graph ? 1 : 0, e->cond_used ? 1 : 0, e->launches, e->attn2_tmax,
                         e->attn2_wsm, e->num_sms, (int64_t)e->attn2_smem, (int64_t)e->mem_smem,
                         e->use_tc ? 1 : 0, e->attn3_tmax, e->use_a4 ? 1 : 0,
                         (int64_t)e->attn4_smem, e->use_m4 ? 1 : 0, (int64_t)e->mem4_smem};
  for (int i = 0; i < n && i < 14; ++i) info[i] = v[i];
  return STGN_OK;
}

// State-only fast-forward (test harness): batches advance topology, rings
// (payloads frozen from the layer cache as it stands), memory and drift, but
// the attention recomputes are not launched, so the layer cache is not
// written. Mirrors the oracle's process_batch(compute=False).
extern "C" int stgn_engine_set_skip_recompute(stgn_engine* e, int on) {
  if (!e) return STGN_ERR_INVALID;
  e->skip_recompute = on != 0;
  drop_graph(e);
  return STGN_OK;
}

// Switch the recompute scope between batches (drops the captured graph).
extern "C" int stgn_engine_set_scope(stgn_engine* e, int scope) {
  if (!e || (scope != STGN_SCOPE_AFFECTED && scope != STGN_SCOPE_DIRECT &&
             scope != STGN_SCOPE_DELTA))
    return STGN_ERR_INVALID;
  if (scope == STGN_SCOPE_DIRECT && std::isfinite(e->cfg.window)) return STGN_ERR_INVALID;
  if (scope == STGN_SCOPE_DELTA && e->g.K == 1 && (e->g.H > 4 || !e->ds_ok))
    return STGN_ERR_INVALID;  // attn_logz keeps 4 heads; the state kernel's smem plan
  e->cfg.scope = scope;
  drop_graph(e);
  return STGN_OK;
}

// Per-CTA start/end/entries/tiles of the last recompute launches (-DA4_PROF
// builds; reading clears them). Returns the entries written (4 per CTA).
extern "C" int stgn_debug_a4_cta(uint64_t* out, int cap) {
#ifdef A4_PROF
  const int n = cap < 4 * 1024 ? cap : 4 * 1024;
  if (cudaMemcpyFromSymbol(out, g_a4_cta, sizeof(uint64_t) * n) != cudaSuccess) return -1;
  static uint64_t zeros[4 * 1024];
  cudaMemcpyToSymbol(g_a4_cta, zeros, sizeof(zeros));
  return n;
#else
  (void)out;
  (void)cap;
  return 0;
#endif
}

// Phase timestamps of CTA 0 of the 128-row recompute kernel (builds with
// -DA4_PROF only; otherwise 0 entries). Each entry: globaltimer_ns << 4 | tag.
extern "C" int stgn_debug_a4_prof(uint64_t* out, int cap) {
#ifdef A4_PROF
  int n = 0;
  if (cudaMemcpyFromSymbol(&n, g_a4_prof_n, sizeof(int)) != cudaSuccess) return -1;
  n = n < cap ? n : cap;
  if (n > 0 && cudaMemcpyFromSymbol(out, g_a4_prof, sizeof(uint64_t) * n) != cudaSuccess) return -1;
  const int zero = 0;
  cudaMemcpyToSymbol(g_a4_prof_n, &zero, sizeof(int));
  return n;
#else
  (void)out;
  (void)cap;
  return 0;
#endif
}

extern "C" int stgn_debug_tc_gemm(int F, int N, int K, const float* W, const float* X, float* D,
                                  int mode, void* stream) {
  if (F < 1 || F > 128 || N < 1 || N > 256 || K < 1) return STGN_ERR_INVALID;
  const int Kp = (K + 7) & ~7, Np = (N + 15) & ~15;
  const size_t smem = (size_t)(256 * Kp + 2 * Np * Kp) * sizeof(float);
  if (smem > 220 * 1024) return STGN_ERR_INVALID;
  CUDA_TRY(cudaFuncSetAttribute((const void*)k_tc_gemm_test,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_tc_gemm_test<<<1, 128, smem, (cudaStream_t)stream>>>(F, N, K, W, X, D, mode);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return STGN_OK;
}
