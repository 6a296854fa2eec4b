// ctx.h -- internal state of a GIST context (the opaque gist_ctx of include/gist.h) and the
// helpers shared by the library's translation units: gist_api.cu (lifecycle, graph load,
// parameters, inspection, kernel entry points), round.cu (subGCNs / subAgg: partition, extract,
// aggregate), plan.cu (the grouped launch plan of one subTrain step), step.cu (the step itself,
// CUDA-graph replay, gist_subtrain) and eval.cu (full-graph / partition-wise evaluation).
#pragma once
#include <algorithm>
#include <mutex>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include <cub/cub.cuh>
#include <nvtx3/nvToolsExt.h>
#include <nccl.h>
#include <nccl_device.h>

#include "../../include/gist.h"
#include "comm.h"
#include "common.cuh"
#include "kernels.h"

using namespace gist;

struct gist_ctx;

namespace gist_impl {

enum State { S_CREATED = 0, S_GRAPH = 1, S_PARAMS = 2, S_PARTITIONED = 3 };

struct LayerShape {
  int nrows = 0, ncols = 0;  // logical rows (self block for SAGE) / cols of the sub block
  int Kp = 0, Np = 0;        // physical (padded) shape
  int half = 0;              // SAGE: physical offset of neighbour rows
  int64_t off = 0;           // float offset in the packed slot buffer
  int32_t* rows = nullptr;   // device unit list (nullptr = identity)
  int32_t* cols = nullptr;
};

struct Slot {
  int index = 0;  // global slot id i
  // views into the rank's contiguous [slots_per_rank x S_max] buffers (Wall / Gall / Mall / Vall / Wball)
  float *W = nullptr, *G = nullptr, *M = nullptr, *V = nullptr;
  bf16* Wb = nullptr;
  // batch schedule (device + pinned host mirror), capacity `cap` steps
  int cap = 0;
  int32_t *desc_dev = nullptr, *desc_host = nullptr;
  std::vector<int> nb_of_step, q_of_step;
  std::vector<int64_t> vol_of_step;
  int cached_epoch = -1;
  std::vector<int32_t> epoch_perm;
  // batch buffers (nb_max rows)
  int32_t *b_nodes = nullptr, *lab_b = nullptr, *b_col = nullptr;
  uint64_t* map64 = nullptr;  // cluster -> (step tag, local-id delta)
  uint8_t* train_b = nullptr;
  float* scale = nullptr;
  int64_t *b_beg = nullptr, *b_end = nullptr, *stats = nullptr;
  // activations (element type T of the precision mode)
  std::vector<void*> C, H, dZ;
  std::vector<uint32_t*> mb;  // BF16: bit-packed ReLU masks of C_l / H_l (l >= 1), words [nb_max x mb_ld[l]]
  void* dC = nullptr;
  float* logits = nullptr;
  float *row_loss = nullptr, *step_loss = nullptr, *loss_acc = nullptr;
  uint32_t* ce_done = nullptr;  // softmax-CE last-CTA counter
  // re-associated last layer (BF16 GraphSAGE): P = H W_bot, AGG = N P, DQ = [dZ | Q = N^T dZ],
  // DZs = dZ / deg (block-diagonal path)
  void *rP = nullptr, *rAGG = nullptr, *rDQ = nullptr, *rDZs = nullptr;
  void* rWc = nullptr;  // [W_top | W_bot] of the last layer, half x 2Np bf16 (refreshed every step)
  // GAT (R21): Z_l = H_l W_l per layer, per-row scalars [s | t | lse | S | dt | ds] (6 x nb_max),
  // and the backward operand G (dlogits, then dH_l of each layer)
  std::vector<void*> gZ;
  std::vector<float*> gsc;
  void* gG = nullptr;
  int last_nb = 0;
};

// Launch plan of one subTrain step for a group of <= kMaxGroup local slots run in lockstep:
// argument blocks of every grouped launch, built once per partition (TMA descriptors encoded once).
template <typename T>
struct StepPlan {
  struct Group {
    int first = 0, count = 0;
    BatchGroup batch;
    std::vector<SpmmGroup<T, T>> fwd_spmm, bwd_spmm;  // per layer (bwd index l produces dZ_{l-1})
    std::vector<GemmPlanTC> fwd_tc, dw_tc, dx_tc;     // BF16 mode
    std::vector<SgemmGroup> fwd_f, dw_f, dx_f;        // FP32 mode
    std::vector<double> fwd_fl, dw_fl, dx_fl;         // algorithmic FLOPs (profiling)
    std::vector<OptRanges> opt_l;                      // per-layer optimizer ranges (layer_opt)
    std::vector<double> fwd_by, bwd_by;               // SpMM compulsory bytes excl. nnz part (profiling)
    std::vector<BdPlan> fwd_bd, bwd_bd;               // block-diagonal tensor-core aggregation (c->bd)
    std::vector<double> bd_fl;                        // its FLOPs per launch (profiling)
    CeGroup<T> ce;
    // re-associated last layer: Z = H W_top + N (H W_bot); backward via Q = N^T dZ
    bool reassoc = false;
    GemmPlanTC ra_p, ra_z, ra_dw, ra_dh;
    RelayoutGroup ra_wc;
    BdPlan ra_fbd, ra_bbd;
    SpmmGroup<T, T> ra_fsp, ra_bsp;
    SpmmGroup<T, float> ra_fsp_f;  // GCN: logits = A_hat P straight into the fp32 logits
    double ra_gemm_fl = 0.0, ra_bd_fl = 0.0, ra_fby = 0.0, ra_bby = 0.0;
  };
  std::vector<Group> groups;
};

}  // namespace gist_impl
using namespace gist_impl;  // (internal header: the context below is built from these types)


struct gist_ctx {
  gist_config cfg{};
  std::vector<int> dims;
  int L = 0, arch = 0, prec = 0;
  cudaStream_t stream = nullptr;
  // dW stream (default; GIST_DW_STREAM=0 disables): the backward dW GEMMs (and, with one
  // lockstep group, the per-layer optimizer steps) run on a side stream, overlapping the rest
  // of the backward chain (dX -> aggregation); joined at the end of the step
  cudaStream_t dws = nullptr;
  // the side stream for this step: dws, except in profiled steps (every prof_stride-th), which
  // run serialised so that the per-kernel event times of the live roofline are not inflated by
  // overlap (ncu's launch list is serialised too)
  cudaStream_t side_now = nullptr;
  // the optimizer runs per layer on the dW stream right after that layer's dW GEMM (overlapping
  // the rest of the backward chain) instead of one pass after the backward; GCN / GraphSAGE
  bool layer_opt = false;
  bool opt_side = false;  // this step's one-pass optimizer already enqueued on the dW stream (early prefetch)
  bool opt_side_ok = false;
  cudaEvent_t ev_dw_fork = nullptr, ev_dw_join = nullptr;
  // this step's batches were built on the dW stream, overlapping the previous step's optimizer
  bool batch_prefetched = false;
  int cur_z = 0;  // host index of the step being enqueued (schedule bookkeeping / profiling only)
  // CUDA graphs of one step, per variant [build * 2 + prefetch] (dropped at every plan rebuild)
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    int64_t nk = 0;  // kernels per replay
  };
  StepGraph graphs[4];
  bool own_stream = false;
  int state = S_CREATED;
  gist_status sticky = GIST_OK;
  std::string err;
  Comm comm;  // NCCL communicator or loopback group (world > 1)
  cudaEvent_t fork_ev = nullptr;
  // graph (relabelled: clusters contiguous)
  int64_t n = 0, nnz = 0;
  int c = 0, k = 0;
  int64_t self_loops = 0;
  int64_t *rp = nullptr, *cstart = nullptr;
  int32_t *col = nullptr, *cid = nullptr, *labels = nullptr;
  int32_t* ccol = nullptr;  // cluster of every edge's neighbour (batch build), or packed codes (pack_ob > 0)
  int pack_ob = 0;          // offset bits of the packed edge codes (0: plain cluster ids)
  uint8_t* split = nullptr;
  void* X = nullptr;  // n x pad8(d0), T
  float* full_scale = nullptr;
  std::vector<int32_t> perm_h;  // new id -> original id
  std::vector<int64_t> cstart_h, cvol_h;  // cluster offsets (new ids) / cluster volumes (sum of degrees)
  int nb_max = 0, max_csize = 0;
  int64_t nnzb_max = 0;
  // block-diagonal tensor-core aggregation (SAGE, BF16): binary intra-cluster blocks
  bf16* blocks = nullptr;
  int bs = 0;
  bool bd = false;
  double block_density = 0.0;
  // global parameters, physical layout (R6): SAGE rows [0,d) self, [pad8(d), pad8(d)+d) neighbour
  std::vector<float*> theta;
  std::vector<int64_t> th_K, th_N;
  // owner-sharded Theta (GIST_THETA_SHARDED): this rank's physical rows [sh_lo, sh_hi) of every
  // layer (replicated: [0, th_K)); xscr = every slot's packed sub-model (m x S_max), of which
  // this rank fills / reads only the rows it owns (the send / receive side of the exchanges);
  // units_h = host copy of the round's hidden-dim partition (the exchange runs are planned on it)
  std::vector<int64_t> sh_lo, sh_hi;
  float* xscr = nullptr;
  std::vector<std::vector<int32_t>> units_h;
  // partition of the current round
  int m = 0;
  std::vector<uint8_t> layer_set;              // set_params: layers written since load (PARAMS once all are)
  std::vector<int32_t*> units;                 // per dim (hidden dims only)
  std::vector<std::vector<int32_t>> offs;      // per dim, m+1
  std::vector<std::vector<LayerShape>> shapes;  // [slot][layer] for all m slots
  int64_t S_max = 0;                           // floats per packed slot buffer
  int slots_per_rank = 0;
  std::vector<Slot> slots;                     // local slots
  float* Wall = nullptr;                       // slots_per_rank * S_max (local slot weights, contiguous)
  float *Gall = nullptr, *Mall = nullptr, *Vall = nullptr;  // same packing: gradients, Adam moments
  std::vector<float*> theta_m, theta_v;  // GIST_OPT_STATE_PERSISTENT: global Adam moments (Theta layout)
  bf16* Wball = nullptr;                       // bf16 shadow of Wall (BF16 mode)
  int nb_max_rows = 0;                         // static row count of every batch launch
  std::vector<int64_t> mb_ld;                  // words per row of Slot::mb[l]
  bool reassoc = false;                        // last SAGE layer re-associated (BF16, L >= 2)
  StepState* dstate = nullptr;                 // device step state (z, t, lr)
  StepState* hstate = nullptr;                 // pinned host staging for it
  int32_t* bctr = nullptr;                     // per-group batch-build counters (BatchGroup::ctr), 2 per slot
  cudaEvent_t hstate_ev = nullptr;
  StepPlan<float> plan_f;
  StepPlan<bf16> plan_b;
  float* Wrecv = nullptr;                      // world * slots_per_rank * S_max (world > 1, ALLGATHER)
  // agg_mode P2P (f2): Theta (+ f3 moments) in one cudaMalloc region; peer_base[r] = rank r's
  // region (opened from its IPC handle; peer_base[rank] = p2p_base); one-word barrier buffer
  char* p2p_base = nullptr;
  // agg_mode SYMM (f2): the same region from ncclMemAlloc, registered as an NCCL symmetric window,
  // with a device communicator (LSA team; NVLS multicast when available) for the device-API stores
  ncclWindow_t win = nullptr;
  ncclDevComm* devcomm = nullptr;  // host copy, passed by value to the scatter kernel
  bool symm_mm = false;             // the device communicator has an NVLS multimem object
  std::vector<char*> peer_base;
  float* barrier_word = nullptr;
  int alloc_m = 0;
  void* sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  uint64_t *keys_a = nullptr, *keys_b = nullptr;
  int32_t *idx_a = nullptr, *idx_b = nullptr, *blk = nullptr, *offs_dev = nullptr;
  int64_t round = 0, step = 0, adam_t = 0;
  int64_t nk = 0, h2d = 0, d2h = 0;
  std::vector<void*> allocs;
  // live profiling (gist_profile): event pairs around launches of sampled steps
  struct ProfRec {
    int cls;
    double work, per_nnz;
    int nnz_slot;  // index into nnz_pin (-1: none)
    cudaEvent_t a, b;
  };
  int prof_stride = 0;
  bool prof_now = false;
  std::vector<ProfRec> prof_pending;
  std::vector<cudaEvent_t> ev_pool;
  int64_t* nnz_pin = nullptr;
  int nnz_pin_cap = 0, nnz_pin_used = 0;
  double prof_ms[GIST_PROF_N] = {0}, prof_work[GIST_PROF_N] = {0};
  int64_t prof_n[GIST_PROF_N] = {0};
};

// ============================================================== helpers ====
namespace gist_impl {

inline gist_status fail(gist_ctx* c, gist_status s, const std::string& msg) {
  if (c) {
    c->err = msg;
    if (s == GIST_E_CUDA || s == GIST_E_NCCL) c->sticky = s;
  }
  return s;
}

// a collective's status: sticky on CUDA / NCCL failures (the message is already in c->err)
inline gist_status coll(gist_ctx* c, gist_status st) {
  if (st == GIST_E_CUDA || st == GIST_E_NCCL) c->sticky = st;
  return st;
}

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      return fail(c, e_ == cudaErrorMemoryAllocation ? GIST_E_OOM : GIST_E_CUDA,           \
                  std::string(#x) + ": " + cudaGetErrorString(e_));                        \
  } while (0)
#define NK(x)                                                                              \
  do {                                                                                     \
    ncclResult_t r_ = (x);                                                                 \
    if (r_ != ncclSuccess) return fail(c, GIST_E_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)
#define TRY(x)                        \
  do {                                \
    gist_status s_ = (x);             \
    if (s_ != GIST_OK) return s_;     \
  } while (0)
#define PRE(c)                                                        \
  do {                                                                \
    if (!(c)) return GIST_E_ARG;                                      \
    if ((c)->sticky != GIST_OK) return (c)->sticky;                   \
    cudaSetDevice((c)->cfg.device);                                   \
  } while (0)
// profiled launch: PL(class, algorithmic work, stream, launch-expression)
#define PL(cls, work, st, expr)                     \
  do {                                              \
    int id_ = prof_begin(c, (st), (cls), (work));   \
    expr;                                           \
    prof_end(c, (st), id_);                         \
    ++c->nk;                                        \
  } while (0)
// launch bookkeeping: every kernel launch of the library goes through LK or PL
#define LK(expr)  \
  do {            \
    expr;         \
    ++c->nk;      \
  } while (0)

// Device memory comes from the device's stream-ordered pool (cudaMallocAsync on the context
// stream), which keeps up to 16 GB reserved after frees: a second context in the same process
// (e.g. bench.py's e2e run after its device-timed run) reuses it instead of paying cudaMalloc /
// page mapping again.  Allocation happens at load / partition time only, never in the step.
inline void configure_pool() {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = 16ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
  });
}
inline gist_status dalloc(gist_ctx* c, void** p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) bytes = 16;
  configure_pool();
  cudaError_t e = cudaMallocAsync(p, bytes, c->stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, GIST_E_OOM, "cudaMalloc(" + std::to_string(bytes) + " bytes) failed: " + cudaGetErrorString(e));
  }
  c->allocs.push_back(*p);
  return GIST_OK;
}
template <typename P>
inline gist_status dalloc_t(gist_ctx* c, P** p, size_t count) {
  return dalloc(c, reinterpret_cast<void**>(p), count * sizeof(P));
}
inline void dfree(gist_ctx* c, void* p) {
  if (!p) return;
  auto it = std::find(c->allocs.begin(), c->allocs.end(), p);
  if (it != c->allocs.end()) c->allocs.erase(it);
  cudaFreeAsync(p, c->stream);
}

inline gist_status check_launch(gist_ctx* c, const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, GIST_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return GIST_OK;
}

inline size_t esize(const gist_ctx* c) { return c->prec == GIST_PREC_BF16 ? 2 : 4; }

inline cudaEvent_t pool_event(gist_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
// opens a profiled launch on stream s (only while c->prof_now)
inline int prof_begin(gist_ctx* c, cudaStream_t s, int cls, double work, double per_nnz = 0.0, int nnz_slot = -1) {
  if (!c->prof_now) return -1;
  gist_ctx::ProfRec r{cls, work, per_nnz, nnz_slot, pool_event(c), pool_event(c)};
  cudaEventRecord(r.a, s);
  c->prof_pending.push_back(r);
  return (int)c->prof_pending.size() - 1;
}
inline void prof_end(gist_ctx* c, cudaStream_t s, int id) {
  if (id >= 0) cudaEventRecord(c->prof_pending[id].b, s);
}
// synchronises and folds pending records into the per-class totals
inline void prof_flush(gist_ctx* c) {
  if (c->prof_pending.empty()) return;
  cudaDeviceSynchronize();
  for (auto& r : c->prof_pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    double w = r.work;
    if (r.nnz_slot >= 0) w += r.per_nnz * (double)c->nnz_pin[r.nnz_slot];
    c->prof_ms[r.cls] += ms;
    c->prof_work[r.cls] += w;
    c->prof_n[r.cls] += 1;
    c->ev_pool.push_back(r.a);
    c->ev_pool.push_back(r.b);
  }
  c->prof_pending.clear();
  c->nnz_pin_used = 0;
}

inline int hidden_block_max(const gist_ctx* c, int l, int m) {
  return (c->dims[l] + m - 1) / m;  // ceil: the largest balanced block (R5)
}

// logical shape of the sub-weight of slot i, layer l (R6)
inline void sub_logical(const gist_ctx* c, int i, int l, int* nrows, int* ncols) {
  auto bsize = [&](int dim) {
    if (dim == 0 || dim == c->L) return c->dims[dim];
    return c->offs[dim][i + 1] - c->offs[dim][i];
  };
  *nrows = bsize(l);
  *ncols = bsize(l + 1);
}

// Host side of R7: cluster permutation of slot i in epoch e; batch p = perm[pq : (p+1)q)
inline void epoch_perm(const gist_ctx* c, int slot, int64_t e, std::vector<int32_t>& out) {
  std::vector<std::pair<uint64_t, int32_t>> kv(c->c);
  for (int j = 0; j < c->c; ++j)
    kv[j] = {philox_key64((uint32_t)j, (uint32_t)e, (uint32_t)slot, PURPOSE_BATCH, c->cfg.batch_seed), j};
  std::sort(kv.begin(), kv.end());
  out.resize(c->c);
  for (int j = 0; j < c->c; ++j) out[j] = kv[j].second;
}

}  // namespace gist_impl

// ---- small helpers used by several translation units
namespace gist_impl {
// NVTX range over one ABI call (host timeline; named after the call) for Nsight-style tracing
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
  Range(const Range&) = delete;
  Range& operator=(const Range&) = delete;
};
inline bool persistent_adam(const gist_ctx* c) {
  return c->cfg.optimizer == GIST_OPT_ADAM && c->cfg.opt_state == GIST_OPT_STATE_PERSISTENT;
}
// Logical rows of Theta_l for input width d (GCN d, GraphSAGE 2d (R2), GAT d + 2 (R21)) and the
// physical rows (second block at pad8(d): SAGE neighbour rows, GAT the two attention rows)
inline int wrows(const gist_ctx* c, int d) {
  return c->arch == GIST_ARCH_SAGE ? 2 * d : (c->arch == GIST_ARCH_GAT ? d + 2 : d);
}
inline int64_t kphys(const gist_ctx* c, int64_t d) {
  return c->arch == GIST_ARCH_SAGE ? 2 * pad8(d) : (c->arch == GIST_ARCH_GAT ? pad8(d) + 8 : pad8(d));
}
inline bool two_blocks(const gist_ctx* c) { return c->arch != GIST_ARCH_GCN; }
inline bool sharded(const gist_ctx* c) { return c->cfg.theta_mode == GIST_THETA_SHARDED; }
// physical rows of Theta_l owned by rank r (contiguous, balanced)
inline int64_t shard_lo(const gist_ctx* c, int l, int r) { return c->th_K[l] * r / c->cfg.world_size; }
inline int64_t rows_here(const gist_ctx* c, int l) { return c->sh_hi[l] - c->sh_lo[l]; }
inline void free_slots(gist_ctx* c) {
  for (auto& s : c->slots)
    if (s.desc_host) cudaFreeHost(s.desc_host);
  c->slots.clear();
}
// cross-file entry points
gist_status alloc_slots(gist_ctx* c, int m);
// shard.cu: the owner-sharded model's exchanges (collectives over the group)
gist_status shard_extract(gist_ctx* c);     // gist_partition: owners' rows -> every slot's rank
gist_status shard_aggregate(gist_ctx* c);   // gist_aggregate: slots' rows -> their owners
gist_status shard_gather_layer(gist_ctx* c, const float* shard, int l, float* full, cudaStream_t s);
template <typename T> gist_status build_plan(gist_ctx* c, StepPlan<T>& P);
void drop_graphs(gist_ctx* c);
}  // namespace gist_impl
