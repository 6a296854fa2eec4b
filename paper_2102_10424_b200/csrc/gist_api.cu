// gist_api.cu -- the C ABI (include/gist.h): context lifecycle, graph load, parameters,
// inspection hooks, live profiling and the kernel-level entry points.  The GIST round lives in
// round.cu (subGCNs / subAgg), plan.cu + step.cu (subTrain) and eval.cu (evaluation); every
// arithmetic step runs in the kernels of kernels.h.
#include "ctx.h"

using namespace gist;
using namespace gist_impl;

bool gist::pdl_enabled() {
  static const bool on = [] { const char* e = std::getenv("GIST_PDL"); return !(e && e[0] == '0'); }();
  return on;
}

// ============================================================ lifecycle ====

extern "C" void gist_config_default(gist_config* cfg) {
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->arch = GIST_ARCH_GCN;
  cfg->optimizer = GIST_OPT_ADAM;
  cfg->beta1 = 0.9f;
  cfg->beta2 = 0.999f;
  cfg->eps = 1e-8f;
  cfg->precision = GIST_PREC_FP32;
  cfg->clusters_per_batch = 1;
  cfg->world_size = 1;
}

extern "C" const char* gist_status_str(gist_status s) {
  switch (s) {
    case GIST_OK: return "GIST_OK";
    case GIST_E_ARG: return "GIST_E_ARG";
    case GIST_E_SHAPE: return "GIST_E_SHAPE";
    case GIST_E_STATE: return "GIST_E_STATE";
    case GIST_E_OOM: return "GIST_E_OOM";
    case GIST_E_CUDA: return "GIST_E_CUDA";
    case GIST_E_NCCL: return "GIST_E_NCCL";
    case GIST_E_UNSUPPORTED: return "GIST_E_UNSUPPORTED";
  }
  return "GIST_E_?";
}

extern "C" const char* gist_last_error(const gist_ctx* c) { return c ? c->err.c_str() : "null context"; }

extern "C" int32_t gist_slot_owner(int32_t slot, int32_t world_size) {
  return world_size > 0 && slot >= 0 ? slot % world_size : -1;
}
extern "C" int32_t gist_slots_per_rank(int32_t m, int32_t world_size) {
  return world_size > 0 && m > 0 ? (m + world_size - 1) / world_size : 0;
}

extern "C" gist_status gist_nccl_unique_id(void* out128) {
  if (!out128) return GIST_E_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return GIST_E_NCCL;
  std::memcpy(out128, &id, sizeof(id));
  return GIST_OK;
}

extern "C" gist_status gist_create(const gist_config* cfg, gist_ctx** out) {
  if (!cfg || !out || !cfg->dims || cfg->num_layers < 1) return GIST_E_ARG;
  *out = nullptr;
  if (cfg->arch != GIST_ARCH_GCN && cfg->arch != GIST_ARCH_SAGE && cfg->arch != GIST_ARCH_GAT) return GIST_E_ARG;
  if (cfg->optimizer != GIST_OPT_SGD && cfg->optimizer != GIST_OPT_ADAM) return GIST_E_ARG;
  if (cfg->precision != GIST_PREC_FP32 && cfg->precision != GIST_PREC_BF16 && cfg->precision != GIST_PREC_TF32)
    return GIST_E_ARG;
  if (cfg->opt_state != GIST_OPT_STATE_RESET && cfg->opt_state != GIST_OPT_STATE_PERSISTENT) return GIST_E_ARG;
  if (cfg->agg_mode != GIST_AGG_ALLGATHER && cfg->agg_mode != GIST_AGG_P2P && cfg->agg_mode != GIST_AGG_SYMM)
    return GIST_E_ARG;
  // SYMM: NCCL symmetric windows need an NCCL communicator (not the loopback test transport); R21's
  // mean of the GAT attention rows needs every copy on every rank
  if (cfg->agg_mode == GIST_AGG_SYMM && (cfg->loopback || cfg->arch == GIST_ARCH_GAT)) return GIST_E_UNSUPPORTED;
  if (cfg->eval_scale != GIST_EVAL_SCALE_NONE && cfg->eval_scale != GIST_EVAL_SCALE_MEAN) return GIST_E_ARG;
  if (cfg->theta_mode != GIST_THETA_REPLICATED && cfg->theta_mode != GIST_THETA_SHARDED) return GIST_E_ARG;
  // the owner-sharded model moves rows point to point; the peer-store subAgg modes write replicas
  if (cfg->theta_mode == GIST_THETA_SHARDED && cfg->agg_mode != GIST_AGG_ALLGATHER) return GIST_E_UNSUPPORTED;
  if (cfg->agg_mode == GIST_AGG_P2P && (cfg->arch == GIST_ARCH_GAT || cfg->world_size > kMaxPeers))
    return GIST_E_UNSUPPORTED;  // R21 needs every copy of the attention rows; PeerDst holds 8 ranks
  if (cfg->clusters_per_batch < 1 || cfg->world_size < 1 || cfg->rank < 0 || cfg->rank >= cfg->world_size)
    return GIST_E_ARG;
  for (int l = 0; l <= cfg->num_layers; ++l)
    if (cfg->dims[l] < 1) return GIST_E_SHAPE;
  // GAT attention passes hold an output row in registers (gat.cu): layer outputs <= kGatMaxWidth
  for (int l = 1; l <= cfg->num_layers && cfg->arch == GIST_ARCH_GAT; ++l)
    if (pad8(cfg->dims[l]) > kGatMaxWidth) return GIST_E_UNSUPPORTED;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= cfg->device || cfg->device < 0) {
    cudaGetLastError();
    return GIST_E_UNSUPPORTED;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess || prop.major != 10) return GIST_E_UNSUPPORTED;
  if (cfg->graph_residency != GIST_GRAPH_DEVICE) return GIST_E_UNSUPPORTED;
  if (cfg->world_size > 1 && !cfg->nccl_unique_id && !cfg->loopback) return GIST_E_ARG;
  gist_ctx* c = new gist_ctx();
  c->cfg = *cfg;
  c->dims.assign(cfg->dims, cfg->dims + cfg->num_layers + 1);
  c->cfg.dims = c->dims.data();
  c->L = cfg->num_layers;
  c->arch = cfg->arch;
  c->prec = cfg->precision;
  c->comm.rank = cfg->rank;
  c->comm.world = cfg->world_size;
  // every error below releases what was created so far through gist_destroy
  auto bail = [&](gist_status st) {
    gist_destroy(c);
    return st;
  };
  cudaSetDevice(cfg->device);
  if (cfg->stream) {
    c->stream = (cudaStream_t)cfg->stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(GIST_E_CUDA);
    c->own_stream = true;
  }
  if (cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming) != cudaSuccess) return bail(GIST_E_CUDA);
  if (const char* e = std::getenv("GIST_DW_STREAM"); !(e && e[0] == '0')) {
    if (cudaStreamCreateWithFlags(&c->dws, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_dw_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_dw_join, cudaEventDisableTiming) != cudaSuccess)
      return bail(GIST_E_CUDA);
  }
  if (cfg->world_size == 1 && cfg->agg_mode == GIST_AGG_SYMM) {  // a one-rank communicator owns the window
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess || ncclCommInitRank(&c->comm.nccl, 1, id, 0) != ncclSuccess)
      return bail(GIST_E_NCCL);
  }
  if (cfg->world_size > 1) {
    if (cfg->loopback) {  // tests: W contexts of one process stand in for W ranks (comm.h)
      if (loopback_join(cfg->loopback, cfg->rank, cfg->world_size) != GIST_OK) return bail(GIST_E_ARG);
      c->comm.lb = cfg->loopback;
    } else {
      ncclUniqueId id;
      std::memcpy(&id, cfg->nccl_unique_id, sizeof(id));
      if (ncclCommInitRank(&c->comm.nccl, cfg->world_size, id, cfg->rank) != ncclSuccess) return bail(GIST_E_NCCL);
    }
  }
  *out = c;
  return GIST_OK;
}


extern "C" void gist_destroy(gist_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->cfg.device);
  cudaDeviceSynchronize();
  free_slots(c);
  for (void* p : c->allocs) cudaFreeAsync(p, c->stream);
  cudaStreamSynchronize(c->stream);
  for (size_t r = 0; r < c->peer_base.size(); ++r)
    if (c->peer_base[r] && c->peer_base[r] != c->p2p_base && !c->comm.lb) cudaIpcCloseMemHandle(c->peer_base[r]);
  // after a failed CUDA / NCCL call (sticky status) a peer may be blocked in a collective: abort the
  // communicator instead of the collective teardown (window deregistration, device communicator,
  // ncclCommDestroy), which would wait for it
  const bool abort = c->sticky != GIST_OK && c->comm.nccl;
  if (c->devcomm) {
    if (!abort) ncclDevCommDestroy(c->comm.nccl, c->devcomm);
    delete c->devcomm;
  }
  if (c->win && !abort) ncclCommWindowDeregister(c->comm.nccl, c->win);
  if (c->p2p_base) {
    if (c->cfg.agg_mode == GIST_AGG_SYMM) {
      if (!abort) ncclMemFree(c->p2p_base);
    } else {
      cudaFree(c->p2p_base);
    }
  }
  if (c->comm.nccl) {
    if (abort) ncclCommAbort(c->comm.nccl);
    else ncclCommDestroy(c->comm.nccl);
  }
  if (c->comm.lb) loopback_leave(c->comm.lb, c->comm.rank);
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  drop_graphs(c);
  if (c->dws) cudaStreamDestroy(c->dws);
  if (c->ev_dw_fork) cudaEventDestroy(c->ev_dw_fork);
  if (c->ev_dw_join) cudaEventDestroy(c->ev_dw_join);
  for (auto& r : c->prof_pending) c->ev_pool.push_back(r.a), c->ev_pool.push_back(r.b);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  if (c->nnz_pin) cudaFreeHost(c->nnz_pin);
  if (c->hstate) cudaFreeHost(c->hstate);
  if (c->hstate_ev) cudaEventDestroy(c->hstate_ev);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

extern "C" void* gist_stream(gist_ctx* c) { return c ? (void*)c->stream : nullptr; }

extern "C" int64_t gist_stat(gist_ctx* c, int32_t which) {
  if (!c) return -1;
  switch (which) {
    case GIST_STAT_ROUND: return c->round;
    case GIST_STAT_STEP: return c->step;
    case GIST_STAT_SELF_LOOPS_DROPPED: return c->self_loops;
    case GIST_STAT_LAST_NNZ_B: {
      if (c->slots.empty()) return 0;
      int64_t st[2] = {0, 0};
      cudaMemcpy(st, c->slots[0].stats, sizeof(st), cudaMemcpyDeviceToHost);
      return st[0];
    }
    case GIST_STAT_LAST_NB: return c->slots.empty() ? 0 : c->slots[0].last_nb;
    case GIST_STAT_KERNELS: return c->nk;
    case GIST_STAT_H2D_BYTES: return c->h2d;
    case GIST_STAT_D2H_BYTES: return c->d2h;
    case GIST_STAT_MAX_NB: return c->nb_max;
    case GIST_STAT_BLOCK_AGG: return c->bd ? 1 : 0;
    case GIST_STAT_BLOCK_DENSITY_PPM: return (int64_t)(c->block_density * 1e6);
    case GIST_STAT_THETA_BYTES: {
      int64_t b = 0;
      for (int l = 0; l < (int)c->sh_lo.size(); ++l) b += rows_here(c, l) * c->th_N[l] * 4;
      return persistent_adam(c) ? 3 * b : b;
    }
  }
  return -1;
}

// ============================================================ load graph ===
// agg_mode P2P: Theta (and the f3 moments) in ONE cudaMalloc region (CUDA IPC
// exports whole cudaMalloc allocations, not stream-ordered pool blocks), laid out identically on
// every rank; the 64-byte IPC handles travel in one ncclAllGather and every rank opens its
// peers' regions (NVLink peer access enabled lazily by the driver).  World 1: the only
// "peer" is the local region, and gist_aggregate reduces to the ALLGATHER path's local scatter.
static gist_status p2p_setup(gist_ctx* c) {
  const int W = c->cfg.world_size, L = c->L;
  const int parts = persistent_adam(c) ? 3 : 1;
  std::vector<size_t> off(L);
  size_t floats = 0;
  for (int l = 0; l < L; ++l) {
    off[l] = floats;
    floats += (size_t)pad8(kphys(c, c->dims[l])) * pad8(c->dims[l + 1]);  // 32-byte aligned layers
  }
  const bool symm = c->cfg.agg_mode == GIST_AGG_SYMM;
  const size_t bytes = symm ? cdiv(floats * 4 * parts, NCCL_WIN_REQUIRED_ALIGNMENT) * NCCL_WIN_REQUIRED_ALIGNMENT
                            : floats * 4 * parts;
  if (symm) {
    // SYMM: ncclMemAlloc + a collective window registration (identical offsets on every rank) and a
    // device communicator; NVLS multicast is requested at W > 1 and dropped if unavailable
    NK(ncclMemAlloc(reinterpret_cast<void**>(&c->p2p_base), bytes));
    NK(ncclCommWindowRegister(c->comm.nccl, c->p2p_base, bytes, &c->win, NCCL_WIN_COLL_SYMMETRIC));
    c->devcomm = new ncclDevComm();
    ncclDevCommRequirements req;
    std::memset(&req, 0, sizeof(req));
    req.lsaMultimem = W > 1;
    if (ncclDevCommCreate(c->comm.nccl, &req, c->devcomm) != ncclSuccess) {
      req.lsaMultimem = false;
      NK(ncclDevCommCreate(c->comm.nccl, &req, c->devcomm));
    }
    c->symm_mm = req.lsaMultimem;
  } else if (cudaMalloc(reinterpret_cast<void**>(&c->p2p_base), bytes) != cudaSuccess) {
    cudaGetLastError();
    c->p2p_base = nullptr;
    return fail(c, GIST_E_OOM, "p2p: cudaMalloc of the Theta region failed");
  }
  float* f = reinterpret_cast<float*>(c->p2p_base);
  if (parts == 3) c->theta_m.assign(L, nullptr), c->theta_v.assign(L, nullptr);
  for (int l = 0; l < L; ++l) {
    c->theta[l] = f + off[l];
    if (parts == 3) c->theta_m[l] = f + floats + off[l], c->theta_v[l] = f + 2 * floats + off[l];
  }
  TRY(dalloc_t(c, &c->barrier_word, 1));
  CK(cudaMemsetAsync(c->barrier_word, 0, 4, c->stream));
  c->peer_base.assign(W, nullptr);
  c->peer_base[c->cfg.rank] = c->p2p_base;
  if (W == 1 || symm) return GIST_OK;  // SYMM: the device API maps the peers
  if (c->comm.lb) {  // loopback ranks share one process: the peers' regions are plain pointers
    std::vector<void*> all;
    gist_status st = comm_exchange_ptr(c->comm, c->p2p_base, all, &c->err);
    if (st != GIST_OK) return fail(c, st, c->err);
    for (int r = 0; r < W; ++r) c->peer_base[r] = static_cast<char*>(all[r]);
    return GIST_OK;
  }
  cudaIpcMemHandle_t mine;
  CK(cudaIpcGetMemHandle(&mine, c->p2p_base));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  char* hd = nullptr;
  TRY(dalloc_t(c, &hd, (size_t)64 * (W + 1)));
  CK(cudaMemcpyAsync(hd + 64 * (1 + c->cfg.rank), &mine, 64, cudaMemcpyHostToDevice, c->stream));
  TRY(coll(c, comm_allgather(c->comm, hd + 64 * (1 + c->cfg.rank), hd + 64, 64, c->stream, &c->err)));
  std::vector<cudaIpcMemHandle_t> all(W);
  CK(cudaMemcpyAsync(all.data(), hd + 64, (size_t)64 * W, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  dfree(c, hd);
  for (int r = 0; r < W; ++r) {
    if (r == c->cfg.rank) continue;
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, all[r], cudaIpcMemLazyEnablePeerAccess));
    c->peer_base[r] = static_cast<char*>(p);
  }
  return GIST_OK;
}

extern "C" gist_status gist_load_graph(gist_ctx* c, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                                       int64_t nnz, const float* X, const int32_t* labels, int32_t num_classes,
                                       const uint8_t* split, const int32_t* cluster_ids, int32_t num_clusters) {
  PRE(c);
  Range nvtx_range("gist_load_graph");
  if (c->state != S_CREATED) return fail(c, GIST_E_STATE, "load_graph: graph already loaded");
  if (n < 1 || n > INT32_MAX - 1 || !row_ptr || (!col_idx && nnz > 0) || !X || !labels || !split || !cluster_ids)
    return fail(c, GIST_E_ARG, "load_graph: null pointer or bad n");
  if (num_classes != c->dims[c->L]) return fail(c, GIST_E_SHAPE, "load_graph: num_classes != d_L");
  if (num_clusters < 1 || num_clusters > n) return fail(c, GIST_E_ARG, "load_graph: bad num_clusters");
  if (c->cfg.clusters_per_batch > num_clusters) return fail(c, GIST_E_ARG, "load_graph: q > num_clusters");
  if (row_ptr[0] != 0 || row_ptr[n] != nnz) return fail(c, GIST_E_ARG, "load_graph: row_ptr[0]/row_ptr[n] mismatch");
  // O(n) checks on the host; the O(nnz) edge checks (range, self loops, intra-cluster count)
  // run on the device after the upload (k_validate_edges)
  for (int64_t v = 0; v < n; ++v) {
    if (row_ptr[v + 1] < row_ptr[v]) return fail(c, GIST_E_ARG, "load_graph: row_ptr decreasing");
    if (cluster_ids[v] < 0 || cluster_ids[v] >= num_clusters)
      return fail(c, GIST_E_ARG, "load_graph: cluster id out of range");
    if (labels[v] < 0 || labels[v] >= num_classes) return fail(c, GIST_E_ARG, "load_graph: label out of range");
    if (split[v] > 3) return fail(c, GIST_E_ARG, "load_graph: split code > 3");
  }
  c->n = n;
  c->c = num_clusters;
  c->k = num_classes;
  // counting sort by cluster (stable in original id): new id -> original id
  std::vector<int64_t> csize(num_clusters, 0);
  for (int64_t v = 0; v < n; ++v) csize[cluster_ids[v]]++;
  c->cstart_h.assign(num_clusters + 1, 0);
  for (int j = 0; j < num_clusters; ++j) {
    if (csize[j] == 0) return fail(c, GIST_E_ARG, "load_graph: empty cluster " + std::to_string(j));
    c->cstart_h[j + 1] = c->cstart_h[j] + csize[j];
  }
  c->perm_h.assign(n, 0);
  std::vector<int32_t> inv(n), cid_new(n), lab_new(n);
  std::vector<uint8_t> split_new(n);
  {
    std::vector<int64_t> pos(c->cstart_h.begin(), c->cstart_h.end() - 1);
    for (int64_t v = 0; v < n; ++v) {
      const int64_t g = pos[cluster_ids[v]]++;
      c->perm_h[g] = (int32_t)v;
      inv[v] = (int32_t)g;
    }
  }
  for (int64_t g = 0; g < n; ++g) {
    const int32_t v = c->perm_h[g];
    cid_new[g] = cluster_ids[v];
    lab_new[g] = labels[v];
    split_new[g] = split[v];
  }
  // largest possible batch (sum of the q largest clusters) and its nnz bound (sum of q largest volumes)
  {
    std::vector<int64_t> sz(csize), vol(num_clusters, 0);
    for (int64_t v = 0; v < n; ++v) vol[cluster_ids[v]] += row_ptr[v + 1] - row_ptr[v];
    c->cvol_h = vol;
    std::sort(sz.rbegin(), sz.rend());
    std::sort(vol.rbegin(), vol.rend());
    int64_t a = 0, b = 0;
    for (int j = 0; j < c->cfg.clusters_per_batch; ++j) a += sz[j], b += vol[j];
    c->nb_max = (int)a;
    c->nnzb_max = b;
    c->max_csize = (int)sz[0];
  }
  cudaStream_t s = c->stream;
  // device copies of the original CSR, then relabel on the device
  int64_t *rp_o = nullptr;
  int32_t *col_o = nullptr, *perm_d = nullptr, *inv_d = nullptr;
  int64_t* deg_new = nullptr;
  TRY(dalloc_t(c, &rp_o, n + 1));
  TRY(dalloc_t(c, &col_o, std::max<int64_t>(nnz, 1)));
  TRY(dalloc_t(c, &perm_d, n));
  TRY(dalloc_t(c, &inv_d, n));
  TRY(dalloc_t(c, &deg_new, n + 1));
  TRY(dalloc_t(c, &c->rp, n + 1));
  CK(cudaMemcpyAsync(rp_o, row_ptr, (n + 1) * 8, cudaMemcpyHostToDevice, s));
  if (nnz > 0) CK(cudaMemcpyAsync(col_o, col_idx, nnz * 4, cudaMemcpyHostToDevice, s));
  {  // edge checks on the device (original ids and cluster ids)
    int32_t* cid_o = nullptr;
    unsigned long long* cnt = nullptr;
    TRY(dalloc_t(c, &cid_o, n));
    TRY(dalloc_t(c, &cnt, 5));
    CK(cudaMemcpyAsync(cid_o, cluster_ids, n * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(cnt, 0, 5 * sizeof(unsigned long long), s));
    LK(validate_edges(rp_o, col_o, cid_o, n, cnt, s));
    unsigned long long h[5] = {0, 0, 0, 0, 0};
    CK(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    dfree(c, cid_o);
    dfree(c, cnt);
    if (h[0] || h[3] || h[4]) {
      dfree(c, rp_o), dfree(c, col_o), dfree(c, perm_d), dfree(c, inv_d), dfree(c, deg_new);
      return fail(c, GIST_E_ARG, h[0] ? "load_graph: col_idx out of range"
                                 : h[3] ? "load_graph: col_idx not strictly increasing within a row (unsorted or duplicate edges)"
                                        : "load_graph: adjacency not symmetric (an edge (u,v) without (v,u))");
    }
    c->self_loops = (int64_t)h[1];
    c->nnz = nnz - c->self_loops;
    double sq = 0.0;
    for (int j = 0; j < num_clusters; ++j) sq += (double)csize[j] * (double)csize[j];
    c->block_density = sq > 0 ? (double)h[2] / sq : 0.0;
  }
  TRY(dalloc_t(c, &c->col, std::max<int64_t>(c->nnz, 1)));
  CK(cudaMemcpyAsync(perm_d, c->perm_h.data(), n * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(inv_d, inv.data(), n * 4, cudaMemcpyHostToDevice, s));
  c->h2d += (n + 1) * 8 + nnz * 4 + n * 8;
  LK(relabel_count(rp_o, col_o, perm_d, n, deg_new, s));
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, deg_new, c->rp, n + 1, s);
    void* tmp = nullptr;
    TRY(dalloc(c, &tmp, tb));
    CK(cudaMemsetAsync(deg_new + n, 0, 8, s));
    cub::DeviceScan::ExclusiveSum(tmp, tb, deg_new, c->rp, n + 1, s);
    ++c->nk;
    CK(cudaStreamSynchronize(s));
    dfree(c, tmp);
  }
  LK(relabel_fill(rp_o, col_o, perm_d, inv_d, c->rp, n, c->col, s));
  // features: X_new[g] = X[perm[g]], padded to pad8(d0), in the mode's element type
  const int d0 = c->dims[0];
  const int64_t ldx = pad8(d0);
  float* x_o = nullptr;
  TRY(dalloc_t(c, &x_o, (size_t)n * d0));
  CK(cudaMemcpyAsync(x_o, X, (size_t)n * d0 * 4, cudaMemcpyHostToDevice, s));
  c->h2d += (int64_t)n * d0 * 4;
  TRY(dalloc(c, &c->X, (size_t)n * ldx * esize(c)));
  if (c->prec == GIST_PREC_BF16)
    LK(gather_rows_f32<bf16>(x_o, d0, perm_d, n, d0, (bf16*)c->X, ldx, s));
  else
    LK(gather_rows_f32<float>(x_o, d0, perm_d, n, d0, (float*)c->X, ldx, s));
  TRY(dalloc_t(c, &c->cid, n));
  TRY(dalloc_t(c, &c->labels, n));
  TRY(dalloc_t(c, &c->split, n));
  TRY(dalloc_t(c, &c->cstart, num_clusters + 1));
  TRY(dalloc_t(c, &c->full_scale, n));
  CK(cudaMemcpyAsync(c->cid, cid_new.data(), n * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(c->labels, lab_new.data(), n * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(c->split, split_new.data(), n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(c->cstart, c->cstart_h.data(), (num_clusters + 1) * 8, cudaMemcpyHostToDevice, s));
  c->h2d += n * 9 + (num_clusters + 1) * 8;
  LK(full_graph_scales(c->rp, n, c->arch, c->full_scale, s));
  TRY(dalloc_t(c, &c->ccol, std::max<int64_t>(c->nnz, 1)));
  c->pack_ob = pack_bits(num_clusters, c->max_csize);
  if (c->pack_ob)
    LK(edge_codes(c->col, c->cid, c->cstart, c->nnz, c->pack_ob, c->ccol, s));
  else
    LK(edge_clusters(c->col, c->cid, c->nnz, c->ccol, s));
  // Block-diagonal tensor-core aggregation: GraphSAGE in BF16 mode when the
  // clusters are small (<= 256 rows) and their intra-cluster blocks dense enough (>= 5%).
  // GIST_BD=0/1 overrides the choice.
  {
    const char* env = std::getenv("GIST_BD");
    const int bs = (int)pad8(c->max_csize);
    const double bytes = (double)num_clusters * bs * bs * 2.0;
    bool want = c->arch == GIST_ARCH_SAGE && c->prec == GIST_PREC_BF16 && c->max_csize <= 256 &&
                c->cfg.clusters_per_batch <= 64 && c->block_density >= 0.05 && bytes <= 8e9;
    if (env)
      want = env[0] == '1' && c->arch == GIST_ARCH_SAGE && c->prec == GIST_PREC_BF16 && c->max_csize <= 256 &&
             c->cfg.clusters_per_batch <= 64;
    if (want) {
      c->bs = bs;
      TRY(dalloc_t(c, &c->blocks, (size_t)num_clusters * bs * bs));
      CK(cudaMemsetAsync(c->blocks, 0, (size_t)num_clusters * bs * bs * 2, s));
      LK(cluster_blocks(c->rp, c->col, c->cid, c->cstart, n, bs, c->blocks, s));
      c->bd = true;
    }
  }
  CK(cudaStreamSynchronize(s));
  TRY(check_launch(c, "load_graph"));
  dfree(c, rp_o);
  dfree(c, col_o);
  dfree(c, perm_d);
  dfree(c, inv_d);
  dfree(c, deg_new);
  dfree(c, x_o);
  // global parameter storage (physical layout)
  c->theta.assign(c->L, nullptr);
  c->th_K.assign(c->L, 0);
  c->th_N.assign(c->L, 0);
  if (c->cfg.agg_mode == GIST_AGG_P2P || c->cfg.agg_mode == GIST_AGG_SYMM) TRY(p2p_setup(c));
  c->sh_lo.assign(c->L, 0);
  c->sh_hi.assign(c->L, 0);
  for (int l = 0; l < c->L; ++l) {
    c->th_K[l] = kphys(c, c->dims[l]);
    c->th_N[l] = pad8(c->dims[l + 1]);
    c->sh_hi[l] = c->th_K[l];
    if (sharded(c)) {  // this rank's physical rows of Theta_l
      c->sh_lo[l] = shard_lo(c, l, c->cfg.rank);
      c->sh_hi[l] = shard_lo(c, l, c->cfg.rank + 1);
      if (c->arch == GIST_ARCH_GAT && l + 1 == c->L) {  // R21 mean: both attention rows on one rank
        for (int r = 1; r < c->cfg.world_size; ++r)
          if (shard_lo(c, l, r) == pad8(c->dims[l]) + 1)
            return fail(c, GIST_E_UNSUPPORTED, "sharded GAT: a shard boundary splits the attention rows");
      }
    }
    const size_t n = (size_t)rows_here(c, l) * c->th_N[l];
    if (!c->p2p_base) TRY(dalloc_t(c, &c->theta[l], std::max<size_t>(n, 1)));
    CK(cudaMemsetAsync(c->theta[l], 0, n * 4, s));
    if (persistent_adam(c) && !c->p2p_base) {  // f3: global moments, same physical layout as Theta
      c->theta_m.resize(c->L, nullptr);
      c->theta_v.resize(c->L, nullptr);
      TRY(dalloc_t(c, &c->theta_m[l], std::max<size_t>(n, 1)));
      TRY(dalloc_t(c, &c->theta_v[l], std::max<size_t>(n, 1)));
    }
  }
  c->state = S_GRAPH;
  return GIST_OK;
}

// ============================================================= params =====
extern "C" gist_status gist_init_params(gist_ctx* c, uint64_t seed) {
  PRE(c);
  Range nvtx_range("gist_init_params");
  if (c->state == S_CREATED || c->state == S_PARTITIONED) return fail(c, GIST_E_STATE, "init_params: bad state");
  for (int l = 0; l < (int)c->theta_m.size(); ++l) {  // f3: moments restart with the parameters
    CK(cudaMemsetAsync(c->theta_m[l], 0, (size_t)rows_here(c, l) * c->th_N[l] * 4, c->stream));
    CK(cudaMemsetAsync(c->theta_v[l], 0, (size_t)rows_here(c, l) * c->th_N[l] * 4, c->stream));
  }
  c->adam_t = 0;
  for (int l = 0; l < c->L; ++l) {
    const int rows = wrows(c, c->dims[l]);
    const int cols = c->dims[l + 1];
    const int fan_in = c->arch == GIST_ARCH_GAT ? c->dims[l] : rows;  // R21: GAT fan_in = d_l
    const float sc = std::sqrt(6.0f / (float)(fan_in + cols));  // fp32, correctly rounded (R11)
    LK(glorot_init(c->theta[l], rows, cols, two_blocks(c), c->dims[l], (int)pad8(c->dims[l]),
                   c->th_N[l], (uint32_t)l, seed, sc, c->stream, c->sh_lo[l], c->sh_hi[l]));
  }
  TRY(check_launch(c, "init_params"));
  c->layer_set.assign(c->L, 1);
  c->state = S_PARAMS;
  return GIST_OK;
}

static int64_t logical_to_phys_row(const gist_ctx* c, int l, int64_t r) {
  if (two_blocks(c) && r >= c->dims[l]) return pad8(c->dims[l]) + (r - c->dims[l]);
  return r;
}

extern "C" gist_status gist_get_params(gist_ctx* c, int32_t layer, float* out) {
  PRE(c);
  if (c->state == S_CREATED) return fail(c, GIST_E_STATE, "get_params: no graph");
  if (layer < 0 || layer >= c->L || !out) return GIST_E_ARG;
  const int64_t K = c->th_K[layer], N = c->th_N[layer];
  std::vector<float> buf(K * N);
  if (sharded(c)) {  // collective: the layer's rows from every rank
    float* full = nullptr;
    TRY(dalloc_t(c, &full, (size_t)K * N));
    const gist_status st = shard_gather_layer(c, c->theta[layer], layer, full, c->stream);
    if (st == GIST_OK) CK(cudaMemcpyAsync(buf.data(), full, K * N * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    dfree(c, full);
    TRY(st);
  } else {
    CK(cudaMemcpyAsync(buf.data(), c->theta[layer], K * N * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  const int64_t rows = wrows(c, c->dims[layer]);
  const int64_t cols = c->dims[layer + 1];
  for (int64_t r = 0; r < rows; ++r)
    std::memcpy(out + r * cols, buf.data() + logical_to_phys_row(c, layer, r) * N, cols * 4);
  return GIST_OK;
}

extern "C" gist_status gist_set_params(gist_ctx* c, int32_t layer, const float* in) {
  PRE(c);
  if (c->state == S_CREATED || c->state == S_PARTITIONED) return fail(c, GIST_E_STATE, "set_params: bad state");
  if (layer < 0 || layer >= c->L || !in) return GIST_E_ARG;
  const int64_t N = c->th_N[layer];
  const int64_t lo = c->sh_lo[layer], K = rows_here(c, layer);  // this rank's physical rows
  std::vector<float> buf(K * N, 0.f);
  const int64_t rows = wrows(c, c->dims[layer]);
  const int64_t cols = c->dims[layer + 1];
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t pr = logical_to_phys_row(c, layer, r);
    if (pr >= lo && pr < lo + K) std::memcpy(buf.data() + (pr - lo) * N, in + r * cols, cols * 4);
  }
  CK(cudaMemcpyAsync(c->theta[layer], buf.data(), K * N * 4, cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->h2d += K * N * 4;
  // the parameters become valid (PARAMS) once every layer was set since the graph load, or
  // init_params ran: a partially set model cannot be trained
  c->layer_set.resize(c->L, 0);
  c->layer_set[layer] = 1;
  if (std::all_of(c->layer_set.begin(), c->layer_set.end(), [](uint8_t v) { return v != 0; })) c->state = S_PARAMS;
  return GIST_OK;
}

// ============================================================ checkpoint ===
// SPEC.md "External Interfaces": "GIST", version u32, arch u8, L u32, dims u32[L+1], then the
// weights row-major f32 (logical layout, layer by layer).  Little-endian hosts only (x86 / ARM).
extern "C" gist_status gist_save_checkpoint(gist_ctx* c, const char* path) {
  PRE(c);
  if (c->state != S_PARAMS) return fail(c, GIST_E_STATE, "save_checkpoint: needs parameters and no open round");
  if (!path) return fail(c, GIST_E_ARG, "save_checkpoint: null path");
  std::string buf("GIST", 4);
  auto put = [&](const void* p, size_t n) { buf.append(static_cast<const char*>(p), n); };
  const uint32_t version = 1, L = (uint32_t)c->L;
  const uint8_t arch = (uint8_t)c->arch;
  put(&version, 4);
  put(&arch, 1);
  put(&L, 4);
  for (int l = 0; l <= c->L; ++l) {
    const uint32_t d = (uint32_t)c->dims[l];
    put(&d, 4);
  }
  for (int l = 0; l < c->L; ++l) {
    std::vector<float> w((size_t)wrows(c, c->dims[l]) * c->dims[l + 1]);
    TRY(gist_get_params(c, l, w.data()));
    put(w.data(), w.size() * 4);
  }
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(c, GIST_E_ARG, std::string("save_checkpoint: cannot open ") + path);
  const size_t wr = std::fwrite(buf.data(), 1, buf.size(), f);
  const int cl = std::fclose(f);
  if (wr != buf.size() || cl != 0) return fail(c, GIST_E_ARG, "save_checkpoint: short write");
  return GIST_OK;
}

extern "C" gist_status gist_load_checkpoint(gist_ctx* c, const char* path) {
  PRE(c);
  if (c->state == S_CREATED || c->state == S_PARTITIONED)
    return fail(c, GIST_E_STATE, "load_checkpoint: needs a graph and no open round");
  if (!path) return fail(c, GIST_E_ARG, "load_checkpoint: null path");
  FILE* f = std::fopen(path, "rb");
  if (!f) return fail(c, GIST_E_ARG, std::string("load_checkpoint: cannot open ") + path);
  std::string buf;
  char tmp[1 << 16];
  size_t got;
  while ((got = std::fread(tmp, 1, sizeof(tmp), f)) > 0) buf.append(tmp, got);
  std::fclose(f);
  size_t pos = 0;
  auto take = [&](void* p, size_t n) {
    if (pos + n > buf.size()) return false;
    std::memcpy(p, buf.data() + pos, n);
    pos += n;
    return true;
  };
  char magic[4];
  uint32_t version = 0, L = 0;
  uint8_t arch = 0;
  if (!take(magic, 4) || std::memcmp(magic, "GIST", 4) != 0 || !take(&version, 4) || version != 1 ||
      !take(&arch, 1) || !take(&L, 4))
    return fail(c, GIST_E_ARG, "load_checkpoint: not a GIST checkpoint (magic / version)");
  if ((int)arch != c->arch || (int)L != c->L) return fail(c, GIST_E_SHAPE, "load_checkpoint: arch or depth differs");
  for (int l = 0; l <= c->L; ++l) {
    uint32_t d = 0;
    if (!take(&d, 4)) return fail(c, GIST_E_ARG, "load_checkpoint: truncated header");
    if ((int)d != c->dims[l]) return fail(c, GIST_E_SHAPE, "load_checkpoint: dims differ");
  }
  std::vector<std::vector<float>> w(c->L);
  for (int l = 0; l < c->L; ++l) {
    w[l].resize((size_t)wrows(c, c->dims[l]) * c->dims[l + 1]);
    if (!take(w[l].data(), w[l].size() * 4)) return fail(c, GIST_E_ARG, "load_checkpoint: truncated weights");
  }
  if (pos != buf.size()) return fail(c, GIST_E_ARG, "load_checkpoint: trailing bytes");
  for (int l = 0; l < c->L; ++l) TRY(gist_set_params(c, l, w[l].data()));
  return GIST_OK;
}

// ====================================================== inspection hooks ===
extern "C" gist_status gist_sub_shape(gist_ctx* c, int32_t slot, int32_t layer, int64_t* rows, int64_t* cols) {
  PRE(c);
  if (c->state != S_PARTITIONED) return fail(c, GIST_E_STATE, "sub_shape: no open round");
  if (slot < 0 || slot >= c->m || layer < 0 || layer >= c->L) return GIST_E_ARG;
  const LayerShape& sh = c->shapes[slot][layer];
  if (rows) *rows = wrows(c, sh.nrows);
  if (cols) *cols = sh.ncols;
  return GIST_OK;
}

static Slot* local_slot(gist_ctx* c, int slot) {
  for (Slot& s : c->slots)
    if (s.index == slot) return &s;
  return nullptr;
}

// physical packed block -> logical row-major
static void phys_to_logical(const gist_ctx* c, const LayerShape& sh, const std::vector<float>& buf, float* out) {
  const int rows = wrows(c, sh.nrows);
  for (int r = 0; r < rows; ++r) {
    const int p = (two_blocks(c) && r >= sh.nrows) ? sh.half + (r - sh.nrows) : r;
    std::memcpy(out + (size_t)r * sh.ncols, buf.data() + (size_t)p * sh.Np, (size_t)sh.ncols * 4);
  }
}

extern "C" gist_status gist_get_sub_params(gist_ctx* c, int32_t slot, int32_t layer, float* out) {
  PRE(c);
  if (c->state != S_PARTITIONED) return fail(c, GIST_E_STATE, "get_sub_params: no open round");
  if (layer < 0 || layer >= c->L || !out) return GIST_E_ARG;
  Slot* sl = local_slot(c, slot);
  if (!sl) return fail(c, GIST_E_ARG, "get_sub_params: slot not on this rank");
  const LayerShape& sh = c->shapes[slot][layer];
  std::vector<float> buf((size_t)sh.Kp * sh.Np);
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(buf.data(), sl->W + sh.off, buf.size() * 4, cudaMemcpyDeviceToHost));
  phys_to_logical(c, sh, buf, out);
  return GIST_OK;
}

template <typename T>
static void copy_rows_out(const void* dev, int nb, int64_t ld, int w, float* out) {
  std::vector<T> buf((size_t)nb * ld);
  cudaMemcpy(buf.data(), dev, buf.size() * sizeof(T), cudaMemcpyDeviceToHost);
  for (int v = 0; v < nb; ++v)
    for (int j = 0; j < w; ++j) {
      if constexpr (sizeof(T) == 4) out[(size_t)v * w + j] = (float)buf[(size_t)v * ld + j];
      else out[(size_t)v * w + j] = __bfloat162float(buf[(size_t)v * ld + j]);
    }
}

extern "C" gist_status gist_get_trace(gist_ctx* c, int32_t slot, int32_t what, int32_t layer, void* out,
                                      int64_t* count) {
  PRE(c);
  if (c->state != S_PARTITIONED) return fail(c, GIST_E_STATE, "get_trace: no open round");
  Slot* sl = local_slot(c, slot);
  if (!sl) return fail(c, GIST_E_ARG, "get_trace: slot not on this rank");
  CK(cudaStreamSynchronize(c->stream));
  const int nb = sl->last_nb;
  const auto& shp = c->shapes[slot];
  int64_t cnt = 0;
  switch (what) {
    case GIST_TRACE_NODES: {
      cnt = nb;
      if (out) {
        std::vector<int32_t> b(nb);
        CK(cudaMemcpy(b.data(), sl->b_nodes, (size_t)nb * 4, cudaMemcpyDeviceToHost));
        for (int v = 0; v < nb; ++v) ((int32_t*)out)[v] = c->perm_h[b[v]];
      }
      break;
    }
    case GIST_TRACE_ACT: {
      if (layer < 1 || layer >= c->L) return GIST_E_ARG;
      const LayerShape& sh = shp[layer];
      cnt = (int64_t)nb * sh.nrows;
      if (out) {
        const void* src = c->arch == GIST_ARCH_SAGE ? sl->C[layer] : sl->H[layer];
        const int64_t ld = c->arch == GIST_ARCH_GAT ? sh.half : sh.Kp;
        if (c->prec == GIST_PREC_BF16) copy_rows_out<bf16>(src, nb, ld, sh.nrows, (float*)out);
        else copy_rows_out<float>(src, nb, ld, sh.nrows, (float*)out);
      }
      break;
    }
    case GIST_TRACE_LOGITS: {
      const LayerShape& sh = shp[c->L - 1];
      cnt = (int64_t)nb * c->k;
      if (out) copy_rows_out<float>(sl->logits, nb, sh.Np, c->k, (float*)out);
      break;
    }
    case GIST_TRACE_GRAD: {
      if (layer < 0 || layer >= c->L) return GIST_E_ARG;
      const LayerShape& sh = shp[layer];
      cnt = (int64_t)wrows(c, sh.nrows) * sh.ncols;
      if (out) {
        std::vector<float> buf((size_t)sh.Kp * sh.Np);
        CK(cudaMemcpy(buf.data(), sl->G + sh.off, buf.size() * 4, cudaMemcpyDeviceToHost));
        phys_to_logical(c, sh, buf, (float*)out);
      }
      break;
    }
    case GIST_TRACE_LOSS: {
      cnt = 1;
      if (out) CK(cudaMemcpy(out, sl->step_loss, 4, cudaMemcpyDeviceToHost));
      break;
    }
    default:
      return GIST_E_ARG;
  }
  if (count) *count = cnt;
  return GIST_OK;
}

// ============================================================ profiling ===
extern "C" gist_status gist_profile(gist_ctx* c, int32_t stride) {
  PRE(c);
  if (stride < 0) return GIST_E_ARG;
  prof_flush(c);
  c->prof_stride = stride;
  for (int k = 0; k < GIST_PROF_N; ++k) c->prof_ms[k] = c->prof_work[k] = 0.0, c->prof_n[k] = 0;
  if (stride > 0 && !c->nnz_pin) {
    c->nnz_pin_cap = 1 << 16;
    CK(cudaMallocHost(&c->nnz_pin, (size_t)c->nnz_pin_cap * 8));
  }
  return GIST_OK;
}

extern "C" gist_status gist_profile_get(gist_ctx* c, int32_t cls, double* ms, int64_t* launches, double* work) {
  PRE(c);
  if (cls < 0 || cls >= GIST_PROF_N) return GIST_E_ARG;
  prof_flush(c);
  if (ms) *ms = c->prof_ms[cls];
  if (launches) *launches = c->prof_n[cls];
  if (work) *work = c->prof_work[cls];
  return GIST_OK;
}

// ===================================================== kernel entry points =
extern "C" gist_status gist_spmm(const int64_t* row_ptr_dev, const int32_t* col_dev, int64_t rows,
                                 const float* rowscale_dev, const float* colscale_dev, int32_t self, const void* H_dev,
                                 void* out_dev, int64_t w, int64_t ld, int32_t dtype, void* stream) {
  if (!row_ptr_dev || !H_dev || !out_dev || w < 0 || ld < w || (ld % 8) != 0) return GIST_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == 0) {
    SpmmArgs<float, float> a;
    a.row_beg = row_ptr_dev; a.row_end = row_ptr_dev + 1; a.col = col_dev; a.rows = rows; a.rowscale = rowscale_dev; a.colscale = colscale_dev;
    a.self = self; a.H = (const float*)H_dev; a.ldh = ld; a.out = (float*)out_dev; a.ldo = ld; a.w = pad8(w);
    spmm<float, float>(a, s);
  } else if (dtype == 1) {
    SpmmArgs<bf16, bf16> a;
    a.row_beg = row_ptr_dev; a.row_end = row_ptr_dev + 1; a.col = col_dev; a.rows = rows; a.rowscale = rowscale_dev; a.colscale = colscale_dev;
    a.self = self; a.H = (const bf16*)H_dev; a.ldh = ld; a.out = (bf16*)out_dev; a.ldo = ld; a.w = pad8(w);
    spmm<bf16, bf16>(a, s);
  } else {
    return GIST_E_ARG;
  }
  return cudaGetLastError() == cudaSuccess ? GIST_OK : GIST_E_CUDA;
}

extern "C" gist_status gist_gemm(int32_t transA, int32_t transB, int64_t M, int64_t N, int64_t K, const void* A_dev,
                                 int64_t lda, const void* B_dev, int64_t ldb, void* C_dev, int64_t ldc, int32_t dtype,
                                 int32_t out_f32, int32_t relu, void* stream) {
  return gist_gemm_reps(transA, transB, M, N, K, A_dev, lda, B_dev, ldb, C_dev, ldc, dtype, out_f32, relu, stream, 1);
}

extern "C" gist_status gist_gemm_reps(int32_t transA, int32_t transB, int64_t M, int64_t N, int64_t K,
                                      const void* A_dev, int64_t lda, const void* B_dev, int64_t ldb, void* C_dev,
                                      int64_t ldc, int32_t dtype, int32_t out_f32, int32_t relu, void* stream,
                                      int32_t reps) {
  if (!A_dev || !B_dev || !C_dev || M < 0 || N < 0 || K < 0 || reps < 1) return GIST_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == 0) {
    for (int r = 0; r < reps; ++r)
      gemm_f32(transA, transB, M, N, K, (const float*)A_dev, lda, (const float*)B_dev, ldb, (float*)C_dev, ldc, relu, s);
  } else if (dtype == 1) {
    if (!gemm_bf16(transA, transB, M, N, K, (const bf16*)A_dev, lda, (const bf16*)B_dev, ldb, C_dev, ldc, out_f32,
                   relu, s, reps))
      return GIST_E_UNSUPPORTED;
  } else if (dtype == 2) {  // TF32 tensor cores: fp32 in, fp32 out
    if (!gemm_tf32(transA, transB, M, N, K, (const float*)A_dev, lda, (const float*)B_dev, ldb, (float*)C_dev, ldc,
                   relu, s, reps))
      return GIST_E_UNSUPPORTED;
  } else {
    return GIST_E_ARG;
  }
  return cudaGetLastError() == cudaSuccess ? GIST_OK : GIST_E_CUDA;
}
