// round.cu -- the per-round steps of Algorithm 1 around subTrain: subGCNs
// (gist_partition: partition keys, sort, blocks, extract, optimizer-state reset; R5, R6, R8) with
// the slot buffers it sizes, and subAgg (gist_aggregate: the collective and the scatter into the
// global model, R9; P2P / SYMM peer stores).
#include "ctx.h"

using namespace gist;
using namespace gist_impl;

// ============================================================ partition ===
namespace gist_impl {
gist_status alloc_slots(gist_ctx* c, int m) {
  free_slots(c);
  for (void* p : {(void*)c->Wall, (void*)c->Gall, (void*)c->Mall, (void*)c->Vall, (void*)c->Wball, (void*)c->Wrecv})
    dfree(c, p);
  c->Wall = c->Gall = c->Mall = c->Vall = c->Wrecv = nullptr;
  c->Wball = nullptr;
  const int W = c->cfg.world_size, r = c->cfg.rank;
  c->slots_per_rank = gist_slots_per_rank(m, W);
  // largest packed slot (every hidden block at ceil(d/m))
  int64_t smax = 0;
  std::vector<int> maxK(c->L), maxN(c->L);
  for (int l = 0; l < c->L; ++l) {
    const int nr = (l == 0) ? c->dims[0] : hidden_block_max(c, l, m);
    const int nc = (l + 1 == c->L) ? c->dims[c->L] : hidden_block_max(c, l + 1, m);
    maxK[l] = (int)kphys(c, nr);
    maxN[l] = (int)pad8(nc);
    smax += (int64_t)maxK[l] * maxN[l];
  }
  c->S_max = smax;
  const size_t tot = (size_t)c->slots_per_rank * smax;
  TRY(dalloc_t(c, &c->Wall, tot));
  TRY(dalloc_t(c, &c->Gall, tot));
  CK(cudaMemsetAsync(c->Wall, 0, tot * 4, c->stream));
  CK(cudaMemsetAsync(c->Gall, 0, tot * 4, c->stream));
  if (c->cfg.optimizer == GIST_OPT_ADAM) {
    TRY(dalloc_t(c, &c->Mall, tot));
    TRY(dalloc_t(c, &c->Vall, tot));
  }
  if (c->prec == GIST_PREC_BF16) {
    TRY(dalloc_t(c, &c->Wball, tot));
    CK(cudaMemsetAsync(c->Wball, 0, tot * 2, c->stream));
  }
  if (W > 1 && c->cfg.agg_mode == GIST_AGG_ALLGATHER && !sharded(c)) TRY(dalloc_t(c, &c->Wrecv, (size_t)W * tot));
  if (c->xscr) dfree(c, c->xscr);
  c->xscr = nullptr;
  if (sharded(c)) TRY(dalloc_t(c, &c->xscr, (size_t)m * smax));  // every slot's packed rows (owned rows only)
  if (c->bctr) dfree(c, c->bctr);
  TRY(dalloc_t(c, &c->bctr, 2 * (size_t)std::max(c->slots_per_rank, 1)));
  if (!c->dstate) {
    TRY(dalloc_t(c, &c->dstate, 1));
    CK(cudaMallocHost(&c->hstate, sizeof(StepState)));
    CK(cudaEventCreateWithFlags(&c->hstate_ev, cudaEventDisableTiming));
  }
  const int nbm = std::max(c->nb_max, 1);
  c->nb_max_rows = nbm;
  const size_t E = esize(c);
  int maxKall = 0;
  for (int l = 0; l < c->L; ++l) maxKall = std::max(maxKall, maxK[l]);
  for (int i = r, j = 0; i < m; i += W, ++j) {
    c->slots.emplace_back();
    Slot& s = c->slots.back();
    s.index = i;
    s.W = c->Wall + (size_t)j * smax;
    s.G = c->Gall + (size_t)j * smax;
    if (c->Mall) s.M = c->Mall + (size_t)j * smax, s.V = c->Vall + (size_t)j * smax;
    if (c->Wball) s.Wb = c->Wball + (size_t)j * smax;
    TRY(dalloc_t(c, &s.b_nodes, nbm));
    TRY(dalloc_t(c, &s.lab_b, nbm));
    TRY(dalloc_t(c, &s.train_b, nbm));
    TRY(dalloc_t(c, &s.scale, nbm));
    TRY(dalloc_t(c, &s.b_beg, nbm));
    TRY(dalloc_t(c, &s.b_end, nbm));
    TRY(dalloc_t(c, &s.stats, 4));  // [0] nnz_b, [1] train rows, [2] batch-build row counter
    TRY(dalloc_t(c, &s.b_col, std::max<int64_t>(c->nnzb_max, 1)));
    TRY(dalloc_t(c, &s.map64, c->c));
    CK(cudaMemsetAsync(s.map64, 0, (size_t)c->c * 8, c->stream));  // tag 0 = never in a batch
    s.C.assign(c->L, nullptr);
    s.H.assign(c->L, nullptr);
    s.dZ.assign(c->L, nullptr);
    s.mb.assign(c->L, nullptr);
    c->mb_ld.assign(c->L, 0);
    for (int l = 1; l < c->L && c->prec == GIST_PREC_BF16; ++l) {
      c->mb_ld[l] = cdiv(maxK[l], 32);
      TRY(dalloc_t(c, &s.mb[l], (size_t)nbm * c->mb_ld[l]));
      CK(cudaMemsetAsync(s.mb[l], 0, (size_t)nbm * c->mb_ld[l] * 4, c->stream));
    }
    for (int l = 0; l < c->L; ++l) {  // zero-initialised: padding columns must read as 0
      TRY(dalloc(c, &s.C[l], (size_t)nbm * maxK[l] * E));
      CK(cudaMemsetAsync(s.C[l], 0, (size_t)nbm * maxK[l] * E, c->stream));
      if (c->arch == GIST_ARCH_GCN && l > 0) {
        TRY(dalloc(c, &s.H[l], (size_t)nbm * maxK[l] * E));
        CK(cudaMemsetAsync(s.H[l], 0, (size_t)nbm * maxK[l] * E, c->stream));
      }
      if (c->arch == GIST_ARCH_GAT) {  // H_l (layer 0: the gathered X_b rows), Z_l, scalars
        const size_t kw = (size_t)(maxK[l] - 8);  // pad8 of the widest input slice
        TRY(dalloc(c, &s.H[l], (size_t)nbm * kw * E));
        CK(cudaMemsetAsync(s.H[l], 0, (size_t)nbm * kw * E, c->stream));
        s.gZ.resize(c->L, nullptr);
        s.gsc.resize(c->L, nullptr);
        TRY(dalloc(c, &s.gZ[l], (size_t)nbm * maxN[l] * E));
        CK(cudaMemsetAsync(s.gZ[l], 0, (size_t)nbm * maxN[l] * E, c->stream));
        TRY(dalloc_t(c, &s.gsc[l], (size_t)6 * nbm + 2 * kw + (size_t)2 * kGatDaChunks * maxN[l]));
      }
      TRY(dalloc(c, &s.dZ[l], (size_t)nbm * maxN[l] * E));
      CK(cudaMemsetAsync(s.dZ[l], 0, (size_t)nbm * maxN[l] * E, c->stream));
    }
    // (only where it pays: the last layer's input slice is >= 256 wide; measured neutral to
    // slightly negative on the Cora-shaped C1 with a 128-wide slice)
    // GIST_REASSOC=1 / 0 forces it on / off (tests exercise both on small shapes)
    const int last_in = c->arch == GIST_ARCH_SAGE ? maxK[c->L - 1] / 2 : maxK[c->L - 1];
    c->reassoc = c->prec == GIST_PREC_BF16 && c->L >= 2 && last_in >= 256;
    if (const char* e = std::getenv("GIST_REASSOC")) c->reassoc = c->prec == GIST_PREC_BF16 && c->L >= 2 && e[0] == '1';
    if (c->arch == GIST_ARCH_GAT) c->reassoc = false;
    if (c->reassoc) {
      const size_t npl = (size_t)maxN[c->L - 1];
      TRY(dalloc(c, &s.rP, (size_t)nbm * npl * E));
      TRY(dalloc(c, &s.rAGG, (size_t)nbm * npl * E));
      TRY(dalloc(c, &s.rDQ, (size_t)nbm * 2 * npl * E));
      TRY(dalloc(c, &s.rDZs, (size_t)nbm * 2 * npl * E));
      TRY(dalloc(c, &s.rWc, (size_t)maxK[c->L - 1] * npl * E));
      CK(cudaMemsetAsync(s.rP, 0, (size_t)nbm * npl * E, c->stream));
      CK(cudaMemsetAsync(s.rAGG, 0, (size_t)nbm * npl * E, c->stream));
      CK(cudaMemsetAsync(s.rDQ, 0, (size_t)nbm * 2 * npl * E, c->stream));
      CK(cudaMemsetAsync(s.rDZs, 0, (size_t)nbm * 2 * npl * E, c->stream));
    }
    if (c->arch == GIST_ARCH_GAT) {
      int gw = 0;
      for (int l = 0; l < c->L; ++l) gw = std::max(gw, maxN[l]);
      TRY(dalloc(c, &s.gG, (size_t)nbm * gw * E));  // dlogits, then dH of each layer
      CK(cudaMemsetAsync(s.gG, 0, (size_t)nbm * gw * E, c->stream));
    }
    TRY(dalloc(c, &s.dC, (size_t)nbm * maxKall * E));
    CK(cudaMemsetAsync(s.dC, 0, (size_t)nbm * maxKall * E, c->stream));
    TRY(dalloc_t(c, &s.logits, (size_t)nbm * maxN[c->L - 1]));
    CK(cudaMemsetAsync(s.logits, 0, (size_t)nbm * maxN[c->L - 1] * 4, c->stream));
    TRY(dalloc_t(c, &s.row_loss, nbm));
    TRY(dalloc_t(c, &s.ce_done, 1));
    CK(cudaMemsetAsync(s.ce_done, 0, 4, c->stream));
    TRY(dalloc_t(c, &s.step_loss, 1));
    TRY(dalloc_t(c, &s.loss_acc, 1));
  }
  c->alloc_m = m;
  return GIST_OK;
}
}  // namespace gist_impl

extern "C" gist_status gist_partition(gist_ctx* c, uint64_t seed, int32_t m) {
  PRE(c);
  Range nvtx_range("gist_partition");
  if (c->state != S_PARAMS) return fail(c, GIST_E_STATE, "partition: needs params and no open round");
  if (m < 1) return fail(c, GIST_E_ARG, "partition: m < 1");
  if (c->arch == GIST_ARCH_GAT && m > kMaxMean) return fail(c, GIST_E_ARG, "partition: GAT supports m <= 128");
  for (int l = 1; l < c->L; ++l)
    if (m > c->dims[l]) return fail(c, GIST_E_ARG, "partition: m exceeds hidden dim " + std::to_string(l));
  cudaStream_t s = c->stream;
  if (m != c->alloc_m) TRY(alloc_slots(c, m));
  c->prof_now = c->prof_stride > 0;
  c->m = m;
  // subGCNs keys / sort / blocks for every hidden dim (R5)
  int dmax = 0;
  for (int l = 1; l < c->L; ++l) dmax = std::max(dmax, c->dims[l]);
  if (c->units.empty()) {
    c->units.assign(c->L + 1, nullptr);
    for (int l = 1; l < c->L; ++l) TRY(dalloc_t(c, &c->units[l], c->dims[l]));
    if (dmax > 0) {
      TRY(dalloc_t(c, &c->keys_a, dmax));
      TRY(dalloc_t(c, &c->keys_b, dmax));
      TRY(dalloc_t(c, &c->idx_a, dmax));
      TRY(dalloc_t(c, &c->idx_b, dmax));
      TRY(dalloc_t(c, &c->blk, dmax));
      c->sort_tmp_bytes = partition_sort(c->keys_a, c->keys_b, c->idx_a, c->idx_b, dmax, nullptr, 0, s);
      TRY(dalloc(c, &c->sort_tmp, c->sort_tmp_bytes));
    }
  }
  if (c->offs_dev) dfree(c, c->offs_dev);
  TRY(dalloc_t(c, &c->offs_dev, (size_t)(m + 1) * (c->L + 1)));
  c->offs.assign(c->L + 1, std::vector<int32_t>());
  std::vector<int32_t> offs_all((size_t)(m + 1) * (c->L + 1), 0);
  for (int l = 0; l <= c->L; ++l) {
    const int d = c->dims[l];
    std::vector<int32_t>& o = c->offs[l];
    o.assign(m + 1, 0);
    if (l == 0 || l == c->L) {
      for (int i = 0; i <= m; ++i) o[i] = 0;  // unused: identity
      continue;
    }
    const int base = d / m, extra = d % m;
    for (int i = 0; i < m; ++i) o[i + 1] = o[i] + base + (i < extra ? 1 : 0);
    std::copy(o.begin(), o.end(), offs_all.begin() + (size_t)l * (m + 1));
  }
  CK(cudaMemcpyAsync(c->offs_dev, offs_all.data(), offs_all.size() * 4, cudaMemcpyHostToDevice, s));
  for (int l = 1; l < c->L; ++l) {
    const int d = c->dims[l];
    PL(GIST_PROF_PARTITION, d * 12.0, s, partition_keys(d, (uint32_t)c->round, (uint32_t)l, seed, c->keys_a, c->idx_a, s));
    PL(GIST_PROF_PARTITION, d * 24.0, s,
       partition_sort(c->keys_a, c->keys_b, c->idx_a, c->idx_b, d, c->sort_tmp, c->sort_tmp_bytes, s));
    PL(GIST_PROF_PARTITION, d * 8.0, s, partition_assign(c->idx_b, d, m, c->blk, s));
    PL(GIST_PROF_PARTITION, d * 4.0 * (m + 1), s,
       partition_compact(c->blk, d, m, c->offs_dev + (size_t)l * (m + 1), c->units[l], s));
  }
  // shapes of every slot (all ranks know the full partition)
  c->shapes.assign(m, std::vector<LayerShape>(c->L));
  for (int i = 0; i < m; ++i) {
    int64_t off = 0;
    for (int l = 0; l < c->L; ++l) {
      LayerShape& sh = c->shapes[i][l];
      sub_logical(c, i, l, &sh.nrows, &sh.ncols);
      sh.half = (int)pad8(sh.nrows);
      sh.Kp = (int)kphys(c, sh.nrows);
      sh.Np = (int)pad8(sh.ncols);
      sh.off = off;
      off += (int64_t)sh.Kp * sh.Np;
      sh.rows = (l == 0) ? nullptr : c->units[l] + c->offs[l][i];
      sh.cols = (l + 1 == c->L) ? nullptr : c->units[l + 1] + c->offs[l + 1][i];
    }
  }
  // extract Theta^(i) for local slots (R6), reset optimizer state (R8)
  if (sharded(c)) TRY(shard_extract(c));  // owner-sharded Theta: the rows come from their owners
  for (Slot& sl : c->slots) {
    if (sharded(c)) break;
    const auto& shp = c->shapes[sl.index];
    for (int l = 0; l < c->L; ++l) {
      const LayerShape& sh = shp[l];
      LayerMap mp;
      mp.rows = sh.rows; mp.nrows = sh.nrows; mp.sage = c->arch == GIST_ARCH_SAGE; mp.gat = c->arch == GIST_ARCH_GAT; mp.half = sh.half;
      mp.glob_half = (int)pad8(c->dims[l]); mp.cols = sh.cols; mp.ncols = sh.ncols; mp.Kp = sh.Kp; mp.Np = sh.Np;
      mp.ldg = c->th_N[l];
      PL(GIST_PROF_PARTITION, (double)sh.Kp * sh.Np * 12.0, s, extract_sub(c->theta[l], mp, sl.W + sh.off, s));
      if (persistent_adam(c)) {  // f3: slice the global moments exactly like the weights
        PL(GIST_PROF_PARTITION, (double)sh.Kp * sh.Np * 12.0, s, extract_sub(c->theta_m[l], mp, sl.M + sh.off, s));
        PL(GIST_PROF_PARTITION, (double)sh.Kp * sh.Np * 12.0, s, extract_sub(c->theta_v[l], mp, sl.V + sh.off, s));
      }
    }
  }
  const int64_t tot_local = (int64_t)c->slots.size() * c->S_max;
  if (c->Mall && tot_local > 0 && !persistent_adam(c)) {  // R8: reset per round
    CK(cudaMemsetAsync(c->Mall, 0, (size_t)tot_local * 4, s));
    CK(cudaMemsetAsync(c->Vall, 0, (size_t)tot_local * 4, s));
  }
  if (c->Wball && tot_local > 0) LK(f32_to_bf16(c->Wall, c->Wball, tot_local, s));
  if (c->prec == GIST_PREC_BF16) TRY(build_plan<bf16>(c, c->plan_b));
  else TRY(build_plan<float>(c, c->plan_f));
  c->prof_now = false;
  TRY(check_launch(c, "partition"));
  if (!persistent_adam(c)) c->adam_t = 0;  // R8 (f3: the counter carries over)
  c->state = S_PARTITIONED;
  return GIST_OK;
}

extern "C" gist_status gist_get_partition(gist_ctx* c, int32_t dim, int32_t* units, int32_t* offs) {
  PRE(c);
  if (c->m == 0 || c->offs.empty()) return fail(c, GIST_E_STATE, "get_partition: no partition yet");
  if (dim < 0 || dim > c->L || !units || !offs) return GIST_E_ARG;
  const int d = c->dims[dim];
  if (dim == 0 || dim == c->L) {
    for (int r = 0; r < d; ++r) units[r] = r;
    for (int i = 0; i <= c->m; ++i) offs[i] = 0;
    offs[c->m] = d;
    return GIST_OK;
  }
  CK(cudaMemcpyAsync(units, c->units[dim], (size_t)d * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  std::copy(c->offs[dim].begin(), c->offs[dim].end(), offs);
  return GIST_OK;
}

// ============================================================ aggregate ===
extern "C" gist_status gist_aggregate(gist_ctx* c) {
  PRE(c);
  Range nvtx_range("gist_aggregate");
  if (c->state != S_PARTITIONED) return fail(c, GIST_E_STATE, "aggregate: no open round");
  cudaStream_t s = c->stream;
  const int W = c->cfg.world_size;
  c->prof_now = c->prof_stride > 0;
  // the weights, and with persistent Adam state (f3) the two moments, travel the same way
  struct Part { float* local; std::vector<float*>* global; };
  std::vector<float*> wvec(c->theta.begin(), c->theta.end());
  std::vector<Part> parts = {{c->Wall, &wvec}};
  if (persistent_adam(c)) parts.push_back({c->Mall, &c->theta_m}), parts.push_back({c->Vall, &c->theta_v});
  if (sharded(c)) {  // owner-sharded Theta: the updated rows go back to their owners
    TRY(shard_aggregate(c));
    c->prof_now = false;
    TRY(check_launch(c, "aggregate"));
    c->round += 1;
    c->state = S_PARAMS;
    return GIST_OK;
  }
  if (c->p2p_base) {  // agg_mode P2P (f2): owners store their blocks into every replica
    // barrier 1: every rank has finished this round's reads of its replica (gist_partition's
    // extraction) before any peer overwrites it
    TRY(coll(c, comm_barrier(c->comm, c->barrier_word, s, &c->err)));
    for (const Part& pt : parts)
      for (int i = c->cfg.rank; i < c->m; i += W) {
        const int j = i / W;
        const float* w = pt.local + (size_t)j * c->S_max;
        for (int l = 0; l < c->L; ++l) {
          const LayerShape& sh = c->shapes[i][l];
          LayerMap mp;
          mp.rows = sh.rows; mp.nrows = sh.nrows; mp.sage = c->arch == GIST_ARCH_SAGE; mp.gat = 0; mp.half = sh.half;
          mp.glob_half = (int)pad8(c->dims[l]); mp.cols = sh.cols; mp.ncols = sh.ncols; mp.Kp = sh.Kp; mp.Np = sh.Np;
          mp.ldg = c->th_N[l];
          const size_t off = (size_t)(reinterpret_cast<char*>((*pt.global)[l]) - c->p2p_base);
          if (c->cfg.agg_mode == GIST_AGG_SYMM) {  // NCCL device API: LSA peer pointers / NVLS multimem
            PL(GIST_PROF_AGGREGATE, (double)sh.Kp * sh.Np * 4.0 * (2.0 + W), s,
               scatter_sub_symm(*c->devcomm, c->win, off, mp, w + sh.off, c->symm_mm, s));
            continue;
          }
          PeerDst pd;
          pd.n = W;
          for (int r = 0; r < W; ++r) pd.dst[r] = reinterpret_cast<float*>(c->peer_base[r] + off);
          PL(GIST_PROF_AGGREGATE, (double)sh.Kp * sh.Np * 4.0 * (2.0 + W), s, scatter_sub_peers(pd, mp, w + sh.off, s));
        }
      }
    // barrier 2: every peer's stores into this replica have completed before anything reads it
    TRY(coll(c, comm_barrier(c->comm, c->barrier_word, s, &c->err)));
    c->prof_now = false;
    TRY(check_launch(c, "aggregate"));
    c->round += 1;
    c->state = S_PARAMS;
    return GIST_OK;
  }
  for (const Part& pt : parts) {
    const float* src = pt.local;
    if (W > 1) {  // subAgg exchange: one all-gather of the packed slot buffers over NVLink
      const int id = prof_begin(c, s, GIST_PROF_COMM, (double)(W - 1) * c->slots_per_rank * c->S_max * 4.0);
      TRY(coll(c, comm_allgather(c->comm, pt.local, c->Wrecv, (size_t)c->slots_per_rank * c->S_max * 4, s, &c->err)));
      prof_end(c, s, id);
      src = c->Wrecv;
    }
    for (int i = 0; i < c->m; ++i) {
      const int rank = gist_slot_owner(i, W), j = i / W;
      const float* w = src + ((size_t)rank * c->slots_per_rank + j) * c->S_max;
      if (W == 1) w = pt.local + (size_t)j * c->S_max;
      for (int l = 0; l < c->L; ++l) {
        const LayerShape& sh = c->shapes[i][l];
        LayerMap mp;
        mp.rows = sh.rows; mp.nrows = sh.nrows; mp.sage = c->arch == GIST_ARCH_SAGE; mp.gat = c->arch == GIST_ARCH_GAT; mp.half = sh.half;
        mp.glob_half = (int)pad8(c->dims[l]); mp.cols = sh.cols; mp.ncols = sh.ncols; mp.Kp = sh.Kp; mp.Np = sh.Np;
        mp.ldg = c->th_N[l];
        PL(GIST_PROF_AGGREGATE, (double)sh.Kp * sh.Np * 12.0, s, scatter_sub((*pt.global)[l], mp, w + sh.off, s));
      }
    }
    if (c->arch == GIST_ARCH_GAT) {  // R21: the last layer's attention rows = mean of the m copies
      const int l = c->L - 1;
      MeanRows mr;
      mr.n = c->m;
      mr.cols = c->dims[c->L];
      mr.ld_dst = c->th_N[l];
      for (int i = 0; i < c->m; ++i) {
        const int rank = gist_slot_owner(i, W), j = i / W;
        const float* w = W == 1 ? pt.local + (size_t)j * c->S_max
                                : src + ((size_t)rank * c->slots_per_rank + j) * c->S_max;
        const LayerShape& sh = c->shapes[i][l];
        mr.src[i] = w + sh.off + (int64_t)sh.half * sh.Np;
        mr.ld_src[i] = sh.Np;
      }
      PL(GIST_PROF_AGGREGATE, 2.0 * c->m * mr.cols * 4.0, s,
         mean_rows((*pt.global)[l] + pad8(c->dims[l]) * c->th_N[l], mr, 2, s));
    }
  }
  c->prof_now = false;
  TRY(check_launch(c, "aggregate"));
  c->round += 1;
  c->state = S_PARAMS;
  return GIST_OK;
}
