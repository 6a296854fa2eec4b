// step.cu -- subTrain: one step of every local sub-GCN as grouped
// lockstep launches (batch build, aggregation, GEMMs, loss, backward, optimizer), captured once
// per variant as a CUDA graph and replayed; the host side of the batch schedule (R7).
#include "ctx.h"

using namespace gist;
using namespace gist_impl;

// ============================================================== step ======
template <typename T>
static void launch_gemm(gist_ctx* c, const GemmPlanTC& tcp, const SgemmGroup& fp, double flops, cudaStream_t s) {
  const int id = prof_begin(c, s, GIST_PROF_GEMM, flops);
  if (c->prec == GIST_PREC_FP32) gemm_f32_group(fp, s);
  else gemm_bf16_launch(tcp, s);  // BF16 or TF32 tcgen05 plan
  prof_end(c, s, id);
  ++c->nk;
}

// One GAT subTrain step (R21) of every slot of group g after the grouped batch build: per slot
// and layer Z = H W (GEMM), attention scores and aggregation; the grouped softmax-CE; then per
// slot and layer the two attention backward passes, dW = H^T dZ (plus the attention rows) and
// dH = dZ W^T.  Dummy batch rows (v >= n_b) carry no neighbours and a zero loss gradient.
template <typename T>
static gist_status gat_group_step(gist_ctx* c, typename StepPlan<T>::Group& g, int nnz_slot, cudaStream_t s) {
  const int L = c->L;
  const int64_t nb = c->nb_max_rows;
  auto layer_args = [&](Slot& sl, int l) {
    const LayerShape& sh = c->shapes[sl.index][l];
    GatLayer<T> a;
    a.row_beg = sl.b_beg; a.row_end = sl.b_end; a.col = sl.b_col; a.rows = nb; a.w = sh.Np;
    a.Z = (const T*)sl.gZ[l]; a.ldz = sh.Np;
    a.a_src = sl.W + sh.off + (int64_t)sh.half * sh.Np;
    a.a_dst = a.a_src + sh.Np;
    float* sc = sl.gsc[l];
    a.s = sc; a.t = sc + nb; a.lse = sc + 2 * nb; a.Srow = sc + 3 * nb; a.dt = sc + 4 * nb; a.ds = sc + 5 * nb;
    return a;
  };
  const int64_t d0p = pad8(c->dims[0]);
  for (int j = 0; j < g.count; ++j) {  // layer-0 input: the batch rows of X
    Slot& sl = c->slots[g.first + j];
    LK(gather_rows_t<T>((const T*)c->X, d0p, sl.b_nodes, nb, d0p, (T*)sl.H[0], d0p, s));
  }
  for (int l = 0; l < L; ++l) {  // ---- a2/a3: forward
    launch_gemm<T>(c, g.fwd_tc[l], g.fwd_f[l], g.fwd_fl[l], s);  // Z = H W (grouped)
    // compulsory bytes: Z read once, H (scores) and the output written once, per-row scalars,
    // 4 B per edge of the batch CSR (the gathered Z rows are served from L2, as for k_spmm)
    double by = 0.0;
    GatGroup<T> G;
    G.n = g.count;
    for (int j = 0; j < g.count; ++j) {
      Slot& sl = c->slots[g.first + j];
      const auto& shp = c->shapes[sl.index];
      const LayerShape& sh = shp[l];
      by += (double)nb * (sh.Np * 2.0 * sizeof(T) + sh.half * sizeof(T) + 32.0);
      GatLayer<T>& a = G.a[j];
      a = layer_args(sl, l);
      a.H = (const T*)sl.H[l]; a.ldh = sh.half; a.kw = sh.half;  // scores = H (W a), fp32 W a
      a.W32 = sl.W + sh.off; a.ldw = sh.Np; a.wa = sl.gsc[l] + 6 * nb;
      if (l + 1 < L) { a.out = (T*)sl.H[l + 1]; a.ldo = shp[l + 1].half; a.relu = 1; }
      else { a.out_f32 = sl.logits; a.ldo = sh.Np; }
    }
    const int id = prof_begin(c, s, GIST_PROF_SPMM, by, 4.0 * g.count, nnz_slot);
    LK(gat_scores<T>(G, s));
    LK(gat_forward<T>(G, s));
    ++c->nk;
    prof_end(c, s, id);
  }
  {  // ---- a4: softmax cross-entropy (grouped), dlogits into gG
    const int id = prof_begin(c, s, GIST_PROF_LOSS, (double)g.count * nb * (g.ce.ld * (4.0 + sizeof(T)) + 17.0));
    softmax_ce<T>(g.ce, s);
    prof_end(c, s, id);
    ++c->nk;
  }
  for (int l = L - 1; l >= 0; --l) {  // ---- a5/a6: backward
    double by = 0.0;  // Z, G (+ mask), dZ once; scalars; two passes over the batch CSR
    GatGroup<T> G;
    G.n = g.count;
    for (int j = 0; j < g.count; ++j) {
      Slot& sl = c->slots[g.first + j];
      const auto& shp = c->shapes[sl.index];
      const LayerShape& sh = shp[l];
      by += (double)nb * (sh.Np * 4.0 * sizeof(T) + 48.0);
      GatLayer<T>& a = G.a[j];
      a = layer_args(sl, l);
      a.G = (const T*)sl.gG; a.ldg = sh.Np;  // dlogits (last layer) or dH_{l+1} (width Np_l)
      if (l + 1 < L) { a.mask = (const T*)sl.H[l + 1]; a.ldm = shp[l + 1].half; }
      a.dZ = (T*)sl.dZ[l]; a.ldd = sh.Np;
      a.da_src = sl.G + sh.off + (int64_t)sh.half * sh.Np;
      a.da_dst = a.da_src + sh.Np;
      a.da_part = sl.gsc[l] + 6 * nb + 2 * sh.half;
    }
    const int id = prof_begin(c, s, GIST_PROF_SPMM, by, 8.0 * g.count, nnz_slot);
    LK(gat_backward<T>(G, s));
    c->nk += 3;
    prof_end(c, s, id);
    if (c->side_now) {  // dW_l only feeds the optimizer: overlap it with the rest of the backward chain
      CK(cudaEventRecord(c->ev_dw_fork, s));
      CK(cudaStreamWaitEvent(c->side_now, c->ev_dw_fork, 0));
    }
    launch_gemm<T>(c, g.dw_tc[l], g.dw_f[l], g.dw_fl[l], c->side_now ? c->side_now : s);  // dW = H^T dZ (rows [0, half))
    if (l > 0) launch_gemm<T>(c, g.dx_tc[l], g.dx_f[l], g.dx_fl[l], s);          // dH = dZ W^T -> gG
  }
  if (c->side_now) {
    CK(cudaEventRecord(c->ev_dw_join, c->side_now));
    CK(cudaStreamWaitEvent(s, c->ev_dw_join, 0));
  }
  return GIST_OK;
}

// a7 for one layer of a group's slots on stream ds (layer_opt)
static gist_status layer_optimizer(gist_ctx* c, const OptRanges& R, cudaStream_t ds) {
  int64_t n = 0;
  for (int j = 0; j < R.count; ++j) n += R.n[j];
  if (c->cfg.optimizer == GIST_OPT_ADAM)
    PL(GIST_PROF_OPTIM, (double)n * (28.0 + (R.Wb[0] ? 2.0 : 0.0)), ds,
       adam_ranges(R, c->cfg.beta1, c->cfg.beta2, c->cfg.eps, c->dstate, ds));
  else
    PL(GIST_PROF_OPTIM, (double)n * (12.0 + (R.Wb[0] ? 2.0 : 0.0)), ds, sgd_ranges(R, c->dstate, ds));
  ++c->nk;
  return GIST_OK;
}

template <typename T>
static gist_status prefetch_batch(gist_ctx* c, typename StepPlan<T>::Group& g, int z, cudaStream_t bs,
                                  bool skip_x = false);
static gist_status run_optimizer_on(gist_ctx* c, cudaStream_t s);

// One subTrain step of every slot of group g, in lockstep: every
// kernel below is one launch over all slots of the group.  early_pf: the next step's batch
// build runs on the main stream right after the last backward aggregation (the last reader of
// this step's batch structures), overlapping dW_0 (and its optimizer) on the dW stream; its copy
// of the X rows into C_0 (which dW_0 reads) follows the join.
template <typename T>
static gist_status run_group_step(gist_ctx* c, typename StepPlan<T>::Group& g, int z, cudaStream_t s,
                                  bool early_pf) {
  const int L = c->L;
  for (int j = 0; j < g.count; ++j) c->slots[g.first + j].last_nb = c->slots[g.first + j].nb_of_step[z];
  int nnz_slot = -1;
  if (c->prof_now && c->nnz_pin_used < c->nnz_pin_cap) nnz_slot = c->nnz_pin_used++;
  // ---- a1: Cluster mini-batch build (unless prefetched during the previous step's optimizer)
  if (!c->batch_prefetched) {
    double vol = 0.0;
    for (int j = 0; j < g.count; ++j) vol += (double)c->slots[g.first + j].vol_of_step[z];
    int id = -1;
    if (c->prof_now)
      id = prof_begin(c, s, GIST_PROF_BATCH, vol * (c->pack_ob ? 12.0 : 16.0) + g.count * c->nb_max_rows * 45.0, 4.0,
                      nnz_slot);
    batch_setup(g.batch, c->cstart, c->rp, s);
    batch_build(g.batch, c->rp, c->col, c->ccol, c->cid, c->cstart, (int)c->c, c->arch, c->labels, c->split,
                c->bd && c->prec == GIST_PREC_BF16 && c->arch == GIST_ARCH_SAGE, c->pack_ob, s);
    prof_end(c, s, id);
    c->nk += 2;
  }
  if (nnz_slot >= 0)  // nnz of the group's first slot; the profile scales it by the group size
    CK(cudaMemcpyAsync(c->nnz_pin + nnz_slot, c->slots[g.first].stats, 8, cudaMemcpyDeviceToHost, s));
  if (c->arch == GIST_ARCH_GAT) return gat_group_step<T>(c, g, nnz_slot, s);
  const double per_nnz = 4.0 * g.count;
  auto spmm_l = [&](const SpmmGroup<T, T>& G, double bytes) {
    int id = -1;
    if (c->prof_now) id = prof_begin(c, s, GIST_PROF_SPMM, bytes, per_nnz, nnz_slot);
    spmm_group<T, T>(G, s);
    prof_end(c, s, id);
    ++c->nk;
  };
  auto bd_l = [&](const BdPlan& P, double flops) {
    const int id = prof_begin(c, s, GIST_PROF_AGG_TC, flops);
    gemm_bd_launch(P, s);
    prof_end(c, s, id);
    ++c->nk;
  };
  const bool bd = c->bd && c->prec == GIST_PREC_BF16 && c->arch == GIST_ARCH_SAGE;
  auto tc_l = [&](const GemmPlanTC& P, double fl) {  // one tcgen05 GEMM launch (BF16 plans only)
    const int id = prof_begin(c, s, GIST_PROF_GEMM, fl);
    gemm_bf16_launch(P, s);
    prof_end(c, s, id);
    ++c->nk;
  };
  // ---- a2/a3: forward
  for (int l = 0; l < L; ++l) {
    if (g.reassoc && l == L - 1 && c->arch != GIST_ARCH_SAGE) {  // GCN: logits = A_hat (H W)
      tc_l(g.ra_p, g.ra_gemm_fl / 3);
      const int id = prof_begin(c, s, GIST_PROF_SPMM, g.ra_fby, per_nnz, nnz_slot);
      spmm_group<T, float>(g.ra_fsp_f, s);
      prof_end(c, s, id);
      ++c->nk;
      continue;
    }
    if (g.reassoc && l == L - 1) {  // Z = H W_top + N (H W_bot)
      // H W_top does not depend on the aggregation of P = H W_bot: on the side stream beside it
      // (the loss kernel adds the two)
      if (c->side_now) {
        CK(cudaEventRecord(c->ev_dw_fork, s));
        CK(cudaStreamWaitEvent(c->side_now, c->ev_dw_fork, 0));
        gemm_bf16_launch(g.ra_z, c->side_now);
        ++c->nk;
      }
      LK(relayout_last(g.ra_wc, s));  // [W_top | W_bot] of this step's weights, for dH below
      ++c->nk;
      tc_l(g.ra_p, g.ra_gemm_fl / 6);
      if (bd) bd_l(g.ra_fbd, g.ra_bd_fl / 2);
      spmm_l(g.ra_fsp, g.ra_fby);
      if (c->side_now) {
        CK(cudaEventRecord(c->ev_dw_join, c->side_now));
        CK(cudaStreamWaitEvent(s, c->ev_dw_join, 0));
      } else {
        tc_l(g.ra_z, g.ra_gemm_fl / 6);
      }
      continue;
    }
    if (bd) bd_l(g.fwd_bd[l], g.bd_fl[l]);
    spmm_l(g.fwd_spmm[l], g.fwd_by[l]);
    launch_gemm<T>(c, g.fwd_tc[l], g.fwd_f[l], g.fwd_fl[l], s);
  }
  // ---- a4: softmax cross-entropy
  {
    const double bytes = (double)g.count * c->nb_max_rows * (g.ce.ld * (4.0 + sizeof(T)) + 17.0);
    const int id = prof_begin(c, s, GIST_PROF_LOSS, bytes);
    softmax_ce<T>(g.ce, s);  // (its last CTA per slot also reduces the step loss)
    prof_end(c, s, id);
    c->nk += 1;
  }
  // ---- a5/a6: backward.  With the dW stream, dW_l (it only feeds the optimizer) overlaps the
  // rest of the backward chain (dX -> aggregation), joined before the optimizer.
  auto fork = [&]() {
    CK(cudaEventRecord(c->ev_dw_fork, s));
    CK(cudaStreamWaitEvent(c->side_now, c->ev_dw_fork, 0));
    return GIST_OK;
  };
  for (int l = L - 1; l >= 0; --l) {
    if (g.reassoc && l == L - 1) {
      // GCN: Q = A_hat dZ; dW = H^T Q; dH = Q W^T.  SAGE: Q = N^T dZ; dW = [H^T dZ; H^T Q];
      // dZ_{l-1} = (dZ W_top^T + Q W_bot^T) * ReLU'
      if (bd && c->arch == GIST_ARCH_SAGE) bd_l(g.ra_bbd, g.ra_bd_fl / 2);
      spmm_l(g.ra_bsp, g.ra_bby);
      // per-layer optimizer: it rewrites W_l, so the fork follows the step's last reader of W_l
      // (GCN's dH = Q W^T reads W; GraphSAGE's reads the relayout copy)
      if (c->layer_opt) tc_l(g.ra_dh, g.ra_gemm_fl / 3);
      cudaStream_t ds = c->side_now ? c->side_now : s;
      if (c->side_now) TRY(fork());
      {
        const int id = prof_begin(c, ds, GIST_PROF_GEMM, g.ra_gemm_fl / 3);
        gemm_bf16_launch(g.ra_dw, ds);
        prof_end(c, ds, id);
        ++c->nk;
      }
      if (c->layer_opt) TRY(layer_optimizer(c, g.opt_l[l], ds));
      if (!c->layer_opt) tc_l(g.ra_dh, g.ra_gemm_fl / 3);
      continue;
    }
    // per-layer optimizer: dW_l and the update of W_l follow dX_l (the step's last reader of W_l)
    if (c->layer_opt && l > 0) launch_gemm<T>(c, g.dx_tc[l], g.dx_f[l], g.dx_fl[l], s);
    cudaStream_t ds = c->side_now ? c->side_now : s;
    if (c->side_now) TRY(fork());
    launch_gemm<T>(c, g.dw_tc[l], g.dw_f[l], g.dw_fl[l], ds);
    if (c->layer_opt) TRY(layer_optimizer(c, g.opt_l[l], ds));
    if (l == 0) {
      // one group, one-pass optimizer: it follows dW_0 on the dW stream, so the next batch's build
      // on the main stream overlaps both (single sub-GCN per GPU: the step's tail is then
      // max(build, dW_0 + optimizer) instead of build + optimizer)
      if (early_pf && !c->layer_opt && c->opt_side_ok) {
        TRY(run_optimizer_on(c, ds));
        c->opt_side = true;
      }
      if (early_pf) TRY(prefetch_batch<T>(c, g, z + 1, s, /*skip_x*/ true));
      break;
    }
    if (!c->layer_opt) launch_gemm<T>(c, g.dx_tc[l], g.dx_f[l], g.dx_fl[l], s);
    if (bd) bd_l(g.bwd_bd[l], g.bd_fl[l]);
    spmm_l(g.bwd_spmm[l], g.bwd_by[l]);
  }
  if (c->side_now) {  // join: the optimizer (or the next step) reads every gradient / weight
    CK(cudaEventRecord(c->ev_dw_join, c->side_now));
    CK(cudaStreamWaitEvent(s, c->ev_dw_join, 0));
  }
  if (early_pf && g.batch.X) {  // dW_0 has read C_0: the next batch's X rows may replace its left half
    LK(batch_xcopy(g.batch, s));
    ++c->nk;
  }
  return GIST_OK;
}

// a1 of the next step for group g on stream bs: the build reads the batch index st->zb (the
// device step state's z still points at the current step while its optimizer runs)
template <typename T>
static gist_status prefetch_batch(gist_ctx* c, typename StepPlan<T>::Group& g, int z, cudaStream_t bs,
                                  bool skip_x) {
  double vol = 0.0;
  for (int j = 0; j < g.count; ++j) vol += (double)c->slots[g.first + j].vol_of_step[z];
  const int id = prof_begin(c, bs, GIST_PROF_BATCH, vol * (c->pack_ob ? 12.0 : 16.0) + g.count * c->nb_max_rows * 45.0);
  batch_setup(g.batch, c->cstart, c->rp, bs);
  BatchGroup bg = g.batch;
  bg.skip_x = skip_x ? 1 : 0;
  batch_build(bg, c->rp, c->col, c->ccol, c->cid, c->cstart, (int)c->c, c->arch, c->labels, c->split,
              c->bd && c->prec == GIST_PREC_BF16 && c->arch == GIST_ARCH_SAGE, c->pack_ob, bs);
  prof_end(c, bs, id);
  c->nk += 2;
  return GIST_OK;
}

// a7 over every local slot at once (the packed buffers are contiguous), then advance the step state
static gist_status run_optimizer_on(gist_ctx* c, cudaStream_t s) {
  const int64_t n = (int64_t)c->slots.size() * c->S_max;
  if (c->cfg.optimizer == GIST_OPT_ADAM)
    PL(GIST_PROF_OPTIM, (double)n * (28.0 + (c->Wball ? 2.0 : 0.0)), s,
       adam_step(c->Wall, c->Gall, c->Mall, c->Vall, n, c->cfg.beta1, c->cfg.beta2, c->cfg.eps, c->dstate, c->Wball,
                 s));
  else
    PL(GIST_PROF_OPTIM, (double)n * (12.0 + (c->Wball ? 2.0 : 0.0)), s,
       sgd_step(c->Wall, c->Gall, n, c->dstate, c->Wball, s));
  ++c->nk;  // (no step_advance launch: the optimizer's last CTA advances the step state)
  return GIST_OK;
}
static gist_status run_optimizer(gist_ctx* c) {
  cudaStream_t s = c->stream;
  if (c->layer_opt && c->arch != GIST_ARCH_GAT) {  // every layer was updated on the dW stream
    PL(GIST_PROF_OPTIM, 16.0, s, step_advance(c->dstate, s));
    ++c->nk;
    return GIST_OK;
  }
  if (c->opt_side) return GIST_OK;  // enqueued after dW_0 on the dW stream (run_group_step)
  return run_optimizer_on(c, s);
}

// host side of R7 for a whole subtrain call: cluster lists, offsets, n_b, tags per step
static gist_status schedule(gist_ctx* c, Slot& sl, int iters, bool* grew) {
  const int q = c->cfg.clusters_per_batch;
  const int per = 3 * q + 4;
  if (iters > sl.cap || !sl.desc_dev) {
    *grew = true;
    CK(cudaStreamSynchronize(c->stream));  // previous uploads / readers of the old buffers are done
    if (sl.desc_host) {
      cudaFreeHost(sl.desc_host);
      dfree(c, sl.desc_dev);
    }
    sl.cap = std::max(iters, 64);
    CK(cudaMallocHost(&sl.desc_host, (size_t)sl.cap * per * 4));
    TRY(dalloc_t(c, &sl.desc_dev, (size_t)sl.cap * per));
  }
  sl.nb_of_step.assign(iters, 0);
  sl.q_of_step.assign(iters, 0);
  sl.vol_of_step.assign(iters, 0);
  const int64_t B = (c->c + q - 1) / q;
  for (int z = 0; z < iters; ++z) {
    const int64_t st = c->step + z;
    const int64_t e = st / B, p = st % B;
    if (sl.cached_epoch != e) {
      epoch_perm(c, sl.index, e, sl.epoch_perm);
      sl.cached_epoch = (int)e;
    }
    int32_t* d = sl.desc_host + (size_t)z * per;
    const int64_t lo = p * q, hi = std::min<int64_t>((p + 1) * q, c->c);
    const int qq = (int)(hi - lo);
    int32_t off = 0;
    int64_t voff = 0;
    int32_t* dv = d + 2 * q + 1;
    for (int k = 0; k < q; ++k) {
      if (k < qq) {
        const int32_t cl = sl.epoch_perm[lo + k];
        d[k] = cl;
        d[q + k] = off;
        dv[k] = (int32_t)voff;
        off += (int32_t)(c->cstart_h[cl + 1] - c->cstart_h[cl]);
        voff += c->cvol_h[cl];
      } else {  // last batch of an epoch may hold fewer clusters
        d[k] = d[qq - 1];
        d[q + k] = off;
        dv[k] = (int32_t)voff;
      }
    }
    d[2 * q] = off;
    dv[q] = (int32_t)voff;
    d[3 * q + 2] = qq;
    d[3 * q + 3] = (int32_t)(uint32_t)(c->step + z + 1);  // unique tag per step (0 = never)
    sl.nb_of_step[z] = off;
    sl.q_of_step[z] = qq;
    sl.vol_of_step[z] = voff;
  }
  return GIST_OK;
}

// One subTrain step of every local slot (every lockstep group), the optimizer, and optionally
// the next step's batch builds on the dW stream, overlapping the optimizer (`prefetch`; every
// reader of this step's batch buffers precedes the fork).  `build`: this step builds its own
// batches (else the previous step prefetched them).  Everything that changes from step to step
// is read by the kernels from the device step state, so the enqueued sequence of a (build,
// prefetch) variant is identical for every step: it is captured once as a CUDA graph and
// replayed (step_graph).
static gist_status enqueue_step(gist_ctx* c, bool build, bool prefetch) {
  cudaStream_t s = c->stream;
  const size_t ng = c->prec == GIST_PREC_BF16 ? c->plan_b.groups.size() : c->plan_f.groups.size();
  c->side_now = c->prof_now ? nullptr : c->dws;
  c->batch_prefetched = !build;
  // GIST_BATCH_PREFETCH=1: the next step's builds during the optimizer (A/B against the early
  // prefetch inside the backward, the default; GAT keeps the late one)
  const char* e_pf = std::getenv("GIST_BATCH_PREFETCH");
  const bool early = prefetch && c->side_now && c->arch != GIST_ARCH_GAT && !(e_pf && e_pf[0] == '1');
  c->opt_side = false;
  c->opt_side_ok = ng == 1;  // the one-pass optimizer covers every group's slots
  for (size_t gi = 0; gi < ng; ++gi) {
    if (c->prec == GIST_PREC_BF16) TRY(run_group_step<bf16>(c, c->plan_b.groups[gi], c->cur_z, s, early));
    else TRY(run_group_step<float>(c, c->plan_f.groups[gi], c->cur_z, s, early));
  }
  if (early) prefetch = false;  // done inside the step
  if (prefetch) {
    CK(cudaEventRecord(c->ev_dw_fork, s));
    CK(cudaStreamWaitEvent(c->dws, c->ev_dw_fork, 0));
    for (size_t gi = 0; gi < ng; ++gi) {
      if (c->prec == GIST_PREC_BF16) TRY(prefetch_batch<bf16>(c, c->plan_b.groups[gi], c->cur_z + 1, c->dws));
      else TRY(prefetch_batch<float>(c, c->plan_f.groups[gi], c->cur_z + 1, c->dws));
    }
  }
  TRY(run_optimizer(c));
  if (prefetch) {
    CK(cudaEventRecord(c->ev_dw_join, c->dws));
    CK(cudaStreamWaitEvent(s, c->ev_dw_join, 0));
  }
  return GIST_OK;
}

namespace gist_impl {
void drop_graphs(gist_ctx* c) {
  for (auto& g : c->graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g.exec = nullptr;
    g.nk = 0;
  }
}
}  // namespace gist_impl

// the step of variant (build, prefetch) as a CUDA graph: captured on first use after every
// plan (re)build, then one cudaGraphLaunch per step (the host enqueue of ~30 launches with
// multi-kilobyte grouped argument blocks was as long as the step itself at one slot per GPU)
static gist_status step_graph(gist_ctx* c, bool build, bool prefetch) {
  gist_ctx::StepGraph& G = c->graphs[(build ? 2 : 0) + (prefetch ? 1 : 0)];
  if (!G.exec) {
    const int64_t nk0 = c->nk;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const gist_status st = enqueue_step(c, build, prefetch);
    cudaGraph_t gr = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c->stream, &gr);
    if (st != GIST_OK) {
      if (gr) cudaGraphDestroy(gr);
      return st;
    }
    CK(e);
    const cudaError_t ei = cudaGraphInstantiate(&G.exec, gr, 0);
    cudaGraphDestroy(gr);
    CK(ei);
    G.nk = c->nk - nk0;
    c->nk = nk0;
  }
  CK(cudaGraphLaunch(G.exec, c->stream));
  c->nk += G.nk;
  return GIST_OK;
}

extern "C" gist_status gist_subtrain(gist_ctx* c, int32_t local_iters, float lr, float* mean_loss) {
  PRE(c);
  Range nvtx_range("gist_subtrain");
  if (c->state != S_PARTITIONED) return fail(c, GIST_E_STATE, "subtrain: call partition first");
  if (local_iters < 0) return fail(c, GIST_E_ARG, "subtrain: local_iters < 0");
  cudaStream_t s = c->stream;
  // host schedule for every local slot; the previous call's uploads must have left the pinned buffers
  CK(cudaEventSynchronize(c->hstate_ev));
  const int per = 3 * c->cfg.clusters_per_batch + 4;
  bool grew = false;
  for (Slot& sl : c->slots) TRY(schedule(c, sl, local_iters, &grew));
  if (grew) {  // descriptor buffers moved: the step plan holds their addresses
    if (c->prec == GIST_PREC_BF16) TRY(build_plan<bf16>(c, c->plan_b));
    else TRY(build_plan<float>(c, c->plan_f));
  }
  for (Slot& sl : c->slots) {
    if (local_iters > 0)
      CK(cudaMemcpyAsync(sl.desc_dev, sl.desc_host, (size_t)local_iters * per * 4, cudaMemcpyHostToDevice, s));
    c->h2d += (int64_t)local_iters * per * 4;
    CK(cudaMemsetAsync(sl.loss_acc, 0, 4, s));
  }
  *c->hstate = StepState{0, (int32_t)c->adam_t, lr, 0u};
  if (!c->slots.empty()) CK(cudaMemsetAsync(c->bctr, 0, c->slots.size() * 2 * sizeof(int32_t), s));
  CK(cudaMemcpyAsync(c->dstate, c->hstate, sizeof(StepState), cudaMemcpyHostToDevice, s));
  CK(cudaEventRecord(c->hstate_ev, s));
  // GIST_BATCH_PREFETCH=0 / GIST_GRAPH=0: A/B switches (prefetch measured +1.4% on C3)
  const char* e_pf = std::getenv("GIST_BATCH_PREFETCH");
  const char* e_gr = std::getenv("GIST_GRAPH");
  const bool prefetch_on = !(e_pf && e_pf[0] == '0'), graphs_on = !(e_gr && e_gr[0] == '0');
  bool prefetched = false;  // step z's batches were built during step z-1's optimizer
  for (int z = 0; z < local_iters; ++z) {
    c->prof_now = c->prof_stride > 0 && ((c->step + z) % c->prof_stride) == 0;
    const bool next_prof = c->prof_stride > 0 && ((c->step + z + 1) % c->prof_stride) == 0;
    for (Slot& sl : c->slots) sl.last_nb = sl.nb_of_step[z];
    c->cur_z = z;
    // profiled steps run eagerly and serialised, and build their own batches
    const bool pf = prefetch_on && c->dws && z + 1 < local_iters && !c->prof_now && !next_prof;
    if (graphs_on && !c->prof_now) TRY(step_graph(c, !prefetched, pf));
    else TRY(enqueue_step(c, !prefetched, pf));
    prefetched = pf;
    c->prof_now = false;
  }
  c->adam_t += local_iters;
  c->step += local_iters;
  TRY(check_launch(c, "subtrain"));
  if (c->prof_stride > 0) prof_flush(c);
  if (mean_loss) {
    std::fill(mean_loss, mean_loss + c->m, 0.f);
    CK(cudaStreamSynchronize(s));
    for (Slot& sl : c->slots) {
      float v = 0.f;
      CK(cudaMemcpy(&v, sl.loss_acc, 4, cudaMemcpyDeviceToHost));
      mean_loss[sl.index] = local_iters > 0 ? v / (float)local_iters : 0.f;
      c->d2h += 4;
    }
  }
  return GIST_OK;
}
