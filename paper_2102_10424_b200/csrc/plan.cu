// plan.cu -- the launch plan of one subTrain step: every grouped launch's
// argument block (tensor maps, per-slot pointers, shapes) built once per partition, for the
// GraphSAGE / GCN paths (block-diagonal aggregation, re-associated last layer) and GAT (R21).
#include "ctx.h"

using namespace gist;
using namespace gist_impl;

namespace gist_impl {
// compulsory bytes of one SpMM launch excluding the nnz-proportional part
template <typename T>
static double spmm_bytes(const SpmmArgs<T, T>& a) {
  const double rw = (double)a.rows * (double)a.w * sizeof(T);
  double b = (double)a.rows * 16 + rw /*H*/ + rw /*out*/;
  if (a.add) b += rw;
  if (a.mask) b += rw;
  if (a.self_out) b += rw;
  if (a.rowscale) b += a.rows * 4.0;
  if (a.colscale) b += a.rows * 4.0;
  if (a.h_index) b += a.rows * 4.0;
  return b;
}

// Builds the launch plan of one subTrain step (every grouped launch's argument block).
template <typename T>
gist_status build_plan(gist_ctx* c, StepPlan<T>& P) {
  drop_graphs(c);  // the captured steps hold the previous plan's argument blocks
  P.groups.clear();
  const int L = c->L, nb = c->nb_max_rows, q = c->cfg.clusters_per_batch;
  const bool sage = c->arch == GIST_ARCH_SAGE;
  const bool tc = c->prec == GIST_PREC_BF16;  // BF16 tensor-core mode (bf16 operands and its fused features)
  const bool tf = c->prec == GIST_PREC_TF32;  // TF32 mode: FP32 storage, step GEMMs on tcgen05 kind::tf32
  // per-layer optimizer on the dW stream for lockstep groups of >= 4 slots (measured: C3 8 slots
  // 9,124 -> 9,178 steps/s; one slot per GPU 258 -> 270 us per step, so one pass there);
  // GIST_LAYER_OPT=0 / 1 forces it off / on (the test switch pinning the two bit-identical); GAT
  // keeps the one pass
  {
    const char* e = std::getenv("GIST_LAYER_OPT");
    c->layer_opt = c->arch != GIST_ARCH_GAT && (e ? e[0] == '1' : c->slots.size() >= 4);
  }
  // slots per lockstep group (GIST_GROUP overrides, <= kMaxGroup): measurements of the
  // L2-footprint / launch-count trade-off
  int gsz = kMaxGroup;
  if (const char* e = std::getenv("GIST_GROUP")) gsz = std::max(1, std::min(kMaxGroup, atoi(e)));
  for (int g0 = 0; g0 < (int)c->slots.size(); g0 += gsz) {
    typename StepPlan<T>::Group g;
    g.first = g0;
    g.count = std::min<int>(gsz, (int)c->slots.size() - g0);
    g.batch.n = g.count;
    g.batch.q = q;
    g.batch.nb_max = nb;
    g.batch.ctr = c->bctr + 2 * g0;
    g.fwd_spmm.assign(L, SpmmGroup<T, T>());
    g.bwd_spmm.assign(L, SpmmGroup<T, T>());
    g.fwd_tc.assign(L, GemmPlanTC());
    g.dw_tc.assign(L, GemmPlanTC());
    g.dx_tc.assign(L, GemmPlanTC());
    g.fwd_f.assign(L, SgemmGroup());
    g.dw_f.assign(L, SgemmGroup());
    g.dx_f.assign(L, SgemmGroup());
    g.fwd_fl.assign(L, 0.0);
    g.dw_fl.assign(L, 0.0);
    g.dx_fl.assign(L, 0.0);
    g.fwd_by.assign(L, 0.0);
    g.bwd_by.assign(L, 0.0);
    g.fwd_bd.assign(L, BdPlan());
    g.bwd_bd.assign(L, BdPlan());
    g.bd_fl.assign(L, 0.0);
    const bool bd = c->bd && tc && sage;
    if (bd) {  // the batch build copies the layer-0 self half [X_b | .] (no self_out in the sparse pass)
      g.batch.X = (const bf16*)c->X;
      g.batch.ldx = pad8(c->dims[0]);
      g.batch.ldxd = c->shapes[c->slots[g0].index][0].Kp;
    }
    g.ce.n = g.count;
    g.ce.rows = nb;
    g.ce.k = c->k;
    g.ce.ld = c->shapes[c->slots[g0].index][L - 1].Np;
    g.reassoc = c->reassoc && tc && L >= 2;
    if (c->arch == GIST_ARCH_GAT) {  // R21: batch build and loss are grouped; the layers run per slot
      for (int j = 0; j < g.count; ++j) {
        Slot& sl = c->slots[g0 + j];
        BatchSlot& b = g.batch.s[j];
        b.desc = sl.desc_dev; b.map64 = sl.map64; b.b_nodes = sl.b_nodes; b.b_beg = sl.b_beg; b.b_end = sl.b_end;
        b.b_col = sl.b_col; b.scale = sl.scale; b.lab_b = sl.lab_b; b.train_b = sl.train_b; b.stats = sl.stats;
        CeSlot<T>& e = g.ce.s[j];
        e.logits = sl.logits; e.dlog = (T*)sl.gG; e.row_loss = sl.row_loss; e.lab = sl.lab_b;
        e.train = sl.train_b; e.stats = sl.stats; e.step_loss = sl.step_loss; e.loss_acc = sl.loss_acc;
        e.done = sl.ce_done;
      }
      // the GEMMs of every layer are grouped over the slots: Z = H W, dW = H^T dZ, dH = dZ W^T
      for (int l = 0; l < L; ++l) {
        std::vector<GemmOp> fw, dw, dx;
        for (int j = 0; j < g.count; ++j) {
          Slot& sl = c->slots[g0 + j];
          const LayerShape& sh = c->shapes[sl.index][l];
          const void* Wl = tc ? (const void*)(sl.Wb + sh.off) : (const void*)(sl.W + sh.off);
          fw.push_back(GemmOp{false, false, nb, sh.Np, sh.half, sl.H[l], sh.half, Wl, sh.Np, sl.gZ[l], sh.Np, !tc,
                              false, nullptr, 0, nullptr, 0});
          dw.push_back(GemmOp{true, false, sh.half, sh.Np, nb, sl.H[l], sh.half, sl.dZ[l], sh.Np, sl.G + sh.off, sh.Np,
                              true, false, nullptr, 0, nullptr, 0});
          if (l > 0)
            dx.push_back(GemmOp{false, true, nb, sh.half, sh.Np, sl.dZ[l], sh.Np, Wl, sh.Np, sl.gG, sh.half, !tc, false,
                                nullptr, 0, nullptr, 0});
          g.fwd_fl[l] += 2.0 * nb * sh.Np * sh.half;
          g.dw_fl[l] += 2.0 * nb * sh.Np * sh.half;
          if (l > 0) g.dx_fl[l] += 2.0 * nb * sh.Np * sh.half;
        }
        if (tc || tf) {
          if (!gemm_tc_prepare(fw.data(), g.count, &g.fwd_tc[l], tf) ||
              !gemm_tc_prepare(dw.data(), g.count, &g.dw_tc[l], tf) ||
              (l > 0 && !gemm_tc_prepare(dx.data(), g.count, &g.dx_tc[l], tf)))
            return fail(c, GIST_E_UNSUPPORTED, "GAT: tcgen05 GEMM plan failed");
        } else {
          for (int j = 0; j < g.count; ++j) {
            g.fwd_f[l].op[j] = fw[j];
            g.dw_f[l].op[j] = dw[j];
            if (l > 0) g.dx_f[l].op[j] = dx[j];
          }
          g.fwd_f[l].n = g.dw_f[l].n = g.count;
          g.dx_f[l].n = l > 0 ? g.count : 0;
        }
      }
      P.groups.push_back(g);
      continue;
    }
    for (int l = 0; l < L; ++l) {
      std::vector<GemmOp> fw, dw, dx;
      std::vector<BdOp> bfw, bbw;
      if (g.reassoc && l == L - 1 && !sage) {
        // Re-associated last GCN layer (Eq. (1): Z = A_hat (H W), width Np instead of
        // the hidden width; A_hat symmetric): forward P = H W, logits = A_hat P; backward
        // Q = A_hat dZ, dW = H^T Q, dH = Q W^T * ReLU'(H).
        std::vector<GemmOp> op_p, op_w, op_h;
        for (int j = 0; j < g.count; ++j) {
          Slot& sl = c->slots[g0 + j];
          const auto& shp = c->shapes[sl.index];
          const LayerShape& sh = shp[l];
          const int64_t Np = sh.Np, Kp = sh.Kp;
          const bf16* Wl = sl.Wb + sh.off;
          const bf16* H = (const bf16*)sl.H[l];
          bf16 *P = (bf16*)sl.rP, *DQ = (bf16*)sl.rDQ;
          op_p.push_back(GemmOp{false, false, nb, Np, Kp, H, Kp, Wl, Np, P, Np, false, false, nullptr, 0, nullptr, 0,
                                nullptr, 0, /*keep_out*/ 1, 0});
          SpmmArgs<T, float>& a = g.ra_fsp_f.a[j];
          a = SpmmArgs<T, float>();
          a.row_beg = sl.b_beg; a.row_end = sl.b_end; a.col = sl.b_col; a.rows = nb;
          a.desc = sl.desc_dev; a.st = c->dstate; a.q = q;
          a.rowscale = sl.scale; a.colscale = sl.scale; a.self = 1;
          a.H = (const T*)P; a.ldh = Np; a.w = Np; a.out = sl.logits; a.ldo = Np;
          SpmmArgs<T, T>& b = g.ra_bsp.a[j];
          b = SpmmArgs<T, T>();
          b.row_beg = sl.b_beg; b.row_end = sl.b_end; b.col = sl.b_col; b.rows = nb;
          b.desc = sl.desc_dev; b.st = c->dstate; b.q = q;
          b.rowscale = sl.scale; b.colscale = sl.scale; b.self = 1;
          b.H = (const T*)DQ; b.ldh = 2 * Np; b.w = Np; b.out = (T*)(DQ + Np); b.ldo = 2 * Np;
          g.ra_fby += (double)nb * Np * 6.0 + nb * 16.0;
          g.ra_bby += spmm_bytes(b);
          op_w.push_back(GemmOp{true, false, Kp, Np, nb, H, Kp, DQ + Np, 2 * Np, sl.G + sh.off, Np, true, false, nullptr,
                                0, nullptr, 0, nullptr, 0, 0, /*stream_a*/ 1});
          GemmOp h{false, true, nb, Kp, Np, DQ + Np, 2 * Np, Wl, Np, sl.dZ[l - 1], shp[l - 1].Np, false, false, nullptr,
                   0, nullptr, 0, nullptr, 0, /*keep_out*/ 1, 0};
          h.mbits_in = sl.mb[l]; h.ldmbi = c->mb_ld[l];
          op_h.push_back(h);
          g.ra_gemm_fl += 2.0 * nb * Np * Kp * 3;
        }
        g.ra_fsp_f.n = g.ra_bsp.n = g.count;
        if (!gemm_bf16_prepare(op_p.data(), g.count, &g.ra_p) || !gemm_bf16_prepare(op_w.data(), g.count, &g.ra_dw) ||
            !gemm_bf16_prepare(op_h.data(), g.count, &g.ra_dh))
          return fail(c, GIST_E_UNSUPPORTED, "re-associated GCN layer: tcgen05 GEMM plan failed");
        g.ce.ld_dlog = 2 * (int64_t)c->shapes[c->slots[g0].index][l].Np;
        for (int j = 0; j < g.count; ++j) g.ce.s[j].dlog = (T*)c->slots[g0 + j].rDQ;
        continue;
      }
      if (g.reassoc && l == L - 1) {
        // Re-associated last GraphSAGE layer (exact algebra of Eq. (2), with the
        // class width far below the hidden width): Z = H W_top + N (H W_bot), so the
        // aggregation runs at the class width Np instead of the hidden width; backward:
        // Q = N^T dZ (width Np), dW_top = H^T dZ, dW_bot = H^T Q, dH = dZ W_top^T + Q W_bot^T.
        std::vector<GemmOp> op_p, op_z, op_w, op_hb;
        std::vector<BdOp> fb, bb;
        for (int j = 0; j < g.count; ++j) {
          Slot& sl = c->slots[g0 + j];
          const auto& shp = c->shapes[sl.index];
          const LayerShape& sh = shp[l];
          const int64_t Np = sh.Np, half = sh.half, Kp = sh.Kp;
          const bf16* Wl = sl.Wb + sh.off;  // [W_top; W_bot], Kp x Np
          const bf16* H = (const bf16*)sl.C[l];  // left half of C_l (written by GEMM l-1)
          bf16 *P = (bf16*)sl.rP, *AGG = (bf16*)sl.rAGG, *DQ = (bf16*)sl.rDQ, *DZs = (bf16*)sl.rDZs;
          op_p.push_back(GemmOp{false, false, nb, Np, half, H, Kp, Wl + half * Np, Np, P, Np, false, false, nullptr, 0,
                                nullptr, 0, nullptr, 0, /*keep_out*/ 1, 0});
          // H W_top alone (independent of the aggregation: it runs on the side stream beside P's
          // aggregation); the loss kernel adds N (H W_bot) in fp32, the same addition as an epilogue's
          op_z.push_back(GemmOp{false, false, nb, Np, half, H, Kp, Wl, Np, sl.logits, Np, true, false, nullptr, 0,
                                nullptr, 0});
          // forward aggregation of P
          SpmmArgs<T, T>& a = g.ra_fsp.a[j];
          a = SpmmArgs<T, T>();
          a.row_beg = sl.b_beg; a.row_end = sl.b_end; a.col = sl.b_col; a.rows = nb;
          a.desc = sl.desc_dev; a.st = c->dstate; a.q = q;
          a.rowscale = sl.scale; a.H = (const T*)P; a.ldh = Np; a.w = Np; a.out = (T*)AGG; a.ldo = Np;
          if (bd) {
            fb.push_back(BdOp{P, Np, (int64_t)nb, Np, (void*)AGG, Np, nullptr, 0, sl.scale, sl.desc_dev, 0, 1});
            a.add = (const T*)AGG; a.ld_add = Np; a.few_nnz = 1; a.early = 1;
          }
          g.ra_fby += spmm_bytes(a);
          // backward: Q = N^T dZ into DQ[:, Np:2Np) (dZ in DQ[:, 0:Np) from the loss kernel)
          SpmmArgs<T, T>& b = g.ra_bsp.a[j];
          b = SpmmArgs<T, T>();
          b.row_beg = sl.b_beg; b.row_end = sl.b_end; b.col = sl.b_col; b.rows = nb;
          b.desc = sl.desc_dev; b.st = c->dstate; b.q = q;
          b.w = Np; b.out = (T*)(DQ + Np); b.ldo = 2 * Np;
          if (bd) {  // N^T = A diag(1/deg): aggregate DZs = dZ / deg (written by the loss kernel)
            bb.push_back(BdOp{DZs, 2 * Np, (int64_t)nb, Np, (void*)(DQ + Np), 2 * Np, nullptr, 0, nullptr, sl.desc_dev, 0, 1});
            b.H = (const T*)DZs; b.ldh = 2 * Np;
            b.add = (const T*)(DQ + Np); b.ld_add = 2 * Np; b.few_nnz = 1; b.early = 1;
          } else {
            b.colscale = sl.scale; b.H = (const T*)DQ; b.ldh = 2 * Np;
          }
          g.ra_bby += spmm_bytes(b);
          op_w.push_back(GemmOp{true, false, half, Np, nb, H, Kp, DQ, 2 * Np, sl.G + sh.off, Np, true, false, nullptr, 0,
                                nullptr, 0, nullptr, 0, 0, /*stream_a*/ 1});
          op_w.push_back(GemmOp{true, false, half, Np, nb, H, Kp, DQ + Np, 2 * Np, sl.G + sh.off + half * Np, Np, true,
                                false, nullptr, 0, nullptr, 0, nullptr, 0, 0, 1});
          // dH = [dZ | Q] [W_top | W_bot]^T (one K = 2 Np GEMM), masked by ReLU'(H) -> dZ_{l-1}
          GemmOp hb{false, true, nb, half, 2 * Np, DQ, 2 * Np, (const bf16*)sl.rWc, 2 * Np, sl.dZ[l - 1],
                    shp[l - 1].Np, false, false, nullptr, 0, nullptr, 0, nullptr, 0, /*keep_out*/ 1, 0};
          hb.mbits_in = sl.mb[l]; hb.ldmbi = c->mb_ld[l];
          op_hb.push_back(hb);
          g.ra_wc.src[j] = Wl;
          g.ra_wc.dst[j] = (bf16*)sl.rWc;
          g.ra_wc.half[j] = (int)half;
          g.ra_wc.Np = (int)Np;
          g.ra_wc.max_half = std::max<int>(g.ra_wc.max_half, (int)half);
          g.ra_gemm_fl += 2.0 * nb * Np * half * 6;
          if (bd) g.ra_bd_fl += 2.0 * q * c->bs * c->bs * Np;
        }
        g.ra_fsp.n = g.ra_bsp.n = g.count;
        g.ra_wc.n = g.count;
        if (bd && (!gemm_bd_prepare(c->blocks, c->c, c->bs, fb.data(), g.count, q, nb, c->cstart, c->dstate, &g.ra_fbd) ||
                   !gemm_bd_prepare(c->blocks, c->c, c->bs, bb.data(), g.count, q, nb, c->cstart, c->dstate, &g.ra_bbd)))
          return fail(c, GIST_E_UNSUPPORTED, "re-associated layer: block-diagonal plan failed");
        if (!gemm_bf16_prepare(op_p.data(), g.count, &g.ra_p) || !gemm_bf16_prepare(op_z.data(), g.count, &g.ra_z) ||
            !gemm_bf16_prepare(op_w.data(), 2 * g.count, &g.ra_dw) ||
            !gemm_bf16_prepare(op_hb.data(), g.count, &g.ra_dh))
          return fail(c, GIST_E_UNSUPPORTED, "re-associated layer: tcgen05 GEMM plan failed");
        // the loss kernel writes dZ into DQ[:, 0:Np) (and dZ / deg for the block-diagonal path)
        g.ce.ld_dlog = 2 * (int64_t)c->shapes[c->slots[g0].index][l].Np;
        for (int j = 0; j < g.count; ++j) {
          Slot& sl = c->slots[g0 + j];
          g.ce.s[j].dlog = (T*)sl.rDQ;
          g.ce.s[j].dlog_s = bd ? (T*)sl.rDZs : nullptr;
          g.ce.s[j].scale_s = sl.scale;
          g.ce.s[j].add = (const T*)sl.rAGG;  // logits = (H W_top) + N (H W_bot)
        }
        continue;
      }
      for (int j = 0; j < g.count; ++j) {
        Slot& sl = c->slots[g0 + j];
        const auto& shp = c->shapes[sl.index];
        const LayerShape& sh = shp[l];
        if (l == 0) {
          BatchSlot& b = g.batch.s[j];
          b.desc = sl.desc_dev; b.map64 = sl.map64; b.b_nodes = sl.b_nodes; b.b_beg = sl.b_beg; b.b_end = sl.b_end;
          b.b_col = sl.b_col; b.scale = sl.scale; b.lab_b = sl.lab_b; b.train_b = sl.train_b; b.stats = sl.stats;
          CeSlot<T>& e = g.ce.s[j];
          e.logits = sl.logits; e.dlog = (T*)sl.dZ[L - 1]; e.row_loss = sl.row_loss; e.lab = sl.lab_b;
          e.train = sl.train_b; e.stats = sl.stats; e.step_loss = sl.step_loss; e.loss_acc = sl.loss_acc;
          e.done = sl.ce_done;
        }
        T* C = (T*)sl.C[l];
        // forward aggregation (a2)
        SpmmArgs<T, T>& a = g.fwd_spmm[l].a[j];
        a.row_beg = sl.b_beg; a.row_end = sl.b_end; a.col = sl.b_col; a.rows = nb;
        a.desc = sl.desc_dev; a.st = c->dstate; a.q = q;
        if (sage) {
          a.rowscale = sl.scale;               // N = D^-1 A (R2)
          a.out = C + sh.half; a.ldo = sh.Kp;   // right half: N H
          a.w = sh.half;
          if (l == 0) {
            a.h_index = sl.b_nodes; a.H = (const T*)c->X; a.ldh = pad8(c->dims[0]);
            a.self_out = C; a.ld_self = sh.Kp;  // left half: gathered X rows
          } else {
            a.H = C; a.ldh = sh.Kp;             // left half written by the previous GEMM epilogue
          }
        } else {
          a.rowscale = sl.scale; a.colscale = sl.scale; a.self = 1;  // D~^-1/2 (A+I) D~^-1/2 (R1)
          a.out = C; a.ldo = sh.Kp; a.w = sh.Kp;
          if (l == 0) { a.h_index = sl.b_nodes; a.H = (const T*)c->X; a.ldh = pad8(c->dims[0]); }
          else { a.H = (const T*)sl.H[l]; a.ldh = sh.Kp; }
        }
        if (bd) {  // intra-cluster part on tensor cores, then the sparse kernel adds the rest in place.
          // Layer 0 reads the batch-local X_b rows the batch build copied into the left half
          // (L2-resident) rather than gathering rows of the global X from HBM.
          bfw.push_back(BdOp{(const bf16*)C, sh.Kp, (int64_t)nb, sh.half, (void*)(C + sh.half), sh.Kp, nullptr, 0,
                             sl.scale, sl.desc_dev, 0, /*keep_out*/ 1});
          a.add = C + sh.half; a.ld_add = sh.Kp;
          a.few_nnz = 1;
          a.early = 1;
          if (l == 0) {
            a.self_out = nullptr; a.h_index = nullptr; a.H = C; a.ldh = sh.Kp;
            g.batch.xdst[j] = (bf16*)C;
          }
          g.bd_fl[l] += 2.0 * q * c->bs * c->bs * sh.half;
        }
        g.fwd_by[l] += spmm_bytes(a);
        // forward contraction (a3)
        const void* Wl = tc ? (const void*)(sl.Wb + sh.off) : (const void*)(sl.W + sh.off);
        if (l + 1 < L) {
          void* out = sage ? sl.C[l + 1] : sl.H[l + 1];
          fw.push_back(GemmOp{false, false, nb, sh.Np, sh.Kp, C, sh.Kp, Wl, sh.Np, out, shp[l + 1].Kp, false, true,
                              nullptr, 0, nullptr, 0, tc ? sl.mb[l + 1] : nullptr, tc ? c->mb_ld[l + 1] : 0,
                              /*keep_out: read by the next aggregation + GEMM*/ 1, /*stream_a*/ 1});
        } else {
          fw.push_back(GemmOp{false, false, nb, sh.Np, sh.Kp, C, sh.Kp, Wl, sh.Np, sl.logits, sh.Np, true, false,
                              nullptr, 0, nullptr, 0});
        }
        g.fwd_fl[l] += 2.0 * nb * sh.Np * sh.Kp;
        // backward: dW_l = C_l^T dZ_l (fp32 into the packed gradient buffer)
        dw.push_back(GemmOp{true, false, sh.Kp, sh.Np, nb, C, sh.Kp, sl.dZ[l], sh.Np, sl.G + sh.off, sh.Np, true, false,
                            nullptr, 0, nullptr, 0, nullptr, 0, 0, /*stream_a: C_l's last read*/ 1});
        g.dw_fl[l] += 2.0 * nb * sh.Np * sh.Kp;
        if (l > 0) {
          // dC_l = dZ_l W_l^T
          // (bd: the epilogue pre-scales the neighbour half by 1/deg of the row: N^T = A diag(1/deg))
          dx.push_back(GemmOp{false, true, nb, sh.Kp, sh.Np, sl.dZ[l], sh.Np, Wl, sh.Np, sl.dC, sh.Kp, false, false,
                              nullptr, 0, bd ? sl.scale : nullptr, sh.half, nullptr, 0, /*keep_out*/ 1, 0});
          g.dx_fl[l] += 2.0 * nb * sh.Np * sh.Kp;
          SpmmArgs<T, T>& b = g.bwd_spmm[l].a[j];
          b.row_beg = sl.b_beg; b.row_end = sl.b_end; b.col = sl.b_col; b.rows = nb;
          b.desc = sl.desc_dev; b.st = c->dstate; b.q = q;
          b.out = (T*)sl.dZ[l - 1]; b.ldo = shp[l - 1].Np;
          if (tc) { b.mbits = sl.mb[l]; b.ld_mbits = c->mb_ld[l]; }  // ReLU mask of C_l / H_l as bits
          if (sage && bd) {  // dZ_{l-1} = (dC_self + A_blocks dC'_neigh + A_inter dC'_neigh) * 1[H_l > 0]
            bbw.push_back(BdOp{(const bf16*)sl.dC + sh.half, sh.Kp, (int64_t)nb, sh.half, sl.dZ[l - 1],
                               shp[l - 1].Np, (const bf16*)sl.dC, sh.Kp, nullptr, sl.desc_dev, 0, /*keep_out*/ 1});
            b.H = (const T*)sl.dC + sh.half; b.ldh = sh.Kp;
            b.add = (const T*)sl.dZ[l - 1]; b.ld_add = shp[l - 1].Np;
            b.mask = (const T*)sl.C[l]; b.ld_mask = sh.Kp;
            b.w = sh.half;
            b.few_nnz = 1;
            b.early = 1;
          } else if (sage) {  // dZ_{l-1} = (dC_self + N^T dC_neigh) * 1[H_l > 0]
            b.colscale = sl.scale; b.H = (const T*)sl.dC + sh.half; b.ldh = sh.Kp;
            b.add = (const T*)sl.dC; b.ld_add = sh.Kp;
            b.mask = (const T*)sl.C[l]; b.ld_mask = sh.Kp;
            b.w = sh.half;
          } else {     // dZ_{l-1} = (A_hat^T dC) * 1[H_l > 0]
            b.rowscale = sl.scale; b.colscale = sl.scale; b.self = 1;
            b.H = (const T*)sl.dC; b.ldh = sh.Kp;
            b.mask = (const T*)sl.H[l]; b.ld_mask = sh.Kp;
            b.w = sh.Kp;
          }
          g.bwd_by[l] += spmm_bytes(b);
        }
      }
      g.fwd_spmm[l].n = g.count;
      g.bwd_spmm[l].n = l > 0 ? g.count : 0;
      if (bd) {
        if (!gemm_bd_prepare(c->blocks, c->c, c->bs, bfw.data(), g.count, q, nb, c->cstart, c->dstate,
                             &g.fwd_bd[l]) ||
            (l > 0 && !gemm_bd_prepare(c->blocks, c->c, c->bs, bbw.data(), g.count, q, nb, c->cstart, c->dstate,
                                       &g.bwd_bd[l])))
          return fail(c, GIST_E_UNSUPPORTED, "block-diagonal aggregation plan failed");
      }
      if (tc || tf) {
        if (tf)  // TF32 mode: every output of the step GEMMs is fp32 (the mode's element type)
          for (auto* v : {&fw, &dw, &dx})
            for (GemmOp& o : *v) o.out_f32 = true;
        if (!gemm_tc_prepare(fw.data(), g.count, &g.fwd_tc[l], tf) ||
            !gemm_tc_prepare(dw.data(), g.count, &g.dw_tc[l], tf) ||
            (l > 0 && !gemm_tc_prepare(dx.data(), g.count, &g.dx_tc[l], tf)))
          return fail(c, GIST_E_UNSUPPORTED, "tcgen05 GEMM plan failed (alignment / driver entry point)");
      } else {
        for (int j = 0; j < g.count; ++j) {
          g.fwd_f[l].op[j] = fw[j];
          g.dw_f[l].op[j] = dw[j];
          if (l > 0) g.dx_f[l].op[j] = dx[j];
        }
        g.fwd_f[l].n = g.dw_f[l].n = g.count;
        g.dx_f[l].n = l > 0 ? g.count : 0;
      }
    }
    g.opt_l.assign(L, OptRanges());
    for (int l = 0; l < L; ++l) {
      OptRanges& R = g.opt_l[l];
      R.count = g.count;
      for (int j = 0; j < g.count; ++j) {
        const Slot& sl = c->slots[g0 + j];
        const LayerShape& sh = c->shapes[sl.index][l];
        R.W[j] = sl.W + sh.off;
        R.G[j] = sl.G + sh.off;
        R.M[j] = sl.M ? sl.M + sh.off : nullptr;
        R.V[j] = sl.V ? sl.V + sh.off : nullptr;
        R.Wb[j] = sl.Wb ? sl.Wb + sh.off : nullptr;
        R.n[j] = (int64_t)sh.Kp * sh.Np;
      }
    }
    P.groups.push_back(g);
  }
  return GIST_OK;
}

template gist_status build_plan<float>(gist_ctx*, StepPlan<float>&);
template gist_status build_plan<bf16>(gist_ctx*, StepPlan<bf16>&);
}  // namespace gist_impl
