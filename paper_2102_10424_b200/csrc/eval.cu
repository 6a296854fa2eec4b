// eval.cu -- evaluation of the global model (boundary, not the hot path): the full-graph forward
// (R1/R2 operator; rows split across ranks at W > 1), partition-wise evaluation (PAPER.md:696-697,
// R20), their per-node logits hook, and the eval_scale MEAN weights (R10).
#include "ctx.h"

using namespace gist;
using namespace gist_impl;

// single GEMM (eval path): FP32 SIMT or BF16 tcgen05
static gist_status gemm_any(gist_ctx* c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                            const void* B, int64_t ldb, void* C, int64_t ldc, bool out_f32, bool relu,
                            cudaStream_t s) {
  if (c->prec == GIST_PREC_FP32) {
    gemm_f32(ta, tb, M, N, K, (const float*)A, lda, (const float*)B, ldb, (float*)C, ldc, relu, s);
  } else if (c->prec == GIST_PREC_TF32) {
    if (!gemm_tf32(ta, tb, M, N, K, (const float*)A, lda, (const float*)B, ldb, (float*)C, ldc, relu, s))
      return fail(c, GIST_E_UNSUPPORTED, "tf32 tensor-core GEMM unavailable for this shape");
  } else if (!gemm_bf16(ta, tb, M, N, K, (const bf16*)A, lda, (const bf16*)B, ldb, C, ldc, out_f32, relu, s)) {
    return fail(c, GIST_E_UNSUPPORTED, "bf16 tensor-core GEMM unavailable for this shape");
  }
  ++c->nk;
  return GIST_OK;
}

// The weights of the evaluation forward: per layer the fp32 weights (Theta_l, or a copy with its W
// rows scaled by 1/m for layers l >= 1 under eval_scale MEAN, R10) and their T-typed GEMM operand
// (the same pointer in FP32 mode, a bf16 copy in BF16 mode).
struct EvalWeights {
  std::vector<float*> w32;
  std::vector<void*> wT;
  std::vector<void*> owned;
};
template <typename T>
static gist_status eval_weights(gist_ctx* c, EvalWeights& ew) {
  cudaStream_t s = c->stream;
  ew.w32.assign(c->L, nullptr);
  ew.wT.assign(c->L, nullptr);
  const bool mean = c->cfg.eval_scale == GIST_EVAL_SCALE_MEAN && c->m > 1;
  for (int l = 0; l < c->L; ++l) {
    const int64_t n = c->th_K[l] * c->th_N[l];
    float* src = c->theta[l];
    if (sharded(c)) {  // owner-sharded Theta: the layer's rows from every rank (collective)
      float* full = nullptr;
      TRY(dalloc_t(c, &full, (size_t)n));
      ew.owned.push_back(full);
      TRY(shard_gather_layer(c, c->theta[l], l, full, s));
      src = full;
    }
    ew.w32[l] = src;
    if (mean && l > 0) {  // hidden input dim d_l is partitioned: scale the W rows (not GAT's a rows)
      const int64_t nw = (c->arch == GIST_ARCH_GAT ? pad8(c->dims[l]) : c->th_K[l]) * c->th_N[l];
      float* w = nullptr;
      TRY(dalloc_t(c, &w, (size_t)n));
      ew.owned.push_back(w);
      LK(scale_prefix_f32(src, w, n, nw, 1.0f / (float)c->m, s));
      ew.w32[l] = w;
    }
    if (sizeof(T) == 2) {
      void* b = nullptr;
      TRY(dalloc(c, &b, (size_t)n * 2));
      ew.owned.push_back(b);
      LK(f32_to_bf16(ew.w32[l], (bf16*)b, n, s));
      ew.wT[l] = b;
    } else {
      ew.wT[l] = ew.w32[l];
    }
  }
  return GIST_OK;
}
static void free_eval_weights(gist_ctx* c, EvalWeights& ew) {
  for (void* p : ew.owned) dfree(c, p);
  ew.owned.clear();
}

// GAT forward of the global model over `rows` rows of a CSR without self loops (R21): layer 0
// reads X0 (ld pad8(d_0)); hidden outputs alternate between bufA / bufB; fp32 logits (ld th_N).
template <typename T>
static gist_status gat_forward_rows(gist_ctx* c, int64_t rows, const int64_t* row_beg, const int64_t* row_end,
                                    const int32_t* col, const T* X0, const EvalWeights& ew, T* bufA, T* bufB,
                                    T* Z, float* sc, float* logits, cudaStream_t s) {
  const T* Hin = X0;
  int64_t ldin = pad8(c->dims[0]);
  T* Hout = bufA;
  for (int l = 0; l < c->L; ++l) {
    const int64_t K = pad8(c->dims[l]), N = c->th_N[l];
    TRY(gemm_any(c, false, false, rows, N, K, Hin, ldin, ew.wT[l], N, Z, N, sizeof(T) == 4, false, s));
    GatGroup<T> G;
    G.n = 1;
    GatLayer<T>& a = G.a[0];
    a.row_beg = row_beg; a.row_end = row_end; a.col = col; a.rows = rows; a.w = N;
    a.Z = Z; a.ldz = N;
    a.a_src = ew.w32[l] + K * N; a.a_dst = a.a_src + N;
    a.s = sc; a.t = sc + rows; a.lse = sc + 2 * rows;
    a.H = Hin; a.ldh = ldin; a.kw = K; a.W32 = ew.w32[l]; a.ldw = N; a.wa = sc + 3 * rows;
    if (l + 1 < c->L) { a.out = Hout; a.ldo = N; a.relu = 1; }
    else { a.out_f32 = logits; a.ldo = N; }
    LK(gat_scores<T>(G, s));
    LK(gat_forward<T>(G, s));
    Hin = Hout;
    ldin = N;
    Hout = Hout == bufA ? bufB : bufA;
  }
  return GIST_OK;
}

// ================================================================ eval ====
// Full-graph forward of the global model (R1/R2 full-graph operator, R10 no scaling).  World > 1
// (GCN / GraphSAGE): the relabelled rows are cut into W blocks of R = ceil(n / W); rank r
// computes the SpMM and GEMM of block r of every layer and one all-gather per hidden layer
// assembles the next layer's input on every rank (its SpMM gathers neighbours from every block);
// the loss / accuracy sums of the blocks are combined with one sum all-reduce.
// GAT runs the whole forward on every rank (its attention needs Z = H W of every neighbour row).
// logits_host (optional): float[n x k] by ORIGINAL node id, assembled on every rank.
template <typename T>
static gist_status eval_t(gist_ctx* c, int code, float* loss, float* acc, float* logits_host) {
  cudaStream_t s = c->stream;
  const int64_t n = c->n;
  const bool sage = c->arch == GIST_ARCH_SAGE;
  const bool gat = c->arch == GIST_ARCH_GAT;
  const int W = gat ? 1 : c->cfg.world_size;
  const int rank = gat ? 0 : c->cfg.rank;
  const int64_t R = cdiv(n, W);
  const int64_t r0 = std::min<int64_t>(n, (int64_t)rank * R);
  const int64_t nr = std::min<int64_t>(n, r0 + R) - r0;  // rows of this rank's block
  const int64_t npad = R * W;
  const int64_t Nl = c->th_N[c->L - 1];
  int64_t maxK = 0;
  for (int l = 0; l < c->L; ++l) maxK = std::max(maxK, c->th_K[l]);
  void *bufA = nullptr, *bufB = nullptr;
  float* logits = nullptr;
  double* out3 = nullptr;
  EvalWeights ew;
  TRY(eval_weights<T>(c, ew));
  TRY(dalloc(c, &bufA, (size_t)npad * maxK * sizeof(T)));
  TRY(dalloc(c, &bufB, (size_t)npad * maxK * sizeof(T)));
  TRY(dalloc_t(c, &logits, (size_t)npad * Nl));
  TRY(dalloc_t(c, &out3, 3));
  T* Cb = (T*)bufA;
  T* Hn = (T*)bufB;
  if (gat) {
    int64_t maxN = 0;
    for (int l = 0; l < c->L; ++l) maxN = std::max(maxN, c->th_N[l]);
    void* Z = nullptr;
    float* sc = nullptr;
    TRY(dalloc(c, &Z, (size_t)n * maxN * sizeof(T)));
    TRY(dalloc_t(c, &sc, (size_t)3 * std::max<int64_t>(n, 1) + 2 * maxK));
    TRY(gat_forward_rows<T>(c, n, c->rp, c->rp + 1, c->col, (const T*)c->X, ew, Cb, Hn, (T*)Z, sc, logits, s));
    CK(cudaStreamSynchronize(s));
    dfree(c, Z);
    dfree(c, sc);
  }
  for (int l = 0; l < c->L && !gat; ++l) {
    const int64_t K = c->th_K[l], N = c->th_N[l];
    const int64_t half = pad8(c->dims[l]);
    SpmmArgs<T, T> a;
    a.row_beg = c->rp + r0; a.row_end = c->rp + r0 + 1; a.col = c->col; a.rows = nr;
    a.row0 = r0; a.h_rows = n;
    a.rowscale = c->full_scale + r0;
    const T* Hin = l == 0 ? (const T*)c->X : (const T*)Hn;
    if (sage) {
      if (l == 0) { a.self_out = Cb + r0 * K; a.ld_self = K; }
      a.H = l == 0 ? Hin : Cb; a.ldh = l == 0 ? half : K;
      a.out = Cb + r0 * K + half; a.ldo = K; a.w = half;
    } else {
      a.colscale = c->full_scale; a.self = 1; a.H = Hin; a.ldh = half; a.out = Cb + r0 * K; a.ldo = K; a.w = K;
    }
    if (nr > 0) LK((spmm<T, T>(a, s)));
    const void* Wl = ew.wT[l];
    if (l + 1 < c->L) {
      // next layer input: GCN H_{l+1} -> Hn; SAGE H_{l+1} -> left half of Hn, which becomes the
      // next concat buffer (swap)
      const int64_t Kn = c->th_K[l + 1];
      if (nr > 0) TRY(gemm_any(c, false, false, nr, N, K, Cb + r0 * K, K, Wl, N, Hn + r0 * Kn, Kn, false, true, s));
      if (sage) std::swap(Cb, Hn);
      T* next = sage ? Cb : Hn;  // the buffer the next layer's SpMM gathers from
      if (W > 1)
        TRY(coll(c, comm_allgather(c->comm, next + (int64_t)rank * R * Kn, next, (size_t)R * Kn * sizeof(T), s,
                                   &c->err)));
    } else if (nr > 0) {
      TRY(gemm_any(c, false, false, nr, N, K, Cb + r0 * K, K, Wl, N, logits + r0 * N, N, true, false, s));
    }
  }
  CK(cudaMemsetAsync(out3, 0, 3 * sizeof(double), s));
  if (nr > 0) LK(eval_rows(logits + r0 * Nl, Nl, nr, c->k, c->labels + r0, c->split + r0, code, out3, s));
  if (W > 1) TRY(coll(c, comm_allreduce_sum(c->comm, out3, 3, true, s, &c->err)));
  double h[3];
  CK(cudaMemcpyAsync(h, out3, sizeof(h), cudaMemcpyDeviceToHost, s));
  if (logits_host) {
    if (W > 1)
      TRY(coll(c, comm_allgather(c->comm, logits + (int64_t)rank * R * Nl, logits, (size_t)R * Nl * 4, s, &c->err)));
    std::vector<float> lg((size_t)n * Nl);
    CK(cudaMemcpyAsync(lg.data(), logits, lg.size() * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int64_t g = 0; g < n; ++g)
      std::memcpy(logits_host + (size_t)c->perm_h[g] * c->k, lg.data() + (size_t)g * Nl, (size_t)c->k * 4);
    c->d2h += (int64_t)n * Nl * 4;
  }
  CK(cudaStreamSynchronize(s));
  TRY(check_launch(c, "eval"));
  if (loss) *loss = h[2] > 0 ? (float)(h[0] / h[2]) : 0.f;
  if (acc) *acc = h[2] > 0 ? (float)(h[1] / h[2]) : 0.f;
  dfree(c, bufA);
  dfree(c, bufB);
  dfree(c, logits);
  dfree(c, out3);
  free_eval_weights(c, ew);
  return GIST_OK;
}

extern "C" gist_status gist_eval(gist_ctx* c, int32_t split_code, float* loss, float* acc) {
  PRE(c);
  Range nvtx_range("gist_eval");
  if (c->state != S_PARAMS) return fail(c, GIST_E_STATE, "eval: needs params and no open round");
  if (split_code < 0 || split_code > 3) return fail(c, GIST_E_ARG, "eval: split code not in 0..3");
  if (c->prec == GIST_PREC_BF16) return eval_t<bf16>(c, split_code, loss, acc, nullptr);
  return eval_t<float>(c, split_code, loss, acc, nullptr);
}

// ==================================================== partition-wise eval (R20) ===
// for wide models the global model is evaluated partition by partition.
// Every partition is a closed subgraph (cut edges dropped), so the local partitions of this
// rank are laid out contiguously (partition order) and processed in row chunks of whole
// partitions: per layer one SpMM over the chunk's partition-induced CSR (layer 0 reads X
// through a row index, no copy) and one GEMM, all buffers chunk-sized.  World > 1:
// partition p is evaluated by rank p mod W and the per-partition sums are all-reduced.
template <typename T>
static gist_status eval_parts_t(gist_ctx* c, int code, const std::vector<int32_t>& part, int np, int64_t max_rows,
                                std::vector<double>& sums, float* logits_host) {
  cudaStream_t s = c->stream;
  const int64_t n = c->n;
  const bool sage = c->arch == GIST_ARCH_SAGE;
  const int W = c->cfg.world_size, rank = c->cfg.rank;
  // local partitions (p mod W == rank) in partition order, nodes ascending (internal ids)
  std::vector<int64_t> cnt(np + 1, 0);
  for (int64_t g = 0; g < n; ++g) ++cnt[part[g] + 1];
  std::vector<int32_t> lparts;
  for (int p = rank; p < np; p += W) lparts.push_back(p);
  const int nlp = (int)lparts.size();
  std::vector<int64_t> lbeg(nlp + 1, 0);
  std::vector<int64_t> fill(np, -1);
  for (int j = 0; j < nlp; ++j) {
    fill[lparts[j]] = lbeg[j];
    lbeg[j + 1] = lbeg[j] + cnt[lparts[j] + 1];
  }
  const int64_t nl = lbeg[nlp];
  std::vector<int32_t> pnode(std::max<int64_t>(nl, 1)), pos(n, -1), rowbase(std::max<int64_t>(nl, 1));
  for (int64_t g = 0; g < n; ++g) {
    const int p = part[g];
    if (fill[p] < 0) continue;
    pos[g] = (int32_t)fill[p];
    pnode[fill[p]++] = (int32_t)g;
  }
  // buffers and chunking
  int64_t maxK = 0;
  for (int l = 0; l < c->L; ++l) maxK = std::max(maxK, c->th_K[l]);
  const int64_t Nl = c->th_N[c->L - 1];
  EvalWeights ew;
  TRY(eval_weights<T>(c, ew));
  const int64_t row_bytes = 2 * maxK * (int64_t)sizeof(T) + Nl * 4;
  if (max_rows <= 0) {
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    max_rows = std::max<int64_t>(1, (int64_t)(fr / 2) / row_bytes);
  }
  std::vector<int> chunk_first{0};  // chunk j = local partitions chunk_first[j] .. chunk_first[j+1]
  for (int j = 0; j < nlp; ++j) {
    const int f = chunk_first.back();
    if (j > f && lbeg[j + 1] - lbeg[f] > max_rows) chunk_first.push_back(j);
  }
  chunk_first.push_back(nlp);
  int64_t max_chunk = 0;
  for (size_t j = 0; j + 1 < chunk_first.size(); ++j) {
    const int64_t k0 = lbeg[chunk_first[j]], k1 = lbeg[chunk_first[j + 1]];
    max_chunk = std::max(max_chunk, k1 - k0);
    for (int64_t r = k0; r < k1; ++r) rowbase[r] = (int32_t)k0;
  }
  // partition-induced CSR (device)
  int32_t *pnode_d = nullptr, *pos_d = nullptr, *part_d = nullptr, *rb_d = nullptr, *pcol = nullptr;
  int64_t *deg = nullptr, *prp = nullptr, *lbeg_d = nullptr;
  float* pscale = nullptr;
  double* out3 = nullptr;
  TRY(dalloc_t(c, &pnode_d, std::max<int64_t>(nl, 1)));
  TRY(dalloc_t(c, &pos_d, n));
  TRY(dalloc_t(c, &part_d, n));
  TRY(dalloc_t(c, &rb_d, std::max<int64_t>(nl, 1)));
  TRY(dalloc_t(c, &deg, nl + 1));
  TRY(dalloc_t(c, &prp, nl + 1));
  TRY(dalloc_t(c, &lbeg_d, nlp + 1));
  TRY(dalloc_t(c, &pscale, std::max<int64_t>(nl, 1)));
  TRY(dalloc_t(c, &out3, 3 * (size_t)std::max(nlp, 1)));
  CK(cudaMemcpyAsync(pnode_d, pnode.data(), nl * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(pos_d, pos.data(), n * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(part_d, part.data(), n * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(rb_d, rowbase.data(), nl * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(lbeg_d, lbeg.data(), (nlp + 1) * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(deg, 0, (nl + 1) * 8, s));
  LK(part_count(c->rp, c->col, pnode_d, part_d, nl, deg, s));
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, deg, prp, nl + 1, s);
    void* tmp = nullptr;
    TRY(dalloc(c, &tmp, tb));
    cub::DeviceScan::ExclusiveSum(tmp, tb, deg, prp, nl + 1, s);
    ++c->nk;
    CK(cudaStreamSynchronize(s));
    dfree(c, tmp);
  }
  int64_t pnnz = 0;
  CK(cudaMemcpy(&pnnz, prp + nl, 8, cudaMemcpyDeviceToHost));
  TRY(dalloc_t(c, &pcol, std::max<int64_t>(pnnz, 1)));
  LK(part_fill(c->rp, c->col, pnode_d, pos_d, part_d, rb_d, prp, nl, pcol, s));
  LK(full_graph_scales(prp, nl, c->arch, pscale, s));
  void *bufA = nullptr, *bufB = nullptr;
  float* logits = nullptr;
  TRY(dalloc(c, &bufA, (size_t)std::max<int64_t>(max_chunk, 1) * maxK * sizeof(T)));
  TRY(dalloc(c, &bufB, (size_t)std::max<int64_t>(max_chunk, 1) * maxK * sizeof(T)));
  TRY(dalloc_t(c, &logits, (size_t)std::max<int64_t>(max_chunk, 1) * Nl));
  void *gX = nullptr, *gZ = nullptr;
  float* gsc = nullptr;
  if (c->arch == GIST_ARCH_GAT) {
    int64_t maxN = 0;
    for (int l = 0; l < c->L; ++l) maxN = std::max(maxN, c->th_N[l]);
    TRY(dalloc(c, &gX, (size_t)std::max<int64_t>(max_chunk, 1) * pad8(c->dims[0]) * sizeof(T)));
    TRY(dalloc(c, &gZ, (size_t)std::max<int64_t>(max_chunk, 1) * maxN * sizeof(T)));
    TRY(dalloc_t(c, &gsc, (size_t)3 * std::max<int64_t>(max_chunk, 1) + 2 * maxK));
  }
  for (size_t j = 0; j + 1 < chunk_first.size(); ++j) {
    const int f = chunk_first[j], e = chunk_first[j + 1];
    const int64_t k0 = lbeg[f], rows = lbeg[e] - k0;
    if (rows == 0) continue;
    T* Cb = (T*)bufA;
    T* Hn = (T*)bufB;
    if (c->arch == GIST_ARCH_GAT) {  // X rows of the chunk gathered, then the GAT layers
      const int64_t d0p = pad8(c->dims[0]);
      LK(gather_rows_t<T>((const T*)c->X, d0p, pnode_d + k0, rows, d0p, (T*)gX, d0p, s));
      TRY(gat_forward_rows<T>(c, rows, prp + k0, prp + k0 + 1, pcol, (const T*)gX, ew, Cb, Hn, (T*)gZ, gsc, logits,
                              s));
    }
    for (int l = 0; l < c->L && c->arch != GIST_ARCH_GAT; ++l) {
      const int64_t K = c->th_K[l], N = c->th_N[l];
      const int64_t half = pad8(c->dims[l]);
      SpmmArgs<T, T> a;
      a.row_beg = prp + k0; a.row_end = prp + k0 + 1; a.col = pcol; a.rows = rows; a.rowscale = pscale + k0;
      const T* Hin = l == 0 ? (const T*)c->X : (const T*)Hn;
      if (l == 0) a.h_index = pnode_d + k0;  // chunk row -> internal node id (rows of X)
      if (sage) {
        if (l == 0) { a.self_out = Cb; a.ld_self = K; }
        a.H = l == 0 ? Hin : Cb; a.ldh = l == 0 ? half : K;
        a.out = Cb + half; a.ldo = K; a.w = half;
      } else {
        a.colscale = pscale + k0; a.self = 1; a.H = Hin; a.ldh = half; a.out = Cb; a.ldo = K; a.w = K;
      }
      LK((spmm<T, T>(a, s)));
      const void* Wl = ew.wT[l];
      if (l + 1 < c->L) {
        TRY(gemm_any(c, false, false, rows, N, K, Cb, K, Wl, N, Hn, c->th_K[l + 1], false, true, s));
        if (sage) std::swap(Cb, Hn);
      } else {
        TRY(gemm_any(c, false, false, rows, N, K, Cb, K, Wl, N, logits, N, true, false, s));
      }
    }
    LK(eval_parts(logits, Nl, c->k, lbeg_d + f, k0, e - f, pnode_d, c->labels, c->split, code, out3 + 3 * f, s));
    if (logits_host) {  // parity hook: chunk logits -> host rows of their nodes (internal ids)
      std::vector<float> lg((size_t)rows * Nl);
      CK(cudaMemcpyAsync(lg.data(), logits, lg.size() * 4, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int64_t i = 0; i < rows; ++i)
        std::memcpy(logits_host + (size_t)pnode[k0 + i] * c->k, lg.data() + (size_t)i * Nl, (size_t)c->k * 4);
    }
  }
  std::vector<double> loc(3 * (size_t)std::max(nlp, 1));
  CK(cudaMemcpyAsync(loc.data(), out3, loc.size() * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  TRY(check_launch(c, "eval_parts"));
  sums.assign(3 * (size_t)np, 0.0);
  for (int j = 0; j < nlp; ++j)
    for (int q = 0; q < 3; ++q) sums[3 * (size_t)lparts[j] + q] = loc[3 * (size_t)j + q];
  if (W > 1) {  // every partition was evaluated by exactly one rank: a sum-all-reduce assembles them
    double* red = nullptr;
    TRY(dalloc_t(c, &red, sums.size()));
    CK(cudaMemcpyAsync(red, sums.data(), sums.size() * 8, cudaMemcpyHostToDevice, s));
    TRY(coll(c, comm_allreduce_sum(c->comm, red, sums.size(), true, s, &c->err)));
    CK(cudaMemcpyAsync(sums.data(), red, sums.size() * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    dfree(c, red);
    if (logits_host) {  // every node's row was written by exactly one rank, zeros elsewhere: exact sum
      float* lr = nullptr;
      TRY(dalloc_t(c, &lr, (size_t)n * c->k));
      CK(cudaMemcpyAsync(lr, logits_host, (size_t)n * c->k * 4, cudaMemcpyHostToDevice, s));
      TRY(coll(c, comm_allreduce_sum(c->comm, lr, (size_t)n * c->k, false, s, &c->err)));
      CK(cudaMemcpyAsync(logits_host, lr, (size_t)n * c->k * 4, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      dfree(c, lr);
    }
  }
  free_eval_weights(c, ew);
  for (void* p : {gX, gZ, (void*)gsc}) if (p) dfree(c, p);
  for (void* p : {(void*)pnode_d, (void*)pos_d, (void*)part_d, (void*)rb_d, (void*)pcol, (void*)deg, (void*)prp,
                  (void*)lbeg_d, (void*)pscale, (void*)out3, bufA, bufB, (void*)logits})
    dfree(c, p);
  return GIST_OK;
}

// partition of every internal node id from the caller's ids (original ids), or the training clusters
static gist_status resolve_parts(gist_ctx* c, const int32_t* part_ids, int32_t num_parts, std::vector<int32_t>& part,
                                 int* np) {
  const int64_t n = c->n;
  part.assign(n, 0);
  *np = num_parts;
  if (part_ids) {
    if (num_parts < 1) return fail(c, GIST_E_ARG, "eval_parts: num_parts < 1");
    for (int64_t g = 0; g < n; ++g) {
      const int32_t p = part_ids[c->perm_h[g]];
      if (p < 0 || p >= num_parts) return fail(c, GIST_E_ARG, "eval_parts: partition id out of range");
      part[g] = p;
    }
  } else {  // the training clusters (contiguous internal id ranges after relabelling)
    *np = (int)c->cstart_h.size() - 1;
    if (num_parts != 0 && num_parts != *np) return fail(c, GIST_E_ARG, "eval_parts: num_parts != clusters");
    for (int p = 0; p < *np; ++p)
      for (int64_t g = c->cstart_h[p]; g < c->cstart_h[p + 1]; ++g) part[g] = p;
  }
  return GIST_OK;
}

extern "C" gist_status gist_eval_parts(gist_ctx* c, int32_t split_code, const int32_t* part_ids, int32_t num_parts,
                                       int64_t max_rows, float* loss, float* acc, float* part_loss,
                                       float* part_acc) {
  PRE(c);
  Range nvtx_range("gist_eval_parts");
  if (c->state != S_PARAMS) return fail(c, GIST_E_STATE, "eval_parts: needs params and no open round");
  if (split_code < 0 || split_code > 3) return fail(c, GIST_E_ARG, "eval_parts: split code not in 0..3");
  std::vector<int32_t> part;
  int np = 0;
  TRY(resolve_parts(c, part_ids, num_parts, part, &np));
  std::vector<double> sums;
  TRY(c->prec == GIST_PREC_BF16 ? eval_parts_t<bf16>(c, split_code, part, np, max_rows, sums, nullptr)
                                : eval_parts_t<float>(c, split_code, part, np, max_rows, sums, nullptr));
  double ls = 0.0, as = 0.0;
  int cntp = 0;
  for (int p = 0; p < np; ++p) {
    const double k = sums[3 * (size_t)p + 2];
    const float lp = k > 0 ? (float)(sums[3 * (size_t)p] / k) : NAN;
    const float ap = k > 0 ? (float)(sums[3 * (size_t)p + 1] / k) : NAN;
    if (part_loss) part_loss[p] = lp;
    if (part_acc) part_acc[p] = ap;
    if (k > 0) ls += sums[3 * (size_t)p] / k, as += sums[3 * (size_t)p + 1] / k, ++cntp;
  }
  if (loss) *loss = cntp ? (float)(ls / cntp) : 0.f;
  if (acc) *acc = cntp ? (float)(as / cntp) : 0.f;
  return GIST_OK;
}

extern "C" gist_status gist_eval_logits(gist_ctx* c, int32_t mode, const int32_t* part_ids, int32_t num_parts,
                                        int64_t max_rows, float* out) {
  PRE(c);
  Range nvtx_range("gist_eval_logits");
  if (c->state != S_PARAMS) return fail(c, GIST_E_STATE, "eval_logits: needs params and no open round");
  if (!out || (mode != 0 && mode != 1)) return fail(c, GIST_E_ARG, "eval_logits: mode not 0/1 or null output");
  if (mode == 0)
    return c->prec == GIST_PREC_BF16 ? eval_t<bf16>(c, 0, nullptr, nullptr, out) : eval_t<float>(c, 0, nullptr, nullptr, out);
  std::vector<int32_t> part;
  int np = 0;
  TRY(resolve_parts(c, part_ids, num_parts, part, &np));
  // internal-id rows, then the original-id order of the output
  std::vector<float> li((size_t)c->n * c->k, 0.f);
  std::vector<double> sums;
  TRY(c->prec == GIST_PREC_BF16 ? eval_parts_t<bf16>(c, 0, part, np, max_rows, sums, li.data())
                                : eval_parts_t<float>(c, 0, part, np, max_rows, sums, li.data()));
  for (int64_t g = 0; g < c->n; ++g)
    std::memcpy(out + (size_t)c->perm_h[g] * c->k, li.data() + (size_t)g * c->k, (size_t)c->k * 4);
  return GIST_OK;
}
