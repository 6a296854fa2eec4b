// kernels.h -- internal launchers of the GIST B200 library.  Every hot-path step
// of subTrain / subGCNs / subAgg runs in one of these kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>

namespace gist {

using bf16 = __nv_bfloat16;

// --------------------------------------------------------------------------
// Aggregation SpMM (Eq. 1/2 sparse factor A_bar H).
//   out[v] = mask(v) * ( add[v] + rowscale[v] * ( self*colscale[v]*H[h(v)] + sum_u colscale[u]*H[h(u)] ) )
// where h(u) = h_index ? h_index[u] : u.  Optionally copies H[h(v)] to self_out[v]
// (GraphSAGE concat [H || N H], R2).  Widths are padded to multiples of 8.
// --------------------------------------------------------------------------
struct StepState;
template <typename TI, typename TO = TI>
struct SpmmArgs {
  const int64_t* row_beg = nullptr;  // row v's neighbours are col[row_beg[v] .. row_end[v])
  const int64_t* row_end = nullptr;  // (plain CSR: row_end = row_ptr + 1)
  const int32_t* col = nullptr;
  int64_t rows = 0;
  const float* rowscale = nullptr;
  const float* colscale = nullptr;
  int self = 0;
  int relu = 0;
  const int32_t* h_index = nullptr;
  const TI* H = nullptr;
  int64_t ldh = 0;
  const TI* add = nullptr;
  int64_t ld_add = 0;
  const TI* mask = nullptr;
  int64_t ld_mask = 0;
  const uint32_t* mbits = nullptr;  // bit-packed form of `mask` (GemmOp::mbits); used instead if set
  int64_t ld_mbits = 0;
  TO* out = nullptr;
  int64_t ldo = 0;
  TI* self_out = nullptr;
  int64_t ld_self = 0;
  int64_t w = 0;  // padded width processed (multiple of 8)
  // row-block launches (row-split eval): local row v is graph row v + row0 for the self term
  // (H row, colscale); neighbours are graph ids.  h_rows = rows of H the gathers may reach
  // (0: rows), for the 32-bit offset choice.
  int64_t row0 = 0, h_rows = 0;
  // batch SpMMs: the step descriptor (marks the launch as a mini-batch pass, not full-graph)
  const int32_t* desc = nullptr;
  const StepState* st = nullptr;
  int q = 0;
  int few_nnz = 0;  // hint: rows have few neighbours (inter-cluster pass): favour occupancy
  // every operand except `add` was written two or more launches back (the inter-cluster pass
  // after its block-diagonal pass): gather before waiting on the predecessor (k_spmm)
  int early = 0;
};
template <typename TI, typename TO> void spmm(const SpmmArgs<TI, TO>& a, cudaStream_t s);

// Grouped launch: the same SpMM for up to kMaxGroup sub-GCN slots in one grid (grid.y = slot).
constexpr int kMaxGroup = 8;
// a grouped tcgen05 GEMM launch may carry two operand sets per slot (re-associated last layer)
constexpr int kMaxGemmOps = 2 * kMaxGroup;
template <typename TI, typename TO = TI>
struct SpmmGroup {
  SpmmArgs<TI, TO> a[kMaxGroup];
  int n = 0;
};
template <typename TI, typename TO> void spmm_group(const SpmmGroup<TI, TO>& G, cudaStream_t s);

// --------------------------------------------------------------------------
// Dense contractions.  C[M x N] = op(A)[M x K] op(B)[K x N].
//   transA: A stored K x M (lda >= M); else M x K.  transB: B stored N x K; else K x N.
// FP32 parity path: SIMT FFMA tiles.  BF16 path: tcgen05 + TMA + TMEM.
// --------------------------------------------------------------------------
void gemm_f32(bool transA, bool transB, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
              const float* B, int64_t ldb, float* C, int64_t ldc, bool relu, cudaStream_t s);
// One operand set of a (grouped) GEMM.  mask (optional, same dtype as the operands):
// out = acc * 1[mask[row, col] > 0] (the ReLU mask of the layer below).
struct GemmOp {
  bool transA, transB;
  int64_t M, N, K;
  const void* A;
  int64_t lda;
  const void* B;
  int64_t ldb;
  void* C;
  int64_t ldc;
  bool out_f32, relu;
  const void* mask;
  int64_t ldm;
  const float* rscale;  // optional per-row scale of the output columns >= rs_from (BF16 path)
  int rs_from;
  // optional (BF16 path): bit-packed ReLU mask of the stored output, bit (col % 32) of word
  // [row * ldmb + col / 32] = 1[out[row, col] > 0] (read by the backward pass instead of out)
  uint32_t* mbits = nullptr;
  int64_t ldmb = 0;
  // L2 residency hints: keep_out = the output is read again by the next kernels (evict_last);
  // stream_a = this is the last read of A for a while (evict_first)
  int keep_out = 0, stream_a = 0;
  // optional (BF16 path): out += add (bf16, ldadd), then out *= 1[bit] with the bit-packed
  // ReLU mask mbits_in (words [row * ldmbi + col / 32]) of the layer below
  const bf16* add = nullptr;
  int64_t ldadd = 0;
  const uint32_t* mbits_in = nullptr;
  int64_t ldmbi = 0;
};
}  // namespace gist
#include <cuda.h>
namespace gist {
struct alignas(64) GemmSlotTC {
  CUtensorMap ma, mb;  // TMA descriptors (128 B each)
  CUtensorMap mc;      // output store map (boxes of 32 rows x 128 B, SWIZZLE_128B); valid if tma_store
  void* C;
  const void* mask;
  const float* rscale;
  uint32_t* mbits;
  const bf16* add;
  const uint32_t* mbits_in;
  int64_t ldc, ldm, ldmb, ldadd, ldmbi;
  int M, N, K, relu, rs_from, tma_store, keep_out, stream_a;
};
struct GemmGroupTC {
  GemmSlotTC s[kMaxGemmOps];
  int n = 0, tm = 0, tn = 0;  // slots, M tiles, N tiles (persistent tile space)
};
// Host-side plan of one grouped tcgen05 GEMM (tensor maps encoded once, launched many times).
struct GemmPlanTC {
  GemmGroupTC G;
  bool a_mn = false, b_mn = false, out_f32 = false, relu = false, mask = false;
  bool pair = false;  // CTA-pair (cta_group::2) kernel
  bool tf32 = false;  // TF32 mode: fp32 operands (kind::tf32), fp32 outputs
  int bn = 128;
  int64_t maxM = 0, maxN = 0;
};
bool gemm_bf16_prepare(const GemmOp* ops, int n, GemmPlanTC* plan);
// tf32 = true: TF32 mode (R13) -- fp32 operands read as tf32, fp32 outputs, relu only
bool gemm_tc_prepare(const GemmOp* ops, int n, GemmPlanTC* plan, bool tf32);
void gemm_bf16_launch(const GemmPlanTC& plan, cudaStream_t s);

// Block-diagonal cluster aggregation on tcgen05 (SAGE, Cluster mini-batches):
//   out[loff_k + r] = rscale[row] * sum_j A_c[r, j] * H[h0 + j]  (+ add[row]),  r < |cluster k|
// with A_c the binary intra-cluster adjacency block of cluster c = bcl[k] (BS x BS bf16,
// precomputed once per graph), h0 = loff_k or cstart[c] (global_rows).  Cluster ids and
// offsets come from the device step descriptor, so the launch is step-invariant.
struct BdOp {
  const bf16* H;
  int64_t ldh, h_rows, N;
  void* C;  // bf16 output
  int64_t ldc;
  const bf16* add;
  int64_t ldadd;
  const float* rscale;
  const int32_t* desc;
  int global_rows;
  int keep_out = 0;  // L2 hint for the output (see GemmOp)
};
struct alignas(64) BdSlot {
  CUtensorMap mb;
  CUtensorMap mc;  // output store map (see GemmSlotTC::mc); valid if tma_store
  void* C;
  const bf16* add;
  const float* rscale;
  const int32_t* desc;
  int64_t ldc, ldadd;
  int N, global_rows, tma_store, keep_out;
};
struct BdGroup {
  CUtensorMap ma;  // all cluster blocks [num_clusters * BS, BS]
  CUtensorMap mat;  // the same, boxes of 64 columns x BS rows (one block's k-block: k_bd_t)
  BdSlot s[kMaxGroup];
  int n = 0, q = 0, bs = 0, tn = 0;
  int64_t rows = 0;  // static batch rows (nb_max): dummy rows [n_b, rows) are zero-filled
  const StepState* st = nullptr;
  const int64_t* cstart = nullptr;
  int blk_bufs = 2;  // k_bd_t: cluster-block buffers in shared memory
};
struct BdPlan {
  BdGroup G;
  int bn = 128;
  bool transposed = false;  // k_bd_t (see gemm_tc.cu)
  int64_t maxN = 0;
};
bool gemm_bd_prepare(const bf16* blocks, int num_clusters, int bs, const BdOp* ops, int n, int q, int64_t rows,
                     const int64_t* cstart, const StepState* st, BdPlan* plan);
void gemm_bd_launch(const BdPlan& plan, cudaStream_t s);
// FP32 SIMT grouped GEMM (grid.z = slot)
struct SgemmGroup {
  GemmOp op[kMaxGroup];
  int n = 0;
};
void gemm_f32_group(const SgemmGroup& g, cudaStream_t s);
// returns false if the shape/alignment is not supported by the tensor-core path
bool gemm_bf16(bool transA, bool transB, int64_t M, int64_t N, int64_t K, const bf16* A, int64_t lda,
               const bf16* B, int64_t ldb, void* C, int64_t ldc, bool out_f32, bool relu, cudaStream_t s,
               int reps = 1);
bool gemm_tf32(bool transA, bool transB, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
               const float* B, int64_t ldb, float* C, int64_t ldc, bool relu, cudaStream_t s, int reps = 1);

// --------------------------------------------------------------------------
// Graph load (relabel nodes so clusters are contiguous) and Cluster mini-batch
// build.
// --------------------------------------------------------------------------
void relabel_count(const int64_t* rp, const int32_t* col, const int32_t* perm, int64_t n, int64_t* deg_new,
                   cudaStream_t s);
void relabel_fill(const int64_t* rp, const int32_t* col, const int32_t* perm, const int32_t* inv,
                  const int64_t* rp_new, int64_t n, int32_t* col_new, cudaStream_t s);
template <typename T>
void gather_rows_f32(const float* src, int64_t ld_src, const int32_t* idx, int64_t n, int64_t w, T* dst,
                     int64_t ld_dst, cudaStream_t s);
// partition-wise eval (R20): partition-induced CSR in partition order, chunk-relative columns
void part_count(const int64_t* rp, const int32_t* col, const int32_t* pnode, const int32_t* part, int64_t n,
                int64_t* deg_new, cudaStream_t s);
void part_fill(const int64_t* rp, const int32_t* col, const int32_t* pnode, const int32_t* pos, const int32_t* part,
               const int32_t* rowbase, const int64_t* rp_new, int64_t n, int32_t* col_new, cudaStream_t s);
void full_graph_scales(const int64_t* rp, int64_t n, int arch, float* scale, cudaStream_t s);

// Device-resident step state: the kernels of one subTrain step read everything that
// changes from step to step from here, so a step is a fixed launch sequence (captured once
// as a CUDA graph and replayed).  z = index of the current step in this call's descriptor
// array, t = optimizer steps taken since the last partition, lr = learning rate of the call.
struct StepState {
  int32_t z, t;
  float lr;
  uint32_t done;   // optimizer CTAs finished this step (the last one advances z, t and resets it)
};
// Per-step batch descriptor (host-built, R7), 3q+4 int32:
//   [bcl(q) | loff(q+1) | voff(q+1) | qq | tag]
// bcl = cluster ids, loff = local row offsets (loff[qq..q] = n_b), voff = offsets of each
// cluster's adjacency segment inside b_col, qq = clusters in this batch, tag = unique
// per slot and step.  map64[c] = (tag << 32) | (uint32)(loff_k - cstart[c]) for the batch's
// clusters: neighbour u is in the batch iff (map64[cid[u]] >> 32) == tag (nothing to reset).
// Rows [n_b, nb_max) are inert dummy rows (no neighbours, scale 0, not train), so every
// launch uses the static row count nb_max.
struct BatchSlot {
  const int32_t* desc;
  uint64_t* map64;
  int32_t* b_nodes;
  int64_t *b_beg, *b_end;
  int32_t* b_col;
  float* scale;
  int32_t* lab_b;
  uint8_t* train_b;
  int64_t* stats;  // [0] nnz_b, [1] train rows, [2] batch-build row counter (int)
};
struct BatchGroup {
  BatchSlot s[kMaxGroup];
  int n = 0, q = 0, nb_max = 0;
  // per-group batch counter {index of the batch to build, finished build CTAs}: the build of
  // step z+1 may run on a side stream while step z's optimizer advances the step state's z, so
  // the builds keep their own index (zeroed per subTrain call; the last build CTA advances it)
  int32_t* ctr = nullptr;
  // optional: copy the batch rows of the feature matrix X (bf16, ldx) into xdst[slot] (ldxd)
  const bf16* X = nullptr;
  int64_t ldx = 0, ldxd = 0;
  bf16* xdst[kMaxGroup] = {};
  // the build leaves the X copy to batch_xcopy (early prefetch: the build overlaps the previous
  // step's dW_0, which still reads the destination)
  int skip_x = 0;
};
void batch_setup(const BatchGroup& G, const int64_t* cstart, const int64_t* rp, cudaStream_t s);
// skip_intra: intra-cluster edges only count towards the degree (they are aggregated by the
// block-diagonal tensor-core path); the batch CSR then holds the inter-cluster edges only.
// ccol[e] = cid[col[e]] (cluster of every edge's neighbour, precomputed at load)
void batch_build(const BatchGroup& G, const int64_t* rp, const int32_t* col, const int32_t* ccol,
                 const int32_t* cid, const int64_t* cstart, int num_clusters, int arch, const int32_t* labels,
                 const uint8_t* split, int skip_intra, int ob, cudaStream_t s);
// the X copy of a batch built with skip_x: rows with b_beg >= 0 (dummy rows untouched, as in the build)
void batch_xcopy(const BatchGroup& G, cudaStream_t s);
// packed edge codes for the batch build: offset bits ob (0 = packing does not apply: use ccol)
int pack_bits(int num_clusters, int64_t max_csize);
void edge_codes(const int32_t* col, const int32_t* cid, const int64_t* cstart, int64_t nnz, int ob, int32_t* code,
                cudaStream_t s);
void edge_clusters(const int32_t* col, const int32_t* cid, int64_t nnz, int32_t* ccol, cudaStream_t s);
// out[5] (zeroed by the caller): edges with col outside [0, n), self loops, intra-cluster edges,
// unsorted / duplicate edges within a row, edges without their reverse (asymmetric A)
void validate_edges(const int64_t* rp, const int32_t* col, const int32_t* cid, int64_t n, unsigned long long* out,
                    cudaStream_t s);
// Binary intra-cluster adjacency blocks: blocks[c][i][j] = 1 iff (cstart[c]+i, cstart[c]+j) is an
// edge (relabelled ids), bf16 [num_clusters x bs x bs], zeroed by the caller.
void cluster_blocks(const int64_t* rp, const int32_t* col, const int32_t* cid, const int64_t* cstart, int64_t n,
                    int bs, bf16* blocks, cudaStream_t s);

// --------------------------------------------------------------------------
// Loss (R4), optimizers (R8), reductions.
// --------------------------------------------------------------------------
template <typename T>
struct CeSlot {
  float* logits;
  T* dlog;
  float* row_loss;
  const int32_t* lab;
  const uint8_t* train;
  const int64_t* stats;
  float *step_loss, *loss_acc;
  uint32_t* done;  // CTAs of this slot finished (the last one reduces the loss and resets it)
  T* dlog_s = nullptr;              // optional second output: dlogits * scale[v] (row scale)
  const float* scale_s = nullptr;
  // optional: logits = logits + add (fp32 addition), written back before the softmax (the
  // re-associated last GraphSAGE layer's N (H W_bot), row stride ld)
  const T* add = nullptr;
};
template <typename T>
struct CeGroup {
  CeSlot<T> s[kMaxGroup];
  int n = 0, rows = 0, k = 0;
  int64_t ld = 0;       // logits row stride
  int64_t ld_dlog = 0;  // dlogits (and dlog_s) row stride; 0 = ld
};
// per slot: dlogits = (softmax - onehot)/n_train on train rows (else 0), row losses
template <typename T> void softmax_ce(const CeGroup<T>& G, cudaStream_t s);
// per slot: step_loss = sum(row_loss)/n_train (0 if none); loss_acc += step_loss
// Adam (R8) over n packed parameters; bias corrections from st->t (device), lr from st->lr
void adam_step(float* W, const float* G, float* M, float* V, int64_t n, float b1, float b2, float eps,
               StepState* st, bf16* Wb, cudaStream_t s);
void sgd_step(float* W, const float* G, int64_t n, StepState* st, bf16* Wb, cudaStream_t s);
// One layer's optimizer over the slots of a lockstep group (grid.y = slot): the same element
// update as adam_step / sgd_step, without the step-state advance (step_advance does it once the
// step's last layer is done).  Launched on the dW stream right after that layer's dW GEMM.
struct OptRanges {
  float* W[kMaxGroup];
  const float* G[kMaxGroup];
  float* M[kMaxGroup];
  float* V[kMaxGroup];
  bf16* Wb[kMaxGroup];
  int64_t n[kMaxGroup];  // elements (multiple of 4)
  int count = 0;
};
void adam_ranges(const OptRanges& R, float b1, float b2, float eps, const StepState* st, cudaStream_t s);
void sgd_ranges(const OptRanges& R, const StepState* st, cudaStream_t s);
void step_advance(StepState* st, cudaStream_t s);
// Re-associated last layer: Wcat[r][c2] = [W_top | W_bot] (half x 2Np, row-major) from the
// bf16 shadow W = [W_top; W_bot] (2 half x Np), so dH = [dZ | Q] Wcat^T is one K = 2 Np GEMM.
struct RelayoutGroup {
  const bf16* src[kMaxGroup];
  bf16* dst[kMaxGroup];
  int half[kMaxGroup];
  int n = 0, Np = 0, max_half = 0;
};
void relayout_last(const RelayoutGroup& G, cudaStream_t s);
void f32_to_bf16(const float* src, bf16* dst, int64_t n, cudaStream_t s);
// dst[i] = src[i] * (i < n_scaled ? s : 1) (eval_scale MEAN: the W rows of a layer, R10)
void scale_prefix_f32(const float* src, float* dst, int64_t n, int64_t n_scaled, float s, cudaStream_t st);

// --------------------------------------------------------------------------
// subGCNs / subAgg / init (R5, R6, R9, R11).
// --------------------------------------------------------------------------
void partition_keys(int d, uint32_t t, uint32_t l, uint64_t seed, uint64_t* keys, int32_t* idx, cudaStream_t s);
// sort (key, idx) pairs ascending; tmp workspace size query when tmp == nullptr
size_t partition_sort(const uint64_t* keys_in, uint64_t* keys_out, const int32_t* idx_in, int32_t* idx_out, int d,
                      void* tmp, size_t tmp_bytes, cudaStream_t s);
void partition_assign(const int32_t* sorted_idx, int d, int m, int32_t* blk, cudaStream_t s);
void partition_compact(const int32_t* blk, int d, int m, const int32_t* offs, int32_t* units, cudaStream_t s);

struct LayerMap {
  const int32_t* rows = nullptr;  // sub row units (nullptr: identity)
  int nrows = 0;                  // logical rows of the sub block (self block for SAGE)
  int sage = 0;
  int gat = 0;                    // GAT (R21): the second block is the two attention rows
  int half = 0;                   // physical offset of the neighbour block in the sub weight (SAGE)
  int glob_half = 0;              // physical offset of the neighbour block in the global weight (SAGE)
  const int32_t* cols = nullptr;  // sub column units (nullptr: identity)
  int ncols = 0;
  int Kp = 0, Np = 0;             // physical sub weight shape
  int64_t ldg = 0;                // global weight physical row stride
  // owner-sharded Theta (GIST_THETA_SHARDED): the global buffer holds physical rows
  // [row_lo, row_hi) only (it points at row row_lo); sub rows of other global rows are skipped
  int64_t row_lo = 0, row_hi = INT64_MAX;
};
void extract_sub(const float* theta, const LayerMap& m, float* w_sub, cudaStream_t s);
void scatter_sub(float* theta, const LayerMap& m, const float* w_sub, cudaStream_t s);
// agg_mode P2P (f2): one read of the block, one store per rank's replica of the layer
constexpr int kMaxPeers = 8;
struct PeerDst {
  float* dst[kMaxPeers];
  int n = 0;
};
void scatter_sub_peers(const PeerDst& d, const LayerMap& m, const float* w_sub, cudaStream_t s);
}  // namespace gist
#include <nccl.h>
#include <nccl_device/core.h>
namespace gist {
// agg_mode SYMM (f2): stores through the NCCL device API into every LSA peer's replica (or one
// multimem.st per element when the window has an NVLS multicast object); `base` = byte offset of
// the layer inside the registered window
void scatter_sub_symm(const ncclDevComm& dc, ncclWindow_t win, size_t base, const LayerMap& m, const float* w_sub,
                      bool multimem, cudaStream_t s);
// (sharded Theta: only physical rows [row_lo, row_hi); theta points at row row_lo)
void glorot_init(float* theta, int rows_logical, int cols, int sage, int d_l, int glob_half, int64_t ldg,
                 uint32_t layer, uint64_t seed, float scale, cudaStream_t s, int64_t row_lo = 0,
                 int64_t row_hi = INT64_MAX);

// eval: per-row CE / argmax correctness over rows with split == code; reduce (deterministic)
void eval_rows(const float* logits, int64_t ld, int64_t n, int k, const int32_t* labels, const uint8_t* split,
               int code, double* out3, cudaStream_t s);

// partition-wise eval: one CTA per partition of a chunk (positions pbeg[p]..pbeg[p+1]; logits row
// = position - k0); out3[3p..3p+2] = (sum CE, correct, count) over rows with split == code
void eval_parts(const float* logits, int64_t ld, int k, const int64_t* pbeg, int64_t k0, int nparts,
                const int32_t* pnode,
                const int32_t* labels, const uint8_t* split, int code, double* out3, cudaStream_t s);

// --------------------------------------------------------------------------
// GAT sub-GCN layer (reading R21; gat.cu).  CSR without self loops (the self
// loop is added by the kernels); dummy batch rows have row_beg = row_end = -1.
// --------------------------------------------------------------------------
template <typename T>
struct GatLayer {
  const int64_t* row_beg = nullptr;
  const int64_t* row_end = nullptr;
  const int32_t* col = nullptr;
  int64_t rows = 0, w = 0;            // rows; padded width (multiple of 8)
  const T* Z = nullptr;               // Z = H W (rows x w)
  int64_t ldz = 0;
  const float* a_src = nullptr;       // attention vectors (fp32 master rows of the weight)
  const float* a_dst = nullptr;
  float *s = nullptr, *t = nullptr, *lse = nullptr;  // per-row scores / log-sum-exp (forward)
  float *Srow = nullptr, *dt = nullptr, *ds = nullptr;  // backward per-row scalars
  T* out = nullptr;                   // forward output (hidden, ReLU if relu) ...
  float* out_f32 = nullptr;           // ... or fp32 logits
  int64_t ldo = 0;
  int relu = 0;
  const T* G = nullptr;               // backward: dL/dout (masked by mask > 0 if mask)
  int64_t ldg = 0;
  const T* mask = nullptr;
  int64_t ldm = 0;
  T* dZ = nullptr;                    // backward output dL/dZ
  int64_t ldd = 0;
  float *da_src = nullptr, *da_dst = nullptr;  // backward output: gradient rows of a_src / a_dst
  float* da_part = nullptr;                    // scratch: 64 x 2 x w partial sums of the above
  // scores re-associated as s = H (W a_src), t = H (W a_dst) (fp32 W a from the fp32 master W), so
  // they do not inherit the rounding of a bf16 Z: layer input H (ld ldh, width kw = padded rows of
  // W), W32 (kw x w, ld ldw) and a 2*kw scratch for [W a_src | W a_dst].  H == nullptr: s = Z a_src.
  const T* H = nullptr;
  int64_t ldh = 0, kw = 0;
  const float* W32 = nullptr;
  int64_t ldw = 0;
  float* wa = nullptr;
};
// one launch per kernel for up to kMaxGroup slots (grid.y = slot)
template <typename T>
struct GatGroup {
  GatLayer<T> a[kMaxGroup];
  int n = 0;
};
template <typename T> void gat_scores(const GatGroup<T>& G, cudaStream_t s);
template <typename T> void gat_forward(const GatGroup<T>& G, cudaStream_t s);
template <typename T> void gat_backward(const GatGroup<T>& G, cudaStream_t s);
constexpr int kGatDaChunks = 64;
constexpr int kGatMaxWidth = 2048;  // widest GAT layer output (padded columns) the attention passes hold
template <typename T>
void gather_rows_t(const T* src, int64_t lds, const int32_t* idx, int64_t rows, int64_t w, T* dst, int64_t ldd,
                   cudaStream_t s);
constexpr int kMaxMean = 128;
struct MeanRows {
  const float* src[kMaxMean];
  int64_t ld_src[kMaxMean];
  int n = 0, cols = 0;
  int64_t ld_dst = 0;
};
void mean_rows(float* dst, const MeanRows& m, int rows, cudaStream_t s);

}  // namespace gist
