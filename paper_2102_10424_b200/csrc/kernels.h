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
  TO* out = nullptr;
  int64_t ldo = 0;
  TI* self_out = nullptr;
  int64_t ld_self = 0;
  int64_t w = 0;  // padded width processed (multiple of 8)
};
template <typename TI, typename TO> void spmm(const SpmmArgs<TI, TO>& a, cudaStream_t s);

// --------------------------------------------------------------------------
// Dense contractions.  C[M x N] = op(A)[M x K] op(B)[K x N].
//   transA: A stored K x M (lda >= M); else M x K.  transB: B stored N x K; else K x N.
// FP32 parity path: SIMT FFMA tiles.  BF16 path: tcgen05 + TMA + TMEM.
// --------------------------------------------------------------------------
void gemm_f32(bool transA, bool transB, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
              const float* B, int64_t ldb, float* C, int64_t ldc, bool relu, cudaStream_t s);
// returns false if the shape/alignment is not supported by the tensor-core path
bool gemm_bf16(bool transA, bool transB, int64_t M, int64_t N, int64_t K, const bf16* A, int64_t lda,
               const bf16* B, int64_t ldb, void* C, int64_t ldc, bool out_f32, bool relu, cudaStream_t s);

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
void full_graph_scales(const int64_t* rp, int64_t n, int arch, float* scale, cudaStream_t s);

// Per-step descriptor (host-built, R7): bcl[q] cluster ids, loff[q+1] local row offsets,
// voff[q+1] offsets of each cluster's adjacency segment inside b_col.
// map64[c] = (tag << 32) | (uint32)(loff_k - cstart[c]) for the batch's clusters: a
// neighbour u is inside the batch iff (map64[cid[u]] >> 32) == tag (no reset needed).
void batch_setup(const int32_t* bcl, const int32_t* loff, const int32_t* voff, int q, const int64_t* cstart,
                 const int64_t* rp, uint32_t tag, uint64_t* map64, int32_t* b_nodes, int64_t* b_beg, int nb,
                 int64_t* stats, cudaStream_t s);
// one pass: in-batch neighbours of row v -> b_col[b_beg[v] .. b_end[v]) (local ids), scale,
// labels, train flags; stats[0] += nnz_b, stats[1] += train rows (integer atomics: deterministic)
void batch_build(const int64_t* rp, const int32_t* col, const int32_t* cid, const uint64_t* map64, uint32_t tag,
                 const int32_t* b_nodes, const int64_t* b_beg, int nb, int arch, const int32_t* labels,
                 const uint8_t* split, int64_t* b_end, int32_t* b_col, float* scale, int32_t* lab_b,
                 uint8_t* train_b, int64_t* stats, cudaStream_t s);

// --------------------------------------------------------------------------
// Loss (R4), optimizers (R8), reductions.
// --------------------------------------------------------------------------
template <typename T>
void softmax_ce(const float* logits, int64_t ld, int nb, int k, const int32_t* lab, const uint8_t* train,
                const int64_t* stats, T* dlog, float* row_loss, cudaStream_t s);
// step_loss[0] = sum(row_loss)/n_train (0 if none); loss_acc[0] += step_loss[0]
void reduce_loss(const float* row_loss, int nb, const int64_t* stats, float* step_loss, float* loss_acc,
                 cudaStream_t s);
void adam_step(float* W, const float* G, float* M, float* V, int64_t n, float lr, float b1, float b2, float eps,
               float bc1, float bc2_sqrt, bf16* Wb, cudaStream_t s);
void sgd_step(float* W, const float* G, int64_t n, float lr, bf16* Wb, cudaStream_t s);
void f32_to_bf16(const float* src, bf16* dst, int64_t n, cudaStream_t s);

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
  int half = 0;                   // physical offset of the neighbour block in the sub weight (SAGE)
  int glob_half = 0;              // physical offset of the neighbour block in the global weight (SAGE)
  const int32_t* cols = nullptr;  // sub column units (nullptr: identity)
  int ncols = 0;
  int Kp = 0, Np = 0;             // physical sub weight shape
  int64_t ldg = 0;                // global weight physical row stride
};
void extract_sub(const float* theta, const LayerMap& m, float* w_sub, cudaStream_t s);
void scatter_sub(float* theta, const LayerMap& m, const float* w_sub, cudaStream_t s);
void glorot_init(float* theta, int rows_logical, int cols, int sage, int d_l, int glob_half, int64_t ldg,
                 uint32_t layer, uint64_t seed, float scale, cudaStream_t s);

// eval: per-row CE / argmax correctness over rows with split == code; reduce (deterministic)
void eval_rows(const float* logits, int64_t ld, int64_t n, int k, const int32_t* labels, const uint8_t* split,
               int code, double* out3, cudaStream_t s);

}  // namespace gist
