/*
 * gist.h -- C ABI of the B200-native GIST hot path (arXiv 2102.10424).
 *
 * GIST = Graph Independent Subnetwork Training.  Algorithm 1:
 *   init Theta; Cluster(G, c); for t in 0..T-1:
 *     subGCNs(Psi, m)            -> gist_partition
 *     zeta x subTrain per sub-GCN -> gist_subtrain
 *     subAgg                      -> gist_aggregate
 * Evaluation of the global model -> gist_eval.
 *
 * Conventions (all entry points):
 *  - Every pointer argument is a HOST pointer unless its name ends in `_dev`.
 *    Inputs are copied before the call returns and never retained; outputs are
 *    caller-allocated with the sizes stated per call.
 *  - Work is stream-ordered on the context stream (gist_config.stream, or a
 *    stream the library creates).  Calls that fill host outputs synchronise
 *    before returning.
 *  - Errors: every call returns a gist_status; a message is available from
 *    gist_last_error().  A CUDA or NCCL failure poisons the context: every
 *    later call returns the same sticky status (GIST_E_CUDA / GIST_E_NCCL).
 *  - State machine: CREATED -> load_graph -> GRAPH -> init_params (or set_params of
 *    every layer) -> PARAMS -> partition -> PARTITIONED -> subtrain* -> aggregate -> PARAMS.
 *    Out-of-order calls return GIST_E_STATE.
 *  - Multi-GPU: one process (context) per GPU.  Slot (sub-GCN) i lives on rank
 *    i mod world_size.  gist_aggregate and gist_eval are collectives: every rank
 *    calls them in the same order (NCCL semantics).
 *  - There is no CPU fallback: a context can only be created on a CUDA device
 *    of compute capability 10.0 (sm_100a); otherwise GIST_E_UNSUPPORTED.
 *
 * Readings R1..R18 (where the paper is silent) are listed in DESIGN.md.
 */
#ifndef GIST_H_
#define GIST_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GIST_ABI_VERSION 1

typedef struct gist_ctx gist_ctx; /* opaque, single owner */

typedef enum {
  GIST_OK = 0,
  GIST_E_ARG = -1,         /* invalid argument (range, null, inconsistent sizes) */
  GIST_E_SHAPE = -2,       /* dims / m / buffer sizes inconsistent */
  GIST_E_STATE = -3,       /* call out of order (see state machine above) */
  GIST_E_OOM = -4,         /* device allocation failed */
  GIST_E_CUDA = -5,        /* CUDA runtime error (sticky) */
  GIST_E_NCCL = -6,        /* NCCL error (sticky) */
  GIST_E_UNSUPPORTED = -7  /* no sm_100 device / feature not built */
} gist_status;

/* Eq. (1); GraphSAGE-mean PAPER.md:246 (R2); GAT PAPER.md:204, 632 (R21: single
 * head, Theta_l = [W; a_src^T; a_dst^T] with logical rows d_l + 2, self loops added, ReLU hidden) */
enum { GIST_ARCH_GCN = 0, GIST_ARCH_SAGE = 1, GIST_ARCH_GAT = 2 };
enum { GIST_OPT_SGD = 0, GIST_OPT_ADAM = 1 };        /* subTrain = SGD step PAPER.md:168; Adam PAPER.md:660,680,690 */
/* R13 precision modes: FP32 parity (FP32 storage, FP32 SIMT GEMMs); BF16 (bf16 activations and GEMM
 * operands on tcgen05, fp32 accumulation, fp32 master weights / gradients / optimizer state);
 * TF32 (FP32 storage everywhere, the GEMMs on tcgen05 kind::tf32: operands rounded to tf32 by the
 * tensor core, fp32 accumulation -- PyTorch's allow_tf32 matmul precision). */
enum { GIST_PREC_FP32 = 0, GIST_PREC_BF16 = 1, GIST_PREC_TF32 = 2 };
enum { GIST_GRAPH_DEVICE = 0 };                     /* the graph is resident in HBM (the only residency built) */
/* Adam state across rounds: RESET = moments and step counter restart at every gist_partition
 * (R8; the default).  PERSISTENT = SURVEY.md §8 f3: global first / second moments
 * shaped like Theta are partitioned, extracted and aggregated with the weights (and
 * all-gathered with them when world_size > 1: 3x subAgg bytes), the step counter carries
 * over; GIST with m = 1 is then plain Adam training without restarts (the paper is silent,
 * PAPER.md:660).  Ignored for SGD. */
enum { GIST_OPT_STATE_RESET = 0, GIST_OPT_STATE_PERSISTENT = 1 };
/* subAgg transport.  ALLGATHER (default): one
 * ncclAllGather of the packed slot buffers, then every rank scatters all m slots into its
 * own replica of Theta.  P2P: Theta (and the f3 moments) live in one cudaMalloc region
 * whose CUDA IPC handle every rank opens at gist_load_graph; gist_aggregate has each owner
 * write its own slots' blocks straight into every rank's replica over NVLink peer stores
 * (one kernel per layer reads a block once and stores it W times), bracketed by two
 * one-word NCCL all-reduces used as barriers (no rank still reads its replica while peers
 * write; no rank reads it before every peer's stores completed).  No receive buffer, no
 * second pass over the gathered bytes.  Not available for GAT (R21 averages the m copies
 * of the attention rows, which needs every copy on every rank): GIST_E_UNSUPPORTED. */
/* SYMM (SURVEY.md §8 f2 with the NCCL device API): Theta (+ f3 moments) in an ncclMemAlloc region
 * registered as an NCCL symmetric window (ncclCommWindowRegister, NCCL_WIN_COLL_SYMMETRIC) with a
 * device communicator (ncclDevCommCreate; NVLS multicast requested at W > 1).  gist_aggregate has
 * each owner's kernel store its slots' blocks into every LSA peer's replica through
 * ncclGetLsaPointer -- or, with multicast, one multimem.st per element that NVSwitch delivers to
 * every replica -- between the same two barriers as P2P.  World 1 uses a one-rank communicator.
 * Not available with the loopback transport or for GAT (GIST_E_UNSUPPORTED). */
enum { GIST_AGG_ALLGATHER = 0, GIST_AGG_P2P = 1, GIST_AGG_SYMM = 2 };
/* Output scaling of the evaluation forward (R10; the theory scales the global
 * model's output by 1/m so that the expected sub-GCN output equals the global one).  NONE
 * (default): Eq. (1) as written.  MEAN: every contraction over a partitioned input dimension
 * (layers l >= 1, input dim d_l) is scaled by 1/m, m of the last gist_partition -- applied to
 * the W rows of those layers (GAT: not to the attention vectors).  Evaluation only; training
 * is unaffected. */
enum { GIST_EVAL_SCALE_NONE = 0, GIST_EVAL_SCALE_MEAN = 1 };
/* Storage of the global model across ranks (SURVEY.md §8(e) alternatives, §8 f2 "variant for C5:
 * owner-sharded Theta with all-to-all re-partition and aggregate"; it takes the place of the
 * paper's parameter server).  REPLICATED (default): every rank holds all of
 * Theta.  SHARDED: rank r holds physical rows [K_l r / W, K_l (r+1) / W) of every Theta_l (and of
 * the f3 moments), ~1/W of the memory; gist_partition sends every owned row of every sub-model
 * to the sub-model's rank and gist_aggregate sends the updated rows back to their owners, both as
 * one grouped point-to-point exchange (ncclSend / ncclRecv) of (W-1)/W of the sub-model bytes --
 * the same values land in the same places, so Theta stays bit-identical to REPLICATED.
 * gist_get_params, gist_save_checkpoint and gist_eval* become collectives (every rank calls
 * them: the rows are gathered for the call); gist_set_params / gist_load_checkpoint and
 * gist_init_params write the local rows only.  Only with agg_mode ALLGATHER. */
enum { GIST_THETA_REPLICATED = 0, GIST_THETA_SHARDED = 1 };

/* Loopback transport (tests): W contexts of ONE process on one device stand in for W ranks.
 * Every collective of gist_aggregate / gist_eval / gist_eval_parts (all-gather, sum all-reduce,
 * barrier, the P2P replica-pointer exchange) is carried out by the host -- stream synchronise,
 * rendezvous of the W calling threads, device-to-device copies -- instead of NCCL, so the
 * library's W > 1 code paths (slot ownership i mod W, packed-buffer offsets, the unpack /
 * scatter of the gathered buffers, peer stores, the row-split eval) run unchanged on one GPU.
 * No kernel ever waits on another rank.  Each rank's context must be driven by its own host
 * thread: a collective returns only once all W ranks have entered it.  Not a multi-GPU
 * transport: across GPUs use NCCL (gist_config.nccl_unique_id).
 *   gist_loopback_create: GIST_E_ARG if world_size < 1.  The group outlives its contexts. */
typedef struct gist_loopback gist_loopback;
gist_status gist_loopback_create(int32_t world_size, gist_loopback** out);
void gist_loopback_destroy(gist_loopback* lb);

typedef struct {
  int32_t arch;               /* GIST_ARCH_* */
  int32_t num_layers;         /* L >= 1 */
  const int32_t* dims;        /* L+1 entries d_0..d_L (d_0 = features, d_L = classes), copied */
  int32_t optimizer;          /* GIST_OPT_* */
  float beta1, beta2, eps;    /* Adam constants; defaults 0.9, 0.999, 1e-8 (R8) */
  int32_t precision;          /* GIST_PREC_* */
  int32_t clusters_per_batch; /* q: clusters unioned into one mini-batch */
  uint64_t batch_seed;        /* Philox key of the per-slot batch schedule (R7) */
  int32_t graph_residency;    /* GIST_GRAPH_* */
  int32_t rank, world_size;   /* this process's rank; number of ranks (1 = no NCCL) */
  int32_t device;             /* CUDA device ordinal */
  const void* nccl_unique_id; /* 128-byte ncclUniqueId from rank 0 when world_size > 1, else NULL */
  void* stream;               /* optional cudaStream_t to order work on; NULL = library-owned */
  int32_t opt_state;          /* GIST_OPT_STATE_* (default RESET) */
  int32_t agg_mode;           /* GIST_AGG_* (default ALLGATHER) */
  gist_loopback* loopback;    /* tests: loopback group of world_size ranks replacing NCCL, or NULL */
  int32_t eval_scale;         /* GIST_EVAL_SCALE_* (default NONE, R10) */
  int32_t theta_mode;         /* GIST_THETA_* (default REPLICATED) */
} gist_config;

/* Fills *cfg with defaults (GCN, Adam .9/.999/1e-8, FP32, q=1, world 1, device 0). */
void gist_config_default(gist_config* cfg);

/* Writes a fresh 128-byte ncclUniqueId into out128 (rank 0 calls it and broadcasts the
 * bytes, e.g. over torch.distributed; every rank passes them as cfg->nccl_unique_id). */
gist_status gist_nccl_unique_id(void* out128);

/* Creates a context on cfg->device.  Errors: GIST_E_ARG (dims), GIST_E_UNSUPPORTED
 * (no CUDA device of compute capability 10.x; a GAT layer wider than 2,048 output units;
 * agg_mode P2P with GAT or more than 8 ranks), GIST_E_NCCL. */
gist_status gist_create(const gist_config* cfg, gist_ctx** out);

/* Loads graph G (n nodes, features X in R^{n x d_0}) and its Cluster
 * partition (METIS is an input here, not computed).
 *  row_ptr[n+1] (int64, non-decreasing, row_ptr[0] = 0, row_ptr[n] = nnz),
 *  col_idx[nnz] (int32 in [0,n), strictly increasing within each row, symmetric adjacency:
 *     every (u,v) has its (v,u); no self loops -- self loops present in the input are dropped
 *     and counted, see gist_stat; violations are rejected on the device with GIST_E_ARG),
 *  X[n*d_0] fp32 row-major, labels[n] int32 in [0,num_classes), num_classes = d_L,
 *  split[n] uint8: 0 train, 1 val, 2 test, 3 none,
 *  cluster_ids[n] int32 in [0,num_clusters), every cluster non-empty.
 * Nodes are relabelled on the device so that clusters are contiguous; every
 * per-node output of this library is keyed by the ORIGINAL node id. */
gist_status gist_load_graph(gist_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                            int64_t nnz, const float* X, const int32_t* labels, int32_t num_classes,
                            const uint8_t* split, const int32_t* cluster_ids, int32_t num_clusters);

/* "randomly initialize GCN": Glorot-uniform from Philox4x32-10,
 * bit-identical to the oracle (R11). */
gist_status gist_init_params(gist_ctx* ctx, uint64_t seed);

/* subGCNs: for every hidden dim l = 1..L-1 a random disjoint
 * partition of [d_l] into m balanced blocks keyed by Philox(seed, round t, l)
 * (R5); d_0 and d_L are not partitioned.  Extracts
 * Theta^(i)_l = [Theta_l]_{D_l^(i) x D_{l+1}^(i)} for this rank's
 * slots and resets their optimizer state (R8).  1 <= m <= min hidden dim. */
gist_status gist_partition(gist_ctx* ctx, uint64_t seed, int32_t m);

/* subTrain: local_iters (zeta) steps for every local
 * slot, each on its own Cluster mini-batch (R7): batch build, forward (Eq. 2),
 * softmax-CE (R4), backward, Adam/SGD with learning rate lr.  The local slots run
 * in lockstep: every kernel of a step is one grouped launch over (up to 8) slots.
 * mean_loss: NULL or float[m]; entries of this rank's slots receive the mean loss
 * over the local_iters steps, others 0. */
gist_status gist_subtrain(gist_ctx* ctx, int32_t local_iters, float lr, float* mean_loss);

/* subAgg: every slot's block replaces its entries of the
 * global Theta (bitwise copy, R9); entries outside all blocks are untouched.
 * Collective: one ncclAllGather of the packed slot buffers when world_size > 1
 * (agg_mode ALLGATHER), or peer stores into every replica between two barriers
 * (agg_mode P2P).  Both give bit-identical Theta.  Increments the round counter t. */
gist_status gist_aggregate(gist_ctx* ctx);

/* Forward of the global model on the full graph (full-graph operator, R1/R2;
 * no output scaling, R10); mean CE loss and accuracy over nodes with
 * split == split_code.  Either output may be NULL.
 * World > 1 (collective): GCN / GraphSAGE rows are split into W blocks of
 * ceil(n / W) relabelled rows; each rank computes its block of every layer, one all-gather
 * per hidden layer assembles the next layer's input, and one sum all-reduce combines the
 * loss / accuracy counts.  GAT runs the whole forward on every rank.
 * Errors: GIST_E_STATE (open round / no params), GIST_E_ARG (split code not in 0..3). */
gist_status gist_eval(gist_ctx* ctx, int32_t split_code, float* loss, float* acc);

/* Partition-wise evaluation of the global model ("for d_i > 4096
 * evaluation must be performed on graph partitions ... F1 score is measured over each
 * partition and averaged"; reading R20).  Every partition is evaluated on its own induced
 * subgraph (cut edges dropped, R1/R2 normalisation inside the partition, R10 no output
 * scaling); its score is the mean CE / accuracy (= single-label micro-F1) over its nodes with
 * split == split_code, and *loss / *acc are the unweighted means over the partitions holding
 * at least one such node (0 if none).
 *   part_ids   host int32[n], ORIGINAL node ids -> partition in [0, num_parts); NULL = the
 *              training clusters of gist_load_graph (num_parts must then be 0 or their count).
 *   max_rows   rows per evaluation chunk (whole partitions per chunk; a partition larger
 *              than max_rows forms its own chunk); <= 0 = sized from free device memory.
 *   part_loss, part_acc  optional host float[num_parts]; NaN for partitions without
 *              evaluated nodes.  Any output may be NULL.
 * World > 1: collective; partition p is evaluated by rank p mod world_size and the
 * per-partition sums are combined with one ncclAllReduce; every rank gets all outputs.
 * Errors: GIST_E_STATE (open round / no params), GIST_E_ARG (bad split code or ids). */
gist_status gist_eval_parts(gist_ctx* ctx, int32_t split_code, const int32_t* part_ids, int32_t num_parts,
                            int64_t max_rows, float* loss, float* acc, float* part_loss, float* part_acc);

/* ---------------- inspection / parity hooks ---------------- */
/* Per-node logits of the global model from exactly the forward that gist_eval (mode 0, the
 * full graph) or gist_eval_parts (mode 1, every partition on its own induced subgraph, R20)
 * runs.  out: host float[n * d_L], row = ORIGINAL node id.  part_ids / num_parts / max_rows
 * as for gist_eval_parts (ignored for mode 0).  Collective like the evaluation it mirrors;
 * every rank receives all rows.  Errors: GIST_E_STATE, GIST_E_ARG (mode, null out, ids). */
gist_status gist_eval_logits(gist_ctx* ctx, int32_t mode, const int32_t* part_ids, int32_t num_parts,
                             int64_t max_rows, float* out);

/* Global Theta_l, logical row-major: rows = d_l (GCN), 2*d_l (SAGE: self rows then
 * neighbour rows) or d_l + 2 (GAT: W rows, then a_src, a_dst), cols = d_{l+1}.
 * out / in: float[rows*cols]. */
gist_status gist_get_params(gist_ctx* ctx, int32_t layer, float* out);
gist_status gist_set_params(gist_ctx* ctx, int32_t layer, const float* in);

/* Model checkpoint file (SPEC.md "External Interfaces"): little-endian binary -- magic "GIST",
 * version u32 (= 1), arch u8 (GIST_ARCH_*), L u32, dims u32[L+1], then every global Theta_l in
 * the logical row-major layout of gist_get_params as f32.  Deterministic bytes for a given model.
 * save: needs parameters and no open round (GIST_E_STATE); I/O failure GIST_E_ARG.
 * load: after gist_load_graph and outside a round; the header must match this context's arch and
 * dims (GIST_E_SHAPE), else GIST_E_ARG for a malformed / short file; the context then holds those
 * parameters (PARAMS, like gist_set_params of every layer). */
gist_status gist_save_checkpoint(gist_ctx* ctx, const char* path);
gist_status gist_load_checkpoint(gist_ctx* ctx, const char* path);

/* Partition of dim `dim` for the current round: units[d_dim] = blocks D^(0..m-1)
 * concatenated (each ascending), offs[m+1] block offsets.  Valid after partition. */
gist_status gist_get_partition(gist_ctx* ctx, int32_t dim, int32_t* units, int32_t* offs);

/* Sub-model Theta^(slot)_layer, logical row-major [|rows| x |cols|] (R6).  Only for
 * slots owned by this rank.  out size: gist_sub_shape(). */
gist_status gist_sub_shape(gist_ctx* ctx, int32_t slot, int32_t layer, int64_t* rows, int64_t* cols);
gist_status gist_get_sub_params(gist_ctx* ctx, int32_t slot, int32_t layer, float* out);

/* Trace of the last subTrain step of a local slot (parity hooks):
 *  GIST_TRACE_NODES   int32[n_b]  original node id of each batch row (batch order)
 *  GIST_TRACE_ACT     float[n_b * w] layer input activation H_layer (layer >= 1, w = width of H_layer)
 *  GIST_TRACE_LOGITS  float[n_b * d_L]
 *  GIST_TRACE_GRAD    float[rows*cols] gradient dL/dTheta^(slot)_layer of that step (logical layout)
 *  GIST_TRACE_LOSS    float[1] the step's loss
 * *count (may be NULL) receives the element count; out may be NULL to query it. */
enum { GIST_TRACE_NODES = 0, GIST_TRACE_ACT = 1, GIST_TRACE_LOGITS = 2, GIST_TRACE_GRAD = 3, GIST_TRACE_LOSS = 4 };
gist_status gist_get_trace(gist_ctx* ctx, int32_t slot, int32_t what, int32_t layer, void* out, int64_t* count);

/* Counters: GIST_STAT_ROUND (t), GIST_STAT_STEP (steps per slot so far),
 * GIST_STAT_SELF_LOOPS_DROPPED, GIST_STAT_LAST_NNZ_B (nnz of the last batch of slot
 * 0 on this rank), GIST_STAT_LAST_NB, GIST_STAT_KERNELS (kernel launches issued
 * by the library so far), GIST_STAT_H2D_BYTES / GIST_STAT_D2H_BYTES (bytes
 * copied so far), GIST_STAT_MAX_NB. */
enum {
  GIST_STAT_ROUND = 0, GIST_STAT_STEP = 1, GIST_STAT_SELF_LOOPS_DROPPED = 2, GIST_STAT_LAST_NNZ_B = 3,
  GIST_STAT_LAST_NB = 4, GIST_STAT_KERNELS = 5, GIST_STAT_H2D_BYTES = 6, GIST_STAT_D2H_BYTES = 7,
  GIST_STAT_MAX_NB = 8, GIST_STAT_BLOCK_AGG = 9 /* 1 if block-diagonal tensor-core aggregation is on */,
  GIST_STAT_BLOCK_DENSITY_PPM = 10 /* intra-cluster block density x 1e6 */,
  GIST_STAT_THETA_BYTES = 11 /* device bytes of this rank's global model storage (Theta + f3 moments) */
};
int64_t gist_stat(gist_ctx* ctx, int32_t which);

/* Live per-kernel-class timing (roofline reporting).  stride > 0: every launch of
 * every stride-th subTrain step (and every partition / aggregate launch) is
 * bracketed by CUDA events on the stream it is launched on; stride = 0 turns it
 * off.  Calling gist_profile resets the counters.  gist_profile_get synchronises
 * and returns, for one class: total event-timed milliseconds, launches, and the
 * algorithmic work of those launches (FLOPs for GEMM = 2 M N K; compulsory
 * bytes for the others: every operand read once, every output written once). */
enum {
  GIST_PROF_BATCH = 0, GIST_PROF_SPMM = 1, GIST_PROF_GEMM = 2, GIST_PROF_LOSS = 3, GIST_PROF_OPTIM = 4,
  GIST_PROF_PARTITION = 5, GIST_PROF_AGGREGATE = 6,
  GIST_PROF_AGG_TC = 7, /* block-diagonal (intra-cluster) aggregation on tensor cores; work = FLOPs */
  GIST_PROF_COMM = 8,   /* subAgg collective (all-gather / barriers); work = bytes received per rank */
  GIST_PROF_N = 9
};
gist_status gist_profile(gist_ctx* ctx, int32_t stride);
gist_status gist_profile_get(gist_ctx* ctx, int32_t cls, double* ms, int64_t* launches, double* work);

/* Sharding layout of the sub-GCN slots (host-only, no device needed; §6 of DESIGN.md):
 * slot i lives on rank gist_slot_owner(i, W) = i mod W as that rank's local slot i / W;
 * every rank contributes gist_slots_per_rank(m, W) = ceil(m / W) equal-size packed slot
 * buffers to the subAgg all-gather, so the gathered buffer of rank r, local slot j is
 * global slot r + W * j (ignored when >= m). */
int32_t gist_slot_owner(int32_t slot, int32_t world_size);
int32_t gist_slots_per_rank(int32_t m, int32_t world_size);

/* cudaStream_t of the context (for timing with CUDA events on the launching stream). */
void* gist_stream(gist_ctx* ctx);

const char* gist_last_error(const gist_ctx* ctx);
const char* gist_status_str(gist_status s);
/* Releases every resource of the context (NULL: no-op).  After a failed CUDA / NCCL call (a
 * sticky GIST_E_CUDA / GIST_E_NCCL status) the NCCL communicator is aborted (ncclCommAbort)
 * rather than destroyed, so a rank whose peers are stuck in a collective does not wait for them. */
void gist_destroy(gist_ctx* ctx);

/* ---------------- kernel-level entry points (benchmark / parity) ----------------
 * Device pointers (`_dev`), stream-ordered on `stream` (cudaStream_t, NULL = legacy).
 * These run exactly the kernels the training step uses. */

/* Aggregation SpMM over a CSR (int64 row_ptr, int32 col):  for v in [0,rows):
 *   out[v,:] = rowscale[v] * ( self * colscale[v] * H[v,:] + sum_{u in N(v)} colscale[u] * H[u,:] )
 * (NULL scale = 1).  H, out: row-major, `ld` elements per row, width w <= ld
 * processed; dtype 0 = fp32, 1 = bf16 (fp32 accumulation).  GCN renorm
 * (R1): rowscale = colscale = (deg+1)^{-1/2}, self = 1; SAGE mean (R2):
 * rowscale = 1/deg, self = 0. */
gist_status gist_spmm(const int64_t* row_ptr_dev, const int32_t* col_dev, int64_t rows,
                      const float* rowscale_dev, const float* colscale_dev, int32_t self,
                      const void* H_dev, void* out_dev, int64_t w, int64_t ld, int32_t dtype, void* stream);

/* C[M x N] = op(A) op(B) (row-major, leading dims lda/ldb/ldc), fp32 or bf16 in,
 * fp32 or bf16 out, fp32 accumulation; trans flags per operand.  dtype 0 = fp32
 * SIMT path, 1 = bf16 tcgen05 path (out fp32 when out_f32 != 0), 2 = tf32 tcgen05 path
 * (fp32 in and out).  relu != 0 applies max(.,0) in the epilogue. */
gist_status gist_gemm(int32_t transA, int32_t transB, int64_t M, int64_t N, int64_t K,
                      const void* A_dev, int64_t lda, const void* B_dev, int64_t ldb,
                      void* C_dev, int64_t ldc, int32_t dtype, int32_t out_f32, int32_t relu, void* stream);
/* The same GEMM launched `reps` times back to back from one plan (the tcgen05 tensor maps are
 * encoded once): device timing of the kernel without per-call host work (tools/gemm_probe.py). */
gist_status gist_gemm_reps(int32_t transA, int32_t transB, int64_t M, int64_t N, int64_t K,
                           const void* A_dev, int64_t lda, const void* B_dev, int64_t ldb,
                           void* C_dev, int64_t ldc, int32_t dtype, int32_t out_f32, int32_t relu, void* stream,
                           int32_t reps);

#ifdef __cplusplus
}
#endif
#endif /* GIST_H_ */
