// shard.cu -- the owner-sharded global model (GIST_THETA_SHARDED; SURVEY.md §8 f2 "variant for
// C5: owner-sharded Theta, with all-to-all re-partition and aggregate", in place of the paper's
// parameter server).  Rank r holds physical rows [K_l r / W, K_l (r+1) / W) of
// every Theta_l.  The subGCNs step (R6) sends every owned row of every sub-model
// to the sub-model's rank; subAgg (R9) sends the updated rows back to their
// owners.  A sub-model's packed rows map to global rows monotonically inside each of its (at most
// two) row blocks, so the rows one owner holds form a few contiguous runs of the packed layout:
// each run travels as one point-to-point message straight from / into its place in the packed
// buffers (comm_alltoallv: grouped ncclSend / ncclRecv).  The same bytes land in the same places
// as with the replicated model, so Theta is bit-identical to GIST_THETA_REPLICATED.
#include "ctx.h"

using namespace gist;
using namespace gist_impl;

namespace {

// Same row placement as glob_row (partition.cu), on the host copy of the partition.
int64_t glob_row_host(const gist_ctx* c, const LayerShape& sh, int l, const int32_t* rows, int p) {
  const int64_t gh = pad8(c->dims[l]);
  if (c->arch == GIST_ARCH_GAT) {
    if (p < sh.nrows) return rows ? rows[p] : p;
    if (p >= sh.half && p < sh.half + 2) return gh + (p - sh.half);
    return -1;
  }
  if (c->arch != GIST_ARCH_SAGE) return p < sh.nrows ? (rows ? rows[p] : p) : -1;
  if (p < sh.nrows) return rows ? rows[p] : p;
  if (p >= sh.half && p < sh.half + sh.nrows) return gh + (rows ? rows[p - sh.half] : p - sh.half);
  return -1;
}

struct Run {
  int owner;   // rank holding these global rows
  int p0, p1;  // packed rows [p0, p1) of the sub-model's layer
};

// runs of slot i, layer l, in packed-row order
std::vector<Run> runs_of(const gist_ctx* c, int i, int l) {
  const LayerShape& sh = c->shapes[i][l];
  const int32_t* rows = (l == 0) ? nullptr : c->units_h[l].data() + c->offs[l][i];
  const int W = c->cfg.world_size;
  std::vector<Run> out;
  for (int p = 0; p < sh.Kp; ++p) {
    const int64_t gr = glob_row_host(c, sh, l, rows, p);
    if (gr < 0) continue;
    int o = W - 1;
    while (o > 0 && shard_lo(c, l, o) > gr) --o;
    if (!out.empty() && out.back().owner == o && out.back().p1 == p) out.back().p1 = p + 1;
    else out.push_back(Run{o, p, p + 1});
  }
  return out;
}

LayerMap layer_map(const gist_ctx* c, int i, int l) {
  const LayerShape& sh = c->shapes[i][l];
  LayerMap mp;
  mp.rows = sh.rows; mp.nrows = sh.nrows; mp.sage = c->arch == GIST_ARCH_SAGE; mp.gat = c->arch == GIST_ARCH_GAT;
  mp.half = sh.half; mp.glob_half = (int)pad8(c->dims[l]); mp.cols = sh.cols; mp.ncols = sh.ncols;
  mp.Kp = sh.Kp; mp.Np = sh.Np; mp.ldg = c->th_N[l];
  mp.row_lo = c->sh_lo[l];
  mp.row_hi = c->sh_hi[l];
  return mp;
}

// the (global buffers, local packed buffers) pairs that travel: Theta, and the f3 moments
struct Part {
  std::vector<float*>* global;
  float* local;
};
std::vector<Part> parts_of(gist_ctx* c) {
  std::vector<Part> v = {{&c->theta, c->Wall}};
  if (persistent_adam(c)) v.push_back({&c->theta_m, c->Mall}), v.push_back({&c->theta_v, c->Vall});
  return v;
}

}  // namespace

namespace gist_impl {

// gist_partition: every rank extracts the rows it owns of EVERY sub-model into xscr (R6), then
// each run goes to the sub-model's rank, into its packed buffer (padding rows stay zero)
gist_status shard_extract(gist_ctx* c) {
  cudaStream_t s = c->stream;
  const int W = c->cfg.world_size, me = c->cfg.rank;
  // the run plan needs the round's partition on the host (hidden dims, ~sum d_l int32)
  c->units_h.assign(c->L + 1, std::vector<int32_t>());
  for (int l = 1; l < c->L; ++l) {
    c->units_h[l].resize(c->dims[l]);
    CK(cudaMemcpyAsync(c->units_h[l].data(), c->units[l], (size_t)c->dims[l] * 4, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  std::vector<std::vector<std::vector<Run>>> R(c->m, std::vector<std::vector<Run>>(c->L));
  for (int i = 0; i < c->m; ++i)
    for (int l = 0; l < c->L; ++l) R[i][l] = runs_of(c, i, l);
  const int64_t tot_local = (int64_t)c->slots.size() * c->S_max;
  for (const Part& pt : parts_of(c)) {
    if (tot_local > 0) CK(cudaMemsetAsync(pt.local, 0, (size_t)tot_local * 4, s));
    for (int i = 0; i < c->m; ++i)
      for (int l = 0; l < c->L; ++l) {
        const LayerShape& sh = c->shapes[i][l];
        PL(GIST_PROF_PARTITION, (double)sh.Kp * sh.Np * 8.0 / W, s,
           extract_sub((*pt.global)[l], layer_map(c, i, l), c->xscr + (size_t)i * c->S_max + sh.off, s));
      }
    std::vector<Xfer> sends, recvs;
    for (int i = 0; i < c->m; ++i) {
      const int o = gist_slot_owner(i, W), j = i / W;
      for (int l = 0; l < c->L; ++l) {
        const LayerShape& sh = c->shapes[i][l];
        for (const Run& r : R[i][l]) {
          const size_t off = (size_t)sh.off + (size_t)r.p0 * sh.Np, bytes = (size_t)(r.p1 - r.p0) * sh.Np * 4;
          if (r.owner == me) sends.push_back(Xfer{o, c->xscr + (size_t)i * c->S_max + off, bytes});
          if (o == me) recvs.push_back(Xfer{r.owner, pt.local + (size_t)j * c->S_max + off, bytes});
        }
      }
    }
    const int id = prof_begin(c, s, GIST_PROF_COMM, 0.0);
    TRY(coll(c, comm_alltoallv(c->comm, sends, recvs, s, &c->err)));
    prof_end(c, s, id);
  }
  return GIST_OK;
}

// gist_aggregate: each slot's rank sends every run back to its owner (into xscr), then every
// rank writes the rows it owns (R9); GAT's last-layer attention rows are the mean of the m
// copies (R21), taken by their owner
gist_status shard_aggregate(gist_ctx* c) {
  cudaStream_t s = c->stream;
  const int W = c->cfg.world_size, me = c->cfg.rank;
  std::vector<std::vector<std::vector<Run>>> R(c->m, std::vector<std::vector<Run>>(c->L));
  for (int i = 0; i < c->m; ++i)
    for (int l = 0; l < c->L; ++l) R[i][l] = runs_of(c, i, l);
  for (const Part& pt : parts_of(c)) {
    std::vector<Xfer> sends, recvs;
    for (int i = 0; i < c->m; ++i) {
      const int o = gist_slot_owner(i, W), j = i / W;
      for (int l = 0; l < c->L; ++l) {
        const LayerShape& sh = c->shapes[i][l];
        for (const Run& r : R[i][l]) {
          const size_t off = (size_t)sh.off + (size_t)r.p0 * sh.Np, bytes = (size_t)(r.p1 - r.p0) * sh.Np * 4;
          if (o == me) sends.push_back(Xfer{r.owner, pt.local + (size_t)j * c->S_max + off, bytes});
          if (r.owner == me) recvs.push_back(Xfer{o, c->xscr + (size_t)i * c->S_max + off, bytes});
        }
      }
    }
    const int id = prof_begin(c, s, GIST_PROF_COMM, 0.0);
    TRY(coll(c, comm_alltoallv(c->comm, sends, recvs, s, &c->err)));
    prof_end(c, s, id);
    for (int i = 0; i < c->m; ++i)
      for (int l = 0; l < c->L; ++l) {
        const LayerShape& sh = c->shapes[i][l];
        PL(GIST_PROF_AGGREGATE, (double)sh.Kp * sh.Np * 8.0 / W, s,
           scatter_sub((*pt.global)[l], layer_map(c, i, l), c->xscr + (size_t)i * c->S_max + sh.off, s));
      }
    if (c->arch == GIST_ARCH_GAT) {  // R21: the last layer's attention rows, if this rank holds them
      const int l = c->L - 1;
      const int64_t ga = pad8(c->dims[l]);  // global physical row of a_src (a_dst follows)
      if (ga >= c->sh_lo[l] && ga + 2 <= c->sh_hi[l]) {
        MeanRows mr;
        mr.n = c->m;
        mr.cols = c->dims[c->L];
        mr.ld_dst = c->th_N[l];
        for (int i = 0; i < c->m; ++i) {
          const LayerShape& sh = c->shapes[i][l];
          mr.src[i] = c->xscr + (size_t)i * c->S_max + sh.off + (int64_t)sh.half * sh.Np;
          mr.ld_src[i] = sh.Np;
        }
        PL(GIST_PROF_AGGREGATE, 2.0 * c->m * mr.cols * 4.0, s,
           mean_rows((*pt.global)[l] + (ga - c->sh_lo[l]) * c->th_N[l], mr, 2, s));
      }  // (gist_load_graph refuses shard boundaries between the two rows)
    }
  }
  return GIST_OK;
}

// all rows of layer l into `full` (th_K x th_N) on every rank: each rank sends its shard to all
gist_status shard_gather_layer(gist_ctx* c, const float* shard, int l, float* full, cudaStream_t s) {
  const int W = c->cfg.world_size, me = c->cfg.rank;
  const int64_t N = c->th_N[l];
  std::vector<Xfer> sends, recvs;
  for (int r = 0; r < W; ++r) {
    sends.push_back(Xfer{r, const_cast<float*>(shard), (size_t)rows_here(c, l) * N * 4});
    const int64_t lo = shard_lo(c, l, r), hi = shard_lo(c, l, r + 1);
    recvs.push_back(Xfer{r, full + lo * N, (size_t)(hi - lo) * N * 4});
  }
  (void)me;
  return coll(c, comm_alltoallv(c->comm, sends, recvs, s, &c->err));
}

}  // namespace gist_impl
