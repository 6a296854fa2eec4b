// graph.cu -- graph relabelling on load and the Cluster mini-batch build
// (SURVEY a1).
//
// On load, nodes are relabelled so that every cluster is a contiguous id range
// (new id = position in the cluster-sorted order).  A mini-batch is then the
// union of q clusters = q id ranges; batch row v maps to new id b_nodes[v], and a
// neighbour u is inside the batch iff map64[cid[u]] carries this step's tag, with
// local id u + delta(cid[u]).  Nothing is cleared between steps (the tag changes).
// The batch adjacency is written into per-row segments b_col[b_beg[v], b_end[v])
// sized by the global degree (segment starts are known before the pass), so the
// build is a single pass with no scan.
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace gist {

// ---------------------------------------------------------------- relabel --
__global__ void k_relabel_count(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                const int32_t* __restrict__ perm, int64_t n, int64_t* __restrict__ deg_new) {
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (g >= n) return;
  const int64_t v = perm[g];
  int cnt = 0;
  for (int64_t e = rp[v] + lane; e < rp[v + 1]; e += 32) cnt += (col[e] != v);
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) deg_new[g] = cnt;
}

__global__ void k_relabel_fill(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                               const int32_t* __restrict__ perm, const int32_t* __restrict__ inv,
                               const int64_t* __restrict__ rp_new, int64_t n, int32_t* __restrict__ col_new) {
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (g >= n) return;
  const int64_t v = perm[g];
  int64_t out = rp_new[g];
  for (int64_t base = rp[v]; base < rp[v + 1]; base += 32) {
    const int64_t e = base + lane;
    const bool in = e < rp[v + 1];
    const int32_t u = in ? col[e] : 0;
    const bool keep = in && u != v;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) col_new[out + __popc(bal & ((1u << lane) - 1))] = inv[u];
    out += __popc(bal);
  }
}

void relabel_count(const int64_t* rp, const int32_t* col, const int32_t* perm, int64_t n, int64_t* deg_new,
                   cudaStream_t s) {
  if (n <= 0) return;
  k_relabel_count<<<(unsigned)cdiv(n, 8), 256, 0, s>>>(rp, col, perm, n, deg_new);
}
void relabel_fill(const int64_t* rp, const int32_t* col, const int32_t* perm, const int32_t* inv,
                  const int64_t* rp_new, int64_t n, int32_t* col_new, cudaStream_t s) {
  if (n <= 0) return;
  k_relabel_fill<<<(unsigned)cdiv(n, 8), 256, 0, s>>>(rp, col, perm, inv, rp_new, n, col_new);
}

// dst[i, 0:w] = src[idx[i], 0:w] (fp32 -> T), zero-filled padding up to ld_dst
template <typename T>
__global__ void k_gather_rows(const float* __restrict__ src, int64_t ld_src, const int32_t* __restrict__ idx,
                              int64_t n, int64_t w, T* __restrict__ dst, int64_t ld_dst) {
  const int64_t i = blockIdx.y;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ld_dst; c += (int64_t)gridDim.x * blockDim.x) {
    float v = c < w ? src[(int64_t)idx[i] * ld_src + c] : 0.f;
    dst[i * ld_dst + c] = Elem<T>::from_f(v);
  }
}
template <typename T>
void gather_rows_f32(const float* src, int64_t ld_src, const int32_t* idx, int64_t n, int64_t w, T* dst,
                     int64_t ld_dst, cudaStream_t s) {
  for (int64_t r0 = 0; r0 < n; r0 += 65535) {
    const int64_t rows = n - r0 < 65535 ? n - r0 : 65535;
    dim3 grid((unsigned)cdiv(ld_dst, 256) > 8 ? 8 : (unsigned)cdiv(ld_dst, 256), (unsigned)rows);
    k_gather_rows<T><<<grid, 256, 0, s>>>(src, ld_src, idx + r0, rows, w, dst + r0 * ld_dst, ld_dst);
  }
}
template void gather_rows_f32<float>(const float*, int64_t, const int32_t*, int64_t, int64_t, float*, int64_t,
                                     cudaStream_t);
template void gather_rows_f32<bf16>(const float*, int64_t, const int32_t*, int64_t, int64_t, bf16*, int64_t,
                                    cudaStream_t);

// ------------------------------------------------ partition-wise eval (R20) --
// Partition-induced graph in partition order: position g holds internal node pnode[g];
// only neighbours in the same partition are kept, as positions relative to the first
// position of g's evaluation chunk (rowbase[g]), so one chunk's rows form a closed CSR.
__global__ void k_part_count(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                             const int32_t* __restrict__ pnode, const int32_t* __restrict__ part, int64_t n,
                             int64_t* __restrict__ deg_new) {
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (g >= n) return;
  const int64_t v = pnode[g];
  const int32_t pv = part[v];
  int cnt = 0;
  for (int64_t e = rp[v] + lane; e < rp[v + 1]; e += 32) {
    const int32_t u = col[e];
    cnt += (u != v) && part[u] == pv;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) deg_new[g] = cnt;
}

__global__ void k_part_fill(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const int32_t* __restrict__ pnode, const int32_t* __restrict__ pos,
                            const int32_t* __restrict__ part, const int32_t* __restrict__ rowbase,
                            const int64_t* __restrict__ rp_new, int64_t n, int32_t* __restrict__ col_new) {
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (g >= n) return;
  const int64_t v = pnode[g];
  const int32_t pv = part[v], base = rowbase[g];
  int64_t out = rp_new[g];
  for (int64_t b = rp[v]; b < rp[v + 1]; b += 32) {
    const int64_t e = b + lane;
    const bool in = e < rp[v + 1];
    const int32_t u = in ? col[e] : 0;
    const bool keep = in && u != v && part[u] == pv;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) col_new[out + __popc(bal & ((1u << lane) - 1))] = pos[u] - base;
    out += __popc(bal);
  }
}

void part_count(const int64_t* rp, const int32_t* col, const int32_t* pnode, const int32_t* part, int64_t n,
                int64_t* deg_new, cudaStream_t s) {
  if (n <= 0) return;
  k_part_count<<<(unsigned)cdiv(n, 8), 256, 0, s>>>(rp, col, pnode, part, n, deg_new);
}
void part_fill(const int64_t* rp, const int32_t* col, const int32_t* pnode, const int32_t* pos, const int32_t* part,
               const int32_t* rowbase, const int64_t* rp_new, int64_t n, int32_t* col_new, cudaStream_t s) {
  if (n <= 0) return;
  k_part_fill<<<(unsigned)cdiv(n, 8), 256, 0, s>>>(rp, col, pnode, pos, part, rowbase, rp_new, n, col_new);
}

// full-graph normalisation scales (R1: (deg+1)^{-1/2}; R2: 1/deg or 0)
__global__ void k_full_scales(const int64_t* __restrict__ rp, int64_t n, int arch, float* __restrict__ scale) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const float deg = (float)(rp[v + 1] - rp[v]);
  scale[v] = arch == 0 ? 1.0f / sqrtf(deg + 1.0f) : (deg > 0.f ? 1.0f / deg : 0.f);
}
void full_graph_scales(const int64_t* rp, int64_t n, int arch, float* scale, cudaStream_t s) {
  if (n <= 0) return;
  k_full_scales<<<(unsigned)cdiv(n, 256), 256, 0, s>>>(rp, n, arch, scale);
}

// ------------------------------------------------------------ batch build --
// grid (cdiv(nb_max, 256), slots)
__global__ void k_batch_setup(const __grid_constant__ BatchGroup G, const int64_t* __restrict__ cstart,
                              const int64_t* __restrict__ rp) {
  pdl_wait();
  pdl_trigger();
  const BatchSlot& S = G.s[blockIdx.y];
  const int q = G.q;
  const int32_t* d = S.desc + (size_t)G.ctr[0] * (3 * q + 4);
  const int32_t* bcl = d;
  const int32_t* loff = d + q;
  const int32_t* voff = d + 2 * q + 1;
  const int qq = d[3 * q + 2];
  const uint32_t tag = (uint32_t)d[3 * q + 3];
  const int nb = loff[q];
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < qq) {
    const int32_t c = bcl[v];
    S.map64[c] = ((uint64_t)tag << 32) | (uint32_t)(loff[v] - (int32_t)cstart[c]);
  }
  if (v == 0) S.stats[0] = S.stats[1] = S.stats[2] = 0;
  if (v >= G.nb_max) return;
  if (v >= nb) {  // inert dummy row: no neighbours, marked by a negative row start
    S.b_nodes[v] = 0;
    S.b_beg[v] = -1;
    return;
  }
  int lo = 0, hi = qq - 1;  // largest k with loff[k] <= v
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (loff[mid] <= v) lo = mid; else hi = mid - 1;
  }
  const int32_t c = bcl[lo];
  const int64_t g = cstart[c] + (v - loff[lo]);
  S.b_nodes[v] = (int32_t)g;
  S.b_beg[v] = voff[lo] + (rp[g] - rp[cstart[c]]);  // row v's segment inside the batch's adjacency space
}
void batch_setup(const BatchGroup& G, const int64_t* cstart, const int64_t* rp, cudaStream_t s) {
  const int n = G.nb_max > G.q ? G.nb_max : G.q;
  launch_pdl(k_batch_setup, dim3((unsigned)cdiv(n > 0 ? n : 1, 256), (unsigned)G.n), 256, 0, s, G, cstart, rp);
}

// One warp per batch row: walk the row's global adjacency 128 entries per round (four
// independent coalesced (col, ccol) load pairs per lane in flight), keep the in-batch
// neighbours (ballot compaction, original order), and write the row's normalisation scale,
// label and train flag.  SMAP: the step's cluster -> local-offset map (q entries, the rest
// "absent") is built in shared memory from the step descriptor by every block, so the
// per-edge membership test is a shared-memory lookup; otherwise the tagged global map64.
// Counters are warp -> block reduced, one integer atomic per block (integer addition:
// deterministic).  grid (<= 2 x 148 / slots, slots), 512 threads; rows dealt by an atomic counter.
constexpr int kBuildRows = 16;
constexpr int32_t kAbsent = INT32_MIN;  // |loff - cstart| < 2^31 - 1: never a real offset
template <bool SMAP, bool PACK>
__global__ void __launch_bounds__(512, 2) k_batch_build(const __grid_constant__ BatchGroup G,
                                                        const int64_t* __restrict__ rp,
                                                        const int32_t* __restrict__ col,
                                                        const int32_t* __restrict__ ccol,
                                                        const int32_t* __restrict__ cid, int arch,
                                                        const int32_t* __restrict__ labels,
                                                        const uint8_t* __restrict__ split, int skip_intra,
                                                        const int64_t* __restrict__ cstart, int num_clusters,
                                                        int ob) {
  extern __shared__ int32_t smap[];  // SMAP: [num_clusters]
  pdl_wait();
  pdl_trigger();
  const BatchSlot& S = G.s[blockIdx.y];
  const int q = G.q;
  const int32_t* d = S.desc + (size_t)G.ctr[0] * (3 * q + 4);
  const int nb = d[2 * q];
  const uint32_t tag = (uint32_t)d[3 * q + 3];
  if (SMAP) {
    for (int i = threadIdx.x; i < num_clusters; i += blockDim.x) smap[i] = kAbsent;
    __syncthreads();
    const int qq = d[3 * q + 2];
    // PACK: local id = local start of the cluster + offset inside it; else u + (loff - cstart)
    for (int k = threadIdx.x; k < qq; k += blockDim.x) smap[d[k]] = d[q + k] - (PACK ? 0 : (int32_t)cstart[d[k]]);
    __syncthreads();
  }
  __shared__ int s_cnt[kBuildRows], s_tr[kBuildRows];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // rows are handed out by a per-slot counter (reset by k_batch_setup): a warp that finishes a
  // short row takes the next one instead of idling until the longest row of its block is done
  int* next_row = reinterpret_cast<int*>(S.stats + 2);
  int cnt_sum = 0, tr_sum = 0;
  for (;;) {
  int v = 0;
  if (lane == 0) v = atomicAdd(next_row, 1);
  v = __shfl_sync(0xffffffffu, v, 0);
  if (v >= G.nb_max) break;
  int cnt = 0, tr = 0;
  if (v < nb) {
    const int64_t g = S.b_nodes[v];
    const int64_t end = rp[g + 1];
    const int64_t out0 = S.b_beg[v];
    int64_t out = out0;
    int intra = 0;  // in-batch intra-cluster neighbours (skip_intra: counted, not stored)
    const int32_t cg = skip_intra ? cid[g] : -1;
    const unsigned lt = (1u << lane) - 1u;
    // R edges per round (R/32 independent (col, ccol) load pairs per lane); the degree tail
    // (lognormal, max ~20x the mean) is what bounds this kernel, so long rows take 256 per
    // round: the longest row's chain of dependent rounds is what the whole launch waits for
    auto walk = [&](auto RT) {
      constexpr int R = decltype(RT)::value;
      for (int64_t base = rp[g]; base < end; base += R) {
        // PACK: u holds the edge code (neighbour cluster << ob) | offset inside it, cc is unused
        int32_t u[R / 32], cc[R / 32], dl[R / 32];
#pragma unroll
        for (int r = 0; r < R / 32; ++r) {  // independent, coalesced loads
          const int64_t e = base + r * 32 + lane;
          if (PACK) {
            u[r] = e < end ? ccol[e] : -1;
          } else {
            u[r] = e < end ? col[e] : -1;
            cc[r] = e < end ? ccol[e] : 0;
          }
        }
        auto clus = [&](int r) { return PACK ? (u[r] >> ob) : cc[r]; };
#pragma unroll
        for (int r = 0; r < R / 32; ++r) {
          if (SMAP) {
            dl[r] = u[r] >= 0 ? smap[clus(r)] : kAbsent;
          } else {
            const uint64_t m = u[r] >= 0 ? S.map64[cc[r]] : 0ull;
            dl[r] = (u[r] >= 0 && (uint32_t)(m >> 32) == tag) ? (int32_t)(uint32_t)m : kAbsent;
          }
        }
#pragma unroll
        for (int r = 0; r < R / 32; ++r) {
          bool in = dl[r] != kAbsent;
          if (skip_intra) {
            const bool ii = in && clus(r) == cg;
            intra += __popc(__ballot_sync(0xffffffffu, ii));
            in &= !ii;
          }
          const unsigned bm = __ballot_sync(0xffffffffu, in);
          if (in) S.b_col[out + __popc(bm & lt)] = (PACK ? (u[r] & ((1 << ob) - 1)) : u[r]) + dl[r];
          out += __popc(bm);
        }
      }
    };
    if (PACK && end - rp[g] > 256) walk(std::integral_constant<int, PACK ? 512 : 256>());
    else if (end - rp[g] > 128) walk(std::integral_constant<int, 256>());
    else walk(std::integral_constant<int, 128>());
    cnt = (int)(out - out0) + intra;  // degree in the batch-induced subgraph
    if (G.X && !G.skip_x) {  // layer-0 self block [X_b | .] of the GraphSAGE concat (R2)
      const uint4* xs = reinterpret_cast<const uint4*>(G.X + g * G.ldx);
      uint4* xd = reinterpret_cast<uint4*>(G.xdst[blockIdx.y] + (int64_t)v * G.ldxd);
      for (int i = lane; i < G.ldx / 8; i += 32) xd[i] = xs[i];
    }
    if (lane == 0) {
      S.b_end[v] = out;
      const float dg = (float)cnt;
      S.scale[v] = arch == 0 ? 1.0f / sqrtf(dg + 1.0f) : (cnt > 0 ? 1.0f / dg : 0.f);
      S.lab_b[v] = labels[g];
      tr = split[g] == 0;
      S.train_b[v] = (uint8_t)tr;
    }
  } else if (lane == 0) {  // inert dummy row
    S.b_end[v] = -1;
    S.scale[v] = 0.f;
    S.lab_b[v] = 0;
    S.train_b[v] = 0;
  }
  cnt_sum += cnt;
  tr_sum += tr;
  }
  if (lane == 0) { s_cnt[w] = cnt_sum; s_tr[w] = tr_sum; }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long a = 0, b = 0;
    for (int k = 0; k < kBuildRows; ++k) a += s_cnt[k], b += s_tr[k];
    if (a) atomicAdd((unsigned long long*)&S.stats[0], (unsigned long long)a);
    if (b) atomicAdd((unsigned long long*)&S.stats[1], (unsigned long long)b);
    // the last CTA of the launch (every CTA has read the batch index by now) advances it
    __threadfence();
    const unsigned total = gridDim.x * gridDim.y;
    if (atomicAdd(reinterpret_cast<unsigned*>(G.ctr + 1), 1u) == total - 1) {
      G.ctr[0] += 1;
      G.ctr[1] = 0;
    }
  }
}
void batch_build(const BatchGroup& G, const int64_t* rp, const int32_t* col, const int32_t* ccol,
                 const int32_t* cid, const int64_t* cstart, int num_clusters, int arch, const int32_t* labels,
                 const uint8_t* split, int skip_intra, int ob, cudaStream_t s) {
  if (G.nb_max <= 0) return;
  // two 512-thread CTAs per SM (launch bounds) shared by the slots; rows are dealt dynamically
  const int per_slot = std::max(1, std::min((int)cdiv(G.nb_max, kBuildRows), 2 * device_sms() / std::max(G.n, 1)));
  const dim3 grid((unsigned)per_slot, (unsigned)G.n);
  const size_t smem = (size_t)num_clusters * 4;
  const char* force = std::getenv("GIST_BATCH_GLOBAL_MAP");  // tests: exercise the global-map path
  if (smem <= 64 * 1024 && !(force && force[0] == '1')) {
    ensure_smem((const void*)k_batch_build<true, false>, 64 * 1024);
    ensure_smem((const void*)k_batch_build<true, true>, 64 * 1024);
    if (ob > 0)
      launch_pdl(k_batch_build<true, true>, grid, kBuildRows * 32, smem, s, G, rp, col, ccol, cid, arch, labels,
                 split, skip_intra, cstart, num_clusters, ob);
    else
      launch_pdl(k_batch_build<true, false>, grid, kBuildRows * 32, smem, s, G, rp, col, ccol, cid, arch, labels,
                 split, skip_intra, cstart, num_clusters, 0);
  } else {  // the packed codes are only built when the shared-memory map applies (pack_bits)
    launch_pdl(k_batch_build<false, false>, grid, kBuildRows * 32, 0, s, G, rp, col, ccol, cid, arch, labels, split,
               skip_intra, cstart, num_clusters, 0);
  }
}

// The layer-0 self block [X_b | .] of a batch built with skip_x (the same copy as the build's):
// one warp per row; rows of the batch built last, dummy rows (b_beg < 0) untouched
__global__ void __launch_bounds__(256) k_batch_xcopy(const __grid_constant__ BatchGroup G) {
  pdl_wait();
  pdl_trigger();
  const BatchSlot& S = G.s[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int nvec = (int)(G.ldx / 8);
  const int wpg = (int)((gridDim.x * blockDim.x) >> 5);
  for (int v = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); v < G.nb_max; v += wpg) {
    if (S.b_beg[v] < 0) continue;
    const uint4* xs = reinterpret_cast<const uint4*>(G.X + (int64_t)S.b_nodes[v] * G.ldx);
    uint4* xd = reinterpret_cast<uint4*>(G.xdst[blockIdx.y] + (int64_t)v * G.ldxd);
    // the row's random HBM read: up to four 16-byte loads per lane in flight before any store
    for (int i0 = 0; i0 < nvec; i0 += 128) {
      uint4 t[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (i0 + 32 * j + lane < nvec) t[j] = __ldg(xs + i0 + 32 * j + lane);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (i0 + 32 * j + lane < nvec) xd[i0 + 32 * j + lane] = t[j];
    }
  }
}
void batch_xcopy(const BatchGroup& G, cudaStream_t s) {
  if (G.nb_max <= 0 || !G.X) return;
  // one row per warp: every row's gather latency overlaps every other's
  const int per_slot = std::max(1, (int)cdiv(G.nb_max, 8));
  launch_pdl(k_batch_xcopy, dim3((unsigned)per_slot, (unsigned)G.n), 256, 0, s, G);
}

// ob > 0: packed per-edge codes (cid[u] << ob) | (u - cstart[cid[u]]) (one array instead of col +
// ccol for the batch build); ob == 0: ccol[e] = cid[col[e]]
__global__ void k_edge_codes(const int32_t* __restrict__ col, const int32_t* __restrict__ cid,
                             const int64_t* __restrict__ cstart, int64_t nnz, int ob, int32_t* __restrict__ code) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = col[e], k = cid[u];
    code[e] = (k << ob) | (int32_t)(u - cstart[k]);
  }
}
void edge_codes(const int32_t* col, const int32_t* cid, const int64_t* cstart, int64_t nnz, int ob, int32_t* code,
                cudaStream_t s) {
  if (nnz <= 0) return;
  k_edge_codes<<<148 * 8, 256, 0, s>>>(col, cid, cstart, nnz, ob, code);
}
int pack_bits(int num_clusters, int64_t max_csize) {
  if ((size_t)num_clusters * 4 > 64 * 1024 || std::getenv("GIST_BATCH_GLOBAL_MAP")) return 0;
  int ob = 1, cb = 1;
  while (((int64_t)1 << ob) < max_csize) ++ob;
  while ((1 << cb) < num_clusters) ++cb;
  return ob + cb <= 31 ? ob : 0;
}

__global__ void k_edge_clusters(const int32_t* __restrict__ col, const int32_t* __restrict__ cid, int64_t nnz,
                                int32_t* __restrict__ ccol) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    ccol[e] = cid[col[e]];
}
// Edge checks of load_graph on the device (one warp per row, original ids): out[0] = edges with
// col out of [0, n), out[1] = self loops, out[2] = non-loop edges inside a cluster, out[3] = edges
// not strictly after their predecessor in the row (unsorted or duplicate), out[4] = edges (v, u)
// whose reverse (u, v) is missing (binary search in row u; the backward SpMM^T reuses the CSR of
// the symmetric A).  Block-reduced integer atomics: deterministic.
__device__ __forceinline__ bool row_has(const int64_t* rp, const int32_t* col, int64_t u, int32_t v) {
  int64_t lo = rp[u], hi = rp[u + 1] - 1;
  while (lo <= hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int32_t x = col[mid];
    if (x == v) return true;
    if (x < v) lo = mid + 1; else hi = mid - 1;
  }
  return false;
}
__global__ void __launch_bounds__(256) k_validate_edges(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                        const int32_t* __restrict__ cid, int64_t n,
                                                        unsigned long long* __restrict__ out) {
  constexpr int NC = 5;
  __shared__ unsigned long long sb[NC];
  if (threadIdx.x < NC) sb[threadIdx.x] = 0;
  __syncthreads();
  const int64_t v = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  unsigned long long c[NC] = {0, 0, 0, 0, 0};
  if (v < n) {
    const int32_t cv = cid[v];
    for (int64_t e = rp[v] + lane; e < rp[v + 1]; e += 32) {
      const int32_t u = col[e];
      if (e > rp[v] && col[e - 1] >= u) ++c[3];
      if (u < 0 || u >= n) { ++c[0]; continue; }
      if (u == v) { ++c[1]; continue; }
      if (cid[u] == cv) ++c[2];
      if (!row_has(rp, col, u, (int32_t)v)) ++c[4];
    }
  }
#pragma unroll
  for (int k = 0; k < NC; ++k)
    for (int o = 16; o; o >>= 1) c[k] += __shfl_xor_sync(0xffffffffu, c[k], o);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NC; ++k)
      if (c[k]) atomicAdd(&sb[k], c[k]);
  __syncthreads();
  if (threadIdx.x < NC && sb[threadIdx.x]) atomicAdd(&out[threadIdx.x], sb[threadIdx.x]);
}
void validate_edges(const int64_t* rp, const int32_t* col, const int32_t* cid, int64_t n, unsigned long long* out,
                    cudaStream_t s) {
  if (n <= 0) return;
  k_validate_edges<<<(unsigned)cdiv(n, 8), 256, 0, s>>>(rp, col, cid, n, out);
}

void edge_clusters(const int32_t* col, const int32_t* cid, int64_t nnz, int32_t* ccol, cudaStream_t s) {
  if (nnz <= 0) return;
  k_edge_clusters<<<148 * 8, 256, 0, s>>>(col, cid, nnz, ccol);
}

// one warp per node g: its intra-cluster neighbours -> 1 in its cluster's block row
__global__ void k_cluster_blocks(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                 const int32_t* __restrict__ cid, const int64_t* __restrict__ cstart, int64_t n,
                                 int bs, bf16* __restrict__ blocks) {
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (g >= n) return;
  const int32_t c = cid[g];
  const int64_t c0 = cstart[c];
  bf16* row = blocks + ((int64_t)c * bs + (g - c0)) * bs;
  for (int64_t e = rp[g] + lane; e < rp[g + 1]; e += 32) {
    const int32_t u = col[e];
    if (cid[u] == c) row[u - c0] = __float2bfloat16_rn(1.0f);
  }
}
void cluster_blocks(const int64_t* rp, const int32_t* col, const int32_t* cid, const int64_t* cstart, int64_t n,
                    int bs, bf16* blocks, cudaStream_t s) {
  if (n <= 0) return;
  k_cluster_blocks<<<(unsigned)cdiv(n, 8), 256, 0, s>>>(rp, col, cid, cstart, n, bs, blocks);
}

}  // namespace gist
