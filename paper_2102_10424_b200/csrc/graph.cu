// graph.cu -- graph relabelling on load and the Cluster mini-batch build
// (SURVEY a1).
//
// On load, nodes are relabelled so that every cluster is a contiguous id range
// (new id = position in the cluster-sorted order).  A mini-batch is then the
// union of q clusters = q id ranges; batch row v maps to new id b_nodes[v] and
// a neighbour u is inside the batch iff map_cl[cid[u]] >= 0, with local id
// map_cl[cid[u]] + (u - cstart[cid[u]]).  No n-sized scratch map has to be
// cleared per step: only the q entries of map_cl are set and reset.
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

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
__global__ void k_batch_nodes(const int32_t* __restrict__ bcl, const int32_t* __restrict__ loff, int q,
                              const int64_t* __restrict__ cstart, int32_t* __restrict__ map_cl,
                              int32_t* __restrict__ b_nodes, int nb) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < q) map_cl[bcl[v]] = loff[v];
  if (v >= nb) return;
  int lo = 0, hi = q - 1;  // largest k with loff[k] <= v
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (loff[mid] <= v) lo = mid; else hi = mid - 1;
  }
  b_nodes[v] = (int32_t)(cstart[bcl[lo]] + (v - loff[lo]));
}
void batch_nodes(const int32_t* bcl, const int32_t* loff, int q, const int64_t* cstart, int32_t* map_cl,
                 int32_t* b_nodes, int nb, cudaStream_t s) {
  const int n = nb > q ? nb : q;
  k_batch_nodes<<<(unsigned)cdiv(n, 256), 256, 0, s>>>(bcl, loff, q, cstart, map_cl, b_nodes, nb);
}

__global__ void k_batch_count(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                              const int32_t* __restrict__ cid, const int32_t* __restrict__ map_cl,
                              const int32_t* __restrict__ b_nodes, int nb, int arch,
                              const int32_t* __restrict__ labels, const uint8_t* __restrict__ split,
                              int32_t* __restrict__ deg_b, float* __restrict__ scale, int32_t* __restrict__ lab_b,
                              uint8_t* __restrict__ train_b) {
  const int v = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (v >= nb) return;
  const int64_t g = b_nodes[v];
  int cnt = 0;
  for (int64_t e = rp[g] + lane; e < rp[g + 1]; e += 32) cnt += map_cl[cid[col[e]]] >= 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) {
    deg_b[v] = cnt;
    const float d = (float)cnt;
    scale[v] = arch == 0 ? 1.0f / sqrtf(d + 1.0f) : (cnt > 0 ? 1.0f / d : 0.f);
    lab_b[v] = labels[g];
    train_b[v] = split[g] == 0;
  }
}
void batch_count(const int64_t* rp, const int32_t* col, const int32_t* cid, const int32_t* map_cl,
                 const int32_t* b_nodes, int nb, int arch, const int32_t* labels, const uint8_t* split,
                 int32_t* deg_b, float* scale, int32_t* lab_b, uint8_t* train_b, cudaStream_t s) {
  if (nb <= 0) return;
  k_batch_count<<<(unsigned)cdiv(nb, 8), 256, 0, s>>>(rp, col, cid, map_cl, b_nodes, nb, arch, labels, split, deg_b,
                                                       scale, lab_b, train_b);
}

// single-CTA deterministic scan of the batch degrees + count of train rows
__global__ void __launch_bounds__(1024) k_batch_scan(const int32_t* __restrict__ deg_b,
                                                     const uint8_t* __restrict__ train_b, int nb,
                                                     int64_t* __restrict__ b_rp, int64_t* __restrict__ stats) {
  using Scan = cub::BlockScan<int64_t, 1024>;
  using Red = cub::BlockReduce<int64_t, 1024>;
  __shared__ typename Scan::TempStorage ts;
  __shared__ typename Red::TempStorage tr;
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  int64_t ntrain = 0;
  for (int base = 0; base < nb; base += 1024) {
    const int v = base + threadIdx.x;
    const int64_t d = v < nb ? deg_b[v] : 0;
    if (v < nb) ntrain += train_b[v];
    int64_t excl, tot;
    Scan(ts).ExclusiveSum(d, excl, tot);
    if (v < nb) b_rp[v] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  const int64_t nt = Red(tr).Sum(ntrain);
  if (threadIdx.x == 0) {
    b_rp[nb] = carry;
    stats[0] = carry;
    stats[1] = nt;
  }
}
void batch_scan(const int32_t* deg_b, const uint8_t* train_b, int nb, int64_t* b_rp, int64_t* stats,
                cudaStream_t s) {
  k_batch_scan<<<1, 1024, 0, s>>>(deg_b, train_b, nb, b_rp, stats);
}

__global__ void k_batch_fill(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                             const int32_t* __restrict__ cid, const int32_t* __restrict__ map_cl,
                             const int64_t* __restrict__ cstart, const int32_t* __restrict__ b_nodes, int nb,
                             const int64_t* __restrict__ b_rp, int32_t* __restrict__ b_col) {
  const int v = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (v >= nb) return;
  const int64_t g = b_nodes[v];
  int64_t out = b_rp[v];
  const int64_t end = rp[g + 1];
  for (int64_t base = rp[g]; base < end; base += 32) {
    const int64_t e = base + lane;
    int32_t loc = -1;
    if (e < end) {
      const int32_t u = col[e];
      const int32_t c = cid[u];
      const int32_t lo = map_cl[c];
      if (lo >= 0) loc = lo + (int32_t)(u - cstart[c]);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, loc >= 0);
    if (loc >= 0) b_col[out + __popc(bal & ((1u << lane) - 1))] = loc;
    out += __popc(bal);
  }
}
void batch_fill(const int64_t* rp, const int32_t* col, const int32_t* cid, const int32_t* map_cl,
                const int64_t* cstart, const int32_t* b_nodes, int nb, const int64_t* b_rp, int32_t* b_col,
                cudaStream_t s) {
  if (nb <= 0) return;
  k_batch_fill<<<(unsigned)cdiv(nb, 8), 256, 0, s>>>(rp, col, cid, map_cl, cstart, b_nodes, nb, b_rp, b_col);
}

__global__ void k_batch_reset(const int32_t* __restrict__ bcl, int q, int32_t* __restrict__ map_cl) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < q) map_cl[bcl[k]] = -1;
}
void batch_reset(const int32_t* bcl, int q, int32_t* map_cl, cudaStream_t s) {
  k_batch_reset<<<(unsigned)cdiv(q, 256), 256, 0, s>>>(bcl, q, map_cl);
}

}  // namespace gist
