// spmm.cu -- aggregation SpMM of Eq. (1)/(2).
//
// One warp owns one output row and one 512-byte column chunk (32 lanes x 16 B).
// Neighbour indices of the row are loaded 32 at a time with one coalesced load,
// broadcast by shuffle, and each neighbour row chunk is gathered with 16-byte
// vector loads (4 fp32 / 8 bf16 per lane), accumulated in fp32 registers in a
// fixed order (deterministic, no atomics).  The normalisation of A_bar is never
// materialised: row/column scale vectors (deg+1)^{-1/2} (GCN renorm, R1) or
// 1/deg (GraphSAGE mean, R2) are applied on the fly; the backward SpMM reuses
// the same CSR with the scales swapped (N^T = A diag(1/deg)).
#include "common.cuh"
#include "kernels.h"

namespace gist {

template <typename T, int UNROLL>
__global__ void __launch_bounds__(256) k_spmm(const SpmmArgs<T> a, int nchunks) {
  constexpr int V = Elem<T>::kVec;
  constexpr int CW = 32 * V;
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t v = wid / nchunks;
  const int chunk = (int)(wid - v * nchunks);
  if (v >= a.rows) return;
  const int64_t c0 = (int64_t)chunk * CW + lane * V;
  const bool active = c0 < a.w;

  float acc[V];
#pragma unroll
  for (int i = 0; i < V; ++i) acc[i] = 0.f;

  const int64_t hv = a.h_index ? (int64_t)a.h_index[v] : v;
  if (a.self && active) {
    float t[V];
    ld16(a.H + hv * a.ldh + c0, t);
    const float s = a.colscale ? a.colscale[v] : 1.f;
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = s * t[i];
  }
  if (a.self_out && active) {
    float t[V];
    ld16(a.H + hv * a.ldh + c0, t);
    st16(a.self_out + v * a.ld_self + c0, t);
  }

  const int64_t beg = a.row_ptr[v], end = a.row_ptr[v + 1];
  for (int64_t base = beg; base < end; base += 32) {
    const int n = (end - base) < 32 ? (int)(end - base) : 32;
    int32_t u = lane < n ? a.col[base + lane] : 0;
    float su = (a.colscale && lane < n) ? a.colscale[u] : 1.f;
    int64_t hu = a.h_index ? (int64_t)(lane < n ? a.h_index[u] : 0) : (int64_t)u;
    int j = 0;
    for (; j + UNROLL <= n; j += UNROLL) {
      float t[UNROLL][V];
      float s[UNROLL];
#pragma unroll
      for (int q = 0; q < UNROLL; ++q) {
        const int64_t r = __shfl_sync(0xffffffffu, hu, j + q);
        s[q] = __shfl_sync(0xffffffffu, su, j + q);
        if (active) ld16(a.H + r * a.ldh + c0, t[q]);
      }
      if (active) {
#pragma unroll
        for (int q = 0; q < UNROLL; ++q)
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] = fmaf(s[q], t[q][i], acc[i]);
      }
    }
    for (; j < n; ++j) {
      const int64_t r = __shfl_sync(0xffffffffu, hu, j);
      const float s = __shfl_sync(0xffffffffu, su, j);
      if (active) {
        float t[V];
        ld16(a.H + r * a.ldh + c0, t);
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = fmaf(s, t[i], acc[i]);
      }
    }
  }
  if (!active) return;
  const float rs = a.rowscale ? a.rowscale[v] : 1.f;
#pragma unroll
  for (int i = 0; i < V; ++i) acc[i] *= rs;
  if (a.add) {
    float t[V];
    ld16(a.add + v * a.ld_add + c0, t);
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] += t[i];
  }
  if (a.mask) {
    float t[V];
    ld16(a.mask + v * a.ld_mask + c0, t);
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = t[i] > 0.f ? acc[i] : 0.f;  // ReLU'(0) = 0 (R3)
  }
  st16(a.out + v * a.ldo + c0, acc);
}

template <typename T>
void spmm(const SpmmArgs<T>& a, cudaStream_t s) {
  if (a.rows <= 0 || a.w <= 0) return;
  constexpr int CW = 32 * Elem<T>::kVec;
  const int nchunks = (int)cdiv(a.w, CW);
  const int64_t warps = a.rows * nchunks;
  const int64_t blocks = cdiv(warps, 8);
  k_spmm<T, 4><<<(unsigned)blocks, 256, 0, s>>>(a, nchunks);
}

template void spmm<float>(const SpmmArgs<float>&, cudaStream_t);
template void spmm<bf16>(const SpmmArgs<bf16>&, cudaStream_t);

}  // namespace gist
