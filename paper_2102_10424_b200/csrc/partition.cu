// partition.cu -- subGCNs, subAgg scatter
// and Glorot init, following readings R5, R6, R9, R11.
//
// Partition of hidden dim l in round t: key_r = Philox(seed; r, t, l, 1) as a
// 64-bit value, pi = units sorted by (key, r) (stable device radix sort on the
// key with the unit index as value), block i = pi[b_i, b_{i+1}) where the first
// d mod m blocks hold ceil(d/m) units, each block re-sorted ascending.
#include <cub/cub.cuh>
#include <nccl.h>
#include <nccl_device.h>

#include "common.cuh"
#include "kernels.h"

namespace gist {

__global__ void k_part_keys(int d, uint32_t t, uint32_t l, uint64_t seed, uint64_t* __restrict__ keys,
                            int32_t* __restrict__ idx) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= d) return;
  keys[r] = philox_key64((uint32_t)r, t, l, PURPOSE_PARTITION, seed);
  idx[r] = r;
}
void partition_keys(int d, uint32_t t, uint32_t l, uint64_t seed, uint64_t* keys, int32_t* idx, cudaStream_t s) {
  k_part_keys<<<(unsigned)cdiv(d, 256), 256, 0, s>>>(d, t, l, seed, keys, idx);
}

size_t partition_sort(const uint64_t* keys_in, uint64_t* keys_out, const int32_t* idx_in, int32_t* idx_out, int d,
                      void* tmp, size_t tmp_bytes, cudaStream_t s) {
  // radix sort is stable: equal keys keep ascending unit order (the (key, r) tie-break of R5)
  size_t bytes = tmp_bytes;
  cub::DeviceRadixSort::SortPairs(tmp, bytes, keys_in, keys_out, idx_in, idx_out, d, 0, 64, s);
  return bytes;
}

__global__ void k_part_assign(const int32_t* __restrict__ sorted_idx, int d, int m, int32_t* __restrict__ blk) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  const int base = d / m, extra = d % m;
  const int big = extra * (base + 1);
  const int b = j < big ? j / (base + 1) : extra + (j - big) / base;
  blk[sorted_idx[j]] = b;
}
void partition_assign(const int32_t* sorted_idx, int d, int m, int32_t* blk, cudaStream_t s) {
  k_part_assign<<<(unsigned)cdiv(d, 256), 256, 0, s>>>(sorted_idx, d, m, blk);
}

// one CTA per block i: stable compaction of {r : blk[r] == i} in ascending r
__global__ void __launch_bounds__(1024) k_part_compact(const int32_t* __restrict__ blk, int d,
                                                       const int32_t* __restrict__ offs, int32_t* __restrict__ units) {
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage ts;
  __shared__ int carry;
  const int i = blockIdx.x;
  if (threadIdx.x == 0) carry = offs[i];
  __syncthreads();
  for (int base = 0; base < d; base += 1024) {
    const int r = base + threadIdx.x;
    const int f = (r < d && blk[r] == i) ? 1 : 0;
    int excl, tot;
    Scan(ts).ExclusiveSum(f, excl, tot);
    if (f) units[carry + excl] = r;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}
void partition_compact(const int32_t* blk, int d, int m, const int32_t* offs, int32_t* units, cudaStream_t s) {
  k_part_compact<<<(unsigned)m, 1024, 0, s>>>(blk, d, offs, units);
}

// physical row of the global weight for sub-weight physical row p (-1 = padding)
__device__ __forceinline__ int64_t glob_row(const LayerMap& m, int p) {
  if (m.gat) {  // R21: rows D_l^(i), then the two attention rows (global rows glob_half, glob_half + 1)
    if (p < m.nrows) return m.rows ? m.rows[p] : p;
    if (p >= m.half && p < m.half + 2) return (int64_t)m.glob_half + (p - m.half);
    return -1;
  }
  if (!m.sage) {
    if (p >= m.nrows) return -1;
    return m.rows ? m.rows[p] : p;
  }
  if (p < m.nrows) return m.rows ? m.rows[p] : p;
  if (p >= m.half && p < m.half + m.nrows) {
    const int r = p - m.half;
    return (int64_t)m.glob_half + (m.rows ? m.rows[r] : r);
  }
  return -1;
}

__global__ void k_extract(const float* __restrict__ theta, const LayerMap m, float* __restrict__ w, int p0) {
  const int p = p0 + blockIdx.y;
  const int64_t gr = glob_row(m, p);
  if (gr >= 0 && (gr < m.row_lo || gr >= m.row_hi)) return;  // another rank's row (sharded Theta)
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < m.Np; q += gridDim.x * blockDim.x) {
    float v = 0.f;
    if (gr >= 0 && q < m.ncols) v = theta[(gr - m.row_lo) * m.ldg + (m.cols ? m.cols[q] : q)];
    w[(int64_t)p * m.Np + q] = v;
  }
}
__global__ void k_scatter(float* __restrict__ theta, const LayerMap m, const float* __restrict__ w, int p0) {
  const int p = p0 + blockIdx.y;
  const int64_t gr = glob_row(m, p);
  if (gr < m.row_lo || gr >= m.row_hi) return;  // padding (gr < 0) or another rank's row
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < m.ncols; q += gridDim.x * blockDim.x)
    theta[(gr - m.row_lo) * m.ldg + (m.cols ? m.cols[q] : q)] = w[(int64_t)p * m.Np + q];
}
static dim3 grid_for(const LayerMap& m, int rows) {
  unsigned gx = (unsigned)cdiv(m.Np, 256);
  return dim3(gx > 16 ? 16 : gx, (unsigned)rows);
}
void extract_sub(const float* theta, const LayerMap& m, float* w_sub, cudaStream_t s) {
  for (int p0 = 0; p0 < m.Kp; p0 += 65535) {
    const int rows = m.Kp - p0 < 65535 ? m.Kp - p0 : 65535;
    k_extract<<<grid_for(m, rows), 256, 0, s>>>(theta, m, w_sub, p0);
  }
}
void scatter_sub(float* theta, const LayerMap& m, const float* w_sub, cudaStream_t s) {
  for (int p0 = 0; p0 < m.Kp; p0 += 65535) {
    const int rows = m.Kp - p0 < 65535 ? m.Kp - p0 : 65535;
    k_scatter<<<grid_for(m, rows), 256, 0, s>>>(theta, m, w_sub, p0);
  }
}

// subAgg over peer memory (agg_mode P2P): the owner reads its block once and
// stores it into every rank's replica (d.dst[r] is rank r's copy of this layer of Theta, a
// peer pointer opened from its CUDA IPC handle; d.dst[rank] is the local one).  Same element
// placement as k_scatter; the system-scope fence orders the peer stores before this thread
// retires, ahead of the NCCL barrier that follows the launch on the stream.
__global__ void k_scatter_peers(const PeerDst d, const LayerMap m, const float* __restrict__ w, int p0) {
  const int p = p0 + blockIdx.y;
  const int64_t gr = glob_row(m, p);
  if (gr < 0) return;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < m.ncols; q += gridDim.x * blockDim.x) {
    const float v = w[(int64_t)p * m.Np + q];
    const int64_t o = gr * m.ldg + (m.cols ? m.cols[q] : q);
    for (int r = 0; r < d.n; ++r) d.dst[r][o] = v;
  }
  __threadfence_system();
}
void scatter_sub_peers(const PeerDst& d, const LayerMap& m, const float* w_sub, cudaStream_t s) {
  for (int p0 = 0; p0 < m.Kp; p0 += 65535) {
    const int rows = m.Kp - p0 < 65535 ? m.Kp - p0 : 65535;
    k_scatter_peers<<<grid_for(m, rows), 256, 0, s>>>(d, m, w_sub, p0);
  }
}

// subAgg through an NCCL symmetric window (agg_mode SYMM): Theta lives in an
// ncclMemAlloc region registered as a symmetric window; the owner of a slot reads each element of its
// block once and stores it into every LSA peer's replica through the device API (ncclGetLsaPointer:
// peer replicas mapped into this process by NCCL), or -- when the communicator has an NVLS
// multicast object (lsaMultimem) -- with one multimem.st that the NVSwitch fans out to every replica.
__global__ void k_scatter_symm(const ncclDevComm dc, ncclWindow_t win, size_t base, const LayerMap m,
                               const float* __restrict__ w, int p0, int mm) {
  const int p = p0 + blockIdx.y;
  const int64_t gr = glob_row(m, p);
  if (gr < 0) return;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < m.ncols; q += gridDim.x * blockDim.x) {
    const float v = w[(int64_t)p * m.Np + q];
    const size_t off = base + (size_t)(gr * m.ldg + (m.cols ? m.cols[q] : q)) * sizeof(float);
    if (mm) {
      float* mp = static_cast<float*>(ncclGetLsaMultimemPointer(win, off, dc));
      asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mp), "f"(v) : "memory");
    } else {
      for (int r = 0; r < dc.lsaSize; ++r) *static_cast<float*>(ncclGetLsaPointer(win, off, r)) = v;
    }
  }
  __threadfence_system();
}
void scatter_sub_symm(const ncclDevComm& dc, ncclWindow_t win, size_t base, const LayerMap& m, const float* w_sub,
                      bool multimem, cudaStream_t s) {
  for (int p0 = 0; p0 < m.Kp; p0 += 65535) {
    const int rows = m.Kp - p0 < 65535 ? m.Kp - p0 : 65535;
    k_scatter_symm<<<grid_for(m, rows), 256, 0, s>>>(dc, win, base, m, w_sub, p0, multimem ? 1 : 0);
  }
}

// Glorot uniform (R11): u = (w0 >> 8) 2^-24, t = 2u - 1 (exact), W = fl32(t * scale).
// Logical (r, c) of Theta_l (SAGE: r < d self rows, r >= d neighbour rows).
__global__ void k_glorot(float* __restrict__ theta, int rows, int cols, int sage, int d_l, int glob_half,
                         int64_t ldg, uint32_t layer, uint64_t seed, float scale, int r0, int64_t row_lo,
                         int64_t row_hi) {
  const int r = r0 + blockIdx.y;
  {  // sharded Theta: only this rank's physical rows
    const int64_t pr = (sage && r >= d_l) ? (int64_t)glob_half + (r - d_l) : (int64_t)r;
    if (pr < row_lo || pr >= row_hi) return;
  }
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += gridDim.x * blockDim.x) {
    const uint64_t flat = (uint64_t)r * (uint64_t)cols + (uint64_t)c;
    const U4 o = philox4x32_10(U4{(uint32_t)flat, layer, (uint32_t)(flat >> 32), PURPOSE_INIT}, (uint32_t)seed,
                               (uint32_t)(seed >> 32));
    const float u = __fmul_rn((float)(o.x >> 8), 5.9604644775390625e-08f);  // 2^-24, exact
    const float t = __fsub_rn(__fmul_rn(2.0f, u), 1.0f);
    const int64_t pr = (sage && r >= d_l) ? (int64_t)glob_half + (r - d_l) : (int64_t)r;
    theta[(pr - row_lo) * ldg + c] = __fmul_rn(t, scale);
  }
}
void glorot_init(float* theta, int rows_logical, int cols, int sage, int d_l, int glob_half, int64_t ldg,
                 uint32_t layer, uint64_t seed, float scale, cudaStream_t s, int64_t row_lo, int64_t row_hi) {
  const unsigned gx = (unsigned)cdiv(cols, 256);
  for (int r0 = 0; r0 < rows_logical; r0 += 65535) {
    const int rows = rows_logical - r0 < 65535 ? rows_logical - r0 : 65535;
    dim3 grid(gx > 16 ? 16 : gx, (unsigned)rows);
    k_glorot<<<grid, 256, 0, s>>>(theta, rows_logical, cols, sage, d_l, glob_half, ldg, layer, seed, scale, r0,
                                  row_lo, row_hi);
  }
}

}  // namespace gist
