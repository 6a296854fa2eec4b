// gat.cu -- GAT sub-GCN layer kernels (reading R21).
//
// One single-head GAT layer on a batch (or full / partition) CSR without self loops:
//   Z = H W (tcgen05 / SIMT GEMM, outside), s = Z a_src, t = Z a_dst          (k_gat_scores)
//   e_ij = LeakyReLU(t_i + s_j), j in N(i) u {i}; alpha = row softmax;
//   out_i = sum_j alpha_ij Z_j, ReLU on hidden layers                          (k_gat_fwd)
// Backward, with G = dL/dout (ReLU mask of the next layer's input applied on read):
//   S_i = sum_j alpha_ij (G_i . Z_j),  dt_i = sum_j alpha_ij slope_ij (G_i . Z_j - S_i)  (k_gat_bwd_rows,
//   which also stores the masked G_i back in place for the column pass)
//   dZ_j = sum_i alpha_ij G_i + ds_j a_src + dt_j a_dst,
//   ds_j = sum_i alpha_ij slope_ij (G_i . Z_j - S_i)      over i in N(j) u {j}   (k_gat_bwd_cols)
// (the adjacency is symmetric, so the column pass walks row j's own neighbour list and
// recomputes alpha_ij from the per-node scalars t_i, s_j, lse_i: no atomics, no transpose);
//   d a_src = Z^T ds, d a_dst = Z^T dt                                          (k_gat_da)
// One warp per row; a lane holds 4 consecutive columns of each 128-column chunk (NV chunks).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace gist {
namespace {

constexpr float kSlope = 0.2f;  // LeakyReLU negative slope (GAT)

__device__ __forceinline__ void ld4(const float* p, float* v) {
  const float4 x = *reinterpret_cast<const float4*>(p);
  v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
__device__ __forceinline__ void ld4(const bf16* p, float* v) {
  const uint2 x = *reinterpret_cast<const uint2*>(p);
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&x.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&x.y));
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
__device__ __forceinline__ void st4(float* p, const float* v) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void st4(bf16* p, const float* v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
  uint2 x;
  x.x = *reinterpret_cast<uint32_t*>(&a);
  x.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = x;
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ float lrelu(float x) { return x > 0.f ? x : kSlope * x; }

// G_i (masked by mask_i > 0 when a mask is given) into registers; columns >= w read as 0
template <typename T, int NV, typename TM = T>
__device__ __forceinline__ void load_row(const T* base, int64_t ld, int64_t r, int64_t w, int lane, float (&x)[NV][4],
                                         const TM* mask = nullptr, int64_t ldm = 0) {
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int64_t c = (int64_t)k * 128 + lane * 4;
    if (c < w) {
      ld4(base + r * ld + c, x[k]);
      if (mask) {
        float m[4];
        ld4(mask + r * ldm + c, m);
#pragma unroll
        for (int q = 0; q < 4; ++q) x[k][q] = m[q] > 0.f ? x[k][q] : 0.f;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) x[k][q] = 0.f;
    }
  }
}

// Two dot products of one row (width w, any w; lane holds 4 consecutive columns of every
// 128-column chunk, the chunks in order -- the summation order of the register-tile kernels)
template <typename T>
__device__ __forceinline__ void dot2(const T* row, int64_t w, const float* u1, const float* u2, int lane, float& p1,
                                     float& p2) {
  p1 = p2 = 0.f;
  for (int64_t c = lane * 4; c < w; c += 128) {
    float x[4];
    ld4(row + c, x);
#pragma unroll
    for (int q = 0; q < 4; ++q) p1 += x[q] * u1[c + q], p2 += x[q] * u2[c + q];
  }
  p1 = warp_sum(p1);
  p2 = warp_sum(p2);
}

// s[v] = Z[v, :] . a_src, t[v] = Z[v, :] . a_dst (one warp per row)
template <typename T>
__global__ void __launch_bounds__(256) k_gat_scores(const __grid_constant__ GatGroup<T> Gp) {
  const GatLayer<T>& a = Gp.a[blockIdx.y];
  const int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= a.rows) return;
  float ps, pt;
  dot2(a.Z + v * a.ldz, a.w, a.a_src, a.a_dst, lane, ps, pt);
  if (lane == 0) a.s[v] = ps, a.t[v] = pt;
}

// wa[k] = W32[k, :] . a_src, wa[kw + k] = W32[k, :] . a_dst (fp32; one warp per row of W)
template <typename T>
__global__ void __launch_bounds__(256) k_gat_wa(const __grid_constant__ GatGroup<T> Gp) {
  const GatLayer<T>& a = Gp.a[blockIdx.y];
  const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= a.kw) return;
  float ps, pt;
  dot2(a.W32 + k * a.ldw, a.w, a.a_src, a.a_dst, lane, ps, pt);
  if (lane == 0) a.wa[k] = ps, a.wa[a.kw + k] = pt;
}

// s[v] = H[v, :] . wa[0:kw], t[v] = H[v, :] . wa[kw:2kw] (any input width kw, e.g. d_0 = 3,703)
template <typename T>
__global__ void __launch_bounds__(256) k_gat_scores_h(const __grid_constant__ GatGroup<T> Gp) {
  const GatLayer<T>& a = Gp.a[blockIdx.y];
  const int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= a.rows) return;
  float ps, pt;
  dot2(a.H + v * a.ldh, a.kw, a.wa, a.wa + a.kw, lane, ps, pt);
  if (lane == 0) a.s[v] = ps, a.t[v] = pt;
}

// neighbours gathered per unrolled round (independent row loads in flight per warp)
template <int NV>
struct Unroll {
  static constexpr int U = NV == 1 ? 8 : (NV == 2 ? 4 : (NV == 4 ? 2 : 1));
};

// lse_i = log sum_{j in N(i) u {i}} exp(e_ij): lane-parallel over the neighbour list (scalars only)
template <typename T>
__device__ __forceinline__ float row_lse(const GatLayer<T>& a, int64_t v, int64_t beg, int64_t end, float tv,
                                         int lane) {
  float m = lane == 0 ? lrelu(tv + a.s[v]) : -INFINITY, l = lane == 0 ? 1.f : 0.f;
  for (int64_t e = beg + lane; e < end; e += 32) {
    const float x = lrelu(tv + a.s[a.col[e]]);
    if (x > m) l = l * expf(m - x) + 1.f, m = x;
    else l += expf(x - m);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), l2 = __shfl_xor_sync(0xffffffffu, l, o);
    const float mm = fmaxf(m, m2);
    l = (m == -INFINITY ? 0.f : l * expf(m - mm)) + (m2 == -INFINITY ? 0.f : l2 * expf(m2 - mm));
    m = mm;
  }
  return m + logf(l);
}

// forward: pass 1 the row's log-sum-exp from the per-node scalars, pass 2 the alpha-weighted
// gather of Z rows, U rows in flight per round
template <typename T, int NV>
__global__ void __launch_bounds__(256) k_gat_fwd(const __grid_constant__ GatGroup<T> Gp) {
  const GatLayer<T>& a = Gp.a[blockIdx.y];
  constexpr int U = Unroll<NV>::U;
  const int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= a.rows) return;
  const int64_t beg = a.row_beg[v], end = a.row_end[v];  // dummy batch rows: beg = end = -1 (self only)
  const float tv = a.t[v];
  const float lse = row_lse(a, v, beg, end, tv, lane);
  float acc[NV][4];
  load_row<T, NV>(a.Z, a.ldz, v, a.w, lane, acc);
  {
    const float a0 = expf(lrelu(tv + a.s[v]) - lse);
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[k][q] *= a0;
  }
  for (int64_t b0 = beg; b0 < end; b0 += 32) {
    const int n = (end - b0) < 32 ? (int)(end - b0) : 32;
    int32_t u = 0;
    float al = 0.f;
    if (lane < n) u = a.col[b0 + lane], al = expf(lrelu(tv + a.s[u]) - lse);
    for (int jj = 0; jj < n; jj += U) {
      float z[U][NV][4], w[U];
#pragma unroll
      for (int r = 0; r < U; ++r) {
        const int src = jj + r < n ? jj + r : jj;
        const int32_t uj = __shfl_sync(0xffffffffu, u, src);
        w[r] = jj + r < n ? __shfl_sync(0xffffffffu, al, src) : 0.f;
        load_row<T, NV>(a.Z, a.ldz, uj, a.w, lane, z[r]);
      }
#pragma unroll
      for (int r = 0; r < U; ++r)
#pragma unroll
        for (int k = 0; k < NV; ++k)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[k][q] += w[r] * z[r][k][q];
    }
  }
  if (lane == 0) a.lse[v] = lse;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int64_t c = (int64_t)k * 128 + lane * 4;
    if (c >= a.w) continue;
    float o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = a.relu ? fmaxf(acc[k][q], 0.f) : acc[k][q];
    if (a.out_f32) st4(a.out_f32 + v * a.ldo + c, o);
    else st4(a.out + v * a.ldo + c, o);
  }
}

// per row i: S_i and dt_i (see the file header); U neighbour rows of Z in flight per round
template <typename T, int NV>
__global__ void __launch_bounds__(256) k_gat_bwd_rows(const __grid_constant__ GatGroup<T> Gp) {
  const GatLayer<T>& a = Gp.a[blockIdx.y];
  constexpr int U = Unroll<NV>::U;
  const int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= a.rows) return;
  const int64_t beg = a.row_beg[v], end = a.row_end[v];
  const float tv = a.t[v], lv = a.lse[v];
  float g[NV][4];
  load_row<T, NV>(a.G, a.ldg, v, a.w, lane, g, a.mask, a.ldm);
  float S = 0.f, Uu = 0.f, V = 0.f;
  auto dot = [&](const float (&z)[NV][4]) {
    float d = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) d += g[k][q] * z[k][q];
    return d;
  };
  {  // self loop
    float z[NV][4];
    load_row<T, NV>(a.Z, a.ldz, v, a.w, lane, z);
    const float d = warp_sum(dot(z));
    const float pre = tv + a.s[v];
    const float al = expf(lrelu(pre) - lv), sl = pre > 0.f ? 1.f : kSlope;
    S += al * d, Uu += al * d * sl, V += al * sl;
  }
  for (int64_t b0 = beg; b0 < end; b0 += 32) {
    const int n = (end - b0) < 32 ? (int)(end - b0) : 32;
    int32_t u = 0;
    float al = 0.f, sl = 0.f;
    if (lane < n) {
      u = a.col[b0 + lane];
      const float pre = tv + a.s[u];
      al = expf(lrelu(pre) - lv);
      sl = pre > 0.f ? 1.f : kSlope;
    }
    for (int jj = 0; jj < n; jj += U) {
      float z[U][NV][4], d[U];
#pragma unroll
      for (int r = 0; r < U; ++r) {
        const int src = jj + r < n ? jj + r : jj;
        load_row<T, NV>(a.Z, a.ldz, __shfl_sync(0xffffffffu, u, src), a.w, lane, z[r]);
      }
#pragma unroll
      for (int r = 0; r < U; ++r) d[r] = dot(z[r]);
#pragma unroll
      for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int r = 0; r < U; ++r) d[r] += __shfl_xor_sync(0xffffffffu, d[r], o);
#pragma unroll
      for (int r = 0; r < U; ++r) {
        const int src = jj + r < n ? jj + r : jj;
        const float alr = jj + r < n ? __shfl_sync(0xffffffffu, al, src) : 0.f;
        const float slr = __shfl_sync(0xffffffffu, sl, src);
        S += alr * d[r], Uu += alr * d[r] * slr, V += alr * slr;
      }
    }
  }
  if (lane == 0) a.Srow[v] = S, a.dt[v] = Uu - S * V;
  if (a.mask) {  // store G_v masked in place (only this warp reads row v here): the column pass
    // then gathers G rows without their masks
    T* gw = const_cast<T*>(a.G) + v * a.ldg;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int64_t c = (int64_t)k * 128 + lane * 4;
      if (c < a.w) st4(gw + c, g[k]);
    }
  }
}

// per row j: dZ_j and ds_j (see the file header); U neighbour rows of G in flight per round
template <typename T, int NV>
__global__ void __launch_bounds__(256) k_gat_bwd_cols(const __grid_constant__ GatGroup<T> Gp) {
  const GatLayer<T>& a = Gp.a[blockIdx.y];
  constexpr int U = Unroll<NV>::U;
  const int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= a.rows) return;
  const int64_t beg = a.row_beg[v], end = a.row_end[v];
  const float sv = a.s[v];
  float z[NV][4], acc[NV][4];
  load_row<T, NV>(a.Z, a.ldz, v, a.w, lane, z);
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[k][q] = 0.f;
  float ds = 0.f;
  auto dot = [&](const float (&g)[NV][4]) {
    float d = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) d += g[k][q] * z[k][q];
    return d;
  };
  {  // self loop
    float g[NV][4];
    load_row<T, NV>(a.G, a.ldg, v, a.w, lane, g);  // masked by the row pass
    const float pre = a.t[v] + sv;
    const float al = expf(lrelu(pre) - a.lse[v]);
    const float d = warp_sum(dot(g));
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[k][q] += al * g[k][q];
    ds += al * (d - a.Srow[v]) * (pre > 0.f ? 1.f : kSlope);
  }
  for (int64_t b0 = beg; b0 < end; b0 += 32) {
    const int n = (end - b0) < 32 ? (int)(end - b0) : 32;
    int32_t u = 0;
    float al = 0.f, sl = 0.f, Su = 0.f;
    if (lane < n) {
      u = a.col[b0 + lane];
      const float pre = a.t[u] + sv;
      al = expf(lrelu(pre) - a.lse[u]);
      sl = pre > 0.f ? 1.f : kSlope;
      Su = a.Srow[u];
    }
    for (int jj = 0; jj < n; jj += U) {
      float g[U][NV][4], d[U];
#pragma unroll
      for (int r = 0; r < U; ++r) {
        const int src = jj + r < n ? jj + r : jj;
        load_row<T, NV>(a.G, a.ldg, __shfl_sync(0xffffffffu, u, src), a.w, lane, g[r]);
      }
#pragma unroll
      for (int r = 0; r < U; ++r) d[r] = dot(g[r]);
#pragma unroll
      for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int r = 0; r < U; ++r) d[r] += __shfl_xor_sync(0xffffffffu, d[r], o);
#pragma unroll
      for (int r = 0; r < U; ++r) {
        const int src = jj + r < n ? jj + r : jj;
        const float alr = jj + r < n ? __shfl_sync(0xffffffffu, al, src) : 0.f;
        const float slr = __shfl_sync(0xffffffffu, sl, src);
        const float Sr = __shfl_sync(0xffffffffu, Su, src);
#pragma unroll
        for (int k = 0; k < NV; ++k)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[k][q] += alr * g[r][k][q];
        ds += alr * (d[r] - Sr) * slr;
      }
    }
  }
  const float dtv = a.dt[v];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int64_t c = (int64_t)k * 128 + lane * 4;
    if (c >= a.w) continue;
    float o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = acc[k][q] + ds * a.a_src[c + q] + dtv * a.a_dst[c + q];
    st4(a.dZ + v * a.ldd + c, o);
  }
  if (lane == 0) a.ds[v] = ds;
}

// d a_src[c] = sum_r ds[r] Z[r, c], d a_dst[c] = sum_r dt[r] Z[r, c], in two deterministic
// phases: k_gat_da_part sums a chunk of rows per CTA (32 columns x 8 row phases, smem-reduced)
// into da_part[chunk][2][w]; k_gat_da_sum adds the chunks in order into the fp32 gradient rows.
template <typename T>
__global__ void __launch_bounds__(256) k_gat_da_part(const __grid_constant__ GatGroup<T> Gp) {
  const GatLayer<T>& a = Gp.a[blockIdx.z];
  __shared__ float sx[8][32], sy[8][32];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + lane;
  const int64_t per = (a.rows + kGatDaChunks - 1) / kGatDaChunks;
  const int64_t r0 = blockIdx.y * per, r1 = r0 + per < a.rows ? r0 + per : a.rows;
  float x = 0.f, y = 0.f;
  if (c < a.w)
    for (int64_t r = r0 + wp; r < r1; r += 8) {
      const float z = Elem<T>::to_f(a.Z[r * a.ldz + c]);
      x += a.ds[r] * z, y += a.dt[r] * z;
    }
  sx[wp][lane] = x, sy[wp][lane] = y;
  __syncthreads();
  if (wp == 0 && c < a.w) {
    float xs = 0.f, ys = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) xs += sx[k][lane], ys += sy[k][lane];
    a.da_part[(int64_t)blockIdx.y * 2 * a.w + c] = xs;
    a.da_part[(int64_t)blockIdx.y * 2 * a.w + a.w + c] = ys;
  }
}
template <typename T>
__global__ void __launch_bounds__(128) k_gat_da_sum(const __grid_constant__ GatGroup<T> Gp) {
  const GatLayer<T>& a = Gp.a[blockIdx.y];
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.w) return;
  float x = 0.f, y = 0.f;
  for (int k = 0; k < kGatDaChunks; ++k) x += a.da_part[(int64_t)k * 2 * a.w + c], y += a.da_part[(int64_t)k * 2 * a.w + a.w + c];
  a.da_src[c] = x;
  a.da_dst[c] = y;
}

}  // namespace

// the attention passes hold a row in registers: output widths up to kGatMaxWidth (gist_create
// refuses wider GAT layers with GIST_E_UNSUPPORTED)
static_assert(kGatMaxWidth == 16 * 128, "GAT_DISPATCH tops out at NV = 16 chunks of 128 columns");
#define GAT_DISPATCH(KERNEL, W, ROWS)                                                            \
  do {                                                                                          \
    if ((ROWS) <= 0 || G.n <= 0) return;                                                        \
    const dim3 grid((unsigned)cdiv((ROWS), 8), (unsigned)G.n);                                  \
    if ((W) <= 128) KERNEL<T, 1><<<grid, 256, 0, s>>>(G);                                       \
    else if ((W) <= 256) KERNEL<T, 2><<<grid, 256, 0, s>>>(G);                                  \
    else if ((W) <= 512) KERNEL<T, 4><<<grid, 256, 0, s>>>(G);                                  \
    else if ((W) <= 1024) KERNEL<T, 8><<<grid, 256, 0, s>>>(G);                                 \
    else KERNEL<T, 16><<<grid, 256, 0, s>>>(G);                                                 \
  } while (0)

template <typename T>
static void group_max(const GatGroup<T>& G, int64_t& w, int64_t& rows, int64_t& kw) {
  w = rows = kw = 0;
  for (int i = 0; i < G.n; ++i) {
    w = std::max(w, G.a[i].w);
    rows = std::max(rows, G.a[i].rows);
    kw = std::max(kw, G.a[i].kw);
  }
}

template <typename T>
void gat_scores(const GatGroup<T>& G, cudaStream_t s) {
  int64_t w, rows, kw;
  group_max(G, w, rows, kw);
  if (G.n <= 0) return;
  if (!G.a[0].H) {
    if (rows > 0) k_gat_scores<T><<<dim3((unsigned)cdiv(rows, 8), (unsigned)G.n), 256, 0, s>>>(G);
    return;
  }
  if (kw > 0) k_gat_wa<T><<<dim3((unsigned)cdiv(kw, 8), (unsigned)G.n), 256, 0, s>>>(G);
  if (rows > 0) k_gat_scores_h<T><<<dim3((unsigned)cdiv(rows, 8), (unsigned)G.n), 256, 0, s>>>(G);
}
template <typename T>
void gat_forward(const GatGroup<T>& G, cudaStream_t s) {
  int64_t w, rows, kw;
  group_max(G, w, rows, kw);
  GAT_DISPATCH(k_gat_fwd, w, rows);
}
template <typename T>
void gat_backward(const GatGroup<T>& G, cudaStream_t s) {
  int64_t w, rows, kw;
  group_max(G, w, rows, kw);
  GAT_DISPATCH(k_gat_bwd_rows, w, rows);
  GAT_DISPATCH(k_gat_bwd_cols, w, rows);
  k_gat_da_part<T><<<dim3((unsigned)cdiv(w, 32), kGatDaChunks, (unsigned)G.n), 256, 0, s>>>(G);
  k_gat_da_sum<T><<<dim3((unsigned)cdiv(w, 128), (unsigned)G.n), 128, 0, s>>>(G);
}
#undef GAT_DISPATCH

// dst[r, :] = src[idx[r], :] (T rows, 16-byte vectors; ld multiples of 8 elements)
template <typename T>
__global__ void k_gather_t(const T* __restrict__ src, int64_t lds, const int32_t* __restrict__ idx, int64_t rows,
                           int64_t vecs, T* __restrict__ dst, int64_t ldd) {
  const int64_t r = blockIdx.y + (int64_t)blockIdx.z * 65535;
  if (r >= rows) return;
  const uint4* s = reinterpret_cast<const uint4*>(src + (int64_t)idx[r] * lds);
  uint4* d = reinterpret_cast<uint4*>(dst + r * ldd);
  for (int64_t i = threadIdx.x; i < vecs; i += blockDim.x) d[i] = s[i];
}
template <typename T>
void gather_rows_t(const T* src, int64_t lds, const int32_t* idx, int64_t rows, int64_t w, T* dst, int64_t ldd,
                   cudaStream_t s) {
  if (rows <= 0) return;
  const int64_t vecs = w / Elem<T>::kVec;
  const dim3 grid(1, (unsigned)std::min<int64_t>(rows, 65535), (unsigned)cdiv(rows, 65535));
  k_gather_t<T><<<grid, 128, 0, s>>>(src, lds, idx, rows, vecs, dst, ldd);
}

// dst[c] = mean over k of srcs[k][c] (sum in slot order, then / n): the last GAT layer's
// shared attention rows at subAgg (R21)
__global__ void k_mean_rows(float* __restrict__ dst, const __grid_constant__ MeanRows m) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m.cols) return;
  const int r = blockIdx.y;
  float acc = 0.f;
  for (int k = 0; k < m.n; ++k) acc += m.src[k][(int64_t)r * m.ld_src[k] + c];
  dst[(int64_t)r * m.ld_dst + c] = acc / (float)m.n;
}
void mean_rows(float* dst, const MeanRows& m, int rows, cudaStream_t s) {
  if (m.n <= 0 || m.cols <= 0 || rows <= 0) return;
  k_mean_rows<<<dim3((unsigned)cdiv(m.cols, 128), (unsigned)rows), 128, 0, s>>>(dst, m);
}

template void gat_scores<float>(const GatGroup<float>&, cudaStream_t);
template void gat_scores<bf16>(const GatGroup<bf16>&, cudaStream_t);
template void gat_forward<float>(const GatGroup<float>&, cudaStream_t);
template void gat_forward<bf16>(const GatGroup<bf16>&, cudaStream_t);
template void gat_backward<float>(const GatGroup<float>&, cudaStream_t);
template void gat_backward<bf16>(const GatGroup<bf16>&, cudaStream_t);
template void gather_rows_t<float>(const float*, int64_t, const int32_t*, int64_t, int64_t, float*, int64_t,
                                   cudaStream_t);
template void gather_rows_t<bf16>(const bf16*, int64_t, const int32_t*, int64_t, int64_t, bf16*, int64_t,
                                  cudaStream_t);

}  // namespace gist
