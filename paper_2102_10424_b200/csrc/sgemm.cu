// sgemm.cu -- FP32-parity dense contraction: C = op(A) op(B) with
// FFMA tiles (128 x 128 x 8 per CTA, 8 x 8 per thread, double-buffered shared
// memory with register prefetch).  Used in GIST_PREC_FP32 mode, where the
// north_star's 1e-4 activation tolerance rules out single-pass TF32/BF16.
// The three operand layouts of the step (Z = C W, dC = dZ W^T, dW = C^T dZ)
// are the (transA, transB) = (0,0), (0,1), (1,0) instantiations.
#include "common.cuh"
#include "kernels.h"

namespace gist {

namespace {
constexpr int BM = 128, BN = 128, BK = 8, PAD = 4;

template <bool TA, bool TB, bool RELU, bool MASK>
__global__ void __launch_bounds__(256) k_sgemm(const __grid_constant__ SgemmGroup G) {
  pdl_wait();
  pdl_trigger();
  const GemmOp& op = G.op[blockIdx.z];  // one sub-GCN slot per grid layer
  const int M = (int)op.M, N = (int)op.N, K = (int)op.K;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= M || n0 >= N) return;
  const float* __restrict__ A = (const float*)op.A;
  const float* __restrict__ B = (const float*)op.B;
  float* __restrict__ C = (float*)op.C;
  const int64_t lda = op.lda, ldb = op.ldb, ldc = op.ldc;
  __shared__ __align__(16) float As[2][BK][BM + PAD];
  __shared__ __align__(16) float Bs[2][BK][BN + PAD];
  const int t = threadIdx.x;
  const int ty = t >> 4, tx = t & 15;

  // per-thread load coordinates
  int am, ak, bk, bn;  // base coordinates of this thread's 4 elements
  if (!TA) { am = t >> 1; ak = (t & 1) * 4; } else { ak = t >> 5; am = (t & 31) * 4; }
  if (!TB) { bk = t >> 5; bn = (t & 31) * 4; } else { bn = t >> 1; bk = (t & 1) * 4; }

  float ra[4], rb[4];
  auto load_tiles = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int m = m0 + am + (TA ? i : 0), k = k0 + ak + (TA ? 0 : i);
      ra[i] = (m < M && k < K) ? (TA ? A[(int64_t)k * lda + m] : A[(int64_t)m * lda + k]) : 0.f;
      int n = n0 + bn + (TB ? 0 : i), kb = k0 + bk + (TB ? i : 0);
      rb[i] = (n < N && kb < K) ? (TB ? B[(int64_t)n * ldb + kb] : B[(int64_t)kb * ldb + n]) : 0.f;
    }
  };
  auto store_tiles = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (!TA) As[buf][ak + i][am] = ra[i]; else As[buf][ak][am + i] = ra[i];
      if (!TB) Bs[buf][bk][bn + i] = rb[i]; else Bs[buf][bk + i][bn] = rb[i];
    }
  };

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  const int nk = (K + BK - 1) / BK;
  load_tiles(0);
  store_tiles(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load_tiles((kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[8], b[8];
      float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
      float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w; a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w; b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (kt + 1 < nk) store_tiles(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (n >= N) continue;
      float v = acc[i][j];
      if (RELU) v = fmaxf(v, 0.f);
      if (MASK && !(((const float*)op.mask)[(int64_t)m * op.ldm + n] > 0.f)) v = 0.f;  // ReLU'(0) = 0 (R3)
      C[(int64_t)m * ldc + n] = v;
    }
  }
}

template <bool TA, bool TB>
void launch(const SgemmGroup& g, int64_t maxM, int64_t maxN, cudaStream_t s) {
  dim3 grid((unsigned)cdiv(maxN, BN), (unsigned)cdiv(maxM, BM), (unsigned)g.n);
  const bool relu = g.op[0].relu, mask = g.op[0].mask != nullptr;
  if (relu && mask) launch_pdl(k_sgemm<TA, TB, true, true>, grid, 256, 0, s, g);
  else if (relu) launch_pdl(k_sgemm<TA, TB, true, false>, grid, 256, 0, s, g);
  else if (mask) launch_pdl(k_sgemm<TA, TB, false, true>, grid, 256, 0, s, g);
  else launch_pdl(k_sgemm<TA, TB, false, false>, grid, 256, 0, s, g);
}
}  // namespace

void gemm_f32_group(const SgemmGroup& g, cudaStream_t s) {
  int64_t maxM = 0, maxN = 0;
  for (int i = 0; i < g.n; ++i) {
    maxM = g.op[i].M > maxM ? g.op[i].M : maxM;
    maxN = g.op[i].N > maxN ? g.op[i].N : maxN;
  }
  if (g.n <= 0 || maxM <= 0 || maxN <= 0) return;
  const bool ta = g.op[0].transA, tb = g.op[0].transB;
  if (!ta && !tb) launch<false, false>(g, maxM, maxN, s);
  else if (!ta && tb) launch<false, true>(g, maxM, maxN, s);
  else if (ta && !tb) launch<true, false>(g, maxM, maxN, s);
  else launch<true, true>(g, maxM, maxN, s);
}

void gemm_f32(bool transA, bool transB, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
              const float* B, int64_t ldb, float* C, int64_t ldc, bool relu, cudaStream_t s) {
  SgemmGroup g;
  g.op[0] = GemmOp{transA, transB, M, N, K, A, lda, B, ldb, C, ldc, true, relu, nullptr, 0, nullptr, 0};
  g.n = 1;
  gemm_f32_group(g, s);
}

}  // namespace gist
