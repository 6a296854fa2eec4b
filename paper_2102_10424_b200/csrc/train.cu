// train.cu -- softmax cross-entropy (R4), Adam / SGD (R8), evaluation reductions.
// All reductions are single-CTA, fixed-order trees: results are deterministic.
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace gist {

// One warp per batch row.  loss_v = logsumexp(z_v) - z_v[y_v] on train rows;
// dlogits_v = (softmax(z_v) - onehot(y_v)) / n_train on train rows, else 0;
// padding columns [k, ld) are written as 0.
template <typename T>
__global__ void k_softmax_ce(const float* __restrict__ logits, int64_t ld, int nb, int k,
                             const int32_t* __restrict__ lab, const uint8_t* __restrict__ train,
                             const int64_t* __restrict__ stats, T* __restrict__ dlog, float* __restrict__ row_loss) {
  const int v = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (v >= nb) return;
  const float* z = logits + (int64_t)v * ld;
  const int64_t nt = stats[1];
  const bool tr = train[v] && nt > 0;
  float mx = -INFINITY;
  for (int c = lane; c < k; c += 32) mx = fmaxf(mx, z[c]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float se = 0.f;
  for (int c = lane; c < k; c += 32) se += expf(z[c] - mx);
#pragma unroll
  for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
  const float lse = mx + logf(se);
  const int y = lab[v];
  const float inv = tr ? 1.0f / (float)nt : 0.f;
  for (int c = lane; c < ld; c += 32) {
    float g = 0.f;
    if (tr && c < k) g = (expf(z[c] - lse) - (c == y ? 1.f : 0.f)) * inv;
    dlog[(int64_t)v * ld + c] = Elem<T>::from_f(g);
  }
  if (lane == 0) row_loss[v] = tr ? lse - z[y] : 0.f;
}

template <typename T>
void softmax_ce(const float* logits, int64_t ld, int nb, int k, const int32_t* lab, const uint8_t* train,
                const int64_t* stats, T* dlog, float* row_loss, cudaStream_t s) {
  if (nb <= 0) return;
  k_softmax_ce<T><<<(unsigned)cdiv(nb, 8), 256, 0, s>>>(logits, ld, nb, k, lab, train, stats, dlog, row_loss);
}
template void softmax_ce<float>(const float*, int64_t, int, int, const int32_t*, const uint8_t*, const int64_t*,
                                float*, float*, cudaStream_t);
template void softmax_ce<bf16>(const float*, int64_t, int, int, const int32_t*, const uint8_t*, const int64_t*,
                               bf16*, float*, cudaStream_t);

__global__ void __launch_bounds__(1024) k_reduce_loss(const float* __restrict__ row_loss, int nb,
                                                      const int64_t* __restrict__ stats, float* __restrict__ step_loss,
                                                      float* __restrict__ loss_acc) {
  using Red = cub::BlockReduce<float, 1024>;
  __shared__ typename Red::TempStorage tr;
  float acc = 0.f;
  for (int v = threadIdx.x; v < nb; v += 1024) acc += row_loss[v];
  const float tot = Red(tr).Sum(acc);
  if (threadIdx.x == 0) {
    const int64_t nt = stats[1];
    const float l = nt > 0 ? tot / (float)nt : 0.f;
    step_loss[0] = l;
    loss_acc[0] += l;
  }
}
void reduce_loss(const float* row_loss, int nb, const int64_t* stats, float* step_loss, float* loss_acc,
                 cudaStream_t s) {
  k_reduce_loss<<<1, 1024, 0, s>>>(row_loss, nb, stats, step_loss, loss_acc);
}

// Adam, PyTorch form (R8): m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
// w -= (lr / bc1) * m / (sqrt(v) / sqrt(bc2) + eps).  Optionally refreshes the bf16 shadow.
__global__ void k_adam(float* __restrict__ W, const float* __restrict__ G, float* __restrict__ M,
                       float* __restrict__ V, int64_t n, float lr, float b1, float b2, float eps, float bc1,
                       float bc2_sqrt, bf16* __restrict__ Wb) {
  const int64_t n4 = n >> 2;
  const float step = lr / bc1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 w = reinterpret_cast<float4*>(W)[i];
    const float4 g = reinterpret_cast<const float4*>(G)[i];
    float4 m = reinterpret_cast<float4*>(M)[i];
    float4 v = reinterpret_cast<float4*>(V)[i];
    float* wp = &w.x; const float* gp = &g.x; float* mp = &m.x; float* vp = &v.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mp[j] = b1 * mp[j] + (1.f - b1) * gp[j];
      vp[j] = b2 * vp[j] + (1.f - b2) * gp[j] * gp[j];
      const float denom = sqrtf(vp[j]) / bc2_sqrt + eps;
      wp[j] = wp[j] - step * (mp[j] / denom);
    }
    reinterpret_cast<float4*>(W)[i] = w;
    reinterpret_cast<float4*>(M)[i] = m;
    reinterpret_cast<float4*>(V)[i] = v;
    if (Wb) {
      reinterpret_cast<__nv_bfloat162*>(Wb)[2 * i] = __floats2bfloat162_rn(w.x, w.y);
      reinterpret_cast<__nv_bfloat162*>(Wb)[2 * i + 1] = __floats2bfloat162_rn(w.z, w.w);
    }
  }
}
void adam_step(float* W, const float* G, float* M, float* V, int64_t n, float lr, float b1, float b2, float eps,
               float bc1, float bc2_sqrt, bf16* Wb, cudaStream_t s) {
  if (n <= 0) return;
  const int64_t blocks = cdiv(n >> 2, 256) < 148 * 8 ? cdiv(n >> 2, 256) : 148 * 8;
  k_adam<<<(unsigned)(blocks > 0 ? blocks : 1), 256, 0, s>>>(W, G, M, V, n, lr, b1, b2, eps, bc1, bc2_sqrt, Wb);
}

__global__ void k_sgd(float* __restrict__ W, const float* __restrict__ G, int64_t n, float lr, bf16* __restrict__ Wb) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float w = W[i] - lr * G[i];
    W[i] = w;
    if (Wb) Wb[i] = __float2bfloat16_rn(w);
  }
}
void sgd_step(float* W, const float* G, int64_t n, float lr, bf16* Wb, cudaStream_t s) {
  if (n <= 0) return;
  const int64_t blocks = cdiv(n, 256) < 148 * 8 ? cdiv(n, 256) : 148 * 8;
  k_sgd<<<(unsigned)blocks, 256, 0, s>>>(W, G, n, lr, Wb);
}

__global__ void k_f32_to_bf16(const float* __restrict__ src, bf16* __restrict__ dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}
void f32_to_bf16(const float* src, bf16* dst, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  const int64_t blocks = cdiv(n, 256) < 148 * 8 ? cdiv(n, 256) : 148 * 8;
  k_f32_to_bf16<<<(unsigned)blocks, 256, 0, s>>>(src, dst, n);
}

// Evaluation: out3 = {sum CE over rows with split==code, #correct (argmax, ties -> lowest index), #rows}
__global__ void __launch_bounds__(1024) k_eval_rows(const float* __restrict__ logits, int64_t ld, int64_t n, int k,
                                                    const int32_t* __restrict__ labels,
                                                    const uint8_t* __restrict__ split, int code,
                                                    double* __restrict__ out3) {
  using Red = cub::BlockReduce<double, 1024>;
  __shared__ typename Red::TempStorage tr;
  double loss = 0.0, corr = 0.0, cnt = 0.0;
  for (int64_t v = threadIdx.x; v < n; v += 1024) {
    if (split[v] != code) continue;
    const float* z = logits + v * ld;
    float mx = -INFINITY;
    int am = 0;
    for (int c = 0; c < k; ++c)
      if (z[c] > mx) { mx = z[c]; am = c; }
    float se = 0.f;
    for (int c = 0; c < k; ++c) se += expf(z[c] - mx);
    loss += (double)(mx + logf(se) - z[labels[v]]);
    corr += am == labels[v];
    cnt += 1.0;
  }
  double a = Red(tr).Sum(loss);
  __syncthreads();
  double b = Red(tr).Sum(corr);
  __syncthreads();
  double c = Red(tr).Sum(cnt);
  if (threadIdx.x == 0) { out3[0] = a; out3[1] = b; out3[2] = c; }
}
void eval_rows(const float* logits, int64_t ld, int64_t n, int k, const int32_t* labels, const uint8_t* split,
               int code, double* out3, cudaStream_t s) {
  k_eval_rows<<<1, 1024, 0, s>>>(logits, ld, n, k, labels, split, code, out3);
}

}  // namespace gist
