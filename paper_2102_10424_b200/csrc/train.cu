// train.cu -- softmax cross-entropy (R4), Adam / SGD (R8), evaluation reductions.
// All reductions are single-CTA, fixed-order trees: results are deterministic.
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace gist {

// One warp per batch row (grid.y = slot).  loss_v = logsumexp(z_v) - z_v[y_v] on train
// rows; dlogits_v = (softmax(z_v) - onehot(y_v)) / n_train on train rows, else 0;
// padding columns [k, ld) are written as 0.  The last CTA of each slot to finish sums the
// row losses in a fixed order (deterministic) into step_loss / loss_acc.
template <typename T>
__global__ void __launch_bounds__(256) k_softmax_ce(const __grid_constant__ CeGroup<T> G) {
  pdl_wait();
  pdl_trigger();
  const CeSlot<T>& S = G.s[blockIdx.y];
  // 8 lanes per row (4 rows per warp): the class count is small (7..47), so a full warp per
  // row left most lanes idle and made the launch instruction-bound
  constexpr int LPR = 8;
  const int gl = threadIdx.x & (LPR - 1);
  const unsigned gmask = ((1u << LPR) - 1u) << ((threadIdx.x & 31) - gl);  // this row's lanes
  const int v = (blockIdx.x * blockDim.x + threadIdx.x) / LPR;
  const int64_t nt = S.stats[1];
  float my_loss = 0.f;  // this row's CE (lane 0 of the row's group)
  if (v < G.rows) {
    const int64_t ld = G.ld;
    const int k = G.k;
    float* zw = S.logits + (int64_t)v * ld;
    if (S.add) {  // logits = partial logits + add (fp32), stored: every later reader sees the sum
      const T* ap = S.add + (int64_t)v * ld;
      for (int c = gl; c < ld; c += LPR) zw[c] = zw[c] + Elem<T>::to_f(ap[c]);
      __syncwarp(gmask);
    }
    const float* z = zw;
    const bool tr = S.train[v] && nt > 0;
    float mx = -INFINITY;
    for (int c = gl; c < k; c += LPR) mx = fmaxf(mx, z[c]);
#pragma unroll
    for (int o = LPR / 2; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(gmask, mx, o, LPR));
    float se = 0.f;
    for (int c = gl; c < k; c += LPR) se += expf(z[c] - mx);
#pragma unroll
    for (int o = LPR / 2; o; o >>= 1) se += __shfl_xor_sync(gmask, se, o, LPR);
    const float lse = mx + logf(se);
    const int y = S.lab[v];
    const float inv = tr ? 1.0f / (float)nt : 0.f;
    const int64_t ldd = G.ld_dlog ? G.ld_dlog : ld;
    const float sv = S.dlog_s ? S.scale_s[v] : 0.f;
    for (int c = gl; c < ld; c += LPR) {
      float g = 0.f;
      if (tr && c < k) g = (expf(z[c] - lse) - (c == y ? 1.f : 0.f)) * inv;
      S.dlog[(int64_t)v * ldd + c] = Elem<T>::from_f(g);
      if (S.dlog_s) S.dlog_s[(int64_t)v * ldd + c] = Elem<T>::from_f(g * sv);
    }
    if (gl == 0 && tr) my_loss = lse - z[y];
  }
  // per-CTA partial sums (fixed order), then the last CTA of the slot adds the gridDim.x partials
  using Red = cub::BlockReduce<float, 256>;
  __shared__ typename Red::TempStorage tr;
  const float part = Red(tr).Sum(my_loss);
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    S.row_loss[blockIdx.x] = part;
    __threadfence();
    s_last = atomicAdd(S.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  float acc = 0.f;
  for (int r = threadIdx.x; r < (int)gridDim.x; r += blockDim.x) acc += __ldcg(S.row_loss + r);
  const float tot = Red(tr).Sum(acc);
  if (threadIdx.x == 0) {
    const float l = nt > 0 ? tot / (float)nt : 0.f;
    S.step_loss[0] = l;
    S.loss_acc[0] += l;
    *S.done = 0;
  }
}

template <typename T>
void softmax_ce(const CeGroup<T>& G, cudaStream_t s) {
  if (G.rows <= 0 || G.n <= 0) return;
  launch_pdl(k_softmax_ce<T>, dim3((unsigned)cdiv(G.rows, 32), (unsigned)G.n), 256, 0, s, G);
}
template void softmax_ce<float>(const CeGroup<float>&, cudaStream_t);
template void softmax_ce<bf16>(const CeGroup<bf16>&, cudaStream_t);


// Called by every CTA of an optimizer launch after its last read of *st: the last CTA to
// finish advances the step state for the next step (replaces a separate 1-thread launch).
__device__ __forceinline__ void advance_if_last(StepState* st) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&st->done, 1u);
    if (prev == gridDim.x - 1) {
      st->z += 1;
      st->t += 1;
      st->done = 0;
      __threadfence();
    }
  }
}

// Adam, PyTorch form (R8): m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
// w -= (lr / bc1) * m / (sqrt(v) / sqrt(bc2) + eps), bc_i = 1 - b_i^t, t from the device
// step state (so the launch is identical every step).  Optionally refreshes the bf16 shadow.
__global__ void k_adam(float* __restrict__ W, const float* __restrict__ G, float* __restrict__ M,
                       float* __restrict__ V, int64_t n, float b1, float b2, float eps, StepState* st,
                       bf16* __restrict__ Wb) {
  pdl_wait();
  pdl_trigger();
  __shared__ float s_step, s_bc2;
  if (threadIdx.x == 0) {
    const double t = (double)(st->t + 1);
    s_step = st->lr / (float)(1.0 - pow((double)b1, t));
    s_bc2 = sqrtf((float)(1.0 - pow((double)b2, t)));
  }
  __syncthreads();
  const float step = s_step, bc2_sqrt = s_bc2;
  const int64_t n4 = n >> 2;
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
  advance_if_last(st);
}
void adam_step(float* W, const float* G, float* M, float* V, int64_t n, float b1, float b2, float eps,
               StepState* st, bf16* Wb, cudaStream_t s) {
  if (n <= 0) return;
  const int64_t blocks = cdiv(n >> 2, 256) < 148 * 8 ? cdiv(n >> 2, 256) : 148 * 8;
  launch_pdl(k_adam, (unsigned)(blocks > 0 ? blocks : 1), 256, 0, s, W, G, M, V, n, b1, b2, eps, st, Wb);
}

__global__ void k_sgd(float* __restrict__ W, const float* __restrict__ G, int64_t n, StepState* st,
                      bf16* __restrict__ Wb) {
  pdl_wait();
  pdl_trigger();
  const float lr = st->lr;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float w = W[i] - lr * G[i];
    W[i] = w;
    if (Wb) Wb[i] = __float2bfloat16_rn(w);
  }
  advance_if_last(st);
}
// per-layer optimizer over a group's slots (OptRanges): identical element arithmetic to k_adam /
// k_sgd, so the update does not depend on whether it runs per layer or in one pass
__global__ void k_adam_ranges(const __grid_constant__ OptRanges R, float b1, float b2, float eps,
                              const StepState* st) {
  pdl_wait();
  pdl_trigger();
  const int z = blockIdx.y;
  __shared__ float s_step, s_bc2;
  if (threadIdx.x == 0) {
    const double t = (double)(st->t + 1);
    s_step = st->lr / (float)(1.0 - pow((double)b1, t));
    s_bc2 = sqrtf((float)(1.0 - pow((double)b2, t)));
  }
  __syncthreads();
  const float step = s_step, bc2_sqrt = s_bc2;
  float* __restrict__ W = R.W[z];
  const float* __restrict__ G = R.G[z];
  float* __restrict__ M = R.M[z];
  float* __restrict__ V = R.V[z];
  bf16* __restrict__ Wb = R.Wb[z];
  const int64_t n4 = R.n[z] >> 2;
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
__global__ void k_sgd_ranges(const __grid_constant__ OptRanges R, const StepState* st) {
  pdl_wait();
  pdl_trigger();
  const int z = blockIdx.y;
  const float lr = st->lr;
  float* __restrict__ W = R.W[z];
  const float* __restrict__ G = R.G[z];
  bf16* __restrict__ Wb = R.Wb[z];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < R.n[z]; i += (int64_t)gridDim.x * blockDim.x) {
    const float w = W[i] - lr * G[i];
    W[i] = w;
    if (Wb) Wb[i] = __float2bfloat16_rn(w);
  }
}
static unsigned ranges_blocks(const OptRanges& R, int per) {
  int64_t mx = 0;
  for (int j = 0; j < R.count; ++j) mx = R.n[j] > mx ? R.n[j] : mx;
  const int64_t b = cdiv(mx / per, 256);
  const int64_t cap = (int64_t)148 * 8 / (R.count > 0 ? R.count : 1);
  return (unsigned)(b < 1 ? 1 : (b < cap ? b : (cap < 1 ? 1 : cap)));
}
void adam_ranges(const OptRanges& R, float b1, float b2, float eps, const StepState* st, cudaStream_t s) {
  if (R.count <= 0) return;
  launch_pdl(k_adam_ranges, dim3(ranges_blocks(R, 4), (unsigned)R.count), 256, 0, s, R, b1, b2, eps, st);
}
void sgd_ranges(const OptRanges& R, const StepState* st, cudaStream_t s) {
  if (R.count <= 0) return;
  launch_pdl(k_sgd_ranges, dim3(ranges_blocks(R, 1), (unsigned)R.count), 256, 0, s, R, st);
}
// the step state's advance once every layer's optimizer has run (per-layer mode)
__global__ void k_step_advance(StepState* st) {
  pdl_wait();
  pdl_trigger();
  st->z += 1;
  st->t += 1;
}
void step_advance(StepState* st, cudaStream_t s) { launch_pdl(k_step_advance, 1, 1, 0, s, st); }

void sgd_step(float* W, const float* G, int64_t n, StepState* st, bf16* Wb, cudaStream_t s) {
  if (n <= 0) return;
  const int64_t blocks = cdiv(n, 256) < 148 * 8 ? cdiv(n, 256) : 148 * 8;
  launch_pdl(k_sgd, (unsigned)blocks, 256, 0, s, W, G, n, st, Wb);
}


__global__ void k_relayout_last(const __grid_constant__ RelayoutGroup G) {
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.y;
  const int half = G.half[j], Np = G.Np, w2 = 2 * Np;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)half * w2) return;
  const int r = (int)(idx / w2), c2 = (int)(idx - (int64_t)r * w2);
  const int srow = c2 < Np ? r : half + r, c = c2 < Np ? c2 : c2 - Np;
  G.dst[j][idx] = G.src[j][(int64_t)srow * Np + c];
}
void relayout_last(const RelayoutGroup& G, cudaStream_t s) {
  if (G.n <= 0 || G.max_half <= 0) return;
  launch_pdl(k_relayout_last, dim3((unsigned)cdiv((int64_t)G.max_half * 2 * G.Np, 256), (unsigned)G.n), 256, 0, s, G);
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

__global__ void k_scale_prefix(const float* __restrict__ src, float* __restrict__ dst, int64_t n, int64_t ns, float s) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = i < ns ? src[i] * s : src[i];
}
void scale_prefix_f32(const float* src, float* dst, int64_t n, int64_t n_scaled, float s, cudaStream_t st) {
  if (n <= 0) return;
  const int64_t blocks = cdiv(n, 256) < 148 * 8 ? cdiv(n, 256) : 148 * 8;
  k_scale_prefix<<<(unsigned)blocks, 256, 0, st>>>(src, dst, n, n_scaled, s);
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

__global__ void __launch_bounds__(256) k_eval_parts(const float* __restrict__ logits, int64_t ld, int k,
                                                    const int64_t* __restrict__ pbeg, int64_t k0,
                                                    const int32_t* __restrict__ pnode,
                                                    const int32_t* __restrict__ labels,
                                                    const uint8_t* __restrict__ split, int code,
                                                    double* __restrict__ out3) {
  using Red = cub::BlockReduce<double, 256>;
  __shared__ typename Red::TempStorage tr;
  const int p = blockIdx.x;
  double loss = 0.0, corr = 0.0, cnt = 0.0;
  for (int64_t r = pbeg[p] + threadIdx.x; r < pbeg[p + 1]; r += 256) {
    const int32_t v = pnode[r];
    if (split[v] != code) continue;
    const float* z = logits + (r - k0) * ld;
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
  if (threadIdx.x == 0) { out3[3 * p] = a; out3[3 * p + 1] = b; out3[3 * p + 2] = c; }
}
void eval_parts(const float* logits, int64_t ld, int k, const int64_t* pbeg, int64_t k0, int nparts,
                const int32_t* pnode, const int32_t* labels, const uint8_t* split, int code, double* out3,
                cudaStream_t s) {
  if (nparts <= 0) return;
  k_eval_parts<<<nparts, 256, 0, s>>>(logits, ld, k, pbeg, k0, pnode, labels, split, code, out3);
}

}  // namespace gist
