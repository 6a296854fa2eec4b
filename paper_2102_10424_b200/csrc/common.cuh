// common.cuh -- shared device/host helpers of the GIST B200 library (product path).
// Not shared with oracle/ (the oracle carries its own Philox; both are pinned to
// the Random123 known-answer vectors).
#pragma once
#include <mutex>
#include <unordered_map>
#include <utility>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>

#define GIST_HD __host__ __device__ __forceinline__

namespace gist {

// ----------------------------------------------------------------------------
// Philox4x32-10 (Random123).  Used for R5 (partition keys), R7 (batch schedule)
// and R11 (init).  Purpose tags live in counter word 3.
// ----------------------------------------------------------------------------
struct U4 { uint32_t x, y, z, w; };

enum : uint32_t { PURPOSE_PARTITION = 1, PURPOSE_BATCH = 2, PURPOSE_INIT = 3 };

GIST_HD U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c.x;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c.z;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// 64-bit sort key (w1 << 32) | w0 of counter (idx, c1, c2, purpose) under a 64-bit seed.
GIST_HD uint64_t philox_key64(uint32_t idx, uint32_t c1, uint32_t c2, uint32_t purpose, uint64_t seed) {
  U4 o = philox4x32_10(U4{idx, c1, c2, purpose}, (uint32_t)seed, (uint32_t)(seed >> 32));
  return ((uint64_t)o.y << 32) | (uint64_t)o.x;
}

GIST_HD int64_t pad8(int64_t w) { return (w + 7) & ~int64_t(7); }
GIST_HD int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ----------------------------------------------------------------------------
// element type traits: fp32 parity mode / bf16 tensor-core mode (R13)
// ----------------------------------------------------------------------------
template <typename T> struct Elem;
template <> struct Elem<float> {
  static constexpr int kVec = 4;  // 16-byte vectors
  __device__ __forceinline__ static float to_f(float v) { return v; }
  __device__ __forceinline__ static float from_f(float v) { return v; }
};
template <> struct Elem<__nv_bfloat16> {
  static constexpr int kVec = 8;
  __device__ __forceinline__ static float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};

// Load / store kVec elements (16 bytes) as fp32 values.
__device__ __forceinline__ void ld16(const float* p, float* v) {
  float4 a = *reinterpret_cast<const float4*>(p);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
__device__ __forceinline__ void unpack8(const uint4& a, float* v) {  // 8 bf16 -> fp32
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x; v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void ld16(const __nv_bfloat16* p, float* v) {
  uint4 a = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x; v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void st16(float* p, const float* v) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void st16(__nv_bfloat16* p, const float* v) {
  uint4 a;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&a);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = a;
}


// ---- programmatic dependent launch (PDL) ------------------------------------------------
// Every kernel of a subTrain step is launched with programmatic stream serialisation: it may
// be scheduled while its predecessor drains, and calls pdl_wait() (griddepcontrol.wait:
// the predecessor grid has completed and its writes are visible) before its first global
// memory access, then pdl_trigger() so its own successor can be scheduled early (the
// successor still launches only once every CTA of this grid has started).  Both are no-ops
// for a kernel launched without the attribute.  GIST_PDL=0 disables the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies per device: set it once per
// (kernel, device) -- a context on a second device must not launch without it.
inline void ensure_smem(const void* kern, int bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, uint64_t> done;  // kernel -> bitmask of devices
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  std::lock_guard<std::mutex> lk(mu);
  uint64_t& m = done[kern];
  if (!(m & bit)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    m |= bit;
  }
}
// SM count of the current device (cached per device)
inline int device_sms() {
  static int n[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int& v = n[dev & 63];
  if (!v) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}
template <typename... P, typename... A>
inline void launch_pdl(void (*kern)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}

}  // namespace gist
