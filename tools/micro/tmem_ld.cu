// TMEM -> register load cost on B200 (the epilogue of the tcgen05 GEMMs): W warps of one CTA per
// SM (warp w reads TMEM lane quarter w % 4) each issue R rounds of tcgen05.ld.32x32b.x{32,128}
// (+ tcgen05.wait::ld), optionally followed by 32 shared-memory stores per 32 columns (the
// epilogue's staging).  Prints cycles per round and per 32 columns, median over CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_ld tools/micro/tmem_ld.cu && /tmp/tmem_ld
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>

template <int X, bool STS>
__global__ void k_tmem(unsigned long long* out, int rounds, float* sink) {
  __shared__ uint32_t slot;
  __shared__ float stg[10][32 * 33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16);
  float acc = 0.f;
  const unsigned long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    const uint32_t col = (uint32_t)((r * X) % 512);
    uint32_t v[X];
    if constexpr (X == 32) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(tmem + col));
    } else {  // four x32 loads back to back, one wait
#pragma unroll
      for (int q = 0; q < X / 32; ++q)
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[32 * q + 0]), "=r"(v[32 * q + 1]), "=r"(v[32 * q + 2]), "=r"(v[32 * q + 3]), "=r"(v[32 * q + 4]),
              "=r"(v[32 * q + 5]), "=r"(v[32 * q + 6]), "=r"(v[32 * q + 7]), "=r"(v[32 * q + 8]), "=r"(v[32 * q + 9]),
              "=r"(v[32 * q + 10]), "=r"(v[32 * q + 11]), "=r"(v[32 * q + 12]), "=r"(v[32 * q + 13]),
              "=r"(v[32 * q + 14]), "=r"(v[32 * q + 15]), "=r"(v[32 * q + 16]), "=r"(v[32 * q + 17]),
              "=r"(v[32 * q + 18]), "=r"(v[32 * q + 19]), "=r"(v[32 * q + 20]), "=r"(v[32 * q + 21]),
              "=r"(v[32 * q + 22]), "=r"(v[32 * q + 23]), "=r"(v[32 * q + 24]), "=r"(v[32 * q + 25]),
              "=r"(v[32 * q + 26]), "=r"(v[32 * q + 27]), "=r"(v[32 * q + 28]), "=r"(v[32 * q + 29]),
              "=r"(v[32 * q + 30]), "=r"(v[32 * q + 31])
            : "r"(tmem + ((col + 32 * q) % 512)));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (STS) {
#pragma unroll
      for (int i = 0; i < X; ++i) stg[warp][(i % 32) * 33 + lane] = __uint_as_float(v[i]);
      __syncwarp();
      acc += stg[warp][lane * 33 + (r & 31)];
      __syncwarp();
    } else {
#pragma unroll
      for (int i = 0; i < X; ++i) acc += __uint_as_float(v[i]);
    }
  }
  const unsigned long long t1 = clock64();
  if (lane == 0 && blockIdx.x < 1024) out[blockIdx.x * 16 + warp] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int X, bool STS>
void run(int warps, int rounds, unsigned long long* d_out, float* sink) {
  k_tmem<X, STS><<<148, 32 * warps>>>(d_out, rounds, sink);
  cudaDeviceSynchronize();
  k_tmem<X, STS><<<148, 32 * warps>>>(d_out, rounds, sink);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<unsigned long long> h(148 * 16);
  cudaMemcpy(h.data(), d_out, h.size() * 8, cudaMemcpyDeviceToHost);
  std::vector<unsigned long long> w;
  for (int b = 0; b < 148; ++b)
    for (int k = 0; k < warps; ++k) w.push_back(h[b * 16 + k]);
  std::sort(w.begin(), w.end());
  const double med = (double)w[w.size() / 2];
  printf("{\"x\": %d, \"sts\": %d, \"warps\": %d, \"rounds\": %d, \"cyc_per_round\": %.1f, \"cyc_per_32col\": %.1f, \"err\": \"%s\"}\n",
         X, STS ? 1 : 0, warps, rounds, med / rounds, med / rounds / (X / 32), cudaGetErrorString(e));
}

int main() {
  unsigned long long* d_out;
  float* sink;
  cudaMalloc(&d_out, 148 * 16 * 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  for (int warps : {1, 4, 8}) {
    run<32, false>(warps, 256, d_out, sink);
    run<128, false>(warps, 64, d_out, sink);
    run<32, true>(warps, 256, d_out, sink);
  }
  return 0;
}
