// Launch-latency floor of a dependent kernel chain on B200: N kernels in one CUDA graph, each
// waiting on its predecessor (griddepcontrol.wait), with and without programmatic dependent
// launch, for small / full-grid / big-smem kernels.  Prints us per kernel.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_small(int* p, int work) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  int v = p[blockIdx.x * blockDim.x + threadIdx.x];
  for (int i = 0; i < work; ++i) v = v * 3 + 1;
  p[blockIdx.x * blockDim.x + threadIdx.x] = v;
}
__global__ void k_smem(int* p, int work) {
  extern __shared__ int sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  int v = p[blockIdx.x * blockDim.x + threadIdx.x] + sm[(threadIdx.x + 1) % blockDim.x];
  for (int i = 0; i < work; ++i) v = v * 3 + 1;
  p[blockIdx.x * blockDim.x + threadIdx.x] = v;
}

template <typename K>
float run(K kern, int grid, int block, int smem, bool pdl, int n, int work, int* buf) {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < n; ++i) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, buf, work);
  }
  cudaStreamEndCapture(s, &g);
  cudaGraphExec_t ge;
  cudaGraphInstantiate(&ge, g, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
  cudaEventRecord(a, s);
  const int R = 20;
  for (int r = 0; r < R; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge); cudaGraphDestroy(g); cudaStreamDestroy(s);
  return ms * 1e3f / (R * n);
}

int main() {
  int* buf;
  cudaMalloc(&buf, 148 * 1024 * 4 * 8);
  cudaMemset(buf, 0, 148 * 1024 * 4 * 8);
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int n = 64;
  for (int pdl = 0; pdl < 2; ++pdl) {
    printf("pdl=%d small 1x32        %.2f us/kernel\n", pdl, run(k_small, 1, 32, 0, pdl, n, 0, buf));
    printf("pdl=%d small 148x256     %.2f us/kernel\n", pdl, run(k_small, 148, 256, 0, pdl, n, 0, buf));
    printf("pdl=%d small 592x256     %.2f us/kernel\n", pdl, run(k_small, 592, 256, 0, pdl, n, 0, buf));
    printf("pdl=%d smem200K 148x320  %.2f us/kernel\n", pdl, run(k_smem, 148, 320, 200 * 1024, pdl, n, 0, buf));
    printf("pdl=%d smem100K 148x320  %.2f us/kernel\n", pdl, run(k_smem, 148, 320, 100 * 1024, pdl, n, 0, buf));
    printf("pdl=%d smem200K 148x320 work2000 %.2f us/kernel\n", pdl, run(k_smem, 148, 320, 200 * 1024, pdl, n, 2000, buf));
    printf("pdl=%d small 148x256 work2000    %.2f us/kernel\n", pdl, run(k_small, 148, 256, 0, pdl, n, 2000, buf));
  }
  return 0;
}
