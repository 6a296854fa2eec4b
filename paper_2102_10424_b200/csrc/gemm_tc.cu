// gemm_tc.cu -- BF16 tcgen05 tensor-core GEMM (placeholder until the sm_100a
// kernel lands; returning false makes BF16 mode report GIST_E_UNSUPPORTED
// instead of silently using another path).
#include "common.cuh"
#include "kernels.h"

namespace gist {

bool gemm_bf16(bool, bool, int64_t, int64_t, int64_t, const bf16*, int64_t, const bf16*, int64_t, void*, int64_t,
               bool, bool, cudaStream_t) {
  return false;
}

}  // namespace gist
