// gemm_tc.cu -- BF16 dense contraction on the 5th-generation tensor cores (sm_100a):
// TMA (cp.async.bulk.tensor, 128-byte swizzle) -> shared-memory ring of STAGES
// -> tcgen05.mma.cta_group::1.kind::f16 (one elected thread) -> fp32 accumulator
// in TMEM -> tcgen05.ld epilogue (ReLU, bf16/fp32 convert) -> global.
//
// The three GEMMs of a GIST step use the operand majorness directly from the
// row-major activations/weights (no transposes are ever materialised):
//   forward  Z  = C  W     A = C  [M x K]  K-major   B = W  [K x N] stored K x N: MN-major
//   input    dC = dZ W^T   A = dZ [M x K]  K-major   B = W  stored N x K:        K-major
//   weight   dW = C^T dZ   A = C  stored K x M: MN-major, B = dZ stored K x N:  MN-major
// Warp roles (128 threads): warp 0 = TMA producer, warp 1 = MMA issuer,
// warp 2 = TMEM allocator; all 4 warps run the epilogue (warp w owns TMEM lanes
// 32w..32w+31 = tile rows).  One output tile (128 x BN) per CTA.
#include <cuda.h>

#include <cstring>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace gist {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 bytes: one SWIZZLE_128B row

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra.uni WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
// UMMA shared-memory descriptor: start, LBO, SBO in 16-byte units; version 1 (sm_100); SWIZZLE_128B.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <int BN>
struct Cfg {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int A_BYTES = BM * BK * 2;  // 16 KB
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
};

template <int BN, bool A_MN, bool B_MN, bool OUT_F32, bool RELU, bool MASK>
__global__ void __launch_bounds__(128, 1) k_gemm_tc(const __grid_constant__ GemmGroupTC G) {
  using CF = Cfg<BN>;
  const GemmSlotTC& S = G.s[blockIdx.z];  // one sub-GCN slot per grid layer
  const int M = S.M, N = S.N, K = S.K;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= M || n0 >= N) return;         // slots may be smaller than the grid (uniform exit)
  const CUtensorMap* mapA = &S.ma;
  const CUtensorMap* mapB = &S.mb;
  void* Cout = S.C;
  const int64_t ldc = S.ldc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + CF::STAGES * CF::STAGE_BYTES);
  uint64_t* empty = full + CF::STAGES;
  uint64_t* accf = empty + CF::STAGES;
  uint32_t* tmem_slot = (uint32_t*)(accf + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < CF::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(mapA);
    prefetch_map(mapB);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(CF::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------ TMA producer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % CF::STAGES;
      const uint32_t ph = (uint32_t)(kb / CF::STAGES) & 1u;
      mbar_wait(&empty[s], ph ^ 1u);
      uint8_t* sa = smem + s * CF::STAGE_BYTES;
      uint8_t* sb = sa + CF::A_BYTES;
      mbar_arrive_expect_tx(&full[s], CF::STAGE_BYTES);
      const int k0 = kb * BK;
      if (!A_MN) {
        tma_load_2d(sa, mapA, &full[s], k0, m0);
      } else {
#pragma unroll
        for (int j = 0; j < BM / 64; ++j) tma_load_2d(sa + j * 8192, mapA, &full[s], m0 + 64 * j, k0);
      }
      if (!B_MN) {
        tma_load_2d(sb, mapB, &full[s], k0, n0);
      } else {
#pragma unroll
        for (int j = 0; j < BN / 64; ++j) tma_load_2d(sb + j * 8192, mapB, &full[s], n0 + 64 * j, k0);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) |
                               ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % CF::STAGES;
      const uint32_t ph = (uint32_t)(kb / CF::STAGES) & 1u;
      mbar_wait(&full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sa = smem_u32(smem + s * CF::STAGE_BYTES);
      const uint32_t sb = sa + CF::A_BYTES;
#pragma unroll
      for (int k = 0; k < BK / 16; ++k) {
        // K-major: advance 16 elements = 32 bytes inside the swizzled row; MN-major: 16 K-rows = 2048 bytes
        const uint64_t ad = A_MN ? make_desc(sa + k * 2048, 8192, 1024) : make_desc(sa + k * 32, 16, 1024);
        const uint64_t bd = B_MN ? make_desc(sb + k * 2048, 8192, 1024) : make_desc(sb + k * 32, 16, 1024);
        umma_bf16(tmem, ad, bd, idesc, (kb | k) != 0);
      }
      umma_commit(&empty[s]);  // frees the smem stage when these MMAs have read it
    }
    umma_commit(accf);  // accumulator complete
  }
  __syncwarp();
  // ------------------------------------------------------------ epilogue (all 4 warps)
  mbar_wait(accf, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = m0 + warp * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
  for (int c = 0; c < BN; c += 16) {
    float v[16];
    tmem_ld16(trow + c, v);
    if (row < M && n0 + c < N) {
      if (RELU) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
      }
      const int col = n0 + c;
      if (MASK) {  // ReLU'(0) = 0 of the layer below (R3): out = acc * 1[mask > 0]
        const bf16* mp = (const bf16*)S.mask + (int64_t)row * S.ldm + col;
        for (int i = 0; i < 16; ++i)
          if (col + i < N && !(__bfloat162float(mp[i]) > 0.f)) v[i] = 0.f;
      }
      if (OUT_F32) {
        float* dst = (float*)Cout + (int64_t)row * ldc + col;
        if (col + 16 <= N && (((uintptr_t)dst & 15) == 0)) {
#pragma unroll
          for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        } else {
          for (int i = 0; i < 16 && col + i < N; ++i) dst[i] = v[i];
        }
      } else {
        bf16* dst = (bf16*)Cout + (int64_t)row * ldc + col;
        if (col + 16 <= N && (((uintptr_t)dst & 15) == 0)) {
          st16(dst, v);
          st16(dst + 8, v + 8);
        } else {
          for (int i = 0; i < 16 && col + i < N; ++i) dst[i] = __float2bfloat16_rn(v[i]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CF::TMEM_COLS));
  }
}

// ------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeFn)p;
  });
  return fn;
}

// 2D bf16 tensor map: inner dim `inner` (contiguous), outer dim `outer`, row stride ld elements
bool make_map(CUtensorMap* map, const void* base, int64_t inner, int64_t outer, int64_t ld, int box_inner,
              int box_outer) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, bool A_MN, bool B_MN, bool OUT_F32, bool RELU, bool MASK>
void launch_tc(const GemmPlanTC& P, cudaStream_t s) {
  auto kern = k_gemm_tc<BN, A_MN, B_MN, OUT_F32, RELU, MASK>;
  static bool attr = false;  // per instantiation
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM);
    attr = true;
  }
  dim3 grid((unsigned)cdiv(P.maxN, BN), (unsigned)cdiv(P.maxM, BM), (unsigned)P.G.n);
  kern<<<grid, 128, Cfg<BN>::SMEM, s>>>(P.G);
}

template <int BN, bool A_MN, bool B_MN>
void dispatch_epi(const GemmPlanTC& P, cudaStream_t s) {
  const int e = (P.out_f32 ? 4 : 0) | (P.relu ? 2 : 0) | (P.mask ? 1 : 0);
  switch (e) {
    case 0: launch_tc<BN, A_MN, B_MN, false, false, false>(P, s); break;
    case 1: launch_tc<BN, A_MN, B_MN, false, false, true>(P, s); break;
    case 2: launch_tc<BN, A_MN, B_MN, false, true, false>(P, s); break;
    case 3: launch_tc<BN, A_MN, B_MN, false, true, true>(P, s); break;
    case 4: launch_tc<BN, A_MN, B_MN, true, false, false>(P, s); break;
    case 5: launch_tc<BN, A_MN, B_MN, true, false, true>(P, s); break;
    case 6: launch_tc<BN, A_MN, B_MN, true, true, false>(P, s); break;
    default: launch_tc<BN, A_MN, B_MN, true, true, true>(P, s); break;
  }
}

template <int BNV>
void dispatch_layout(const GemmPlanTC& P, cudaStream_t s) {
  if (!P.a_mn && P.b_mn) dispatch_epi<BNV, false, true>(P, s);
  else if (!P.a_mn && !P.b_mn) dispatch_epi<BNV, false, false>(P, s);
  else if (P.a_mn && P.b_mn) dispatch_epi<BNV, true, true>(P, s);
  else dispatch_epi<BNV, true, false>(P, s);
}

}  // namespace

bool gemm_bf16_prepare(const GemmOp* ops, int n, GemmPlanTC* P) {
  if (!get_encode() || n < 1 || n > kMaxGroup) return false;
  const GemmOp& o0 = ops[0];
  P->a_mn = o0.transA;     // A stored K x M
  P->b_mn = !o0.transB;    // B stored K x N
  P->out_f32 = o0.out_f32;
  P->relu = o0.relu;
  P->mask = o0.mask != nullptr;
  P->maxM = P->maxN = 0;
  int64_t maxN = 0;
  for (int i = 0; i < n; ++i) maxN = ops[i].N > maxN ? ops[i].N : maxN;
  P->bn = maxN > 128 ? 256 : 128;
  P->G.n = n;
  for (int i = 0; i < n; ++i) {
    const GemmOp& o = ops[i];
    if (o.transA != o0.transA || o.transB != o0.transB || o.out_f32 != o0.out_f32 || o.relu != o0.relu ||
        (o.mask != nullptr) != P->mask)
      return false;
    if (o.K <= 0 || ((uintptr_t)o.A & 15) || ((uintptr_t)o.B & 15) || (o.lda % 8) || (o.ldb % 8)) return false;
    GemmSlotTC& S = P->G.s[i];
    bool ok = P->a_mn ? make_map(&S.ma, o.A, o.M, o.K, o.lda, 64, 64) : make_map(&S.ma, o.A, o.K, o.M, o.lda, 64, BM);
    ok = ok && (P->b_mn ? make_map(&S.mb, o.B, o.N, o.K, o.ldb, 64, 64)
                        : make_map(&S.mb, o.B, o.K, o.N, o.ldb, 64, P->bn));
    if (!ok) return false;
    S.C = o.C;
    S.ldc = o.ldc;
    S.mask = o.mask;
    S.ldm = o.ldm;
    S.M = (int)o.M;
    S.N = (int)o.N;
    S.K = (int)o.K;
    P->maxM = o.M > P->maxM ? o.M : P->maxM;
    P->maxN = o.N > P->maxN ? o.N : P->maxN;
  }
  return true;
}

void gemm_bf16_launch(const GemmPlanTC& P, cudaStream_t s) {
  if (P.G.n <= 0 || P.maxM <= 0 || P.maxN <= 0) return;
  if (P.bn == 256) dispatch_layout<256>(P, s);
  else dispatch_layout<128>(P, s);
}

bool gemm_bf16(bool transA, bool transB, int64_t M, int64_t N, int64_t K, const bf16* A, int64_t lda, const bf16* B,
               int64_t ldb, void* C, int64_t ldc, bool out_f32, bool relu, cudaStream_t s) {
  if (!get_encode()) return false;
  if (M == 0 || N == 0) return true;  // nothing to do (also the availability probe)
  GemmOp o{transA, transB, M, N, K, A, lda, B, ldb, C, ldc, out_f32, relu, nullptr, 0};
  GemmPlanTC P;
  if (!gemm_bf16_prepare(&o, 1, &P)) return false;
  gemm_bf16_launch(P, s);
  return true;
}

}  // namespace gist
