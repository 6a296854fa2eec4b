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

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace gist {
namespace {

constexpr int BM = 128;
// epilogue warps: two per TMEM lane quarter, each owning half of the tile's columns
constexpr int kEpiWarps = 8;
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;
constexpr int BK = 64;  // 64 bf16 = 128 bytes: one SWIZZLE_128B row (TF32: 32 fp32, the same 128 bytes)

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
// L2 eviction-priority policies (createpolicy; used as .L2::cache_hint operands)
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st16_hint(bf16* p, const float* v, uint64_t pol) {
  uint4 a;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&a);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
               "r"(a.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
// GIST_GEMM_TRACE (debug builds only, tools/gemm_trace.py): %globaltimer at the phases of
// each CTA's first tile -- entry, after the PDL wait, first TMA issue, first stage landed,
// last MMA of the tile issued, accumulator ready in the epilogue, epilogue done, exit.
#ifdef GIST_GEMM_TRACE
__device__ unsigned long long g_gemm_trace[1024][16];
__device__ __forceinline__ void gtrace(int k) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (blockIdx.x < 1024) g_gemm_trace[blockIdx.x][k] = t;
}
#else
__device__ __forceinline__ void gtrace(int) {}
#endif
// TMA store of one staged box (shared -> global; out-of-bounds rows/columns are clipped)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, const void* src, int x, int y, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(map),
               "r"(smem_u32(src)), "r"(x), "r"(y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---- CTA-pair (cta_group::2) primitives: two CTAs of a cluster on one TPC share one
// 256-row MMA; each holds its 128 rows of A and half of B's columns in shared memory.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2-SM TMA load into this CTA's shared memory; the transaction bytes are counted on the
// leader CTA's (rank 0) barrier at the same offset (peer bit cleared)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// MMA completion -> arrive on the barrier at this offset in BOTH CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// arrive on the leader CTA's barrier at this offset (local for the leader, remote for the peer)
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile(
      "{\n.reg .b32 ra;\nmapa.shared::cluster.u32 ra, %0, 0;\nmbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra.uni WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// UMMA shared-memory descriptor: start, LBO, SBO in 16-byte units; version 1 (sm_100); layout type
// SWIZZLE_128B (2) or, for MN-major 32-bit (tf32) operands, SWIZZLE_128B_BASE32B (1): the only
// shared-memory layout UMMA accepts for MN-major tf32 (32-byte swizzle atoms, 4-row K groups).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
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
// TF32 mode (R13): fp32 operands read as tf32 by the tensor cores, fp32 accumulation; K = 8 per MMA
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
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

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// split tcgen05.ld: issue now, wait later; the wait names the destination registers as in-out
// operands, so no read of them can be scheduled above it
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

template <int BN, int ST = (BN == 256 ? 4 : (BN == 64 ? 8 : 6))>
struct Cfg {
  static constexpr int STAGES = ST;
  static constexpr int A_BYTES = BM * BK * 2;  // 16 KB
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // epilogue staging for TMA stores: 4 warps x 2 buffers x (32 rows x 128 B)
  static constexpr int EPI_BYTES = kEpiWarps * 4096;  // one 32 x 128 B box per epilogue warp
  static constexpr int SMEM_BASE = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
};

// Epilogue options (runtime, warp-uniform): ReLU, ReLU-mask of the layer below, a per-row
// scale on columns >= rs_from, an added bf16 matrix.
struct Epi {
  void* C;
  int64_t ldc;
  int relu;
  const bf16* mask;
  int64_t ldm;
  const float* rscale;
  int rs_from;
  const bf16* add;
  int64_t ldadd;
  uint32_t* mbits;
  int64_t ldmb;
  const CUtensorMap* mc;  // TMA store map of C, or nullptr (direct stores)
  int clip;               // rows >= rows_valid lie outside mc (TMA clips them): every warp may use it
  int keep;               // L2 evict_last hint on the output stores
  const uint32_t* mbits_in;  // bit-packed ReLU mask applied after add (words [row * ldmbi + col / 32])
  int64_t ldmbi;
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Epilogue of one 16-column chunk of one output row: v = accumulator values.
// `pre`: the chunk's 16 `add` values (two 16-byte vectors) loaded ahead of time, or nullptr.
template <bool OUT_F32, bool STORE = true>
__device__ __forceinline__ void epi_chunk(const Epi& E, float sc, int64_t row, int col, int N, float* v,
                                          const uint4* pre, const uint32_t* mw_pre = nullptr) {
  const bool full16 = col + 16 <= N;
  if (E.rscale) {  // per-row scale of the columns >= rs_from (sc = rscale[row], loaded once per tile)
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (col + i >= E.rs_from) v[i] *= sc;
  }
  if (E.add) {
    const bf16* ap = E.add + row * E.ldadd + col;
    if (pre) {
      float t[16];
      unpack8(pre[0], t);
      unpack8(pre[1], t + 8);
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] += t[i];
    } else if (full16 && ((((uintptr_t)ap) & 15) == 0)) {
      float t[16];
      ld16(ap, t);
      ld16(ap + 8, t + 8);
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] += t[i];
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (col + i < N) v[i] += __bfloat162float(ap[i]);
    }
  }
  if (E.relu) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
  }
  if (E.mbits_in) {  // ReLU'(0) = 0 of the layer below (R3), bit-packed (col % 16 == 0 here)
    const uint32_t wd = (mw_pre ? *mw_pre : E.mbits_in[row * E.ldmbi + (col >> 5)]) >> (col & 31);
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (!((wd >> i) & 1u)) v[i] = 0.f;
  }
  if (E.mask) {  // ReLU'(0) = 0 of the layer below (R3): out = acc * 1[mask > 0]
    const bf16* mp = E.mask + row * E.ldm + col;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (col + i < N && !(__bfloat162float(mp[i]) > 0.f)) v[i] = 0.f;
  }
  if (!STORE) return;  // staged for a TMA store by the caller
  if (OUT_F32) {
    float* dst = (float*)E.C + row * E.ldc + col;
    if (full16 && (((uintptr_t)dst & 15) == 0)) {
#pragma unroll
      for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (col + i < N) dst[i] = v[i];
    }
  } else {
    bf16* dst = (bf16*)E.C + row * E.ldc + col;
    if (full16 && (((uintptr_t)dst & 15) == 0)) {
      if (E.keep) {
        const uint64_t pol = policy_evict_last();
        st16_hint(dst, v, pol);
        st16_hint(dst + 8, v + 8, pol);
      } else {
        st16(dst, v);
        st16(dst + 8, v + 8);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (col + i < N) dst[i] = __float2bfloat16_rn(v[i]);
    }
  }
}

// One output tile of a persistent GEMM: where its operands start, where it writes.
struct Tile {
  bool valid;  // tile exists
  bool mma;    // false: zero-fill only (inert dummy rows of a batch)
  const CUtensorMap *ma, *mb;
  int a_row, b_col, b_k0, K;  // TMA coordinates
  int64_t out_row0;
  int rows_valid, n0, N;
  int stream_a;  // evict_first hint on the A loads
  Epi E;
};

// The scalar fields of a slot (everything after its tensor maps), copied from the kernel
// parameters into shared memory before the PDL wait: a tile decode then reads shared memory
// instead of the parameter bank, whose per-slot fields (dynamically indexed) miss the constant
// cache -- ~0.5 us of serial misses in the producer's first decode and again in the epilogue.
// (compact: 16 of them fit next to the largest ring + staging configuration)
struct SlotTailTC {
  void* C;
  const void* mask;
  const float* rscale;
  uint32_t* mbits;
  const bf16* add;
  const uint32_t* mbits_in;
  int32_t ldc, ldm, ldmb, ldadd, ldmbi;
  int32_t M, N, K, rs_from;
  uint8_t relu, tma_store, keep_out, stream_a;
};
static_assert(sizeof(SlotTailTC) == 88, "compact tail");
struct BdTail {
  void* C;
  const bf16* add;
  const float* rscale;
  const int32_t* desc;
  int64_t ldc, ldadd;
  int N, global_rows, tma_store, keep_out;
};
static_assert(offsetof(BdSlot, C) == 2 * sizeof(CUtensorMap), "BdSlot tail");
static_assert(offsetof(BdSlot, keep_out) - offsetof(BdSlot, C) == offsetof(BdTail, keep_out), "tail");
template <class Tail, class Slot>
__device__ __forceinline__ void copy_tails(const Slot* slots, int n, Tail* dst, size_t off) {
  static_assert(sizeof(Tail) % 8 == 0, "tail words");
  constexpr int W = (int)(sizeof(Tail) / 8);
  for (int i = threadIdx.x; i < n * W; i += blockDim.x) {
    const int z = i / W, w = i - z * W;
    reinterpret_cast<uint64_t*>(dst + z)[w] = reinterpret_cast<const uint64_t*>(reinterpret_cast<const char*>(slots + z) + off)[w];
  }
}

// Plain grouped GEMM: tiles (slot, m-tile, n-tile), n fastest.
template <int BN>
struct ProbPlain {
  using Group = GemmGroupTC;
  static constexpr bool kTmaEpi = true;  // epilogue staging + TMA stores
  static __device__ __forceinline__ int ydim(const Group& G) { return G.tm; }
  static __device__ __forceinline__ int count(const Group& G) { return G.n * G.tm * G.tn; }
  // shared scratch (int32 words): the slots' scalar tails
  static constexpr int kTailWords = (int)(kMaxGemmOps * sizeof(SlotTailTC) / 4);
  static constexpr int kScratchWords = kTailWords;
  static __device__ __forceinline__ void stage_tail(const Group& G, int32_t* sd) {
    if ((int)threadIdx.x < G.n) {  // one slot per thread (leading dimensions < 2^31 elements)
      const GemmSlotTC& S = G.s[threadIdx.x];
      SlotTailTC& t = reinterpret_cast<SlotTailTC*>(sd)[threadIdx.x];
      t.C = S.C; t.mask = S.mask; t.rscale = S.rscale; t.mbits = S.mbits; t.add = S.add; t.mbits_in = S.mbits_in;
      t.ldc = (int32_t)S.ldc; t.ldm = (int32_t)S.ldm; t.ldmb = (int32_t)S.ldmb; t.ldadd = (int32_t)S.ldadd;
      t.ldmbi = (int32_t)S.ldmbi;
      t.M = S.M; t.N = S.N; t.K = S.K; t.rs_from = S.rs_from;
      t.relu = (uint8_t)S.relu; t.tma_store = (uint8_t)S.tma_store; t.keep_out = (uint8_t)S.keep_out;
      t.stream_a = (uint8_t)S.stream_a;
    }
  }
  static __device__ __forceinline__ void stage(const Group&, int32_t*) {}
  // the tensor maps of this CTA's first tile, fetched while the predecessor drains
  static __device__ __forceinline__ void prefetch(const Group& G, int t) {
    if (t >= count(G)) return;
    const GemmSlotTC& S = G.s[t / (G.tm * G.tn)];
    prefetch_map(&S.ma);
    prefetch_map(&S.mb);
    if (S.tma_store) prefetch_map(&S.mc);
  }
  static __device__ __forceinline__ Tile decode(const Group& G, int t, const int32_t* sd) {
    const int per = G.tm * G.tn;
    const int z = t / per, r = t - z * per;
    return decode_y(G, z, r / G.tn, r % G.tn, sd);
  }
  // tile (slot z, 128-row tile y, n-tile nt)
  static __device__ __forceinline__ Tile decode_y(const Group& G, int z, int y, int nt, const int32_t* sd) {
    Tile T;
    const SlotTailTC& S = reinterpret_cast<const SlotTailTC*>(sd)[z];
    const int m0 = y * BM, n0 = nt * BN;
    T.valid = T.mma = m0 < S.M && n0 < S.N;
    T.ma = &G.s[z].ma;
    T.mb = &G.s[z].mb;
    T.a_row = m0;
    T.b_col = n0;
    T.b_k0 = 0;
    T.K = S.K;
    T.out_row0 = m0;
    T.rows_valid = S.M - m0;
    T.n0 = n0;
    T.N = S.N;
    T.E = Epi{S.C, S.ldc, S.relu, (const bf16*)S.mask, S.ldm, S.rscale, S.rs_from, S.add, S.ldadd, S.mbits, S.ldmb,
                 S.tma_store ? &G.s[z].mc : nullptr, 1, S.keep_out, S.mbits_in, S.ldmbi};
    T.stream_a = S.stream_a;
    return T;
  }
};

// Block-diagonal cluster aggregation: tiles (slot, [cluster k, m-tile] | dummy tile, n-tile).
template <int BN>
struct ProbBd {
  using Group = BdGroup;
  // TMA-staged stores for every 32-row lane quarter inside its cluster (a tile's last quarter
  // may cross the cluster end: direct stores there, E.clip = 0); a 3-stage ring leaves room
  static constexpr bool kTmaEpi = true;
  static __device__ __forceinline__ int mt_per(const Group& G) { return (G.bs + BM - 1) / BM; }
  static __device__ __forceinline__ int ydim(const Group& G) {
    return G.q * mt_per(G) + (int)((G.rows + BM - 1) / BM);
  }
  static __device__ __forceinline__ int count(const Group& G) { return G.n * ydim(G) * G.tn; }
  // shared scratch: the slots' scalar tails, then this step's descriptors of every slot
  static constexpr int kMaxDesc = 3 * 64 + 4;
  static constexpr int kTailWords = (int)(kMaxGroup * sizeof(BdTail) / 4);
  static constexpr int kScratchWords = kTailWords + kMaxDesc * kMaxGroup;
  static __device__ __forceinline__ void stage_tail(const Group& G, int32_t* sd) {
    copy_tails(G.s, G.n, reinterpret_cast<BdTail*>(sd), offsetof(BdSlot, C));
  }
  static __device__ __forceinline__ void prefetch(const Group& G, int) {
    prefetch_map(&G.ma);
    prefetch_map(&G.s[0].mb);
  }
  static __device__ __forceinline__ void stage(const Group& G, int32_t* sd) {
    const int per = 3 * G.q + 4;
    const int z = G.st->z;
    const BdTail* tl = reinterpret_cast<const BdTail*>(sd);
    int32_t* sdesc = sd + kTailWords;
    for (int i = threadIdx.x; i < G.n * per; i += blockDim.x)
      sdesc[i] = tl[i / per].desc[(size_t)z * per + (i % per)];
  }
  static __device__ __forceinline__ Tile decode(const Group& G, int t, const int32_t* sdesc) {
    const int per = ydim(G) * G.tn;
    const int z = t / per, r = t - z * per;
    return decode_y(G, z, r / G.tn, r % G.tn, sdesc);
  }
  static __device__ __forceinline__ Tile decode_y(const Group& G, int z, int y, int nt, const int32_t* sd) {
    Tile T;
    const int n0 = nt * BN;
    const BdTail& S = reinterpret_cast<const BdTail*>(sd)[z];
    const int q = G.q, mp = mt_per(G);
    const int32_t* d = sd + kTailWords + z * (3 * q + 4);
    T.ma = &G.ma;
    T.mb = &G.s[z].mb;
    T.n0 = n0;
    T.N = S.N;
    T.E = Epi{S.C, S.ldc, 0, nullptr, 0, S.rscale, 0, S.add, S.ldadd, nullptr, 0, S.tma_store ? &G.s[z].mc : nullptr, 0,
              S.keep_out, nullptr, 0};
    T.stream_a = 0;
    T.b_col = n0;
    T.K = G.bs;
    if (y >= q * mp) {  // inert dummy rows [n_b, rows): zeros
      const int64_t r0 = (int64_t)d[2 * q] + (int64_t)(y - q * mp) * BM;
      T.mma = false;
      T.out_row0 = r0;
      T.rows_valid = (int)((G.rows - r0) < BM ? (G.rows - r0) : BM);
      T.valid = T.rows_valid > 0 && n0 < S.N;
      return T;
    }
    const int k = y / mp, mt = y - k * mp;
    T.valid = T.mma = false;
    if (k >= d[3 * q + 2]) return T;
    const int c = d[k], r0 = d[q + k], size = d[q + k + 1] - r0;
    if (mt * BM >= size || n0 >= S.N) return T;
    T.valid = T.mma = true;
    T.a_row = c * G.bs + mt * BM;
    T.b_k0 = S.global_rows ? (int)G.cstart[c] : r0;
    T.out_row0 = r0 + mt * BM;
    T.rows_valid = size - mt * BM;
    return T;
  }
};

// Epilogue of one MMA tile by one epilogue warp (its TMEM lane quarter lq, columns
// [c0w, c0w + CW)): waits for the accumulator, then TMEM -> registers -> (scale, add, ReLU,
// mask, ReLU-mask bits) -> TMA-staged or direct stores.  Shared by the 1-CTA and CTA-pair kernels.
template <int BN, bool OUT_F32, bool TMA_EPI>
__device__ __forceinline__ void epi_tile(const Tile& T, uint32_t tmem_acc, uint64_t* accf_b, uint32_t aph, int lq,
                                         int lane, int c0w, uint8_t* stg) {
  constexpr int CW = BN / (kEpiWarps / 4);  // columns per epilogue warp
  const int r = lq * 32 + lane;
    const int64_t row = T.out_row0 + r;
    const bool live = r < T.rows_valid;
    const float sc = (T.E.rscale && live) ? T.E.rscale[row] : 1.f;  // before the wait: overlaps the MMA
    // `add` is read one 32-column chunk ahead (the first before the accumulator wait), so its
    // latency overlaps the MMA / the previous chunk instead of serialising the epilogue
    const bf16* arow = T.E.add ? T.E.add + row * T.E.ldadd + T.n0 : nullptr;
    const bool avec = arow && live && ((((uintptr_t)arow) & 15) == 0) && ((T.E.ldadd & 7) == 0);
    uint4 cur[4], nxt[4];
    bool cur_ok = avec && c0w + 32 <= T.N - T.n0;
    // the ReLU-mask words of this warp's columns, also ahead of the wait (one per 32 columns)
    constexpr int MW = CW / 32;
    uint32_t mw[MW];
    const bool mpre = T.E.mbits_in && live;
    if (mpre)
#pragma unroll
      for (int i = 0; i < MW; ++i)
        mw[i] = T.n0 + c0w + 32 * i < T.N ? T.E.mbits_in[row * T.E.ldmbi + ((T.n0 + c0w) >> 5) + i] : 0u;
    if (cur_ok)
#pragma unroll
      for (int i = 0; i < 4; ++i) cur[i] = __ldg(reinterpret_cast<const uint4*>(arow + c0w) + i);
    mbar_wait(accf_b, aph);
    if (lq == 2 && c0w == 0 && lane == 0) gtrace(5);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t trow = tmem_acc + ((uint32_t)(lq * 32) << 16);
    // TMA-store path: this warp's 32 rows are staged (128-byte rows, SWIZZLE_128B: 16-byte
    // chunk j of row r at r*128 + ((j ^ (r & 7)) * 16), bank-conflict free) and written by
    // one cp.async.bulk.tensor per 32 x 128 B box, so stores are full lines instead of one
    // 16-byte piece of 32 different rows per instruction.
    const bool tma = TMA_EPI && T.E.mc && (T.E.clip || lq * 32 + 32 <= T.rows_valid);
    constexpr int CPB = OUT_F32 ? 32 : 64;  // columns per 128-byte box row
#pragma unroll 1
    for (int c = c0w; c < c0w + CW; c += 32) {
      // warp-uniform: the tile's remaining columns all lie beyond N (nothing to store; a
      // staged-but-never-stored box would also break the buffer accounting below)
      if (T.n0 + c >= T.N) break;
      const bool nxt_ok = avec && c + 32 < c0w + CW && c + 64 <= T.N - T.n0;
      if (nxt_ok)
#pragma unroll
        for (int i = 0; i < 4; ++i) nxt[i] = __ldg(reinterpret_cast<const uint4*>(arow + c + 32) + i);
      float v[32];
      tmem_ld32(trow + c, v);
      const bool trc = lq == 2 && c0w == 0 && lane == 0 && c == 0;
      if (trc) gtrace(8);
      if (tma) {
        const int cb = c % CPB;  // column of this piece inside its box
        uint8_t* buf = stg;
        if (cb == 0) {  // the previous box's TMA store must have finished reading the buffer
          if (lane == 0) bulk_wait_read0();
          __syncwarp();
        }
        if (live && T.n0 + c < T.N) {
          epi_chunk<OUT_F32, false>(T.E, sc, row, T.n0 + c, T.N, v, cur_ok ? cur : nullptr, mpre ? mw : nullptr);
          if (T.n0 + c + 16 < T.N)
            epi_chunk<OUT_F32, false>(T.E, sc, row, T.n0 + c + 16, T.N, v + 16, cur_ok ? cur + 2 : nullptr, mpre ? mw : nullptr);
        }
        uint8_t* rbase = buf + lane * 128;
        if (OUT_F32) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(rbase + ((j ^ (lane & 7)) * 16)) =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 pk;
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
            for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[8 * j + 2 * i], v[8 * j + 2 * i + 1]);
            const int jj = (cb / 8) + j;  // 16-byte chunk index inside the 128-byte row
            *reinterpret_cast<uint4*>(rbase + ((jj ^ (lane & 7)) * 16)) = pk;
          }
        }
        if (cb + 32 == CPB || c + 32 == c0w + CW || T.n0 + c + 32 >= T.N) {  // box complete: store it
          if (lq == 2 && c0w == 0 && lane == 0) gtrace(9);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (T.E.keep) tma_store_2d_hint(T.E.mc, buf, T.n0 + c - cb, (int)(T.out_row0 + lq * 32), policy_evict_last());
            else tma_store_2d(T.E.mc, buf, T.n0 + c - cb, (int)(T.out_row0 + lq * 32));
            bulk_commit();
            if (lq == 2 && c0w == 0) gtrace(10);
          }
        }
        if (live && T.n0 + c < T.N && T.E.mbits) {
          uint32_t bits = 0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float sv = OUT_F32 ? v[i] : __bfloat162float(__float2bfloat16_rn(v[i]));
            bits |= (T.n0 + c + i < T.N && sv > 0.f) ? (1u << i) : 0u;
          }
          T.E.mbits[row * T.E.ldmb + ((T.n0 + c) >> 5)] = bits;
        }
      } else if (live && T.n0 + c < T.N) {
        epi_chunk<OUT_F32>(T.E, sc, row, T.n0 + c, T.N, v, cur_ok ? cur : nullptr, mpre ? mw : nullptr);
        if (T.n0 + c + 16 < T.N)
          epi_chunk<OUT_F32>(T.E, sc, row, T.n0 + c + 16, T.N, v + 16, cur_ok ? cur + 2 : nullptr, mpre ? mw : nullptr);
        if (T.E.mbits) {  // sign bits of the values as stored (bf16-rounded on the bf16 path)
          uint32_t bits = 0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float sv = OUT_F32 ? v[i] : __bfloat162float(__float2bfloat16_rn(v[i]));
            bits |= (T.n0 + c + i < T.N && sv > 0.f) ? (1u << i) : 0u;
          }
          T.E.mbits[row * T.E.ldmb + ((T.n0 + c) >> 5)] = bits;
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) cur[i] = nxt[i];
      cur_ok = nxt_ok;
#pragma unroll
      for (int i = 0; i + 1 < MW; ++i) mw[i] = mw[i + 1];
    }
}

// inert dummy rows of a batch: exact zeros (no MMA); et = thread index among the epilogue warps
template <int BN, bool OUT_F32>
__device__ __forceinline__ void zero_fill_tile(const Tile& T, int et) {
  for (int idx = et; idx < BM * BN; idx += 32 * kEpiWarps) {
    const int rr = idx / BN, cc = T.n0 + idx % BN;
    if (rr < T.rows_valid && cc < T.N) {
      const int64_t row = T.out_row0 + rr;
      if (OUT_F32) ((float*)T.E.C)[row * T.E.ldc + cc] = 0.f;
      else ((bf16*)T.E.C)[row * T.E.ldc + cc] = __float2bfloat16_rn(0.f);
    }
  }
}

// Persistent warp-specialised tcgen05 GEMM: grid = min(tiles, #SMs), kGemmThreads threads.
// warp 0: TMA producer (one lane) into an ST-deep shared-memory ring; warp 1: MMA issuer
// (one lane) into one of two TMEM accumulators; warps 2..9: epilogue, two per TMEM lane quarter
// splitting the columns (TMEM -> registers ->
// global), releasing the accumulator to the MMA warp, so the epilogue of tile i overlaps the
// main loop of tile i+1 and the CTA set-up (barriers, TMEM allocation) is paid once per SM.
// TF: TF32 mode -- operands are fp32 (4 bytes): a 128-byte swizzle row holds BKE = 32 K elements,
// an MN-major TMA box is 32 elements wide (4 per 128-row tile, 4 KB apart), one MMA covers K = 8
// (+32 bytes K-major, +1 KB MN-major).  The ring, its byte counts and the epilogue are unchanged.
template <int BN, int ST, bool A_MN, bool B_MN, bool OUT_F32, class Prob, bool TF = false>
__global__ void __launch_bounds__(kGemmThreads, 1) k_gemm_persist(const __grid_constant__ typename Prob::Group G) {
  using CF = Cfg<BN, ST>;
  constexpr int BKE = TF ? 32 : BK;            // K elements per k-block (128 bytes)
  constexpr int MNB = TF ? 32 : 64;            // MN elements per MN-major box (128 bytes)
  constexpr uint32_t BOXB = (uint32_t)MNB * BKE * (TF ? 4 : 2);  // bytes per MN-major box
  constexpr uint32_t KSTEP_MN = TF ? 1024u : 2048u;            // MN-major descriptor advance per MMA
  // MN-major tf32: SWIZZLE_128B_BASE32B (layout 1, K groups of 4 rows = 512 B); bf16: SWIZZLE_128B
  constexpr uint32_t MN_LAYOUT = TF ? 1u : 2u, MN_SBO = TF ? 512u : 1024u;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int EPI = Prob::kTmaEpi ? CF::EPI_BYTES : 0;
  uint64_t* full = (uint64_t*)(smem + CF::STAGES * CF::STAGE_BYTES + EPI);  // after the epilogue staging
  uint64_t* empty = full + CF::STAGES;
  uint64_t* accf = empty + CF::STAGES;  // [2]
  uint64_t* acce = accf + 2;            // [2]
  uint32_t* tmem_slot = (uint32_t*)(acce + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t TCOLS = 2 * BN < 32 ? 32 : 2 * BN;  // two accumulators
  __shared__ __align__(16) int32_t sdesc[Prob::kScratchWords];

  if (threadIdx.x == 0) {
    gtrace(0);
    for (int s = 0; s < CF::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], kEpiWarps);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) Prob::prefetch(G, blockIdx.x);
  Prob::stage_tail(G, sdesc);
  __syncthreads();  // the tails are read by other threads from here on (ProbBd::stage, decode)
  if (threadIdx.x == 0) gtrace(12);
  // prologue above (barriers, TMEM, tensor-map prefetch) overlaps the predecessor kernel's
  // tail under PDL; everything below may read what it wrote
  pdl_wait();
  pdl_trigger();
  Prob::stage(G, sdesc);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int total = Prob::count(G);
  if (threadIdx.x == 0) gtrace(1);

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      uint32_t it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const Tile T = Prob::decode(G, t, sdesc);
        if (!T.mma) continue;
        const int nk = (T.K + BKE - 1) / BKE;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % CF::STAGES;
          const uint32_t ph = (it / CF::STAGES) & 1u;
          mbar_wait(&empty[s], ph ^ 1u);
          uint8_t* sa = smem + s * CF::STAGE_BYTES;
          uint8_t* sb = sa + CF::A_BYTES;
          mbar_arrive_expect_tx(&full[s], CF::STAGE_BYTES);
          if (it == 0) gtrace(2);
          const int k0 = kb * BKE;
          if (T.stream_a) {  // last read of A for a while: evict first
            const uint64_t pol = policy_evict_first();
            if (!A_MN) {
              tma_load_2d_hint(sa, T.ma, &full[s], k0, T.a_row, pol);
            } else {
#pragma unroll
              for (int j = 0; j < BM / MNB; ++j)
                tma_load_2d_hint(sa + j * BOXB, T.ma, &full[s], T.a_row + MNB * j, k0, pol);
            }
          } else if (!A_MN) {
            tma_load_2d(sa, T.ma, &full[s], k0, T.a_row);
          } else {
#pragma unroll
            for (int j = 0; j < BM / MNB; ++j)
              tma_load_2d(sa + j * BOXB, T.ma, &full[s], T.a_row + MNB * j, k0);
          }
          if (!B_MN) {
            tma_load_2d(sb, T.mb, &full[s], T.b_k0 + k0, T.b_col);
          } else {
#pragma unroll
            for (int j = 0; j < BN / MNB; ++j)
              tma_load_2d(sb + j * BOXB, T.mb, &full[s], T.b_col + MNB * j, T.b_k0 + k0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      // c_format F32 (bit 4); a/b format BF16 = 1 or TF32 = 2 (bits 7-9, 10-12); majorness; N >> 3; M >> 4
      constexpr uint32_t fmt = TF ? 2u : 1u;
      constexpr uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((A_MN ? 1u : 0u) << 15) |
                                 ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      uint32_t it = 0, tc = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const Tile T = Prob::decode(G, t, sdesc);
        if (!T.mma) continue;
        const uint32_t b = tc & 1u, aph = (tc >> 1) & 1u;
        mbar_wait(&acce[b], aph ^ 1u);  // the epilogue has drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dacc = tmem + b * BN;
        const int nk = (T.K + BKE - 1) / BKE;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % CF::STAGES;
          const uint32_t ph = (it / CF::STAGES) & 1u;
          mbar_wait(&full[s], ph);
          if (it == 0) gtrace(3);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(smem + s * CF::STAGE_BYTES);
          const uint32_t sb = sa + CF::A_BYTES;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            // K-major: +32 bytes per MMA (K16 bf16 / K8 tf32) inside the swizzled row; MN-major:
            // +16 (bf16) / +8 (tf32) K-rows of 128 bytes; LBO = one MN box
            const uint64_t ad = A_MN ? make_desc(sa + k * KSTEP_MN, BOXB, MN_SBO, MN_LAYOUT) : make_desc(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_desc(sb + k * KSTEP_MN, BOXB, MN_SBO, MN_LAYOUT) : make_desc(sb + k * 32, 16, 1024);
            if constexpr (TF) umma_tf32(dacc, ad, bd, idesc, (kb | k) != 0);
            else umma_bf16(dacc, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[s]);  // frees the stage once these MMAs have read it
        }
        umma_commit(&accf[b]);  // accumulator b complete
        if (tc == 0) gtrace(4);
        ++tc;
      }
    }
  } else {  // ---------------------------------------------- epilogue warps 2 .. 1 + kEpiWarps
    const int ew = warp - 2;
    const int lq = warp & 3;  // TMEM lane quarter this warp may access
    const int r = lq * 32 + lane;
    constexpr int CW = BN / (kEpiWarps / 4);  // columns per epilogue warp
    const int c0w = (ew >> 2) * CW;           // this warp's first column inside the tile
    uint8_t* stg = smem + CF::STAGES * CF::STAGE_BYTES + ew * 4096;  // this warp's staging box
    uint32_t tc = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const Tile T = Prob::decode(G, t, sdesc);
      if (!T.valid) continue;
      if (!T.mma) {  // zero-fill (dummy rows)
        zero_fill_tile<BN, OUT_F32>(T, threadIdx.x - 64);
        continue;
      }
      const uint32_t b = tc & 1u, aph = (tc >> 1) & 1u;
      epi_tile<BN, OUT_F32, Prob::kTmaEpi>(T, tmem + b * BN, &accf[b], aph, lq, lane, c0w, stg);
      if (tc == 0 && ew == 0 && lane == 0) gtrace(6);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[b]);
      ++tc;
    }
    if (lane == 0) bulk_wait_read0();  // the staging buffers are read before the CTA exits
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) gtrace(7);
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
  }
}

// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes 256 x BN tiles
// (two consecutive 128-row tiles y = 2p, 2p+1 of the same slot and n-tile).  Each CTA stages
// its own 128 rows of A and HALF of B's columns, so a ring stage is 16 + BN/4 KB instead of
// 16 + BN/2 KB: with the same shared memory the ring is 1.5x deeper and each SM pulls 1/3
// fewer operand bytes through L2 per FLOP.  The leader (rank 0) issues the 256-row MMA and
// multicasts its completions to both CTAs; both CTAs' producers count their TMA bytes on the
// leader's full barrier; both CTAs' epilogues drain their own TMEM rows and arrive on the
// leader's accumulator-empty barrier.  Same arithmetic as k_gemm_persist.
template <int BN, int ST, bool A_MN, bool B_MN, bool OUT_F32, class Prob>
__global__ void __launch_bounds__(kGemmThreads, 1) k_gemm_pair(const __grid_constant__ typename Prob::Group G) {
  constexpr int BNH = BN / 2;
  constexpr int A_BYTES = BM * BK * 2, B_BYTES = BNH * BK * 2, STAGE = A_BYTES + B_BYTES;
  constexpr int EPI = Prob::kTmaEpi ? kEpiWarps * 4096 : 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + ST * STAGE + EPI);
  uint64_t* empty = full + ST;
  uint64_t* accf = empty + ST;  // [2]
  uint64_t* acce = accf + 2;    // [2]  (leader: both CTAs' epilogue warps arrive)
  uint32_t* tmem_slot = (uint32_t*)(acce + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  constexpr uint32_t TCOLS = 2 * BN < 32 ? 32 : 2 * BN;
  __shared__ __align__(16) int32_t sdesc[Prob::kScratchWords];

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], 2 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {  // paired TMEM allocation: same warp, same destination offset in both CTAs
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  cluster_sync_all();  // both CTAs' barriers initialised before any cross-CTA arrival
  Prob::stage_tail(G, sdesc);
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  Prob::stage(G, sdesc);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int yd = Prob::ydim(G);
  const int yp_n = (yd + 1) / 2;
  const int per2 = yp_n * G.tn;
  const int total2 = G.n * per2;
  // this CTA's 128-row tile and the leader's (which carries the pair's B operand and K)
  auto decode2 = [&](int p, Tile& T0, Tile& Ts) {
    const int z = p / per2, rr = p - z * per2, yp = rr / G.tn, nt = rr - yp * G.tn;
    T0 = Prob::decode_y(G, z, 2 * yp, nt, sdesc);
    if (leader) {
      Ts = T0;
    } else if (2 * yp + 1 < yd) {
      Ts = Prob::decode_y(G, z, 2 * yp + 1, nt, sdesc);
    } else {
      Ts = T0;
      Ts.valid = Ts.mma = false;
    }
  };

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------- TMA producer (both CTAs)
      uint32_t it = 0;
      for (int p = pair; p < total2; p += npairs) {
        Tile T0, Ts;
        decode2(p, T0, Ts);
        if (!T0.mma) continue;
        const int a_row = Ts.mma ? Ts.a_row : T0.a_row + BM;  // rows past the tile: never stored
        const int b_col = T0.b_col + (int)rank * BNH;
        const int nk = (T0.K + BK - 1) / BK;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % ST;
          const uint32_t ph = (it / ST) & 1u;
          mbar_wait(&empty[s], ph ^ 1u);
          uint8_t* sa = smem + s * STAGE;
          uint8_t* sb = sa + A_BYTES;
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * STAGE);  // both CTAs' bytes
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d_pair(sa, T0.ma, &full[s], k0, a_row);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d_pair(sa + j * 8192, T0.ma, &full[s], a_row + 64 * j, k0);
          }
          if (!B_MN) {
            tma_load_2d_pair(sb, T0.mb, &full[s], T0.b_k0 + k0, b_col);
          } else {
#pragma unroll
            for (int j = 0; j < BNH / 64; ++j)
              tma_load_2d_pair(sb + j * 8192, T0.mb, &full[s], b_col + 64 * j, T0.b_k0 + k0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ------------------------------------ MMA issuer (leader only)
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) |
                                 ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)((2 * BM) >> 4) << 24);
      uint32_t it = 0, tc = 0;
      for (int p = pair; p < total2; p += npairs) {
        Tile T0, Ts;
        decode2(p, T0, Ts);
        if (!T0.mma) continue;
        const uint32_t b = tc & 1u, aph = (tc >> 1) & 1u;
        mbar_wait_cluster(&acce[b], aph ^ 1u);  // both CTAs' epilogues drained accumulator b
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dacc = tmem + b * BN;
        const int nk = (T0.K + BK - 1) / BK;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % ST;
          const uint32_t ph = (it / ST) & 1u;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(smem + s * STAGE);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? make_desc(sa + k * 2048, 8192, 1024) : make_desc(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_desc(sb + k * 2048, 8192, 1024) : make_desc(sb + k * 32, 16, 1024);
            umma_bf16_pair(dacc, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit_pair(&empty[s]);  // frees stage s in both CTAs
        }
        umma_commit_pair(&accf[b]);  // accumulator b complete in both CTAs
        ++tc;
      }
    }
  } else {  // ---------------------------------------------- epilogue warps 2 .. 1 + kEpiWarps
    const int ew = warp - 2;
    const int lq = warp & 3;
    constexpr int CW = BN / (kEpiWarps / 4);
    const int c0w = (ew >> 2) * CW;
    uint8_t* stg = smem + ST * STAGE + ew * 4096;
    uint32_t tc = 0;
    for (int p = pair; p < total2; p += npairs) {
      Tile T0, Ts;
      decode2(p, T0, Ts);
      if (!T0.mma) {  // no MMA for this pair: zero-fill own dummy rows, if any
        if (Ts.valid && !Ts.mma) zero_fill_tile<BN, OUT_F32>(Ts, threadIdx.x - 64);
        continue;
      }
      const uint32_t b = tc & 1u, aph = (tc >> 1) & 1u;
      if (Ts.valid && Ts.mma) {
        epi_tile<BN, OUT_F32, Prob::kTmaEpi>(Ts, tmem + b * BN, &accf[b], aph, lq, lane, c0w, stg);
      } else {  // this CTA's half lies past the problem: nothing to store, still drain in order
        mbar_wait(&accf[b], aph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&acce[b]);
      ++tc;
    }
    if (lane == 0) bulk_wait_read0();
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // the peer's shared memory / TMEM may be read until the leader is done
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
  }
}

// ---- Block-diagonal aggregation, transposed (intra-cluster part of Eq. (2)) ----
// out[r0 + r][f] = scale[r0 + r] * sum_k Blk_c[r][k] H[h0 + k][f] (+ add[r0 + r][f]).  The cluster
// block is symmetric (A symmetric), so the MMA computes the transpose D[f][r] = sum_k
// H[h0 + k][f] Blk_c[k][r]: M = 128 features (A = H^T, read in place: MN-major), N = BSN = pad16(bs)
// rows of the cluster (B = Blk_c, K-major), K = bs.  One unit = (slot, batch cluster, 128-feature
// tile) covers every row of the cluster -- no partly filled 128-row tiles, no re-read of H per row
// tile -- and the block stays in shared memory for the unit's neighbours (double-buffered across
// clusters; a CTA owns a contiguous unit range, feature tiles fastest, so it loads each of its ~2
// blocks once): 2-3x fewer operand bytes through L2 than the row-tile kernel.  The epilogue
// transposes each 32-row chunk of the accumulator through shared memory so that every store and
// residual load covers 8 rows x 64 contiguous bytes; TMEM loads are double-buffered.  Dummy rows
// [n_b, rows) of every slot are zero-filled.  Phase trace: tools/bdt_trace.py (-DGIST_GEMM_TRACE;
// the epilogue, ~1 us per 32-row chunk, paces the kernel).
#ifdef GIST_GEMM_TRACE
// k_bd_t phase trace (debug builds): [cta][unit slot 0..8 | 9 = CTA][phase] %globaltimer
__device__ unsigned long long g_bdt_trace[160][10][8];
__device__ __forceinline__ void btrace(int slot, int ph) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (blockIdx.x < 160 && slot < 10) g_bdt_trace[blockIdx.x][slot][ph] = t;
}
#else
__device__ __forceinline__ void btrace(int, int) {}
#endif
constexpr int kBdtStages = 4;
constexpr int kBdtAStage = BM * BK * 2;  // 128 features x 64 rows (two 64 x 64 MN-major boxes)
constexpr int kBdtSmemMax = 220 * 1024;  // dynamic shared memory cap (the descriptors are static)
constexpr int kBdtStg = kEpiWarps * 32 * 32 * 4;  // epilogue transpose buffers
__device__ __forceinline__ void st_bf16(bf16* p, float v, int keep, uint64_t pol) {
  const unsigned short h = __bfloat16_as_ushort(__float2bfloat16_rn(v));
  if (keep) asm volatile("st.global.L2::cache_hint.b16 [%0], %1, %2;" ::"l"(p), "h"(h), "l"(pol) : "memory");
  else asm volatile("st.global.b16 [%0], %1;" ::"l"(p), "h"(h) : "memory");
}

template <bool ADD>
__global__ void __launch_bounds__(kGemmThreads, 1) k_bd_t(const __grid_constant__ BdGroup G) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int bs = G.bs, BSN = (bs + 15) & ~15, KB = (bs + BK - 1) / BK;
  const uint32_t BREG = (uint32_t)KB * BSN * 128;  // one cluster block: KB k-blocks of BSN rows x 128 B
  const uint32_t NBUF = (uint32_t)G.blk_bufs;      // 1 or 2 block buffers
  uint8_t* sblk = smem + kBdtStages * kBdtAStage;
  float* stg_all = (float*)(sblk + NBUF * BREG);  // epilogue transposes: 32 x 32 fp32 per warp
  uint64_t* full = (uint64_t*)((uint8_t*)stg_all + kBdtStg);
  uint64_t* empty = full + kBdtStages;
  uint64_t* accf = empty + kBdtStages;  // [2]
  uint64_t* acce = accf + 2;            // [2]
  uint64_t* bfull = acce + 2;           // [2]
  uint64_t* bempty = bfull + 2;         // [2]
  uint32_t* tmem_slot = (uint32_t*)(bempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t TCOLS = 512;  // two accumulators of <= 256 columns
  constexpr int per_max = ProbBd<128>::kMaxDesc;
  __shared__ int32_t sd[kMaxGroup * per_max];
  __shared__ __align__(16) BdTail stl[kMaxGroup];  // the slots' scalar fields (no dynamic param reads)
  if (threadIdx.x == 0) btrace(9, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kBdtStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], kEpiWarps);
      mbar_init(&bfull[b], 1);
      mbar_init(&bempty[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    prefetch_map(&G.mat);
    for (int z = 0; z < G.n; ++z) prefetch_map(&G.s[z].mb);
  }
  copy_tails(G.s, G.n, stl, offsetof(BdSlot, C));
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const int q = G.q, per = 3 * q + 4;
  {  // this step's batch descriptors of every slot (the step index is read after the PDL wait)
    const int zst = G.st->z;
    for (int i = threadIdx.x; i < G.n * per; i += blockDim.x)
      sd[i] = G.s[i / per].desc[(size_t)zst * per + (i % per)];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) btrace(9, 1);
  int FT = 0;
  for (int z = 0; z < G.n; ++z) FT = max(FT, (stl[z].N + BM - 1) / BM);
  const int U = G.n * q * FT;
  const int u0 = (int)((int64_t)blockIdx.x * U / gridDim.x), u1 = (int)((int64_t)(blockIdx.x + 1) * U / gridDim.x);
  struct Unit {
    bool ok;
    int z, c, r0, size, f0, h0;
  };
  auto decode = [&](int u) {
    Unit t;
    t.z = u / (q * FT);
    const int rem = u - t.z * q * FT, k = rem / FT;
    t.f0 = (rem - k * FT) * BM;
    const int32_t* d = sd + t.z * per;
    t.ok = k < d[3 * q + 2] && t.f0 < stl[t.z].N;
    t.c = d[k];
    t.r0 = d[q + k];
    t.size = d[q + k + 1] - t.r0;
    t.h0 = stl[t.z].global_rows ? (int)G.cstart[t.c] : t.r0;
    return t;
  };

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------------- TMA producer
      uint32_t it = 0, nbl = 0;
      int cur = -1;
      for (int u = u0; u < u1; ++u) {
        const Unit t = decode(u);
        if (!t.ok) continue;
        btrace(u - u0, 0);
        if (t.c != cur) {  // the next cluster block into the other buffer
          const uint32_t bb = nbl % NBUF, bph = (nbl / NBUF) & 1u;
          mbar_wait(&bempty[bb], bph ^ 1u);
          btrace(u - u0, 7);
          mbar_arrive_expect_tx(&bfull[bb], (uint32_t)KB * bs * 128);
          for (int kb = 0; kb < KB; ++kb)
            tma_load_2d(sblk + bb * BREG + (uint32_t)kb * BSN * 128, &G.mat, &bfull[bb], kb * BK, t.c * bs);
          cur = t.c;
          ++nbl;
        }
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % kBdtStages;
          mbar_wait(&empty[s], ((it / kBdtStages) & 1u) ^ 1u);
          uint8_t* sa = smem + s * kBdtAStage;
          mbar_arrive_expect_tx(&full[s], kBdtAStage);
#pragma unroll
          for (int j = 0; j < BM / 64; ++j) tma_load_2d(sa + j * 8192, &G.s[t.z].mb, &full[s], t.f0 + 64 * j, t.h0 + kb * BK);
        }
        btrace(u - u0, 1);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------------------- MMA issuer
      // F32 accumulate, bf16 A/B, A MN-major (features contiguous in H), B K-major, N = BSN, M = 128
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(BSN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);
      uint32_t it = 0, tc = 0, nbl = 0;
      int cur = -1;
      for (int u = u0; u < u1; ++u) {
        const Unit t = decode(u);
        if (!t.ok) continue;
        if (t.c != cur) {
          if (cur >= 0) umma_commit(&bempty[(nbl - 1) % NBUF]);  // the previous block is free once read
          mbar_wait(&bfull[nbl % NBUF], (nbl / NBUF) & 1u);
          cur = t.c;
          ++nbl;
        }
        const uint32_t sbk = smem_u32(sblk + ((nbl - 1) % NBUF) * BREG);
        const uint32_t b = tc & 1u;
        mbar_wait(&acce[b], ((tc >> 1) & 1u) ^ 1u);
        btrace(u - u0, 2);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dacc = tmem + b * 256;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % kBdtStages;
          mbar_wait(&full[s], (it / kBdtStages) & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(smem + s * kBdtAStage);
          const uint32_t sb = sbk + (uint32_t)kb * BSN * 128;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(dacc, make_desc(sa + k * 2048, 8192, 1024), make_desc(sb + k * 32, 16, 1024), idesc, (kb | k) != 0);
          umma_commit(&empty[s]);
        }
        umma_commit(&accf[b]);
        btrace(u - u0, 3);
        ++tc;
      }
    }
  } else {  // ---------------------------------------------- epilogue warps 2 .. 9
    // warp (lane quarter lq, half) drains 32-column chunks ch = half, half + 2, ... of the
    // accumulator: lane f holds feature f0 + 32 lq + f of the chunk's 32 rows; the chunk goes
    // through shared memory (16-byte groups XOR-swizzled by row: conflict-free both ways) so that
    // lane r then owns row 32 ch + r with its 32 features -- one row scale, 16-byte residual loads
    // and stores (the row-tile kernel's epilogue arithmetic: (acc * scale) + add, then bf16)
    const int ew = warp - 2, lq = warp & 3, half = ew >> 2;
    const int nch = (BSN + 31) / 32;  // <= 8 (BSN <= 256): at most kCh = 4 chunks per warp
    constexpr int kCh = 4;
    float* stg = stg_all + ew * 1024;
    // After the transpose, pass p of a chunk has lane l on row 8 p + l / 4, features 8 (l % 4) ..
    // +7 of the warp's 32: every store / residual load instruction covers 8 rows x 64 contiguous
    // bytes.  The operands of those rows (residual groups under ADD, else row scales) are loaded
    // for the next unit while this one drains (ADD: for this unit, before the accumulator wait).
    const int pr = lane >> 2, pj = lane & 3;
    struct Ops {
      float sc[ADD ? 1 : kCh][4];
    };
    auto load_ops = [&](const Unit& t, Ops& o) {  // row scales of the unit's chunks (!ADD)
      const BdTail& S = stl[t.z];
#pragma unroll
      for (int k = 0; k < kCh; ++k) {
        const int ch = half + 2 * k;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int r = ch * 32 + 8 * p + pr;
          if constexpr (!ADD) o.sc[k][p] = (S.rscale && ch < nch && r < t.size) ? __ldg(S.rscale + t.r0 + r) : 1.f;
        }
      }
    };
    // ADD: the residual groups of chunk k (lane: row 8 p + l / 4, features 8 (l % 4) .. +7)
    auto load_add = [&](const Unit& t, int k, uint4 (&a)[4]) {
      const BdTail& S = stl[t.z];
      const int fc = t.f0 + lq * 32, ch = half + 2 * k;
      const bool jl = fc + 8 * pj + 8 <= S.N;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int r = ch * 32 + 8 * p + pr;
        a[p] = (ch < nch && r < t.size && jl)
                   ? __ldg(reinterpret_cast<const uint4*>(S.add + (int64_t)(t.r0 + r) * S.ldadd + fc + 8 * pj))
                   : make_uint4(0u, 0u, 0u, 0u);
      }
    };
    auto next_unit = [&](int u) {
      for (; u < u1; ++u)
        if (decode(u).ok) break;
      return u;
    };
    Ops cur, nxt;
    int u = next_unit(u0);
    if (!ADD && u < u1) load_ops(decode(u), cur);
    uint32_t tc = 0;
    for (; u < u1;) {
      const Unit t = decode(u);
      const int un = next_unit(u + 1);
      // ADD: the residual groups of chunk k in A[k], issued one chunk ahead (distinct registers
      // per chunk: no copy that would wait for an in-flight load)
      uint4 A[ADD ? kCh : 1][4];
      if constexpr (ADD) load_add(t, 0, A[0]);
      else if (un < u1) load_ops(decode(un), nxt);
      const BdTail& S = stl[t.z];
      const int fc = t.f0 + lq * 32;  // this warp's first feature
      const bool jl = fc + 8 * pj + 8 <= S.N;
      const int keep = S.keep_out;
      const uint64_t pol = keep ? policy_evict_last() : 0ull;
      int nk = 0;  // this warp's chunks: ch = half + 2 k inside the cluster
#pragma unroll
      for (int k = 0; k < kCh; ++k) nk += (half + 2 * k < nch && (half + 2 * k) * 32 < t.size) ? 1 : 0;
      const uint32_t b = tc & 1u;
      mbar_wait(&accf[b], (tc >> 1) & 1u);
      if (lane == 0 && ew == 0) btrace(u - u0, 4);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t trow = tmem + b * 256 + ((uint32_t)(lq * 32) << 16);
      uint32_t va[32], vb[32];
      if (nk > 0) {
        tmem_ld32_issue(trow + half * 32, va);
        tmem_wait_ld(va);
      }
      auto chunk = [&](int k, uint32_t (&v)[32], const uint4 (&a)[4]) {
        const int ch = half + 2 * k;
        // v[i] = D[feature lane][row i] -> [row i][feature lane], 16-byte group g of row i at
        // physical group g ^ (i & 7) (conflict-free stores and loads)
#pragma unroll
        for (int i = 0; i < 32; ++i) stg[i * 32 + ((((lane >> 2) ^ (i & 7)) << 2) | (lane & 3))] = __uint_as_float(v[i]);
        __syncwarp();
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int rr = 8 * p + pr, r = ch * 32 + rr;
          float o[8];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float4 qv = *reinterpret_cast<const float4*>(stg + rr * 32 + (((2 * pj + h) ^ (rr & 7)) << 2));
            o[4 * h] = qv.x; o[4 * h + 1] = qv.y; o[4 * h + 2] = qv.z; o[4 * h + 3] = qv.w;
          }
          if (r < t.size && jl) {
            if constexpr (!ADD) {
              if (S.rscale)
#pragma unroll
                for (int i = 0; i < 8; ++i) o[i] *= cur.sc[k][p];
            } else {
              float tt[8];
              unpack8(a[p], tt);
#pragma unroll
              for (int i = 0; i < 8; ++i) o[i] += tt[i];
            }
            bf16* cp = (bf16*)S.C + (int64_t)(t.r0 + r) * S.ldc + fc + 8 * pj;
            if (keep) st16_hint(cp, o, pol);
            else st16(cp, o);
          }
        }
        __syncwarp();
      };
#pragma unroll
      for (int k = 0; k < kCh; ++k) {
        if (k >= nk) break;
        if (k == 0 && lane == 0 && ew == 0 && u == u0) btrace(8, 0);
        if constexpr (ADD) {  // registers go to the residual prefetch; TMEM loads are short (~170 cycles)
          if (k > 0) {
            tmem_ld32_issue(trow + (half + 2 * k) * 32, va);
            tmem_wait_ld(va);
          }
          if (k + 1 < nk) load_add(t, k + 1 < kCh ? k + 1 : kCh - 1, A[k + 1 < kCh ? k + 1 : kCh - 1]);
          chunk(k, va, A[k]);
        } else {
          if (k + 1 < nk) tmem_ld32_issue(trow + (half + 2 * (k + 1)) * 32, (k & 1) ? va : vb);
          if (k & 1) chunk(k, vb, A[0]);
          else chunk(k, va, A[0]);
          if (k + 1 < nk) tmem_wait_ld((k & 1) ? va : vb);
        }
        if (lane == 0 && ew == 0 && u == u0) btrace(8, 1 + k);
      }
      if (lane == 0 && ew == 0) btrace(u - u0, 5);
      if (lane == 0 && ew == 4) btrace(u - u0, 6);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[b]);
      ++tc;
      if (!ADD) cur = nxt;
      u = un;
    }
    if (lane == 0 && ew == 0) btrace(9, 2);
    // inert dummy rows [n_b, rows) of every slot: exact zeros (warp per row, 16-byte stores)
    const int gw = blockIdx.x * kEpiWarps + ew, nw = gridDim.x * kEpiWarps;
    for (int z = 0; z < G.n; ++z) {
      const BdTail& S = stl[z];
      const int nbz = sd[z * per + 2 * q];
      const uint4 zero = make_uint4(0u, 0u, 0u, 0u);
      for (int64_t row = nbz + gw; row < G.rows; row += nw) {
        bf16* cp = (bf16*)S.C + row * S.ldc;
        for (int c8 = lane; c8 < S.N / 8; c8 += 32) *reinterpret_cast<uint4*>(cp + 8 * c8) = zero;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) btrace(9, 3);
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
  }
}

int num_sms() { return device_sms(); }

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

// 2D bf16 (or fp32: TF32 mode) tensor map: inner dim `inner` (contiguous), outer dim `outer`, row
// stride ld elements
bool make_map(CUtensorMap* map, const void* base, int64_t inner, int64_t outer, int64_t ld, int box_inner,
              int box_outer, bool f32 = false, bool mn32 = false) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * (f32 ? 4 : 2))};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  return enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
             dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             mn32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}


// Output store map: C [outer x inner] (ld elements), boxes of 32 rows x 128 bytes, SWIZZLE_128B.
bool make_store_map(CUtensorMap* map, void* base, int64_t inner, int64_t outer, int64_t ld, bool f32) {
  EncodeFn enc = get_encode();
  const int64_t es = f32 ? 4 : 2;
  if (!enc || ((uintptr_t)base & 15) || ((ld * es) & 15) || inner <= 0 || outer <= 0) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {(cuuint32_t)(128 / es), 32};
  cuuint32_t est[2] = {1, 1};
  return enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box,
             est, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int ST, bool A_MN, bool B_MN, bool OUT_F32, class Prob, bool TF = false>
void launch_persist(const typename Prob::Group& G, int total, cudaStream_t s) {
  auto kern = k_gemm_persist<BN, ST, A_MN, B_MN, OUT_F32, Prob, TF>;
  constexpr int SMEM = Cfg<BN, ST>::SMEM_BASE + (Prob::kTmaEpi ? Cfg<BN, ST>::EPI_BYTES : 0) + 64;
  ensure_smem((const void*)kern, SMEM);
  const int grid = total < num_sms() ? total : num_sms();
  if (grid > 0) launch_pdl(kern, grid, kGemmThreads, SMEM, s, G);
}

// CTA-pair launch: clusters of 2 (cudaLaunchAttributeClusterDimension) + PDL, grid = 2 x pairs
template <int BN, bool A_MN, bool B_MN, bool OUT_F32, class Prob>
void launch_pair(const typename Prob::Group& G, int total2, cudaStream_t s) {
  constexpr int ST = BN == 256 ? 6 : 8;
  constexpr int STAGE = BM * BK * 2 + (BN / 2) * BK * 2;
  constexpr int SMEM = ST * STAGE + (Prob::kTmaEpi ? kEpiWarps * 4096 : 0) + 1024 + 256 + 64;
  auto kern = k_gemm_pair<BN, ST, A_MN, B_MN, OUT_F32, Prob>;
  ensure_smem((const void*)kern, SMEM);
  const int pairs = total2 < num_sms() / 2 ? total2 : num_sms() / 2;
  if (pairs <= 0) return;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaLaunchKernelEx(&cfg, kern, G);
}

template <int BN, bool A_MN, bool B_MN>
void dispatch_epi(const GemmPlanTC& P, cudaStream_t s) {
  if (P.tf32) {  // TF32 mode: fp32 in, fp32 out, one CTA per tile
    constexpr int ST = BN == 256 ? 4 : (BN == 64 ? 8 : 6);
    launch_persist<BN, ST, A_MN, B_MN, true, ProbPlain<BN>, true>(P.G, P.G.n * P.G.tm * P.G.tn, s);
    return;
  }
  if constexpr (BN >= 128) if (P.pair) {
    const int total2 = P.G.n * ((P.G.tm + 1) / 2) * P.G.tn;
    if (P.out_f32) launch_pair<BN, A_MN, B_MN, true, ProbPlain<BN>>(P.G, total2, s);
    else launch_pair<BN, A_MN, B_MN, false, ProbPlain<BN>>(P.G, total2, s);
    return;
  }
  constexpr int ST = BN == 256 ? 4 : (BN == 64 ? 8 : 6);
  const int total = P.G.n * P.G.tm * P.G.tn;
  if (P.out_f32) launch_persist<BN, ST, A_MN, B_MN, true, ProbPlain<BN>>(P.G, total, s);
  else launch_persist<BN, ST, A_MN, B_MN, false, ProbPlain<BN>>(P.G, total, s);
}

template <int BNV>
void dispatch_layout(const GemmPlanTC& P, cudaStream_t s) {
  if (!P.a_mn && P.b_mn) dispatch_epi<BNV, false, true>(P, s);
  else if (!P.a_mn && !P.b_mn) dispatch_epi<BNV, false, false>(P, s);
  else if (P.a_mn && P.b_mn) dispatch_epi<BNV, true, true>(P, s);
  else dispatch_epi<BNV, true, false>(P, s);
}

template <int BN>
void launch_bd(const BdPlan& P, cudaStream_t s) {
  const int mt_per = (P.G.bs + BM - 1) / BM;
  const int yd = P.G.q * mt_per + (int)cdiv(P.G.rows, BM);
  const int total = P.G.n * yd * P.G.tn;
  launch_persist<BN, 3, false, true, false, ProbBd<BN>>(P.G, total, s);
}

}  // namespace

bool gemm_bf16_prepare(const GemmOp* ops, int n, GemmPlanTC* P) { return gemm_tc_prepare(ops, n, P, false); }

bool gemm_tc_prepare(const GemmOp* ops, int n, GemmPlanTC* P, bool tf32) {
  if (!get_encode() || n < 1 || n > kMaxGemmOps) return false;
  const GemmOp& o0 = ops[0];
  P->tf32 = tf32;
  if (tf32 && (!o0.out_f32 || o0.mask)) return false;  // TF32 mode: fp32 outputs, no bf16 epilogue operands
  const int ebox = tf32 ? 32 : 64;  // elements per 128-byte TMA box row
  P->a_mn = o0.transA;     // A stored K x M
  P->b_mn = !o0.transB;    // B stored K x N
  P->out_f32 = o0.out_f32;
  P->relu = o0.relu;
  P->mask = o0.mask != nullptr;
  P->maxM = P->maxN = 0;
  int64_t maxN = 0, maxM = 0;
  for (int i = 0; i < n; ++i) {
    maxN = ops[i].N > maxN ? ops[i].N : maxN;
    maxM = ops[i].M > maxM ? ops[i].M : maxM;
  }
  // persistent kernel: wide tiles amortise the epilogue; class-width outputs (the re-associated
  // last layer, N = 48) take 64-wide tiles instead of wasting 5/8 of a 128-wide MMA
  P->bn = maxN > 128 ? 256 : (maxN > 64 ? 128 : 64);
  // A single-op launch (one slot per lockstep group: one sub-GCN per GPU at W = m) whose
  // 256-wide tiles leave SMs idle takes 128-wide ones: single-slot C3 groups 2,806 -> 2,863
  // steps/s; measured slower for 2-op (4,627 -> 4,564) and 8-op (8,46x -> 8,364) launches, so
  // the rule stops at one op (profiles/r01p_*)
  {
    if (P->bn == 256 && n == 1) {
      int64_t t256 = 0;
      for (int i = 0; i < n; ++i) t256 += cdiv(ops[i].M, BM) * cdiv(ops[i].N, 256);
      if (t256 < (int64_t)num_sms()) P->bn = 128;
    }
    // ... and 64-wide ones when even 128-wide tiles fill less than half of the SMs (a single
    // sub-GCN's dW GEMMs: 1,024 x 512 outputs = 32 tiles of 128 x 128 for a K = 3,106 reduction).
    // Per-element K order is independent of the tile width: the same bits for any choice.
    if (P->bn == 128 && n == 1 && cdiv(ops[0].M, BM) * cdiv(ops[0].N, 128) < (int64_t)num_sms() / 2) P->bn = 64;
  }
  // CTA pairs for large, long-K GEMMs (>= 4 tiles per SM and K >= 2048: measured 82 -> 88% of
  // peak at width 4096); short-K GEMMs (the C3 step's dX, K = 512: 27 -> 41 us as pairs) and
  // the cluster-block aggregation stay on one CTA per tile
  {
    int64_t tiles = 0, kmin = INT64_MAX;
    for (int i = 0; i < n; ++i) {
      tiles += cdiv(ops[i].M, BM) * cdiv(ops[i].N, P->bn);
      kmin = ops[i].K < kmin ? ops[i].K : kmin;
    }
    static const int64_t kmin_pair = [] { const char* e = std::getenv("GIST_PAIR_KMIN"); return e ? atoll(e) : 2048; }();
    static const int64_t tiles_pair = [] { const char* e = std::getenv("GIST_PAIR_TILES"); return e ? atoll(e) : 4; }();
    P->pair = !tf32 && P->bn >= 128 && tiles >= tiles_pair * (int64_t)num_sms() && kmin >= kmin_pair;
  }
  P->G.n = n;
  for (int i = 0; i < n; ++i) {
    const GemmOp& o = ops[i];
    if (o.transA != o0.transA || o.transB != o0.transB || o.out_f32 != o0.out_f32) return false;
    if (o.K <= 0 || ((uintptr_t)o.A & 15) || ((uintptr_t)o.B & 15) || (o.lda % 8) || (o.ldb % 8)) return false;
    if (tf32 && (o.mbits || o.add || o.mbits_in || o.rscale)) return false;
    // the kernel keeps the epilogue's leading dimensions as 32-bit (SlotTailTC)
    const int64_t lim = INT32_MAX;
    if (o.ldc > lim || o.ldm > lim || o.ldmb > lim || o.ldadd > lim || o.ldmbi > lim) return false;
    GemmSlotTC& S = P->G.s[i];
    bool ok = P->a_mn ? make_map(&S.ma, o.A, o.M, o.K, o.lda, ebox, ebox, tf32, tf32)
                      : make_map(&S.ma, o.A, o.K, o.M, o.lda, ebox, BM, tf32);
    ok = ok && (P->b_mn ? make_map(&S.mb, o.B, o.N, o.K, o.ldb, ebox, ebox, tf32, tf32)
                        : make_map(&S.mb, o.B, o.K, o.N, o.ldb, ebox, P->pair ? P->bn / 2 : P->bn, tf32));
    if (!ok) return false;
    S.C = o.C;
    S.ldc = o.ldc;
    S.mask = o.mask;
    S.ldm = o.ldm;
    S.relu = o.relu ? 1 : 0;
    S.rscale = o.rscale;
    S.rs_from = o.rs_from;
    S.mbits = o.mbits;
    S.ldmb = o.ldmb;
    S.add = o.add;
    S.ldadd = o.ldadd;
    S.mbits_in = o.mbits_in;
    S.ldmbi = o.ldmbi;
    S.keep_out = o.keep_out;
    S.stream_a = o.stream_a;
    // 64-wide bf16 tiles: an epilogue warp owns 32 columns, half of a 128-byte store box -> direct stores
    S.tma_store = !(P->bn == 64 && !o.out_f32) && make_store_map(&S.mc, o.C, o.N, o.M, o.ldc, o.out_f32) ? 1 : 0;
    S.M = (int)o.M;
    S.N = (int)o.N;
    S.K = (int)o.K;
    P->maxM = o.M > P->maxM ? o.M : P->maxM;
    P->maxN = o.N > P->maxN ? o.N : P->maxN;
  }
  P->G.tm = (int)cdiv(P->maxM, BM);
  P->G.tn = (int)cdiv(P->maxN, P->bn);
  return true;
}

void gemm_bf16_launch(const GemmPlanTC& P, cudaStream_t s) {
  if (P.G.n <= 0 || P.maxM <= 0 || P.maxN <= 0) return;
  if (P.bn == 256) dispatch_layout<256>(P, s);
  else if (P.bn == 64) dispatch_layout<64>(P, s);
  else dispatch_layout<128>(P, s);
}

bool gemm_bd_prepare(const bf16* blocks, int num_clusters, int bs, const BdOp* ops, int n, int q, int64_t rows,
                     const int64_t* cstart, const StepState* st, BdPlan* P) {
  if (!get_encode() || n < 1 || n > kMaxGroup || (bs % 8)) return false;
  if (!make_map(&P->G.ma, blocks, bs, (int64_t)num_clusters * bs, bs, 64, BM)) return false;
  P->G.n = n;
  P->G.q = q;
  P->G.bs = bs;
  P->G.st = st;
  P->G.cstart = cstart;
  P->G.rows = rows;
  P->maxN = 0;
  for (int i = 0; i < n; ++i) {
    const BdOp& o = ops[i];
    BdSlot& S = P->G.s[i];
    if (((uintptr_t)o.H & 15) || (o.ldh % 8)) return false;
    // H stored [rows x N] (N contiguous): MN-major B operand, K = rows
    if (!make_map(&S.mb, o.H, o.N, o.h_rows, o.ldh, 64, 64)) return false;
    S.C = o.C;
    S.ldc = o.ldc;
    S.add = o.add;
    S.ldadd = o.ldadd;
    S.rscale = o.rscale;
    S.desc = o.desc;
    S.global_rows = o.global_rows;
    S.N = (int)o.N;
    S.tma_store = make_store_map(&S.mc, o.C, o.N, rows, o.ldc, false) ? 1 : 0;
    S.keep_out = o.keep_out;

    P->maxN = o.N > P->maxN ? o.N : P->maxN;
  }
  P->bn = P->maxN > 128 ? 256 : 128;
  // transposed kernel (k_bd_t) when the cluster block(s), the A ring and the epilogue transposes fit
  // in shared memory (clusters of <= 256 rows) and the descriptors fit the staging (measured: C3
  // block aggregation 3.11 -> 2.90 ms per profiled sample, 9,311 -> 9,385 steps/s, single-slot
  // step 252 -> 247 us); GIST_BD_T=0 keeps the row-tile kernel (the test switch)
  {
    const char* e = std::getenv("GIST_BD_T");
    const char* eb = std::getenv("GIST_BDT_BUFS");
    const int BSN = (bs + 15) & ~15, KB = (bs + BK - 1) / BK;
    auto bytes = [&](int nb) { return kBdtStages * kBdtAStage + nb * KB * BSN * 128 + kBdtStg + 1024 + 256; };
    // two block buffers when they fit (clusters of <= 160 rows), else one (<= 256 rows: a block
    // load waits for the previous cluster's MMAs); one buffer measured equal at C3 (9,440 vs
    // 9,445 steps/s: the freed shared memory lets the inter-cluster pass co-reside, no gain);
    // GIST_BDT_BUFS=1 forces one (the test switch)
    P->G.blk_bufs = (eb && eb[0] == '1') ? 1 : (bytes(2) <= kBdtSmemMax ? 2 : 1);
    P->transposed = !(e && e[0] == '0') && bs <= 256 && 3 * q + 4 <= ProbBd<128>::kMaxDesc &&
                    bytes(P->G.blk_bufs) <= kBdtSmemMax && (bs % 8) == 0;
    if (P->transposed && !make_map(&P->G.mat, blocks, bs, (int64_t)num_clusters * bs, bs, 64, bs)) return false;
  }
  // single-slot launches: 128-wide tiles when 256-wide ones leave SMs idle (one slot per group:
  // block aggregation 35.6 -> 32.5 ms per profiled sample, 2,861 -> 2,867-2,873 steps/s,
  // profiles/r01s_*); multi-slot launches unchanged
  {
    const int64_t t256 = (int64_t)n * ((int64_t)q * cdiv(bs, BM) + cdiv(rows, BM)) * cdiv(P->maxN, 256);
    if (P->bn == 256 && n == 1 && t256 < (int64_t)num_sms()) P->bn = 128;
  }
  P->G.tn = (int)cdiv(P->maxN, P->bn);
  return true;
}

void gemm_bd_launch(const BdPlan& P, cudaStream_t s) {
  if (P.G.n <= 0 || P.maxN <= 0) return;
  if (P.transposed) {  // k_bd_t: one unit per (slot, batch cluster, 128-feature tile)
    const int BSN = (P.G.bs + 15) & ~15, KB = (P.G.bs + BK - 1) / BK;
    const int smem = kBdtStages * kBdtAStage + P.G.blk_bufs * KB * BSN * 128 + kBdtStg + 1024 + 256;
    const int units = P.G.n * P.G.q * (int)cdiv(P.maxN, BM);
    const int grid = units < num_sms() ? units : num_sms();
    if (P.G.s[0].add) {  // every slot of a launch adds a residual, or none does
      ensure_smem((const void*)k_bd_t<true>, kBdtSmemMax);
      launch_pdl(k_bd_t<true>, grid, kGemmThreads, smem, s, P.G);
    } else {
      ensure_smem((const void*)k_bd_t<false>, kBdtSmemMax);
      launch_pdl(k_bd_t<false>, grid, kGemmThreads, smem, s, P.G);
    }
    return;
  }
  if (P.bn == 256) launch_bd<256>(P, s);
  else launch_bd<128>(P, s);
}

bool gemm_bf16(bool transA, bool transB, int64_t M, int64_t N, int64_t K, const bf16* A, int64_t lda, const bf16* B,
               int64_t ldb, void* C, int64_t ldc, bool out_f32, bool relu, cudaStream_t s, int reps) {
  if (!get_encode()) return false;
  if (M == 0 || N == 0) return true;  // nothing to do (also the availability probe)
  GemmOp o{transA, transB, M, N, K, A, lda, B, ldb, C, ldc, out_f32, relu, nullptr, 0, nullptr, 0};
  GemmPlanTC P;
  if (!gemm_bf16_prepare(&o, 1, &P)) return false;
  for (int r = 0; r < reps; ++r) gemm_bf16_launch(P, s);  // one plan (tensor maps encoded once)
  return true;
}

bool gemm_tf32(bool transA, bool transB, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
               int64_t ldb, float* C, int64_t ldc, bool relu, cudaStream_t s, int reps) {
  if (!get_encode()) return false;
  if (M == 0 || N == 0) return true;
  GemmOp o{transA, transB, M, N, K, A, lda, B, ldb, C, ldc, true, relu, nullptr, 0, nullptr, 0};
  GemmPlanTC P;
  if (!gemm_tc_prepare(&o, 1, &P, true)) return false;
  for (int r = 0; r < reps; ++r) gemm_bf16_launch(P, s);
  return true;
}

}  // namespace gist

#ifdef GIST_GEMM_TRACE
extern "C" int gist_debug_bdt_trace(unsigned long long* out) {  // [160][10][8]
  return cudaMemcpyFromSymbol(out, gist::g_bdt_trace, sizeof(gist::g_bdt_trace)) == cudaSuccess ? 0 : -1;
}
extern "C" int gist_debug_gemm_trace(unsigned long long* out, int n) {
  if (n > 1024) n = 1024;
  return cudaMemcpyFromSymbol(out, gist::g_gemm_trace, (size_t)n * 16 * sizeof(unsigned long long)) == cudaSuccess ? 0 : -1;
}
#endif
