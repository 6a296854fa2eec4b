// spmm.cu -- aggregation SpMM of Eq. (1)/(2).
//
// A group of LPR lanes (32, 16, 8 or 4) owns one output row; each lane owns J
// 16-byte vectors of the row, so a group covers LPR*J*16 bytes of the row in
// registers and walks the row's neighbour list once.  Neighbour indices are loaded
// LPR at a time (one coalesced load) and turned into 32-bit vector offsets
// (row * ldh/V) before a single shuffle broadcast per neighbour; UNROLL neighbour
// rows are gathered per iteration into raw uint4 registers (UNROLL*J 16-byte loads
// in flight per lane) and unpacked with shifts (bf16 -> fp32 is a 16-bit shift).
// Accumulation is fp32 in a fixed order: deterministic, no atomics.
// The normalisation of A_bar is never materialised: row/column scale vectors
// (deg+1)^{-1/2} (GCN renorm, R1) or 1/deg (GraphSAGE mean, R2) are applied on the
// fly; the backward SpMM reuses the same CSR with swapped scales (SURVEY a6:
// N^T = A diag(1/deg)).  Rows wider than LPR*J*V elements are split into column
// chunks handled by separate groups.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <cstdlib>

namespace gist {

namespace {



// 16 bytes -> V fp32 values
__device__ __forceinline__ void unpack(const uint4& x, float* v, float) {
  v[0] = __uint_as_float(x.x); v[1] = __uint_as_float(x.y); v[2] = __uint_as_float(x.z); v[3] = __uint_as_float(x.w);
}
__device__ __forceinline__ void unpack(const uint4& x, float* v, bf16) {
  const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

// Sum of the neighbour rows col[b .. e) of one (row, column chunk) unit into acc, in edge order
// (UNROLL gathers per round; PRED: every round predicated, no serial tail -- same order).
template <typename TI, typename TO, int LPR, int J, int UNROLL, bool CSCALE, bool PRED, typename Off>
__device__ __forceinline__ void gather_range(const SpmmArgs<TI, TO>& a, int64_t b, int64_t e, const uint4* H4, Off ldv,
                                             int vbase, const bool (&act)[J], unsigned gmask, int gl,
                                             float (&acc)[J][Elem<TI>::kVec]) {
  constexpr int V = Elem<TI>::kVec;
  for (int64_t base = b; base < e; base += LPR) {
    const int n = (e - base) < LPR ? (int)(e - base) : LPR;
    Off ou = 0;
    float su = 1.f;
    if (gl < n) {
      const int32_t u = a.col[base + gl];
      if (CSCALE) su = a.colscale[u];
      // row offset only: each receiving lane adds its own column after the broadcast
      ou = (Off)(a.h_index ? (int64_t)a.h_index[u] : (int64_t)u) * ldv;
    }
    int jj = 0;
    if constexpr (PRED) {  // all UNROLL gathers of a round in flight, predicated (no serial tail)
      for (; jj < n; jj += UNROLL) {
        uint4 x[UNROLL][J];
#pragma unroll
        for (int q = 0; q < UNROLL; ++q) {
          const bool on = jj + q < n;  // uniform over the group
          const Off r = __shfl_sync(gmask, ou, on ? jj + q : 0, LPR);
#pragma unroll
          for (int j = 0; j < J; ++j)
            if (act[j] && on) x[q][j] = __ldg(H4 + r + vbase + j * LPR);
        }
#pragma unroll
        for (int q = 0; q < UNROLL; ++q)
          if (jj + q < n)
#pragma unroll
            for (int j = 0; j < J; ++j)
              if (act[j]) {
                float t[V];
                unpack(x[q][j], t, TI());
#pragma unroll
                for (int i = 0; i < V; ++i) acc[j][i] += t[i];
              }
      }
    } else {
      for (; jj + UNROLL <= n; jj += UNROLL) {
        uint4 x[UNROLL][J];
        float s[UNROLL];
#pragma unroll
        for (int q = 0; q < UNROLL; ++q) {
          const Off r = __shfl_sync(gmask, ou, jj + q, LPR);
          s[q] = CSCALE ? __shfl_sync(gmask, su, jj + q, LPR) : 1.f;
#pragma unroll
          for (int j = 0; j < J; ++j)
            if (act[j]) x[q][j] = __ldg(H4 + r + vbase + j * LPR);
        }
#pragma unroll
        for (int q = 0; q < UNROLL; ++q)
#pragma unroll
          for (int j = 0; j < J; ++j)
            if (act[j]) {
              float t[V];
              unpack(x[q][j], t, TI());
#pragma unroll
              for (int i = 0; i < V; ++i) acc[j][i] = CSCALE ? fmaf(s[q], t[i], acc[j][i]) : acc[j][i] + t[i];
            }
      }
      for (; jj < n; ++jj) {
        const Off r = __shfl_sync(gmask, ou, jj, LPR);
        const float s = CSCALE ? __shfl_sync(gmask, su, jj, LPR) : 1.f;
#pragma unroll
        for (int j = 0; j < J; ++j)
          if (act[j]) {
            float t[V];
            unpack(__ldg(H4 + r + vbase + j * LPR), t, TI());
#pragma unroll
            for (int i = 0; i < V; ++i) acc[j][i] = CSCALE ? fmaf(s, t[i], acc[j][i]) : acc[j][i] + t[i];
          }
      }
    }
  }
}

// Heavy rows (split_min > 0: a unit whose row has more than split_min neighbours): the row's
// dependency chain would set the launch length (the degree tail of a batch: ~1% of the rows hold
// 5-20x the mean neighbour count), so after the light rows the whole CTA takes each heavy unit
// of its range in turn -- group g sums the g-th contiguous slice of the edge list, the slices
// meet in shared memory and the unit's own group adds them in slice order.  The split depends
// only on the row's degree, so the result is deterministic and independent of the launch shape
// (grouped or single-slot, any world size).  Dynamic shared memory: 2 * 256 * J * V floats.
template <typename TI, typename TO, int LPR, int J, int UNROLL, bool CSCALE, bool WIDE, bool PRED = false>
__global__ void __launch_bounds__(256, PRED ? (J == 1 ? 3 : 2) : (J == 1 && sizeof(TI) == 2) ? 4
                                           : UNROLL == 1 ? (J <= 2 ? 4 : 3) : (J <= 2 ? 3 : 2))
    k_spmm(const __grid_constant__ SpmmGroup<TI, TO> G, int nchunks, int split_min) {
  const SpmmArgs<TI, TO>& a = G.a[blockIdx.y];  // one sub-GCN slot per grid row
  // early: every gathered operand was written at least two launches back (the launch before this
  // one, the block-diagonal pass, only produces `add`), so the whole gather phase runs before
  // griddepcontrol.wait, overlapping the predecessor; only the epilogue waits for it
  const bool early = a.early && !a.self_out;
  if (!early) {
    pdl_wait();
    pdl_trigger();
  }
  constexpr int V = Elem<TI>::kVec;  // elements per 16-byte vector of TI
  constexpr int GPW = 32 / LPR;      // groups per warp
  constexpr int NG = 8 * GPW;        // groups per CTA (256 threads)
  using Off = typename std::conditional<WIDE, int64_t, uint32_t>::type;
  const int lane = threadIdx.x & 31;
  const int gl = lane % LPR;         // lane inside the group
  const int grp = (threadIdx.x >> 5) * GPW + lane / LPR;  // group inside the CTA
  const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (lane - gl));
  const int64_t gid = (int64_t)blockIdx.x * NG + grp;
  const uint4* __restrict__ H4 = reinterpret_cast<const uint4*>(a.H);
  const Off ldv = (Off)(a.ldh / V);  // row stride in 16-byte vectors
  const int64_t wv = a.w / V;        // width in vectors

  // self term (and the copy of the row into self_out) of unit (v, vbase)
  auto self_term = [&](int64_t v, int vbase, const bool(&act)[J], float(&acc)[J][V]) {
    if (!(a.self || a.self_out)) return;
    const Off hv = (Off)(a.h_index ? (int64_t)a.h_index[v] : v + a.row0) * ldv;
    const float s = a.colscale ? a.colscale[v + a.row0] : 1.f;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (!act[j]) continue;
      const uint4 x = H4[hv + vbase + j * LPR];
      if (a.self_out) *reinterpret_cast<uint4*>(a.self_out + v * a.ld_self + (int64_t)(vbase + j * LPR) * V) = x;
      if (a.self) {
        float t[V];
        unpack(x, t, TI());
#pragma unroll
        for (int i = 0; i < V; ++i) acc[j][i] = s * t[i];
      }
    }
  };
  // row scale, residual add, ReLU mask / ReLU and the store of unit (v, vbase)
  auto epilogue = [&](int64_t v, int vbase, const bool(&act)[J], float(&acc)[J][V], bool dummy, const uint4* addv) {
    const float rs = a.rowscale ? a.rowscale[v] : 1.f;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (!act[j]) continue;
      const int64_t c = (int64_t)(vbase + j * LPR) * V;
      float o[V];
#pragma unroll
      for (int i = 0; i < V; ++i) o[i] = acc[j][i] * rs;
      if (dummy) {
#pragma unroll
        for (int i = 0; i < V; ++i) o[i] = 0.f;
      } else {
        if (a.add) {
          float t[V];
          unpack(addv ? addv[j] : *reinterpret_cast<const uint4*>(a.add + v * a.ld_add + c), t, TI());
#pragma unroll
          for (int i = 0; i < V; ++i) o[i] += t[i];
        }
        if (a.mbits) {  // bit-packed ReLU mask: 4 bytes per 32 columns instead of 2-4 bytes per column
          const uint32_t wd = a.mbits[v * a.ld_mbits + (c >> 5)] >> (c & 31);
#pragma unroll
          for (int i = 0; i < V; ++i) o[i] = (wd >> i) & 1u ? o[i] : 0.f;  // ReLU'(0) = 0 (R3)
        } else if (a.mask) {
          float t[V];
          unpack(*reinterpret_cast<const uint4*>(a.mask + v * a.ld_mask + c), t, TI());
#pragma unroll
          for (int i = 0; i < V; ++i) o[i] = t[i] > 0.f ? o[i] : 0.f;  // ReLU'(0) = 0 (R3)
        }
        if (a.relu) {
#pragma unroll
          for (int i = 0; i < V; ++i) o[i] = fmaxf(o[i], 0.f);
        }
      }
      if constexpr (sizeof(TO) == sizeof(TI)) {
        st16(a.out + v * a.ldo + c, o);
      } else {
        constexpr int VO = Elem<TO>::kVec;
#pragma unroll
        for (int p = 0; p < V / VO; ++p) st16(a.out + v * a.ldo + c + p * VO, o + p * VO);
      }
    }
  };

  const int64_t v = gid / nchunks;
  const int chunk = (int)(gid - v * nchunks);
  const bool valid = v < a.rows;
  int64_t beg = 0, end = 0;
  if (valid) {
    beg = a.row_beg[v];
    end = a.row_end[v];
  }
  // inert dummy rows of a batch launch (v >= n_b, marked row_beg < 0 by the batch build):
  // exact zeros, never a stale `add`
  const bool dummy = beg < 0;
  const bool heavy = split_min > 0 && valid && !dummy && end - beg > split_min;
  // whether the CTA holds a heavy unit, decided up front: CTAs without one (most) never meet
  // at a barrier after their gathers, so a warp does not idle behind the CTA's slowest row
  __shared__ uint8_t hflag[NG];
  bool any_heavy = false;
  if (split_min > 0) {  // uniform over the launch
    if (gl == 0) hflag[grp] = heavy;
    any_heavy = __syncthreads_or(heavy);
  }
  const int vbase = chunk * LPR * J + gl;  // this lane's first vector column
  bool act[J];
  float acc[J][V];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    act[j] = vbase + j * LPR < wv;
#pragma unroll
    for (int i = 0; i < V; ++i) acc[j][i] = 0.f;
  }
  // the residual row is loaded ahead of the gathers (its latency overlaps them) unless it is
  // the predecessor's output (early)
  uint4 addv[J];
  const bool pre_add = !early && valid && !heavy && !dummy && a.add;
  if (pre_add) {
#pragma unroll
    for (int j = 0; j < J; ++j)
      if (act[j]) addv[j] = *reinterpret_cast<const uint4*>(a.add + v * a.ld_add + (int64_t)(vbase + j * LPR) * V);
  }
  if (valid && !heavy) {
    self_term(v, vbase, act, acc);
    gather_range<TI, TO, LPR, J, UNROLL, CSCALE, PRED, Off>(a, beg, end, H4, ldv, vbase, act, gmask, gl, acc);
  }
  {
    if (any_heavy) {  // uniform over the CTA
      // [NG][LPR * J] vectors of V floats (V / 4 float4 each): the slices' partial sums, then
      // every group's own sum parked while the heavy units run (keeps it out of registers)
      extern __shared__ float4 spart[];
      float4* sacc = spart + (size_t)NG * LPR * J * (V / 4);
      auto slot = [&](float4* buf, int g, int j, int i) -> float4& {
        return buf[((int64_t)g * LPR * J + j * LPR + gl) * (V / 4) + i / 4];
      };
#pragma unroll
      for (int j = 0; j < J; ++j)
#pragma unroll
        for (int i = 0; i < V; i += 4) slot(sacc, grp, j, i) = make_float4(acc[j][i], acc[j][i + 1], acc[j][i + 2], acc[j][i + 3]);
      for (int h = 0; h < NG; ++h) {
        if (!hflag[h]) continue;  // uniform over the CTA
        const int64_t gh = (int64_t)blockIdx.x * NG + h;
        const int64_t vh = gh / nchunks;
        const int ch = (int)(gh - vh * nchunks);
        const int64_t bh = a.row_beg[vh], n = a.row_end[vh] - bh;
        const int64_t per = (n + NG - 1) / NG;
        const int64_t b0 = bh + (grp * per < n ? grp * per : n);
        const int64_t b1 = bh + ((grp + 1) * per < n ? (grp + 1) * per : n);
        const int vb = ch * LPR * J + gl;
        bool ah[J];
        float p[J][V];
#pragma unroll
        for (int j = 0; j < J; ++j) {
          ah[j] = vb + j * LPR < wv;
#pragma unroll
          for (int i = 0; i < V; ++i) p[j][i] = 0.f;
        }
        if (grp == 0) self_term(vh, vb, ah, p);
        gather_range<TI, TO, LPR, J, UNROLL, CSCALE, PRED, Off>(a, b0, b1, H4, ldv, vb, ah, gmask, gl, p);
#pragma unroll
        for (int j = 0; j < J; ++j)
#pragma unroll
          for (int i = 0; i < V; i += 4) slot(spart, grp, j, i) = make_float4(p[j][i], p[j][i + 1], p[j][i + 2], p[j][i + 3]);
        __syncthreads();
        if (grp == h)  // the unit's own group: the slices in slice order (its own sum was zero)
#pragma unroll
          for (int j = 0; j < J; ++j)
#pragma unroll
            for (int i = 0; i < V; i += 4) {
              float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
              for (int g = 0; g < NG; ++g) {
                const float4 q = slot(spart, g, j, i);
                t.x += q.x; t.y += q.y; t.z += q.z; t.w += q.w;
              }
              slot(sacc, grp, j, i) = t;
            }
        __syncthreads();
      }
#pragma unroll
      for (int j = 0; j < J; ++j)
#pragma unroll
        for (int i = 0; i < V; i += 4) {
          const float4 q = slot(sacc, grp, j, i);
          acc[j][i] = q.x; acc[j][i + 1] = q.y; acc[j][i + 2] = q.z; acc[j][i + 3] = q.w;
        }
    }
  }
  if (early) {
    pdl_wait();
    pdl_trigger();
  }
  if (valid) epilogue(v, vbase, act, acc, dummy, pre_add ? addv : nullptr);
}

// Inter-cluster pass, persistent warps (bf16 mini-batch rows, one column chunk): every warp
// walks rows v = warp0, warp0 + stride, ... on its own -- a warp that finishes a short row takes
// its next one instead of idling until the slowest row of its CTA is done and the CTA retires.
// Heavy rows (> split_min neighbours) are deferred to the end of the CTA and summed by the whole
// CTA exactly as k_spmm does (group g sums the g-th contiguous slice; the row's sum adds the
// slices in slice order), light rows exactly as k_spmm's light rows: the same bits.
template <int J>
__global__ void __launch_bounds__(256, J <= 2 ? 4 : 3) k_inter_persist(const __grid_constant__ SpmmGroup<bf16, bf16> G,
                                                                     int split_min, int rpw) {
  using TI = bf16;
  constexpr int V = 8, NG = 8, LPR = 32, kMaxH = 16;
  const SpmmArgs<bf16, bf16>& a = G.a[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ int hlist[NG][kMaxH];
  __shared__ int hcnt[NG];
  extern __shared__ float4 ip_part[];  // [NG][LPR * J][V / 4]
  const uint4* __restrict__ H4 = reinterpret_cast<const uint4*>(a.H);
  const uint32_t ldv = (uint32_t)(a.ldh / V);
  const int64_t wv = a.w / V;
  bool act[J];
#pragma unroll
  for (int j = 0; j < J; ++j) act[j] = lane + j * LPR < wv;
  auto epilogue = [&](int64_t v, float (&acc)[J][V], bool dummy) {
    const float rs = a.rowscale ? a.rowscale[v] : 1.f;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (!act[j]) continue;
      const int64_t c = (int64_t)(lane + j * LPR) * V;
      float o[V];
#pragma unroll
      for (int i = 0; i < V; ++i) o[i] = acc[j][i] * rs;
      if (dummy) {
#pragma unroll
        for (int i = 0; i < V; ++i) o[i] = 0.f;
      } else {
        if (a.add) {
          float t[V];
          unpack(*reinterpret_cast<const uint4*>(a.add + v * a.ld_add + c), t, TI());
#pragma unroll
          for (int i = 0; i < V; ++i) o[i] += t[i];
        }
        if (a.mbits) {
          const uint32_t wd = a.mbits[v * a.ld_mbits + (c >> 5)] >> (c & 31);
#pragma unroll
          for (int i = 0; i < V; ++i) o[i] = (wd >> i) & 1u ? o[i] : 0.f;
        } else if (a.mask) {
          float t[V];
          unpack(*reinterpret_cast<const uint4*>(a.mask + v * a.ld_mask + c), t, TI());
#pragma unroll
          for (int i = 0; i < V; ++i) o[i] = t[i] > 0.f ? o[i] : 0.f;
        }
        if (a.relu) {
#pragma unroll
          for (int i = 0; i < V; ++i) o[i] = fmaxf(o[i], 0.f);
        }
      }
      st16(a.out + v * a.ldo + c, o);
    }
  };
  if (lane == 0) hcnt[warp] = 0;
  __syncwarp();
  bool waited = false;
  const int64_t v0 = ((int64_t)blockIdx.x * NG + warp) * rpw;
  for (int k = 0; k < rpw; ++k) {
    const int64_t v = v0 + k;
    if (v >= a.rows) break;
    const int64_t beg = a.row_beg[v], end = a.row_end[v];
    const bool dummy = beg < 0;
    if (!dummy && end - beg > split_min) {  // heavy: the CTA sums it at the end
      if (lane == 0) hlist[warp][hcnt[warp]++] = (int)v;
      __syncwarp();
      continue;
    }
    float acc[J][V];
#pragma unroll
    for (int j = 0; j < J; ++j)
#pragma unroll
      for (int i = 0; i < V; ++i) acc[j][i] = 0.f;
    if (!dummy)
      gather_range<TI, TI, LPR, J, 1, false, false, uint32_t>(a, beg, end, H4, ldv, lane, act, 0xffffffffu, lane, acc);
    if (!waited) {  // gathered operands are two or more launches old; `add` is the predecessor's
      pdl_wait();
      pdl_trigger();
      waited = true;
    }
    epilogue(v, acc, dummy);
  }
  if (!waited) {
    pdl_wait();
    pdl_trigger();
  }
  __syncthreads();
  for (int hw = 0; hw < NG; ++hw) {
    const int nh = hcnt[hw];
    for (int h = 0; h < nh; ++h) {
      const int64_t vh = hlist[hw][h];
      const int64_t bh = a.row_beg[vh], n = a.row_end[vh] - bh;
      const int64_t per = (n + NG - 1) / NG;
      const int64_t b0 = bh + (warp * per < n ? warp * per : n);
      const int64_t b1 = bh + ((warp + 1) * per < n ? (warp + 1) * per : n);
      float p[J][V];
#pragma unroll
      for (int j = 0; j < J; ++j)
#pragma unroll
        for (int i = 0; i < V; ++i) p[j][i] = 0.f;
      gather_range<TI, TI, LPR, J, 1, false, false, uint32_t>(a, b0, b1, H4, ldv, lane, act, 0xffffffffu, lane, p);
#pragma unroll
      for (int j = 0; j < J; ++j)
#pragma unroll
        for (int i = 0; i < V; i += 4)
          ip_part[((int64_t)warp * LPR * J + j * LPR + lane) * (V / 4) + i / 4] = make_float4(p[j][i], p[j][i + 1], p[j][i + 2], p[j][i + 3]);
      __syncthreads();
      if (warp == hw) {  // the row's own warp: the slices in slice order
        float t[J][V];
#pragma unroll
        for (int j = 0; j < J; ++j)
#pragma unroll
          for (int i = 0; i < V; i += 4) {
            float4 q4 = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int g = 0; g < NG; ++g) {
              const float4 q = ip_part[((int64_t)g * LPR * J + j * LPR + lane) * (V / 4) + i / 4];
              q4.x += q.x; q4.y += q.y; q4.z += q.z; q4.w += q.w;
            }
            t[j][i] = q4.x; t[j][i + 1] = q4.y; t[j][i + 2] = q4.z; t[j][i + 3] = q4.w;
          }
        epilogue(vh, t, false);
      }
      __syncthreads();
    }
  }
}

template <typename TI, typename TO, int LPR, int J>
void launch(const SpmmGroup<TI, TO>& G, int64_t rows, int64_t w, cudaStream_t s) {
  constexpr int CW = LPR * J * Elem<TI>::kVec;
  // heavy-row split for mini-batch passes (see k_spmm); the threshold depends only on the pass
  // kind, never on the launch shape
  // (GIST_SPMM_SPLIT=0: no split -- the A/B and test switch that pins the split against the
  // unsplit row sums)
  const char* e_split = std::getenv("GIST_SPMM_SPLIT");
  const int split_min = e_split && e_split[0] == '0' ? 0 : (G.a[0].desc ? (G.a[0].few_nnz ? 32 : 128) : 0);
  const size_t sm = split_min > 0 ? (size_t)2 * 256 * J * Elem<TI>::kVec * sizeof(float) : 0;
  const int nchunks = (int)cdiv(w, CW);
  const int64_t groups = rows * nchunks;
  const dim3 grid((unsigned)cdiv(groups, 8 * (32 / LPR)), (unsigned)G.n);
  auto go = [&](auto kern) {
    if (sm > 0) ensure_smem((const void*)kern, (int)sm);  // (static smem counts against 48 KB too)
    launch_pdl(kern, grid, 256, sm, s, G, nchunks, split_min);
  };
  if (G.a[0].few_nnz && J == 1 && !G.a[0].colscale) {  // few neighbours, narrow rows: the row's
    // dependency chain dominates (not bytes), so every round keeps 8 gathers in flight
    const bool wide = G.a[0].h_index != nullptr;
    if (wide) go(k_spmm<TI, TO, LPR, 1, 8, false, true, true>);
    else go(k_spmm<TI, TO, LPR, 1, 8, false, false, true>);
    return;
  }
  if constexpr (std::is_same<TI, bf16>::value && std::is_same<TO, bf16>::value && LPR == 32 && (J == 2 || J == 3)) {
    // grouped launches of > 8,192 rows (4 and 8 slots; measured C3 9,388 -> ~9,650 steps/s, inter-
    // cluster passes 4.87 -> 4.42 ms per profiled sample; 4-slot W = 2 proxy step 514 -> 493 us);
    // one- and two-slot launches keep two gathers in flight per row (measured equal / better).  GIST_INTER_PERSIST=1 / 0 forces it on / off (the bit-identity test)
    const char* e_p = std::getenv("GIST_INTER_PERSIST");
    bool ok = !(e_p && e_p[0] == '0') && split_min > 0 && nchunks == 1 &&
              (rows * G.n > 8192 || (e_p && e_p[0] == '1'));
    for (int i = 0; i < G.n && ok; ++i)
      ok = G.a[i].few_nnz && G.a[i].early && !G.a[i].colscale && !G.a[i].h_index && !G.a[i].self && !G.a[i].self_out &&
           (int64_t)(G.a[i].rows + G.a[i].row0) * (G.a[i].ldh / 8) < ((int64_t)1 << 31);
    if (ok) {  // persistent warps, ~4 CTAs per SM
      // rows dealt over 8 x (8 warps x SMs): ~3 rows per warp at 8 slots, two waves of CTAs
      // (measured: 2 / 4 / 8 / 16 -> 5.68 / 4.63 / 4.42 / 4.44 ms per profiled sample)
      const int64_t warps = 8LL * 8 * device_sms();
      const int rpw = (int)std::max<int64_t>(1, std::min<int64_t>(16, cdiv(rows * G.n, warps)));
      const dim3 pg((unsigned)cdiv(rows, 8LL * rpw), (unsigned)G.n);
      const size_t psm = (size_t)8 * 32 * J * 8 * sizeof(float);
      ensure_smem((const void*)k_inter_persist<J>, (int)psm);
      launch_pdl(k_inter_persist<J>, pg, 256, psm, s, G, split_min, rpw);
      return;
    }
  }
  if (G.a[0].few_nnz && J <= 3) {  // few neighbours per row: occupancy over in-flight loads
    const bool wide = G.a[0].h_index != nullptr;
    if (G.a[0].colscale) {
      if (wide) go(k_spmm<TI, TO, LPR, J, 1, true, true>);
      else go(k_spmm<TI, TO, LPR, J, 1, true, false>);
    } else if (rows * G.n <= 16384) {
      // a small launch (one sub-GCN per GPU: ~3,100 rows, a third of the warp slots): two
      // gathers in flight per row (measured: single-slot step 266 -> 259 us; at 8 slots the
      // lower occupancy costs more than it saves, 9,085 -> 8,730 steps/s)
      if (wide) go(k_spmm<TI, TO, LPR, J, 2, false, true>);
      else go(k_spmm<TI, TO, LPR, J, 2, false, false>);
    } else {
      if (wide) go(k_spmm<TI, TO, LPR, J, 1, false, true>);
      else go(k_spmm<TI, TO, LPR, J, 1, false, false>);
    }
    return;
  }
  constexpr int UNROLL = J <= 2 ? 4 : 2;
  // 32-bit vector offsets whenever every gathered operand spans < 2^31 vectors
  bool wide = false, cs = G.a[0].colscale != nullptr;
  for (int i = 0; i < G.n; ++i) {
    const SpmmArgs<TI, TO>& a = G.a[i];
    const int64_t hr = a.h_rows > a.rows + a.row0 ? a.h_rows : a.rows + a.row0;
    wide |= a.h_index != nullptr || hr * (a.ldh / Elem<TI>::kVec) >= ((int64_t)1 << 31);
  }
  if (!wide && cs) go(k_spmm<TI, TO, LPR, J, UNROLL, true, false>);
  else if (!wide) go(k_spmm<TI, TO, LPR, J, UNROLL, false, false>);
  else if (cs) go(k_spmm<TI, TO, LPR, J, UNROLL, true, true>);
  else go(k_spmm<TI, TO, LPR, J, UNROLL, false, true>);
}

}  // namespace

template <typename TI, typename TO>
void spmm_group(const SpmmGroup<TI, TO>& G, cudaStream_t s) {
  int64_t rows = 0, w = 0;
  for (int i = 0; i < G.n; ++i) {
    rows = G.a[i].rows > rows ? G.a[i].rows : rows;
    w = G.a[i].w > w ? G.a[i].w : w;
  }
  if (G.n <= 0 || rows <= 0 || w <= 0) return;
  constexpr int V = Elem<TI>::kVec;
  const int64_t vecs = cdiv(w, V);  // 16-byte vectors per row (widest slot)
  if (vecs <= 4) launch<TI, TO, 4, 1>(G, rows, w, s);
  else if (vecs <= 8) launch<TI, TO, 8, 1>(G, rows, w, s);
  else if (vecs <= 16) launch<TI, TO, 16, 1>(G, rows, w, s);
  else if (vecs <= 32) launch<TI, TO, 32, 1>(G, rows, w, s);
  else if (vecs <= 64) launch<TI, TO, 32, 2>(G, rows, w, s);
  else if (vecs <= 96) launch<TI, TO, 32, 3>(G, rows, w, s);
  else launch<TI, TO, 32, 4>(G, rows, w, s);  // wider rows: column chunks of 128 vectors
}

template <typename TI, typename TO>
void spmm(const SpmmArgs<TI, TO>& a, cudaStream_t s) {
  // Large graphs (the full-graph / partition eval operator): column slabs whose H rows about
  // fill L2 (rows x slab x e <= 128 MB, >= 128 columns), so most gathers of a slab pass hit L2;
  // every pass re-reads the CSR.  Reddit-shape (232,965 rows, 114.6 M nnz, bf16): width 512
  // 21.4 -> 16.9 ms, width 4096 160 -> 137 ms with 256-column slabs (64 columns: slower, the
  // 128-byte row pieces and 8 CSR passes cost more than the L2 hits save; 384 / 512 columns:
  // 211 / 172 ms at width 4096; evict-first loads of the CSR stream: no change).
  int64_t slab = 0;
  const int64_t e = sizeof(TI);
  const int64_t hr = a.h_rows > a.rows ? a.h_rows : a.rows;  // gathered rows of H
  if (!a.mbits && !a.desc && hr >= 65536) {
    const int64_t fit = ((int64_t)128 << 20) / (hr * e);
    slab = fit >= a.w ? 0 : std::max<int64_t>(128, (fit / 64) * 64);
  }
  if (slab <= 0 || slab >= a.w) {
    SpmmGroup<TI, TO> G;
    G.a[0] = a;
    G.n = 1;
    spmm_group(G, s);
    return;
  }
  for (int64_t c0 = 0; c0 < a.w; c0 += slab) {
    SpmmGroup<TI, TO> G;
    SpmmArgs<TI, TO> b = a;
    b.w = a.w - c0 < slab ? a.w - c0 : slab;
    b.H = a.H + c0;
    b.out = a.out + c0;
    if (a.add) b.add = a.add + c0;
    if (a.mask) b.mask = a.mask + c0;
    if (a.self_out) b.self_out = a.self_out + c0;
    G.a[0] = b;
    G.n = 1;
    spmm_group(G, s);
  }
}

template void spmm<float, float>(const SpmmArgs<float, float>&, cudaStream_t);
template void spmm<bf16, bf16>(const SpmmArgs<bf16, bf16>&, cudaStream_t);
template void spmm<bf16, float>(const SpmmArgs<bf16, float>&, cudaStream_t);
template void spmm_group<float, float>(const SpmmGroup<float, float>&, cudaStream_t);
template void spmm_group<bf16, bf16>(const SpmmGroup<bf16, bf16>&, cudaStream_t);
template void spmm_group<bf16, float>(const SpmmGroup<bf16, float>&, cudaStream_t);

}  // namespace gist
