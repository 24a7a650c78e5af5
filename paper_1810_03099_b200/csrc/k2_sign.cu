// k2_sign.cu — A5 reference table and K2 sign.
//
// sign (reference SPEC.md:360-368): values[k] = cosine(doc, reference_k),
// where cosine is the reference's exact merge-join (ngram.hpp:184-202,
// empty -> 0, clamped to <= 1). With unit reference columns r_k and
// x_d = w_d/||w_d||, cosine(doc, ref_k) = sum_t x_d[t] * r_k[t].
//
// HBM layout: the K reference vectors are compacted to their term union U:
// R[u*K + k] (fp32, ~U*K*4 bytes: 330 KB at configs[1], L2-resident) and the
// per-term row u lives in TermInfo.ref_row next to idf (one 8-byte gather per
// document nonzero). The kernel is warp-per-segment (256 nonzeros of one
// document, see sign_kernel): coalesced row loads, TermInfo gathers, a hit
// queue for the nonzeros in U, float4 gathers of R rows, fixed-order sums.
// The norm is fused and the unit signature for the compare kernel is written
// in the same pass.
//
// Algorithmic bytes per signature: 8*nnz_d (CSR rows) + 4*K (S row) + 4
// (inv_norm); the transposed unit copy for K3, TermInfo and R gathers are
// L2 traffic. R rows are padded to Kp = roundup(K,4) floats.

#include <algorithm>

#include "kernels.cuh"

namespace refsig_gpu {
namespace {

__device__ __forceinline__ void ref_range(const RefArgs& r, uint32_t k, const uint2*& e, uint32_t& n) {
  if (r.start) {
    e = r.ent + r.start[k];
    n = r.n[k];
  } else {
    const uint32_t d = r.ids[k];
    e = r.ent + r.doc_off[d];
    n = r.nnz[d];
  }
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void ref_reset_kernel(TermInfo* __restrict__ info, uint32_t vocab) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < vocab; t += gridDim.x * blockDim.x)
    info[t].ref_row = -1;
}

// A5 in ONE launch: CTA k per reference vector (all K CTAs are co-resident:
// K <= 256 CTAs of 256 threads). Row numbering needs no claims: the j-th
// entry of reference k owns row base_k + j (base_k = entries of references
// 0..k-1), and a term's canonical row is the smallest row of any reference
// holding it — atomicMin on info[t].ref_row as unsigned (-1 = none = max),
// fire-and-forget, so the result does not depend on scheduling.
//   pass 1: weights (count * idf, or explicit), the squared norm in a fixed
//           order, the atomicMin of every entry's row, and the zeroing of the
//           CTA's own rows;
//   grid barrier (arrival counter; CTAs are co-resident);
//   pass 2: R[row(t)*Kp + k] = w / ||w_k|| through the canonical row (read
//           from L2: this CTA's L1 may hold the pre-barrier line), and the
//           count of canonical rows (|U|).
// Rows of terms that are not canonical stay zero and are never referenced.
// Needs info[].ref_row == -1 (count() leaves it so; a replaced reference is
// reset first) and counter[0,1,3] == 0, which the last CTA restores.
constexpr int kRefIpt2 = 4;
__global__ void __launch_bounds__(256) ref_build_kernel(RefArgs r, TermInfo* __restrict__ info,
                                                        float* __restrict__ R, uint32_t* __restrict__ counter) {
  // counter: [0] barrier arrivals, [1] finished CTAs, [2] |U| (output), [3] |U| accumulator
  __shared__ float red[8];
  __shared__ uint32_t ured[8];
  const uint32_t k = blockIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  pdl_wait();
  uint32_t base = 0;  // entries of references 0..k-1
  for (uint32_t q = threadIdx.x; q < k; q += 256) {
    const uint2* eq;
    uint32_t nq;
    ref_range(r, q, eq, nq);
    base += nq;
  }
  base = warp_sum_u32(base);
  if (lane == 0) ured[wid] = base;
  __syncthreads();
  base = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) base += ured[w];
  const uint2* e;
  uint32_t n;
  ref_range(r, k, e, n);
  float sq = 0.0f;
  for (uint32_t p0 = 0; p0 < n; p0 += 256 * kRefIpt2) {
    uint2 x[kRefIpt2];
#pragma unroll
    for (int j = 0; j < kRefIpt2; ++j) {
      const uint32_t i = p0 + j * 256 + threadIdx.x;
      x[j] = i < n ? e[i] : make_uint2(0xFFFFFFFFu, 0u);
    }
#pragma unroll
    for (int j = 0; j < kRefIpt2; ++j) {
      if (x[j].x == 0xFFFFFFFFu) continue;
      const uint32_t row = base + p0 + j * 256 + threadIdx.x;
      atomicMin(reinterpret_cast<unsigned int*>(&info[x[j].x].ref_row), row);
      const float w = r.explicit_w ? __uint_as_float(x[j].y) : static_cast<float>(x[j].y) * info[x[j].x].idf;
      sq = fmaf(w, w, sq);
      float4* rr = reinterpret_cast<float4*>(R + static_cast<size_t>(row) * r.Kp);
      for (uint32_t q = 0; q < r.Kp / 4; ++q) rr[q] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
  }
  sq = warp_sum(sq);
  if (lane == 0) red[wid] = sq;
  __threadfence();  // row minima and zeroed rows visible before the arrival
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(counter, 1u);
    while (static_cast<uint32_t>(ld_acquire(reinterpret_cast<const int*>(counter))) < gridDim.x) __nanosleep(64);
  }
  __syncthreads();
  float tot = 0.0f;
#pragma unroll
  for (int w = 0; w < 8; ++w) tot += red[w];
  const float inv = tot > 0.0f ? 1.0f / sqrtf(tot) : 0.0f;
  uint32_t canon = 0;
  for (uint32_t p0 = 0; p0 < n; p0 += 256 * kRefIpt2) {
    uint2 x[kRefIpt2];
#pragma unroll
    for (int j = 0; j < kRefIpt2; ++j) {
      const uint32_t i = p0 + j * 256 + threadIdx.x;
      x[j] = i < n ? e[i] : make_uint2(0xFFFFFFFFu, 0u);
    }
    uint32_t row[kRefIpt2];
#pragma unroll
    for (int j = 0; j < kRefIpt2; ++j)
      row[j] = x[j].x == 0xFFFFFFFFu ? 0u : static_cast<uint32_t>(__ldcg(&info[x[j].x].ref_row));
#pragma unroll
    for (int j = 0; j < kRefIpt2; ++j) {
      if (x[j].x == 0xFFFFFFFFu) continue;
      const float w = r.explicit_w ? __uint_as_float(x[j].y) : static_cast<float>(x[j].y) * info[x[j].x].idf;
      R[static_cast<size_t>(row[j]) * r.Kp + k] = w * inv;
      canon += row[j] == base + p0 + j * 256 + threadIdx.x;
    }
  }
  canon = warp_sum_u32(canon);
  __syncthreads();  // ured reuse
  if (lane == 0) ured[wid] = canon;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) c += ured[w];
    atomicAdd(counter + 3, c);
    __threadfence();
    if (atomicAdd(counter + 1, 1u) == gridDim.x - 1) {
      counter[2] = atomicAdd(counter + 3, 0u);
      counter[0] = 0;
      counter[1] = 0;
      counter[3] = 0;
    }
  }
}

// K2 is an SpMM, S = X_hit * R, with X_hit the doc rows restricted to the
// union U (hits). Per step of 128 nonzeros (4 per lane): coalesced row loads,
// TermInfo gathers, ||w||^2, and the hits appended to a per-warp queue in
// shared memory (ballot + prefix popcount; queue order = ascending term id).
// Then lane l takes hits l, l+32, ... and adds w * R[row][c0 .. c0+KW) into
// its own KW accumulators with float4 loads of the row (all lanes busy, KW/4
// independent 16-byte loads per hit in flight). After the document, the 32
// per-lane vectors are transposed through shared memory and lane k adds column
// k over the lanes in lane order. Columns are processed in slabs of KW <= 32.
// Work split: documents of > kSignLongTokens tokens get a CTA (8 warps take
// interleaved steps; the 8 column vectors are added in warp order), shorter
// ones a warp. Every sum has a fixed order: signatures do not depend on
// scheduling.
// K2_HINT (A/B): 0 plain __ldg / gathers, 1 count entries L1::no_allocate,
// 2 entries and TermInfo gathers L1::no_allocate, 3 entries L1::evict_first
// and TermInfo gathers L1::evict_last.
#ifndef REFSIG_K2_HINT
#define REFSIG_K2_HINT 0
#endif
__device__ __forceinline__ uint2 sign_ent(const uint2* p) {
#if REFSIG_K2_HINT >= 3
  return ld_ef(p);
#elif REFSIG_K2_HINT >= 1
  return ld_na(p);
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ TermInfo sign_info(const TermInfo* p) {
#if REFSIG_K2_HINT >= 3
  return ld_el(p);
#elif REFSIG_K2_HINT >= 2
  return ld_na(p);
#else
  return *p;
#endif
}
constexpr int kSignWarps = 8;
#ifndef REFSIG_K2_U
#define REFSIG_K2_U 4
#endif
constexpr int kSignU = REFSIG_K2_U;                  // count entries per lane per step (K <= 32 warp path)
constexpr uint32_t kSignStep = 32 * kSignU;
constexpr uint32_t kSignStepC = 128;                 // K > 32 (sign_col_kernel)

// Hit walk by column groups (REFSIG_K2_CG, default): CG_L = KW/4 lanes per
// hit, one float4 of its R row each, CG_H = 32/CG_L hits per pass. A warp load
// then touches CG_H rows (~1.6 L1 wavefronts per 80-byte row) instead of 32
// (one wavefront per lane: 5 per hit at KW = 20): configs[1] sign 40.9 ->
// 35.3 us. (The rest of K2 there is about half per-document latency, half
// TermInfo gathers + R rows; K2.) Lane (g, j) keeps
// the 4 column sums of group j over the hits g, g + CG_H, ... of the
// document; sign_cg_columns adds them over g in a fixed order.
#ifndef REFSIG_K2_CG
#define REFSIG_K2_CG 1
#endif
template <int KW>
struct SignCG {
  static constexpr int L = KW / 4;   // lanes per hit
  static constexpr int H = 32 / L;   // hits per pass (warp)
  static constexpr int H2 = 16 / L;  // hits per pass (16-lane half)
};
#if REFSIG_K2_CG
template <int KW>
using SignAcc = float[4];
#else
template <int KW>
using SignAcc = float[KW];
#endif

template <int KW>
__device__ __forceinline__ void sign_slab_steps(const SignArgs& a, const uint2* __restrict__ e, uint32_t n,
                                                uint32_t s0, uint32_t stride, uint32_t c0, uint32_t lane, int2* qw,
                                                SignAcc<KW>& acc, float& sq, bool do_sq) {
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t c = s0 * kSignStep; c < n; c += stride * kSignStep) {
    uint2 x[kSignU];
#pragma unroll
    for (int u = 0; u < kSignU; ++u) {
      const uint32_t i = c + 32u * u + lane;
      x[u] = i < n ? sign_ent(e + i) : make_uint2(0u, 0u);
    }
    TermInfo ti[kSignU];
#pragma unroll
    for (int u = 0; u < kSignU; ++u) ti[u] = (c + 32u * u + lane < n) ? sign_info(a.info + x[u].x) : TermInfo{0.0f, -1};
    uint32_t qn = 0;
#pragma unroll
    for (int u = 0; u < kSignU; ++u) {
      const float w = static_cast<float>(x[u].y) * ti[u].idf;
      if (do_sq) sq = fmaf(w, w, sq);
      const uint32_t hits = __ballot_sync(0xffffffffu, ti[u].ref_row >= 0);
      if (ti[u].ref_row >= 0)  // the R row's element offset, computed once per hit
        qw[qn + __popc(hits & lt)] = make_int2(static_cast<int>(static_cast<uint32_t>(ti[u].ref_row) * a.Kp),
                                               __float_as_int(w));
      qn += __popc(hits);
    }
    __syncwarp();
#if REFSIG_K2_CG
    {
      constexpr uint32_t L = SignCG<KW>::L, H = SignCG<KW>::H;
      const uint32_t g = lane / L, j = lane - g * L;
      if (g < H) {
        const float* __restrict__ Rj = a.R + c0 + 4 * j;
        uint32_t h = g;
        for (; h + H < qn; h += 2 * H) {  // two rows in flight per lane
          const int2 h0 = qw[h], h1 = qw[h + H];
          const float4 r0 = __ldg(reinterpret_cast<const float4*>(Rj + static_cast<uint32_t>(h0.x)));
          const float4 r1 = __ldg(reinterpret_cast<const float4*>(Rj + static_cast<uint32_t>(h1.x)));
          const float w0 = __int_as_float(h0.y), w1 = __int_as_float(h1.y);
          acc[0] = fmaf(w0, r0.x, acc[0]);
          acc[1] = fmaf(w0, r0.y, acc[1]);
          acc[2] = fmaf(w0, r0.z, acc[2]);
          acc[3] = fmaf(w0, r0.w, acc[3]);
          acc[0] = fmaf(w1, r1.x, acc[0]);
          acc[1] = fmaf(w1, r1.y, acc[1]);
          acc[2] = fmaf(w1, r1.z, acc[2]);
          acc[3] = fmaf(w1, r1.w, acc[3]);
        }
        if (h < qn) {
          const int2 h0 = qw[h];
          const float4 r0 = __ldg(reinterpret_cast<const float4*>(Rj + static_cast<uint32_t>(h0.x)));
          const float w0 = __int_as_float(h0.y);
          acc[0] = fmaf(w0, r0.x, acc[0]);
          acc[1] = fmaf(w0, r0.y, acc[1]);
          acc[2] = fmaf(w0, r0.z, acc[2]);
          acc[3] = fmaf(w0, r0.w, acc[3]);
        }
      }
    }
#else
    for (uint32_t h = lane; h < qn; h += 32) {
      const int2 hv = qw[h];
      const float w = __int_as_float(hv.y);
      const float4* __restrict__ r4 = reinterpret_cast<const float4*>(a.R + static_cast<uint32_t>(hv.x) + c0);
      constexpr int G = KW / 4 < 8 ? KW / 4 : 8;  // float4 loads in flight per group
#pragma unroll
      for (int j0 = 0; j0 < KW / 4; j0 += G) {
        float4 r[G];
#pragma unroll
        for (int j = 0; j < G; ++j)
          r[j] = (c0 + 4u * (j0 + j) < a.Kp) ? __ldg(r4 + j0 + j) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
        for (int j = 0; j < G; ++j) {
          acc[4 * (j0 + j) + 0] = fmaf(w, r[j].x, acc[4 * (j0 + j) + 0]);
          acc[4 * (j0 + j) + 1] = fmaf(w, r[j].y, acc[4 * (j0 + j) + 1]);
          acc[4 * (j0 + j) + 2] = fmaf(w, r[j].z, acc[4 * (j0 + j) + 2]);
          acc[4 * (j0 + j) + 3] = fmaf(w, r[j].w, acc[4 * (j0 + j) + 3]);
        }
      }
    }
#endif
    __syncwarp();
  }
}

// Column sums of the column-group accumulators: col[0] = column `lane` (0
// past KW) = sum over the hit slots g = 0 .. CG_H-1 of lane (g, lane/4)'s
// component lane%4. tw: >= 128 floats of this warp.
template <int KW>
__device__ __forceinline__ float sign_cg_columns(const float (&acc)[4], uint32_t lane, float* tw) {
  constexpr uint32_t L = SignCG<KW>::L, H = SignCG<KW>::H;
  reinterpret_cast<float4*>(tw)[lane] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  __syncwarp();
  float x = 0.0f;
  if (lane < static_cast<uint32_t>(KW)) {
#pragma unroll
    for (uint32_t g = 0; g < H; ++g) x += tw[g * L * 4 + lane];
  }
  __syncwarp();
  return x;
}

// Lane-order column sums of the warp's KW-vectors: col[t] = column
// 32*t + lane (0 past KW). tw: 32*(KW+1) floats of this warp.
template <int KW, int CPL>
__device__ __forceinline__ void sign_transpose_sum(const float (&acc)[KW], uint32_t lane, float* tw,
                                                   float (&col)[CPL]) {
#pragma unroll
  for (int k = 0; k < KW; ++k) tw[lane * (KW + 1) + k] = acc[k];
  __syncwarp();
#pragma unroll
  for (int t = 0; t < CPL; ++t) {
    float x = 0.0f;
    const uint32_t k = 32u * t + lane;
    if (k < static_cast<uint32_t>(KW)) {
#pragma unroll 8
      for (int l = 0; l < 32; ++l) x += tw[l * (KW + 1) + k];
    }
    col[t] = x;
  }
  __syncwarp();
}

// Short documents (<= kSignHalfTokens tokens, the tail of the LPT order): two
// per warp, one per 16-lane half. Same arithmetic as the warp path per
// half (64 nonzeros per step, a per-half hit queue, lane-per-hit
// accumulation, a 16-row transpose-sum in lane order), but the per-document
// fixed cost (transpose, norms, S/ST epilogue) is shared by two documents.
// The signature-norm sum keeps the warp path's order exactly (column
// squares, then the xor butterfly: the 16-lane halves hold columns k and
// k+16, whose sum is the warp path's first butterfly level), so ST equals
// what refsig_gpu_set_signatures rebuilds from S.
template <int KW>
__device__ __forceinline__ void sign_half_docs(const SignArgs& a, uint32_t q, uint32_t lane, float* tw) {
  static_assert(KW <= 32, "half-warp path: KW <= 32");
  const uint32_t h = lane >> 4, hl = lane & 15;
  const bool has = q < a.n_docs;
  const uint32_t d = has ? a.order[q] : 0u;
  const uint2* __restrict__ e = a.ent + a.doc_off[d];
  const uint32_t n = has ? a.nnz[d] : 0u;
  const uint32_t nmax = max(n, __shfl_xor_sync(0xffffffffu, n, 16));
  int2* qw = reinterpret_cast<int2*>(tw) + h * 64;
  const uint32_t lt = (1u << hl) - 1u;
#if REFSIG_K2_CG
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#else
  float acc[KW];
#pragma unroll
  for (int k = 0; k < KW; ++k) acc[k] = 0.0f;
#endif
  float sq = 0.0f;
  for (uint32_t c = 0; c < nmax; c += 64) {
    uint2 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = c + 16u * u + hl;
      x[u] = i < n ? sign_ent(e + i) : make_uint2(0u, 0u);
    }
    TermInfo ti[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) ti[u] = (c + 16u * u + hl < n) ? sign_info(a.info + x[u].x) : TermInfo{0.0f, -1};
    uint32_t qn = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float w = static_cast<float>(x[u].y) * ti[u].idf;
      sq = fmaf(w, w, sq);
      const uint32_t mine = (__ballot_sync(0xffffffffu, ti[u].ref_row >= 0) >> (16 * h)) & 0xffffu;
      if (ti[u].ref_row >= 0)
        qw[qn + __popc(mine & lt)] = make_int2(static_cast<int>(static_cast<uint32_t>(ti[u].ref_row) * a.Kp),
                                               __float_as_int(w));
      qn += __popc(mine);
    }
    __syncwarp();
#if REFSIG_K2_CG
    {
      constexpr uint32_t L = SignCG<KW>::L, H2 = SignCG<KW>::H2;
      const uint32_t g = hl / L, j = hl - g * L;
      if (g < H2) {
        const float* __restrict__ Rj = a.R + 4 * j;
        for (uint32_t hh = g; hh < qn; hh += H2) {
          const int2 hv = qw[hh];
          const float4 r = __ldg(reinterpret_cast<const float4*>(Rj + static_cast<uint32_t>(hv.x)));
          const float w = __int_as_float(hv.y);
          acc[0] = fmaf(w, r.x, acc[0]);
          acc[1] = fmaf(w, r.y, acc[1]);
          acc[2] = fmaf(w, r.z, acc[2]);
          acc[3] = fmaf(w, r.w, acc[3]);
        }
      }
    }
#else
    const uint32_t qmax = max(qn, __shfl_xor_sync(0xffffffffu, qn, 16));
    for (uint32_t hh = hl; hh < qmax; hh += 16) {
      if (hh < qn) {
        const int2 hv = qw[hh];
        const float w = __int_as_float(hv.y);
        const float4* __restrict__ r4 = reinterpret_cast<const float4*>(a.R + static_cast<uint32_t>(hv.x));
#pragma unroll
        for (int j = 0; j < KW / 4; ++j) {
          const float4 r = __ldg(r4 + j);
          acc[4 * j + 0] = fmaf(w, r.x, acc[4 * j + 0]);
          acc[4 * j + 1] = fmaf(w, r.y, acc[4 * j + 1]);
          acc[4 * j + 2] = fmaf(w, r.z, acc[4 * j + 2]);
          acc[4 * j + 3] = fmaf(w, r.w, acc[4 * j + 3]);
        }
      }
    }
#endif
    __syncwarp();
  }
#if REFSIG_K2_CG
  // half h's column-group sums at tw[h][16][4]; lane hl adds columns hl and
  // hl+16 over the half's hit slots in order
  float* th = tw + h * 64;
  reinterpret_cast<float4*>(th)[hl] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  __syncwarp();
  float col0 = 0.0f, col1 = 0.0f;
  {
    constexpr uint32_t L = SignCG<KW>::L, H2 = SignCG<KW>::H2;
    if (hl < static_cast<uint32_t>(KW)) {
#pragma unroll
      for (uint32_t g = 0; g < H2; ++g) col0 += th[g * L * 4 + hl];
    }
    if (hl + 16 < static_cast<uint32_t>(KW)) {
#pragma unroll
      for (uint32_t g = 0; g < H2; ++g) col1 += th[g * L * 4 + hl + 16];
    }
  }
#else
  // transpose-sum: half h's 16 KW-vectors at tw[h][16][KW+1]; lane hl sums
  // columns hl and hl+16 over the half's 16 rows in lane order
  float* th = tw + h * 16 * (KW + 1);
#pragma unroll
  for (int k = 0; k < KW; ++k) th[hl * (KW + 1) + k] = acc[k];
  __syncwarp();
  float col0 = 0.0f, col1 = 0.0f;
  if (hl < static_cast<uint32_t>(KW)) {
#pragma unroll 8
    for (int l = 0; l < 16; ++l) col0 += th[l * (KW + 1) + hl];
  }
  if (hl + 16 < static_cast<uint32_t>(KW)) {
#pragma unroll 8
    for (int l = 0; l < 16; ++l) col1 += th[l * (KW + 1) + hl + 16];
  }
#endif
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  const float inv = sq > 0.0f ? 1.0f / sqrtf(sq) : 0.0f;
  const float v0 = fminf(col0 * inv, 1.0f), v1 = fminf(col1 * inv, 1.0f);  // ngram.hpp:201 clamp
  const bool k0ok = hl < a.K, k1ok = hl + 16 < a.K;
  float ss = (k0ok ? v0 * v0 : 0.0f) + (k1ok ? v1 * v1 : 0.0f);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv_s = ss > 0.0f ? 1.0f / sqrtf(ss) : 0.0f;  // SPEC.md:372 all-zero -> 0
  if (has) {
    if (hl == 0) a.inv_norm[d] = inv;
    if (k0ok) {
      a.S[static_cast<size_t>(d) * a.K + hl] = v0;
      a.ST[static_cast<size_t>(hl) * a.ld + d] = v0 * inv_s;
    }
    if (k1ok) {
      a.S[static_cast<size_t>(d) * a.K + hl + 16] = v1;
      a.ST[static_cast<size_t>(hl + 16) * a.ld + d] = v1 * inv_s;
    }
  }
  __syncwarp();
}

// The zero pad columns [n_docs, ld) of ST (the tile kernels read whole 128-column
// panels), written by block 0 of the sign launch instead of a memset node
// between the reference build and this PDL launch.
__device__ __forceinline__ void sign_zero_pad(const SignArgs& a) {
  if (blockIdx.x != 0) return;
  const uint32_t pad = a.ld - a.n_docs;
  for (uint32_t idx = threadIdx.x; idx < pad * a.K; idx += blockDim.x)
    a.ST[static_cast<size_t>(idx / pad) * a.ld + a.n_docs + idx % pad] = 0.0f;
}

template <int KW>
#ifndef REFSIG_K2_MINB
#define REFSIG_K2_MINB 4
#endif
__global__ void __launch_bounds__(256, KW <= 24 ? REFSIG_K2_MINB : (KW <= 32 ? 3 : 2)) sign_kernel(SignArgs a) {
  constexpr int CPL = (KW + 31) / 32;  // columns per lane
  // per-warp area: the 128-entry hit queue, then the 32 x (KW+1) transpose
  constexpr int TW = 32 * (KW + 1) > 2 * static_cast<int>(kSignStep) ? 32 * (KW + 1) : 2 * kSignStep;
  extern __shared__ __align__(16) float tsm_dyn[];  // [kSignWarps][TW]
  __shared__ float red[kSignWarps][32 * CPL + 1];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* tw = tsm_dyn + wid * TW;
  int2* qw = reinterpret_cast<int2*>(tw);
  pdl_wait();
  sign_zero_pad(a);
  const bool cta = blockIdx.x < a.n_long;  // one long document per CTA
  {
    const uint32_t warp_blocks = static_cast<uint32_t>(ceil_div(a.n_half - a.n_long, kSignWarps));
    if (blockIdx.x >= a.n_long + warp_blocks) {  // two short documents per warp
      const uint32_t pair = (blockIdx.x - a.n_long - warp_blocks) * kSignWarps + wid;
      sign_half_docs<KW>(a, a.n_half + 2 * pair + (lane >> 4), lane, tw);
      return;
    }
  }
  uint32_t q;
  if (cta) {
    q = blockIdx.x;
  } else {
    q = a.n_long + (blockIdx.x - a.n_long) * kSignWarps + wid;
    if (q >= a.n_half) return;
  }
  const uint32_t d = a.order[q];
  const uint2* __restrict__ e = a.ent + a.doc_off[d];
  const uint32_t n = a.nnz[d];
  const uint32_t s0 = cta ? wid : 0u, stride = cta ? kSignWarps : 1u;
  float sq = 0.0f, inv = 0.0f, ss = 0.0f;
  for (uint32_t c0 = 0; c0 < a.K; c0 += KW) {
    float col[CPL];
#if REFSIG_K2_CG
    static_assert(CPL == 1, "column groups: KW <= 32");
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    sign_slab_steps<KW>(a, e, n, s0, stride, c0, lane, qw, acc, sq, c0 == 0);
    col[0] = sign_cg_columns<KW>(acc, lane, tw);
#else
    float acc[KW];
#pragma unroll
    for (int k = 0; k < KW; ++k) acc[k] = 0.0f;
    sign_slab_steps<KW>(a, e, n, s0, stride, c0, lane, qw, acc, sq, c0 == 0);
    sign_transpose_sum<KW, CPL>(acc, lane, tw, col);
#endif
    if (c0 == 0) sq = warp_sum(sq);
    if (cta) {  // add the 8 warps' columns (and norms) in warp order
#pragma unroll
      for (int t = 0; t < CPL; ++t) red[wid][32 * t + lane] = col[t];
      if (c0 == 0 && lane == 0) red[wid][32 * CPL] = sq;
      __syncthreads();
#pragma unroll
      for (int t = 0; t < CPL; ++t) {
        float x = 0.0f;
#pragma unroll
        for (int u = 0; u < kSignWarps; ++u) x += red[u][32 * t + lane];
        col[t] = x;
      }
      if (c0 == 0) {
        float x = 0.0f;
#pragma unroll
        for (int u = 0; u < kSignWarps; ++u) x += red[u][32 * CPL];
        sq = x;
      }
      __syncthreads();
    }
    if (c0 == 0) {
      inv = sq > 0.0f ? 1.0f / sqrtf(sq) : 0.0f;
      if (lane == 0 && wid == 0) a.inv_norm[d] = inv;
    }
#pragma unroll
    for (int t = 0; t < CPL; ++t) {
      const uint32_t kk = 32u * t + lane, k = c0 + kk;
      if (kk < static_cast<uint32_t>(KW) && k < a.K) {
        const float v = fminf(col[t] * inv, 1.0f);  // ngram.hpp:201 clamp
        if (wid == 0 || !cta) a.S[static_cast<size_t>(d) * a.K + k] = v;
        ss = fmaf(v, v, ss);
      }
    }
  }
  if (cta && wid != 0) return;
  ss = warp_sum(ss);
  const float inv_s = ss > 0.0f ? 1.0f / sqrtf(ss) : 0.0f;  // SPEC.md:372 all-zero -> 0
  __syncwarp();
  for (uint32_t k = lane; k < a.K; k += 32)
    a.ST[static_cast<size_t>(k) * a.ld + d] = a.S[static_cast<size_t>(d) * a.K + k] * inv_s;  // own writes
}

// K > 32: lane k owns columns k, k+32, ... (KS = Kp/32 slabs, Kp =
// roundup(K,32) so every lane load is in bounds): per step the hits are queued
// as above — with the R row's element offset row*Kp precomputed once per hit
// instead of by every lane — padded to a multiple of kSignColG with zero-weight
// entries, and every lane walks the queue (broadcast LDS.128 = two hits),
// kSignColG hits = kSignColG*KS coalesced 128-byte row loads in flight, each
// address one IMAD.WIDE from the lane's base. No transpose; each step's
// column sums are added to the running total (two-level summation). Dense
// lane-per-hit accumulators would need 64+ registers per lane and read whole
// 256-byte rows per hit.
constexpr int kSignColG = 8;
template <int KS>
__device__ __forceinline__ void signc_steps(const SignArgs& a, const uint2* __restrict__ e, uint32_t n, uint32_t s0,
                                            uint32_t stride, uint32_t lane, int2* qw, float (&acc)[KS], float& sq) {
  const uint32_t lt = (1u << lane) - 1u;
  const float* __restrict__ Rl = a.R + lane;  // this lane's column within each 32-column slab
  for (uint32_t c = s0 * kSignStepC; c < n; c += stride * kSignStepC) {
    uint2 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = c + 32u * u + lane;
      x[u] = i < n ? sign_ent(e + i) : make_uint2(0u, 0u);
    }
    TermInfo ti[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) ti[u] = (c + 32u * u + lane < n) ? sign_info(a.info + x[u].x) : TermInfo{0.0f, -1};
    uint32_t qn = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float w = static_cast<float>(x[u].y) * ti[u].idf;
      sq = fmaf(w, w, sq);
      const uint32_t hits = __ballot_sync(0xffffffffu, ti[u].ref_row >= 0);
      if (ti[u].ref_row >= 0)
        qw[qn + __popc(hits & lt)] = make_int2(static_cast<int>(static_cast<uint32_t>(ti[u].ref_row) * a.Kp),
                                               __float_as_int(w));
      qn += __popc(hits);
    }
    const uint32_t qp = (qn + kSignColG - 1) & ~static_cast<uint32_t>(kSignColG - 1);
    if (lane < qp - qn) qw[qn + lane] = make_int2(0, 0);  // row 0 exists when qn > 0; weight 0 adds +0
    __syncwarp();
    float part[KS];
#pragma unroll
    for (int t = 0; t < KS; ++t) part[t] = 0.0f;
    for (uint32_t h = 0; h < qp; h += kSignColG) {
      int2 hv[kSignColG];
#pragma unroll
      for (int j = 0; j < kSignColG; j += 2) {
        const int4 v = *reinterpret_cast<const int4*>(qw + h + j);
        hv[j] = make_int2(v.x, v.y);
        hv[j + 1] = make_int2(v.z, v.w);
      }
      float r[kSignColG][KS];
#pragma unroll
      for (int j = 0; j < kSignColG; ++j) {
        const float* __restrict__ row = Rl + static_cast<uint32_t>(hv[j].x);
#pragma unroll
        for (int t = 0; t < KS; ++t) r[j][t] = __ldg(row + 32 * t);
      }
#pragma unroll
      for (int j = 0; j < kSignColG; ++j)
#pragma unroll
        for (int t = 0; t < KS; ++t) part[t] = fmaf(__int_as_float(hv[j].y), r[j][t], part[t]);
    }
#pragma unroll
    for (int t = 0; t < KS; ++t) acc[t] += part[t];
    __syncwarp();
  }
}

template <int KS>
__global__ void __launch_bounds__(256) sign_col_kernel(SignArgs a) {
  __shared__ __align__(16) int2 queue[kSignWarps][kSignStepC];
  __shared__ float red[kSignWarps][32 * KS + 1];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int2* qw = queue[wid];
  pdl_wait();
  sign_zero_pad(a);
  const bool cta = blockIdx.x < a.n_long;  // one long document per CTA
  uint32_t q;
  if (cta) {
    q = blockIdx.x;
  } else {
    q = a.n_long + (blockIdx.x - a.n_long) * kSignWarps + wid;
    if (q >= a.n_docs) return;
  }
  const uint32_t d = a.order[q];
  const uint2* __restrict__ e = a.ent + a.doc_off[d];
  const uint32_t n = a.nnz[d];
  float acc[KS];
#pragma unroll
  for (int t = 0; t < KS; ++t) acc[t] = 0.0f;
  float sq = 0.0f;
  signc_steps<KS>(a, e, n, cta ? wid : 0u, cta ? kSignWarps : 1u, lane, qw, acc, sq);
  sq = warp_sum(sq);
  if (cta) {  // add the 8 warps' columns (and norms) in warp order
#pragma unroll
    for (int t = 0; t < KS; ++t) red[wid][32 * t + lane] = acc[t];
    if (lane == 0) red[wid][32 * KS] = sq;
    __syncthreads();
    if (wid != 0) return;
#pragma unroll
    for (int t = 0; t < KS; ++t) {
      float x = 0.0f;
#pragma unroll
      for (int u = 0; u < kSignWarps; ++u) x += red[u][32 * t + lane];
      acc[t] = x;
    }
    float x = 0.0f;
#pragma unroll
    for (int u = 0; u < kSignWarps; ++u) x += red[u][32 * KS];
    sq = x;
  }
  const float inv = sq > 0.0f ? 1.0f / sqrtf(sq) : 0.0f;
  if (lane == 0) a.inv_norm[d] = inv;
  float v[KS], ss = 0.0f;
#pragma unroll
  for (int t = 0; t < KS; ++t) {
    const uint32_t k = 32u * t + lane;
    v[t] = fminf(acc[t] * inv, 1.0f);  // ngram.hpp:201 clamp
    if (k < a.K) {
      a.S[static_cast<size_t>(d) * a.K + k] = v[t];
      ss = fmaf(v[t], v[t], ss);
    }
  }
  ss = warp_sum(ss);
  const float inv_s = ss > 0.0f ? 1.0f / sqrtf(ss) : 0.0f;  // SPEC.md:372 all-zero -> 0
#pragma unroll
  for (int t = 0; t < KS; ++t) {
    const uint32_t k = 32u * t + lane;
    if (k < a.K) a.ST[static_cast<size_t>(k) * a.ld + d] = v[t] * inv_s;
  }
}

// Unit-signature transpose for externally supplied signatures (multi-GPU:
// the all-gathered S of every rank). Same arithmetic and order as the sign
// kernels' epilogue (per-lane fmaf over columns lane, lane+32, ..., then the
// xor-butterfly warp sum), so ST is bit-identical to a single-GPU sign().
__global__ void __launch_bounds__(256) st_from_s_kernel(const float* __restrict__ S, uint32_t n_docs, uint32_t K,
                                                        uint32_t ld, float* __restrict__ ST) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); d < n_docs; d += nw) {
    float ss = 0.0f;
    for (uint32_t k = lane; k < K; k += 32) {
      const float v = S[static_cast<size_t>(d) * K + k];
      ss = fmaf(v, v, ss);
    }
    ss = warp_sum(ss);
    const float inv_s = ss > 0.0f ? 1.0f / sqrtf(ss) : 0.0f;
    for (uint32_t k = lane; k < K; k += 32) ST[static_cast<size_t>(k) * ld + d] = S[static_cast<size_t>(d) * K + k] * inv_s;
  }
}

}  // namespace

void launch_st_from_s(const float* S, uint32_t n_docs, uint32_t K, uint32_t ld, float* ST, cudaStream_t s) {
  if (!n_docs) return;
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>(ceil_div(n_docs, 8), 148ull * 16));
  st_from_s_kernel<<<g, 256, 0, s>>>(S, n_docs, K, ld, ST);
  note_launch();
}

void launch_ref_reset(TermInfo* info, uint32_t vocab, cudaStream_t s) {
  uint32_t g = (vocab + 255) / 256;
  if (g > 4096) g = 4096;
  ref_reset_kernel<<<g, 256, 0, s>>>(info, vocab);
  note_launch();
}

void launch_ref_build(const RefArgs& r, TermInfo* info, uint32_t vocab, uint32_t* counter, float* R,
                      uint64_t n_entries_max, cudaStream_t s) {
  (void)vocab;
  (void)n_entries_max;
  launch_pdl(ref_build_kernel, dim3(r.K), dim3(256), 0, s, r, info, R, counter);
  note_launch();
}

template <int KW>
void launch_sign_kw(const SignArgs& a, unsigned g, cudaStream_t s) {
  constexpr int TW = 32 * (KW + 1) > 2 * static_cast<int>(kSignStep) ? 32 * (KW + 1) : 2 * kSignStep;
  constexpr size_t smem = sizeof(float) * kSignWarps * TW;
  ensure_smem(sign_kernel<KW>, smem);
  launch_pdl(sign_kernel<KW>, dim3(g), dim3(32 * kSignWarps), smem, s, a);
}

void launch_sign(const SignArgs& a, cudaStream_t s) {
  if (a.n_docs == 0) return;
  const unsigned g = static_cast<unsigned>(a.n_long + ceil_div(a.n_docs - a.n_long, kSignWarps));
  // K <= 32: documents [n_half, n_docs) of the order go two per warp
  const unsigned g_half = static_cast<unsigned>(a.n_long + ceil_div(a.n_half - a.n_long, kSignWarps) +
                                                ceil_div(a.n_docs - a.n_half, 2 * kSignWarps));
  if (a.K > 32) {  // column-owner variant, Kp = roundup(K, 32)
    switch (a.Kp / 32) {
      case 2: launch_pdl(sign_col_kernel<2>, dim3(g), dim3(32 * kSignWarps), 0, s, a); break;
      case 3: launch_pdl(sign_col_kernel<3>, dim3(g), dim3(32 * kSignWarps), 0, s, a); break;
      case 4: launch_pdl(sign_col_kernel<4>, dim3(g), dim3(32 * kSignWarps), 0, s, a); break;
      case 5: launch_pdl(sign_col_kernel<5>, dim3(g), dim3(32 * kSignWarps), 0, s, a); break;
      case 6: launch_pdl(sign_col_kernel<6>, dim3(g), dim3(32 * kSignWarps), 0, s, a); break;
      case 7: launch_pdl(sign_col_kernel<7>, dim3(g), dim3(32 * kSignWarps), 0, s, a); break;
      default: launch_pdl(sign_col_kernel<8>, dim3(g), dim3(32 * kSignWarps), 0, s, a); break;
    }
    note_launch();
    return;
  }
  // lane-per-hit slab width: K rounded up to 4
  const uint32_t kw = (a.K + 3) & ~3u;
  switch (kw) {
    case 4: launch_sign_kw<4>(a, g_half, s); break;
    case 8: launch_sign_kw<8>(a, g_half, s); break;
    case 12: launch_sign_kw<12>(a, g_half, s); break;
    case 16: launch_sign_kw<16>(a, g_half, s); break;
    case 20: launch_sign_kw<20>(a, g_half, s); break;
    case 24: launch_sign_kw<24>(a, g_half, s); break;
    case 28: launch_sign_kw<28>(a, g_half, s); break;
    default: launch_sign_kw<32>(a, g_half, s); break;
  }
  note_launch();
}

}  // namespace refsig_gpu
