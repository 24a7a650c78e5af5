// k3_pairs.cu — all-pairs kernels: MRC signature compare (K3), Hamming
// compare (K4b), and the deterministic emitter shared by both.
//
// Reference semantics:
//   compare(a,b) = cosine of the signature vectors, 0 if either is all-zero
//                  (SPEC.md:369-377); match <=> score >= tau.
//   hamming(a,b) = popcount(a ^ b) (simhash.hpp:47); match <=> hd <= max_dist.
//   pairs are i<j in lexicographic order.
//
// Design: a compare kernel evaluates 128x128 pair tiles of the upper triangle
// (all tiles for a query-vs-DB join) and writes one bit per pair into a
// row-major pair bitmap (words_per_row = ceil(cols/128)*4), plus per-row match
// counts. An exclusive scan of the counts gives each row's output offset and
// the emitter turns set bits into sorted keys (i<<32 | j). No atomics decide
// output positions, so the candidate list is sorted and identical for every
// launch configuration without a device sort.
//
// MRC tile kernel (CUDA cores): see the comment above mrc_bitmap_kernel2.

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace refsig_gpu {
namespace {

constexpr int kKC = 32;  // K chunk staged in shared memory

// Tile t -> (bi, bj): triangle (bi <= bj, row-major) or rectangle.
__device__ __forceinline__ void tile_coords(uint32_t t, uint32_t nbr, uint32_t nbc, bool triangle, uint32_t& bi,
                                            uint32_t& bj) {
  if (!triangle) {
    bi = t / nbc;
    bj = t - bi * nbc;
    return;
  }
  const double nb = nbc;
  double x = (nb + 0.5) - sqrt((nb + 0.5) * (nb + 0.5) - 2.0 * t);
  int64_t b = static_cast<int64_t>(x);
  auto S = [&](int64_t r) { return r * static_cast<int64_t>(nbc) - r * (r - 1) / 2; };
  if (b < 0) b = 0;
  while (b + 1 <= static_cast<int64_t>(nbc) && S(b + 1) <= static_cast<int64_t>(t)) ++b;
  while (b > 0 && S(b) > static_cast<int64_t>(t)) --b;
  bi = static_cast<uint32_t>(b);
  bj = bi + static_cast<uint32_t>(t - S(b));
}

// Valid-column mask for the 32 columns starting at lo in row i.
__device__ __forceinline__ uint32_t col_mask(uint32_t lo, uint32_t i, const PairGrid& g) {
  uint32_t m = 0xffffffffu;
  if (lo >= g.n_cols) return 0u;
  if (lo + 32 > g.n_cols) m >>= (lo + 32 - g.n_cols);
  if (g.triangle && lo <= i) {
    const uint32_t first = i + 1 - lo;  // first valid bit
    m = first >= 32 ? 0u : (m & (0xffffffffu << first));
  }
  return m;
}

// ---- K3 on CUDA cores (K > 41; the tensor-core kernel is k3_tc.cu) ------------
// Persistent CTAs walk a contiguous range of tiles; (tile, K-chunk) stages
// stream through shared memory with cp.async (16 B chunks of the transposed
// unit signatures ST[k][ld]). Thread (ty,tx) owns rows ty*8..+7 and columns
// tx*8..+7 of the 128x128 tile; shared memory stores each panel in "split"
// order (columns c%8<4 in the first half) so both float4 loads of a thread are
// bank-conflict free while its 8 columns stay contiguous. The inner loop is
// 2+2 LDS.128 and 32 FFMA2 (fma.rn.f32x2, scalar-broadcast A) per k.

__device__ __forceinline__ uint32_t split_pos(uint32_t c) {  // smem slot of panel column c
  return (c & 4u) ? 64u + (c >> 3) * 4u + (c & 3u) : (c >> 3) * 4u + (c & 3u);
}

// d = a*b + c on both fp32 lanes (FFMA2); `a` is broadcast (SASS scalar operand).
__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) {
  float2 aa = make_float2(a, a);
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&aa)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

struct MrcArgs {
  const float* STr;
  const float* STc;
  uint32_t ldr, ldc;
  uint32_t K;
  float tau;
  PairGrid g;
  uint32_t nbr, nbc;
  uint64_t n_tiles;
  uint32_t* bitmap;
  uint32_t* rowcnt;
};

// mbarrier ring, warp-local epilogue: no CTA-wide barrier in the main loop: a 4-stage ring
// of (tile, K-chunk) items where each stage has a "full" mbarrier (256
// arrivals: every thread's cp.async.mbarrier.arrive) and an "empty" mbarrier
// (8 arrivals: one per warp after its last read). A stage is refilled two
// items ahead, so warps may drift up to two items apart and one warp's
// epilogue overlaps the others' FFMA2 stream. The epilogue stays in the warp:
// a warp owns 16 whole tile rows (ty = 2w, 2w+1); each lane packs its 8 row
// bytes into two words, a 4x4 byte transpose inside each lane quad (2 SHFL +
// 2 PRMT per word) gives lane (ty, 4q+i) word q of rows ty*8+i and ty*8+4+i,
// which it stores directly. Row match counts stay in registers until the CTA
// moves to the next row panel (one atomic per row per panel, not per tile).
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared.b64 st, [%0]; }" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{ .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      "@!p bra W; }" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
               : "memory");
}

constexpr int mrc2_stages(int KC) { return KC > 0 && KC <= 24 ? 4 : 3; }

template <int KC>
__global__ void __launch_bounds__(256, 2) mrc_bitmap_kernel2(MrcArgs a) {
  constexpr int S = mrc2_stages(KC);  // ring stages (2 CTAs/SM must fit)
  constexpr int D = S - 2;             // refill distance: warps may drift D items apart
  extern __shared__ __align__(16) float smem[];
  __shared__ __align__(8) uint64_t full_bar[S], empty_bar[S];
  const uint32_t kcm = KC > 0 ? static_cast<uint32_t>(KC) : (a.K < kKC ? a.K : kKC);
  const uint32_t panel = kcm * kTile;
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const uint32_t lane = tid & 31;
  const uint32_t t_begin = static_cast<uint32_t>(a.n_tiles * blockIdx.x / gridDim.x);
  const uint32_t t_end = static_cast<uint32_t>(a.n_tiles * (blockIdx.x + 1) / gridDim.x);
  if (t_begin >= t_end) return;
  const uint32_t nchunks = KC > 0 ? (a.K / KC) : (a.K + kKC - 1) / kKC;
  const uint32_t items = (t_end - t_begin) * nchunks;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 256);
      mbar_init(&empty_bar[i], 8);
    }
  }
  __syncthreads();

  uint32_t bi, bj;
  tile_coords(t_begin + a.g.tile0, a.nbr, a.nbc, a.g.triangle, bi, bj);
  uint32_t li = bi, lj = bj, lchunk = 0;
  constexpr int kSlots = KC > 0 ? (2 * KC + 7) / 8 : 2 * kKC / 8;
  const uint32_t cm = tid & 31, kr = tid >> 5, sp = split_pos(4 * cm);
  auto issue = [&](uint32_t st) {
    const uint32_t k0 = lchunk * kcm;
    const uint32_t kc = KC > 0 ? static_cast<uint32_t>(KC) : min(kcm, a.K - k0);
    const float* baseA = a.STr + static_cast<size_t>(k0) * a.ldr + li * kTile + 4 * cm;
    const float* baseB = a.STc + static_cast<size_t>(k0) * a.ldc + lj * kTile + 4 * cm;
    float* sbase = smem + 2 * st * panel + sp;
#pragma unroll
    for (int u = 0; u < kSlots; ++u) {
      const uint32_t k = kr + 8 * u;
      if (k < kcm) {
        if (KC > 0 || k < kc) cp_async16(sbase + k * kTile, baseA + static_cast<size_t>(k) * a.ldr);
      } else if (k < 2 * kcm) {
        const uint32_t kk = k - kcm;
        if (KC > 0 || kk < kc) cp_async16(sbase + panel + kk * kTile, baseB + static_cast<size_t>(kk) * a.ldc);
      }
    }
    cp_async_mbar_arrive(&full_bar[st]);
    if (++lchunk == nchunks) {
      lchunk = 0;
      if (++lj == a.nbc) {
        ++li;
        lj = a.g.triangle ? li : 0;
      }
    }
  };

  // byte-transpose selectors (lane-constant)
  const uint32_t qi = tx & 3;
  const uint32_t sel1 = (qi & 1) ? 0x3715u : 0x6240u;
  const uint32_t sel2 = (qi & 2) ? 0x3276u : 0x5410u;
  auto transpose = [&](uint32_t v) {
    const uint32_t p = __shfl_xor_sync(0xffffffffu, v, 1);
    v = __byte_perm(v, p, sel1);
    const uint32_t q = __shfl_xor_sync(0xffffffffu, v, 2);
    return __byte_perm(v, q, sel2);
  };
  uint32_t cntA = 0, cntB = 0;  // matches of rows ty*8+qi and ty*8+4+qi in the current row panel (this lane's words)
  auto flush_counts = [&](uint32_t pbi) {
    cntA += __shfl_xor_sync(0xffffffffu, cntA, 4);
    cntA += __shfl_xor_sync(0xffffffffu, cntA, 8);
    cntB += __shfl_xor_sync(0xffffffffu, cntB, 4);
    cntB += __shfl_xor_sync(0xffffffffu, cntB, 8);
    if (tx < 4) {
      const uint32_t r0 = pbi * kTile + ty * 8 + qi;
      if (cntA && r0 < a.g.n_rows) atomicAdd(a.rowcnt + r0, cntA);
      if (cntB && r0 + 4 < a.g.n_rows) atomicAdd(a.rowcnt + r0 + 4, cntB);
    }
    cntA = cntB = 0;
  };

  float2 acc[8][4];
  for (uint32_t j = 0; j < D && j < items; ++j) issue(j);
  uint32_t chunk = 0;
  for (uint32_t it = 0; it < items; ++it) {
    const uint32_t st = it % S;
    if (it + D < items) {
      const uint32_t j = it + D, sj = j % S;
      if (j >= S) mbar_wait(&empty_bar[sj], ((j / S) - 1) & 1u);
      issue(sj);
    }
    mbar_wait(&full_bar[st], (it / S) & 1u);
    const float* A = smem + 2 * st * panel;
    const float* B = A + panel;
    auto kstep = [&](uint32_t k, bool first) {
      const float4 a0 = *reinterpret_cast<const float4*>(A + k * kTile + ty * 4);
      const float4 a1 = *reinterpret_cast<const float4*>(A + k * kTile + 64 + ty * 4);
      const float4 b0 = *reinterpret_cast<const float4*>(B + k * kTile + tx * 4);
      const float4 b1 = *reinterpret_cast<const float4*>(B + k * kTile + 64 + tx * 4);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                            make_float2(b1.z, b1.w)};
      const float2 nt = make_float2(-a.tau, -a.tau);
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = ffma2(av[r], bv[c], first ? nt : acc[r][c]);
    };
    if constexpr (KC > 0) {
      if (KC == static_cast<int>(kKC) && chunk != 0) {
#pragma unroll
        for (uint32_t k = 0; k < KC; ++k) kstep(k, false);
      } else {
        kstep(0, true);
#pragma unroll
        for (uint32_t k = 1; k < KC; ++k) kstep(k, false);
      }
    } else {
      const uint32_t kc = min(kcm, a.K - chunk * kcm);
      uint32_t k = 0;
      if (chunk == 0) kstep(k++, true);
#pragma unroll 4
      for (; k < kc; ++k) kstep(k, false);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[st]);
    if (++chunk == nchunks) {
      chunk = 0;
      // rows ty*8 + 0..3 -> wA (byte r = row r), rows ty*8 + 4..7 -> wB; bit c
      // of a byte = column tx*8 + c; match = NOT sign(dot - tau)
      uint32_t wA = 0, wB = 0;
#pragma unroll
      for (int r = 3; r >= 0; --r)
#pragma unroll
        for (int c = 3; c >= 0; --c) {
          wA = __funnelshift_l(__float_as_uint(acc[r][c].y), wA, 1);
          wA = __funnelshift_l(__float_as_uint(acc[r][c].x), wA, 1);
        }
#pragma unroll
      for (int r = 7; r >= 4; --r)
#pragma unroll
        for (int c = 3; c >= 0; --c) {
          wB = __funnelshift_l(__float_as_uint(acc[r][c].y), wB, 1);
          wB = __funnelshift_l(__float_as_uint(acc[r][c].x), wB, 1);
        }
      wA = transpose(~wA);  // lane (ty, 4q+qi): word q of row ty*8+qi
      wB = transpose(~wB);  //                   word q of row ty*8+4+qi
      const uint32_t q = tx >> 2;
      const uint32_t rA = bi * kTile + ty * 8 + qi, rB = rA + 4;
      const uint32_t c0 = bj * kTile + 32 * q;
      if ((a.g.triangle && bj == bi) || bj + 1 == a.nbc) {  // diagonal / last column tile
        wA &= col_mask(c0, rA, a.g);
        wB &= col_mask(c0, rB, a.g);
      }
      if (rA < a.g.n_rows) a.bitmap[static_cast<size_t>(rA) * a.g.words_per_row + bj * 4 + q] = wA;
      if (rB < a.g.n_rows) a.bitmap[static_cast<size_t>(rB) * a.g.words_per_row + bj * 4 + q] = wB;
      cntA += __popc(wA);
      cntB += __popc(wB);
      const uint32_t pbi = bi;
      if (++bj == a.nbc) {
        ++bi;
        bj = a.g.triangle ? bi : 0;
      }
      if (bi != pbi || it + 1 == items) flush_counts(pbi);
    }
  }
}

// Hamming tile: warp w handles rows (w&1)*64 + lane and (w&1)*64 + 32 + lane
// (two rows per thread: every broadcast LDS.128 of two column fingerprints
// serves four pairs, half the shared-memory traffic of one row per thread —
// the kernel was MIO-throttled) and word w>>1 (32 columns).
__global__ void __launch_bounds__(256) hamming_bitmap_kernel(const uint64_t* __restrict__ fr,
                                                             const uint64_t* __restrict__ fc, int max_dist,
                                                             PairGrid g, uint32_t nbr, uint32_t nbc,
                                                             uint32_t* __restrict__ bitmap,
                                                             uint32_t* __restrict__ rowcnt) {
  __shared__ __align__(16) uint2 Fc[kTile];
  uint32_t bi, bj;
  tile_coords(blockIdx.x + g.tile0, nbr, nbc, g.triangle, bi, bj);
  const uint32_t row0 = bi * kTile, col0 = bj * kTile;
  if (threadIdx.x < kTile) {
    const uint32_t j = col0 + threadIdx.x;
    const uint64_t v = j < g.n_cols ? fc[j] : 0ull;
    Fc[threadIdx.x] = make_uint2(static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t iA = row0 + (w & 1) * 64 + lane, iB = iA + 32;
  const uint64_t a64 = iA < g.n_rows ? fr[iA] : 0ull, b64 = iB < g.n_rows ? fr[iB] : 0ull;
  const uint32_t al = static_cast<uint32_t>(a64), ah = static_cast<uint32_t>(a64 >> 32);
  const uint32_t bl = static_cast<uint32_t>(b64), bh = static_cast<uint32_t>(b64 >> 32);
  const int thr = max_dist + 1;
  const int wi = w >> 1;
  uint32_t bitsA = 0, bitsB = 0;
  // Columns 31..0 of this word: shift in the sign of (hd - thr) so column b
  // ends at bit b (one funnel shift per pair).
#pragma unroll
  for (int b = 31; b >= 0; b -= 2) {
    const uint4 y = *reinterpret_cast<const uint4*>(&Fc[wi * 32 + b - 1]);  // cols b-1, b
    const int a1 = __popc(al ^ y.z) + __popc(ah ^ y.w) - thr;
    const int b1 = __popc(bl ^ y.z) + __popc(bh ^ y.w) - thr;
    bitsA = __funnelshift_l(static_cast<uint32_t>(a1), bitsA, 1);
    bitsB = __funnelshift_l(static_cast<uint32_t>(b1), bitsB, 1);
    const int a0 = __popc(al ^ y.x) + __popc(ah ^ y.y) - thr;
    const int b0 = __popc(bl ^ y.x) + __popc(bh ^ y.y) - thr;
    bitsA = __funnelshift_l(static_cast<uint32_t>(a0), bitsA, 1);
    bitsB = __funnelshift_l(static_cast<uint32_t>(b0), bitsB, 1);
  }
  if (iA < g.n_rows) {
    const uint32_t v = bitsA & col_mask(col0 + wi * 32, iA, g);
    bitmap[static_cast<size_t>(iA) * g.words_per_row + bj * 4 + wi] = v;
    if (v) atomicAdd(rowcnt + iA, __popc(v));
  }
  if (iB < g.n_rows) {
    const uint32_t v = bitsB & col_mask(col0 + wi * 32, iB, g);
    bitmap[static_cast<size_t>(iB) * g.words_per_row + bj * 4 + wi] = v;
    if (v) atomicAdd(rowcnt + iB, __popc(v));
  }
}

// The set bits of `word` as ascending column ids col + b at dst[0..): the
// word is bit-reversed once, then each bit is one FLO + one XOR; two bits per
// loop step (the loop runs max-over-lanes times, so its overhead counts).
#ifndef REFSIG_EMIT_PAIRLOOP
#define REFSIG_EMIT_PAIRLOOP 1
#endif
template <class T>
__device__ __forceinline__ void expand_word(uint32_t word, uint32_t col, T* dst) {
#if REFSIG_EMIT_PAIRLOOP
  uint32_t rw = __brev(word);
  while (rw) {
    const uint32_t b0 = __clz(rw);
    rw ^= 0x80000000u >> b0;
    dst[0] = col + b0;
    if (!rw) break;
    const uint32_t b1 = __clz(rw);
    rw ^= 0x80000000u >> b1;
    dst[1] = col + b1;
    dst += 2;
  }
#else
  for (; word; word &= word - 1) *dst++ = col + (__ffs(word) - 1);
#endif
}

// Warp per row: the row's set bits as ascending column ids at
// out[rowstart[i] ..). A row is read in batches of 128 words (4096 columns),
// lane l loading words c + 32k + l (k = 0..3: four coalesced 128-byte loads;
// the next batch's loads are in flight during this batch's expansion). Slice
// k (32 words, 1024 columns) is expanded on its own: the lanes' popcounts of
// slices (0,1) and (2,3) are scanned as packed 16-bit pairs (two warp scans
// per batch); a sparse slice (<= 128 matches) is stored by the lanes
// directly, a denser one through a per-warp shared stage (each lane expands
// its word at its exclusive offset, then the warp copies the stage out with
// contiguous 128-byte stores: one sequential output stream per row; a slice
// never exceeds the 1024-entry stage).
// Rows: warp w of the grid takes row w first; with `persistent`, later rows
// come from a counter (rows differ by orders of magnitude in matches).
constexpr uint32_t kEmitWarps = 8;
constexpr uint32_t kEmitDirect = 128;  // default (sweep 32..1024 at c1 and c3); REFSIG_EMIT_DIRECT overrides
__global__ void __launch_bounds__(256) emit_kernel(const uint32_t* __restrict__ bitmap, PairGrid g,
                                                   const uint32_t* __restrict__ rowcnt,
                                                   const uint64_t* __restrict__ rowstart, uint32_t* __restrict__ out,
                                                   uint64_t capacity, uint32_t* __restrict__ ctr, int persistent,
                                                   uint32_t direct_max) {
  // ctr[0]: next row ticket, ctr[1]: finished CTAs; both zero at launch, and
  // the last CTA to finish zeroes them again (no memset node between the scan
  // and this PDL launch)
  __shared__ uint32_t stage_all[kEmitWarps][1024];
  pdl_wait();
  const uint32_t lane = threadIdx.x & 31;
  uint32_t* stage = stage_all[threadIdx.x >> 5];
  const uint32_t wpr = g.words_per_row;
  const uint32_t n_warps = gridDim.x * kEmitWarps;
  uint32_t r = blockIdx.x * kEmitWarps + (threadIdx.x >> 5);
  for (;;) {
    const uint32_t i = g.row_begin + r;
    if (i >= g.row_end) break;
    if (persistent) {  // next row's ticket, fetched while this row is expanded
      uint32_t t = 0;
      if (lane == 0) t = atomicAdd(ctr, 1u);
      r = n_warps + __shfl_sync(0xffffffffu, t, 0);
    } else {
      r = ~0u - g.row_begin;  // one row per warp
    }
    uint32_t remaining = rowcnt[i];
    if (remaining == 0) continue;
    uint64_t base = rowstart[i];
    const uint32_t* row = bitmap + static_cast<size_t>(i) * wpr;
    uint32_t c = g.triangle ? (i / kTile) * 4 : 0;  // first written word
    uint32_t nx[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) nx[k] = c + 32 * k + lane < wpr ? row[c + 32 * k + lane] : 0u;
    for (; c < wpr && remaining; c += 128) {
      uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        w[k] = nx[k];
        nx[k] = c + 128 + 32 * k + lane < wpr ? row[c + 128 + 32 * k + lane] : 0u;
      }
      // inclusive scans of (n0 | n1 << 16) and (n2 | n3 << 16): counts <= 1024 per field
      const uint32_t p01 = warp_inclusive_scan(__popc(w[0]) | (__popc(w[1]) << 16), static_cast<int>(lane));
      const uint32_t p23 = warp_inclusive_scan(__popc(w[2]) | (__popc(w[3]) << 16), static_cast<int>(lane));
      const uint32_t t01 = __shfl_sync(0xffffffffu, p01, 31), t23 = __shfl_sync(0xffffffffu, p23, 31);
      if ((t01 | t23) == 0) continue;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t pk = k < 2 ? p01 : p23, tk = k < 2 ? t01 : t23, sh = (k & 1) * 16;
        const uint32_t inc = (pk >> sh) & 0xffffu, tot = (tk >> sh) & 0xffffu;
        if (tot == 0) continue;
        uint32_t word = w[k];
        const uint32_t ex = inc - __popc(word);
        const uint32_t col = (c + 32 * k + lane) * 32u;
        if (base + tot > capacity) {  // overflow: exact positions, writes below capacity only
          uint64_t pos = base + ex;
          for (; word; word &= word - 1, ++pos)
            if (pos < capacity) out[pos] = col + (__ffs(word) - 1);
        } else if (tot <= direct_max) {
          expand_word(word, col, out + base + ex);
        } else {
          expand_word(word, col, stage + ex);
          __syncwarp();
          uint32_t* dst = out + base;
          for (uint32_t e = lane; e < tot; e += 32) dst[e] = stage[e];
          __syncwarp();
        }
        base += tot;
        remaining -= tot;
      }
    }
  }
  if (persistent) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
        ctr[0] = 0;
        ctr[1] = 0;
      }
    }
  }
}

// Few wide rows (a query batch against a large database: 10k rows of 31k
// words at configs[4]): warp-per-row leaves ~1.2 rows per warp and a 2-row
// tail. Here a CTA takes a row and its 8 warps take consecutive 128-word
// batches in rounds (warp w: batch 8r + w); a round's output offsets come
// from the warps' batch totals through shared memory, then each warp expands
// its batch exactly as emit_kernel does (direct stores for sparse slices,
// staged coalesced stores for dense ones).
__global__ void __launch_bounds__(256) emit_wide_kernel(const uint32_t* __restrict__ bitmap, PairGrid g,
                                                        const uint32_t* __restrict__ rowcnt,
                                                        const uint64_t* __restrict__ rowstart,
                                                        uint32_t* __restrict__ out, uint64_t capacity,
                                                        uint32_t direct_max) {
  __shared__ uint32_t stage_all[kEmitWarps][1024];
  __shared__ uint32_t wtot[2][kEmitWarps];
  pdl_wait();
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* stage = stage_all[wid];
  const uint32_t i = g.row_begin + blockIdx.x;
  if (i >= g.row_end || rowcnt[i] == 0) return;  // CTA-uniform
  const uint32_t wpr = g.words_per_row;
  uint64_t row_base = rowstart[i];
  const uint32_t* row = bitmap + static_cast<size_t>(i) * wpr;
  const uint32_t c_first = g.triangle ? (i / kTile) * 4 : 0;
  uint32_t par = 0;
  for (uint32_t r0 = c_first; r0 < wpr; r0 += 128 * kEmitWarps, par ^= 1) {
    const uint32_t c = r0 + 128 * wid;
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = c + 32 * k + lane < wpr ? row[c + 32 * k + lane] : 0u;
    const uint32_t p01 = warp_inclusive_scan(__popc(w[0]) | (__popc(w[1]) << 16), static_cast<int>(lane));
    const uint32_t p23 = warp_inclusive_scan(__popc(w[2]) | (__popc(w[3]) << 16), static_cast<int>(lane));
    const uint32_t t01 = __shfl_sync(0xffffffffu, p01, 31), t23 = __shfl_sync(0xffffffffu, p23, 31);
    if (lane == 0) wtot[par][wid] = (t01 & 0xffffu) + (t01 >> 16) + (t23 & 0xffffu) + (t23 >> 16);
    __syncthreads();  // (wtot double-buffered by round parity: one barrier per round)
    uint64_t base = row_base;
    uint32_t round_total = 0;
#pragma unroll
    for (uint32_t u = 0; u < kEmitWarps; ++u) {
      const uint32_t x = wtot[par][u];
      base += u < wid ? x : 0u;
      round_total += x;
    }
    row_base += round_total;
    if ((t01 | t23) == 0) continue;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t pk = k < 2 ? p01 : p23, tk = k < 2 ? t01 : t23, sh = (k & 1) * 16;
      const uint32_t inc = (pk >> sh) & 0xffffu, tot = (tk >> sh) & 0xffffu;
      if (tot == 0) continue;
      uint32_t word = w[k];
      const uint32_t ex = inc - __popc(word);
      const uint32_t col = (c + 32 * k + lane) * 32u;
      if (base + tot > capacity) {  // overflow: exact positions, writes below capacity only
        uint64_t pos = base + ex;
        for (; word; word &= word - 1, ++pos)
          if (pos < capacity) out[pos] = col + (__ffs(word) - 1);
      } else if (tot <= direct_max) {
        expand_word(word, col, out + base + ex);
      } else {
        expand_word(word, col, stage + ex);
        __syncwarp();
        uint32_t* dst = out + base;
        for (uint32_t e = lane; e < tot; e += 32) dst[e] = stage[e];
        __syncwarp();
      }
      base += tot;
    }
  }
}

// keys[k] = (i << 32) | cols[k] for the pairs of row i (warp per row).
__global__ void __launch_bounds__(256) cols_to_keys_kernel(const uint64_t* __restrict__ rowstart, uint32_t row_begin,
                                                           uint32_t row_end, const uint32_t* __restrict__ cols,
                                                           uint64_t* __restrict__ keys) {
  const uint32_t i = row_begin + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= row_end) return;
  const uint64_t hi = static_cast<uint64_t>(i) << 32;
  const uint64_t e = rowstart[i + 1];
  for (uint64_t k = rowstart[i] + (threadIdx.x & 31); k < e; k += 32) keys[k] = hi | cols[k];
}

int sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// Tiles of row panels [row_begin/128, ceil(row_end/128)); sets g.tile0.
uint64_t n_tiles(PairGrid& g, uint32_t& nbr, uint32_t& nbc) {
  nbr = static_cast<uint32_t>(ceil_div(g.n_rows, kTile));
  nbc = static_cast<uint32_t>(ceil_div(g.n_cols, kTile));
  const uint64_t p0 = g.row_begin / kTile, p1 = ceil_div(g.row_end, kTile);
  if (g.row_end <= g.row_begin || p1 <= p0) return 0;
  if (g.triangle) {
    auto S = [&](uint64_t r) { return r * nbc - r * (r - 1) / 2; };
    g.tile0 = static_cast<uint32_t>(S(p0));
    return S(p1) - S(p0);
  }
  g.tile0 = static_cast<uint32_t>(p0 * nbc);
  return (p1 - p0) * nbc;
}

// u32 -> u16 column ids (n_cols <= 65536): two per thread per step, one
// 32-bit store (the input may start at any element of the CSR array).
__global__ void __launch_bounds__(256) narrow_cols_kernel(const uint32_t* __restrict__ in, uint64_t n,
                                                          uint16_t* __restrict__ out) {
  const uint64_t n2 = n / 2;
  uint32_t* o32 = reinterpret_cast<uint32_t*>(out);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n2;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    o32[i] = in[2 * i] | (in[2 * i + 1] << 16);
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) out[n - 1] = static_cast<uint16_t>(in[n - 1]);
}

}  // namespace

__global__ void rebase_rowptr_kernel(const uint64_t* __restrict__ in, uint64_t n, uint64_t* __restrict__ out) {
  const uint64_t base = in[0];
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i] - base;
}

// Small host -> device values passed as kernel parameters (no copy engine:
// a small cudaMemcpyAsync can queue behind a large staged upload on the same
// engine and stall the compute stream for the length of that upload).
struct ParamWords {
  uint32_t v[kParamWords];
};
__global__ void param_words_kernel(ParamWords p, uint32_t n, uint32_t* __restrict__ dst) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = p.v[i];
}

void launch_param_words(const uint32_t* host_src, uint32_t n, uint32_t* dst, cudaStream_t s) {
  ParamWords p;
  for (uint32_t i = 0; i < n && i < kParamWords; ++i) p.v[i] = host_src[i];
  param_words_kernel<<<1, 256, 0, s>>>(p, n < kParamWords ? n : kParamWords, dst);
  note_launch();
}

// Device words -> mapped pinned host memory by a kernel (again no copy engine).
__global__ void words_to_host_kernel(const uint32_t* __restrict__ src, uint32_t n, uint32_t* __restrict__ dst) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// Device-to-device copy on the SMs (a cudaMemcpyAsync D2D would take a copy
// engine, where it can queue behind a staged host upload).
__global__ void copy_words_kernel(const uint32_t* __restrict__ src, uint64_t n, uint32_t* __restrict__ dst) {
  const uint64_t n4 = n / 4;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n4; i += stride) d4[i] = s4[i];
  for (uint64_t i = n4 * 4 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    dst[i] = src[i];
}

void launch_copy_words(const uint32_t* src, uint64_t n, uint32_t* dst, cudaStream_t s) {
  if (!n) return;
  const uint64_t blocks = std::min<uint64_t>(ceil_div(n, 1024), 148ull * 8);
  copy_words_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(src, n, dst);
  note_launch();
}

void launch_words_to_host(const uint32_t* src, uint32_t n, uint32_t* mapped_dst, cudaStream_t s) {
  words_to_host_kernel<<<1, 32, 0, s>>>(src, n, mapped_dst);
  note_launch();
}

void launch_rebase_rowptr(const uint64_t* in, uint64_t n, uint64_t* out, cudaStream_t s) {
  if (!n) return;
  const uint64_t blocks = std::min<uint64_t>(ceil_div(n, 256), 148ull * 8);
  rebase_rowptr_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(in, n, out);
  note_launch();
}

void launch_narrow_cols(const uint32_t* in, uint64_t n, uint16_t* out, cudaStream_t s) {
  if (!n) return;
  const uint64_t blocks = std::min<uint64_t>(ceil_div(n / 2 + 1, 256), 148ull * 16);
  narrow_cols_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(in, n, out);
  note_launch();
}

void launch_mrc_bitmap(const float* ST_rows, uint32_t ld_rows, const float* ST_cols, uint32_t ld_cols, uint32_t K,
                       float tau, const PairGrid& g_in, uint32_t* bitmap, uint32_t* rowcnt, cudaStream_t s) {
  PairGrid g = g_in;
  uint32_t nbr, nbc;
  const uint64_t t = n_tiles(g, nbr, nbc);
  if (t == 0 || K == 0) return;
  const uint32_t kc = K < kKC ? K : kKC;
  uint64_t grid = static_cast<uint64_t>(sms()) * 2;
  if (grid > t) grid = t;
  MrcArgs a{ST_rows, ST_cols, ld_rows, ld_cols, K, tau, g, nbr, nbc, t, bitmap, rowcnt};
  const dim3 gr(static_cast<unsigned>(grid));
  const int kt = K == 20 ? 20 : K == 10 ? 10 : K == 16 ? 16 : K % 32 == 0 ? 32 : 0;
  const size_t smem2 = (2ull * mrc2_stages(kt) * kc * kTile) * sizeof(float);
  {
    const int mx = 8 * kKC * kTile * 4;
    ensure_smem(mrc_bitmap_kernel2<0>, mx);
    ensure_smem(mrc_bitmap_kernel2<10>, mx);
    ensure_smem(mrc_bitmap_kernel2<16>, mx);
    ensure_smem(mrc_bitmap_kernel2<20>, mx);
    ensure_smem(mrc_bitmap_kernel2<32>, mx);
  }
  if (K == 20)
    mrc_bitmap_kernel2<20><<<gr, 256, smem2, s>>>(a);
  else if (K == 10)
    mrc_bitmap_kernel2<10><<<gr, 256, smem2, s>>>(a);
  else if (K == 16)
    mrc_bitmap_kernel2<16><<<gr, 256, smem2, s>>>(a);
  else if (K % 32 == 0)
    mrc_bitmap_kernel2<32><<<gr, 256, smem2, s>>>(a);
  else
    mrc_bitmap_kernel2<0><<<gr, 256, smem2, s>>>(a);
  note_launch();
}

void launch_hamming_bitmap(const uint64_t* f_rows, const uint64_t* f_cols, int max_dist, const PairGrid& g_in,
                           uint32_t* bitmap, uint32_t* rowcnt, cudaStream_t s) {
  PairGrid g = g_in;
  uint32_t nbr, nbc;
  const uint64_t t = n_tiles(g, nbr, nbc);
  if (t == 0) return;
  hamming_bitmap_kernel<<<static_cast<unsigned>(t), 256, 0, s>>>(f_rows, f_cols, max_dist, g, nbr, nbc, bitmap,
                                                                 rowcnt);
  note_launch();
}

void launch_cols_to_keys(const uint64_t* rowstart, uint32_t row_begin, uint32_t row_end, const uint32_t* cols,
                         uint64_t* keys, cudaStream_t s) {
  if (row_end <= row_begin) return;
  cols_to_keys_kernel<<<static_cast<unsigned>(ceil_div(row_end - row_begin, 8)), 256, 0, s>>>(rowstart, row_begin,
                                                                                            row_end, cols, keys);
  note_launch();
}

void launch_emit_pairs(const uint32_t* bitmap, const PairGrid& g, const uint32_t* rowcnt, const uint64_t* rowstart,
                       uint32_t* out, uint64_t capacity, uint32_t* counter, cudaStream_t s) {
  if (g.row_end <= g.row_begin) return;
  // one row per warp; persistent warps (at most 7 CTAs of 8 warps per SM, 32 KB
  // of stages each) when there are many more rows than resident warps
  const uint64_t rows = g.row_end - g.row_begin;
  const uint64_t need = ceil_div(rows, kEmitWarps);
  const uint64_t resident = static_cast<uint64_t>(sms()) * 7;
  const int persistent = need > 4 * resident ? 1 : 0;
  const uint64_t blocks = persistent ? resident : need;
  static const uint32_t direct_max = [] {
    const char* m = std::getenv("REFSIG_EMIT_DIRECT");
    return m ? static_cast<uint32_t>(std::atoi(m)) : kEmitDirect;
  }();
  // few rows of many batches each (fewer than ~2 rows per resident warp, >= 8 batches per row):
  // a CTA per row (REFSIG_EMIT_WIDE=0/1 forces the choice, for measurement and tests)
  static const int wide_mode = [] {
    const char* m = std::getenv("REFSIG_EMIT_WIDE");
    return m ? std::atoi(m) : -1;
  }();
  const bool wide = wide_mode == 1 ||
                    (wide_mode != 0 && rows < 2 * resident * kEmitWarps && g.words_per_row >= 128u * kEmitWarps);
  if (wide) {
    launch_pdl(emit_wide_kernel, dim3(static_cast<unsigned>(rows)), dim3(32 * kEmitWarps), 0, s, bitmap, g, rowcnt,
               rowstart, out, capacity, direct_max);
    note_launch();
    return;
  }
  launch_pdl(emit_kernel, dim3(static_cast<unsigned>(blocks)), dim3(32 * kEmitWarps), 0, s, bitmap, g, rowcnt,
             rowstart, out, capacity, counter, persistent, direct_max);
  note_launch();
}

}  // namespace refsig_gpu
