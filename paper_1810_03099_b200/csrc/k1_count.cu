// k1_count.cu — K1: per-document term counting (sort + run-length encode),
// document frequency and smoothed IDF.
//
// Restates, per document and in parallel over documents:
//   extract_3grams' std::sort + RLE      reference ngram.hpp:170-178
//   NgramVector::from_entries (merge dups, sorted by id)   ngram.hpp:62-75
// so the (id,count) rows are bit-identical to the reference's entries().
// df is SPEC.md:214-222's doc_freq; idf is SURVEY.md Appendix A3.
//
// Layout: tokens u32[T] + doc_off u64[N+1] in HBM. Output is a *padded* CSR:
// doc d's sorted rows live at ent[doc_off[d] .. doc_off[d]+nnz[d]) (uint2 =
// {id,count}, the reference GramCount of ngram.hpp:48-53), so no inter-doc
// prefix sum is needed on the hot path; launch_compact_csr produces the
// compact CSR only when a caller asks for it.
//
// Sort: a bitonic network kept in registers. A group of W warps sorts
// P = 32*IPT*W keys, IPT consecutive keys per thread (blocked layout):
// compare-exchange distances j < IPT are register ops, IPT <= j < 32*IPT are
// one SHFL + one predicated IMNMX per key, and j >= 32*IPT (multi-warp
// groups only) go through shared memory. Run-length encoding is done in
// registers too (neighbour via SHFL, positions via warp/block scans, run ends
// via a suffix-min of the next head). Work plan (host-built at upload):
//   <= 64 tokens: warp per doc, 64-key sort;
//   65..128 / 129..256: one warp per doc sorting 128 / 256 keys in
//     registers (IPT 4 / 8);
//   257..8192: one CTA of 2/4/8/16/32 warps per doc, 8 keys per thread
//     (group_sort_kernel; 8 keys per thread beat 16 and 4 at every size);
//   > 8192: bitonic sort in a global scratch region.

#include <cmath>
#include <cstdlib>

#include "kernels.cuh"

namespace refsig_gpu {
namespace {

constexpr uint32_t kInf = 0xFFFFFFFFu;

// df increments: one atomic per (doc, term) run head into one of R replicas
// of the df array (replica = CTA index mod R). Zipf-head terms occur in nearly
// every document, so a single array serialises thousands of atomics on a few
// L2 addresses; replicas divide that contention by R. The idf kernel sums the
// replicas (measured: a shared-memory aggregation cache was slower — shared
// atomics cost ~2 cycles per lane).
// The replica base is computed once per CTA (df_replica) and kept in a
// register: recomputing the modulo per run head cost ~25 instructions each.
__device__ __forceinline__ uint32_t* df_replica(const CountArgs& a) {
  return a.df + static_cast<size_t>(blockIdx.x % a.df_reps) * a.vocab;
}

__device__ __forceinline__ uint32_t next_pow2(uint32_t x) {
  return x <= 1 ? 1u : (1u << (32 - __clz(x - 1)));
}

// ---------------------------------------------------------------------------
// Register bitonic sort. T = 32*W threads of one CTA sort P = T*IPT keys,
// thread t holding [t*IPT, t*IPT+IPT) (blocked layout; W = 1 is one warp).
// Distances j < IPT are register ops, IPT <= j < 32*IPT shuffles, j >= 32*IPT
// (W > 1 only) go through shared memory (sm: IPT*T words, element-major so
// both the stores and the partner loads are conflict-free). Every stage is a
// template instance, so all register indices are compile-time constants.
// Direction normalisation: from merge level K = IPT on, a thread's sort
// direction is uniform over its keys, so a thread in a descending block holds
// its keys complemented (one XOR per key per level, composed with the
// previous level's) and every compare-exchange of the level sorts ascending —
// the register stages then need no direction selects. The last level
// (K = P) is ascending everywhere, which restores the keys.
// BAR = 0: the CTA barrier; BAR > 0: named barrier BAR over the T threads of
// a sub-group (two independent sorts in one CTA, group_split_kernel).
template <int BAR, int T>
__device__ __forceinline__ void group_barrier() {
  if constexpr (BAR == 0) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(BAR), "r"(T) : "memory");
  }
}

template <int IPT, int T, int K, int J, bool NORM, int BAR = 0>
__device__ __forceinline__ void gbitonic_stage(uint32_t (&v)[IPT], uint32_t t, uint32_t* sm) {
  if constexpr (J >= 32 * IPT) {
    constexpr uint32_t tj = J / IPT;
    group_barrier<BAR, T>();
#pragma unroll
    for (int q = 0; q < IPT; ++q) sm[q * T + t] = v[q];
    group_barrier<BAR, T>();
    const bool take_min = NORM ? (t & tj) == 0 : ((t & tj) == 0) == (((t * IPT) & K) == 0);
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      const uint32_t y = sm[q * T + (t ^ tj)];
      v[q] = take_min ? min(v[q], y) : max(v[q], y);
    }
  } else if constexpr (J >= IPT) {
    constexpr uint32_t lj = J / IPT;
    const bool take_min = NORM ? (t & lj) == 0 : ((t & lj) == 0) == (((t * IPT) & K) == 0);
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      const uint32_t y = __shfl_xor_sync(0xffffffffu, v[q], lj);
      v[q] = take_min ? min(v[q], y) : max(v[q], y);
    }
  } else {
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      if ((q & J) == 0) {
        const int l = q | J;
        const uint32_t lo = min(v[q], v[l]), hi = max(v[q], v[l]);
        if constexpr (NORM) {
          v[q] = lo;
          v[l] = hi;
        } else {  // K < IPT: the direction depends on q only (compile-time)
          const bool asc = (q & K) == 0;
          v[q] = asc ? lo : hi;
          v[l] = asc ? hi : lo;
        }
      }
    }
  }
  if constexpr (J > 1) gbitonic_stage<IPT, T, K, J / 2, NORM, BAR>(v, t, sm);
}

template <int IPT, int T, int K, int KMAX, int BAR = 0>
__device__ __forceinline__ void gbitonic_level(uint32_t (&v)[IPT], uint32_t t, uint32_t* sm, uint32_t& cur) {
  if constexpr (K >= IPT) {
    const uint32_t want = ((t * IPT) & K) ? 0xffffffffu : 0u;  // descending block: hold complements
    const uint32_t x = want ^ cur;
#pragma unroll
    for (int q = 0; q < IPT; ++q) v[q] ^= x;
    cur = want;
    gbitonic_stage<IPT, T, K, K / 2, true, BAR>(v, t, sm);
  } else {
    gbitonic_stage<IPT, T, K, K / 2, false, BAR>(v, t, sm);
  }
  if constexpr (K < KMAX) gbitonic_level<IPT, T, 2 * K, KMAX, BAR>(v, t, sm, cur);
}

template <int IPT, int T, int BAR = 0>
__device__ __forceinline__ void gbitonic_sort(uint32_t (&v)[IPT], uint32_t t, uint32_t* sm) {
  uint32_t cur = 0;
  gbitonic_level<IPT, T, 2, T * IPT, BAR>(v, t, sm, cur);
}

// Multi-warp sort whose warp-local levels (K <= 32*IPT: registers and
// shuffles only, no CTA barrier) are skipped by warps holding only padding:
// an all-kInf block is sorted in either direction, so such a warp just takes
// the representation level 32*IPT expects (complemented in descending
// blocks). Requires warp w to hold keys [w*32*IPT, (w+1)*32*IPT) of the
// document (see group_sort_kernel's load order).
template <int IPT, int T>
__device__ __forceinline__ void gbitonic_sort_skip(uint32_t (&v)[IPT], uint32_t t, uint32_t* sm, bool live) {
  constexpr uint32_t KW = 32 * IPT;
  uint32_t cur = 0;
  if (live) {
    gbitonic_level<IPT, T, 2, KW>(v, t, sm, cur);
  } else {
    cur = ((t * IPT) & KW) ? 0xffffffffu : 0u;
#pragma unroll
    for (int q = 0; q < IPT; ++q) v[q] = kInf ^ cur;
  }
  if constexpr (KW < T * IPT) gbitonic_level<IPT, T, 2 * KW, T * IPT>(v, t, sm, cur);
}

template <int IPT>
__device__ __forceinline__ void bitonic_regs(uint32_t (&v)[IPT], uint32_t lane) {
  gbitonic_sort<IPT, 32>(v, lane, nullptr);
}

// Warp inclusive scan / suffix min.
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, uint32_t lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= static_cast<uint32_t>(o)) x += y;
  }
  return x;
}
__device__ __forceinline__ uint32_t warp_suffix_min_excl(uint32_t x, uint32_t lane) {
  // min over lanes > lane
  uint32_t r = __shfl_down_sync(0xffffffffu, x, 1);
  if (lane == 31) r = kInf;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_down_sync(0xffffffffu, r, o);
    if (lane + o < 32) r = min(r, y);
  }
  return r;
}

// RLE of the sorted keys (blocked, IPT per thread, first `len` valid) of a
// group of W warps; writes (id,count) rows at ent[0..nnz) and bumps df.
// Returns nnz (valid in every thread). sm: >= 3*W+2 words (W > 1).
template <int IPT, int W>
__device__ __forceinline__ uint32_t rle_regs(const uint32_t (&v)[IPT], uint32_t t, uint32_t len, uint2* ent,
                                             const CountArgs& ca, uint32_t* sm) {
  const uint32_t lane = threadIdx.x & 31, w = t >> 5;
  // predecessor of v[0]
  uint32_t prev = __shfl_up_sync(0xffffffffu, v[IPT - 1], 1);
  if constexpr (W > 1) {
    if (lane == 31) sm[w] = v[IPT - 1];
    __syncthreads();
    if (lane == 0) prev = w > 0 ? sm[w - 1] : kInf;
  } else {
    if (lane == 0) prev = kInf;
  }
  const uint32_t base = t * IPT;
  uint32_t* const dfr = df_replica(ca);
  uint32_t hmask = 0;  // bit q: key q starts a run
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const uint32_t p = q == 0 ? prev : v[q - 1];
    if (base + q < len && (base + q == 0 || v[q] != p)) hmask |= 1u << q;
  }
  const uint32_t nh = __popc(hmask);
  const uint32_t first = hmask ? base + (__ffs(hmask) - 1) : kInf;
  // exclusive position of this thread's first head; total; next head after this thread
  uint32_t incl = warp_incl_scan(nh, lane);
  uint32_t next = warp_suffix_min_excl(first, lane);
  uint32_t total, pos;
  if constexpr (W > 1) {
    uint32_t* wsum = sm + W;      // [W] head counts per warp
    uint32_t* wmin = sm + 2 * W;  // [W] first head of each warp
    __syncthreads();
    if (lane == 31) wsum[w] = incl;
    const uint32_t wfirst = __reduce_min_sync(0xffffffffu, first);
    if (lane == 0) wmin[w] = wfirst;
    __syncthreads();
    uint32_t before = 0, tot = 0, after = kInf;
#pragma unroll
    for (int u = 0; u < W; ++u) {
      const uint32_t c = wsum[u];
      before += (u < static_cast<int>(w)) ? c : 0u;
      tot += c;
      if (u > static_cast<int>(w)) after = min(after, wmin[u]);
    }
    pos = before + incl - nh;
    total = tot;
    next = min(next, after);
    __syncthreads();
  } else {
    pos = incl - nh;
    total = __shfl_sync(0xffffffffu, incl, 31);
  }
  if (next == kInf) next = len;
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    if (hmask & (1u << q)) {
      const uint32_t rest = hmask & ~((2u << q) - 1);  // heads after q in this thread
      const uint32_t end = rest ? base + (__ffs(rest) - 1) : next;
      ent[pos] = make_uint2(v[q], end - (base + q));
#ifndef REFSIG_K1_NO_DF  // (timing experiment only: df left unset)
      atomicAdd(dfr + v[q], 1u);
#endif
      ++pos;
    }
  }
  return total;
}

// Branch-free key load: out-of-range ids are clamped (the error flag is
// raised once per warp after the sort, see flag_bad), padding is kInf.
__device__ __forceinline__ uint32_t load_key(const CountArgs& a, uint64_t b, uint32_t i, uint32_t len,
                                             uint32_t& bad) {
  const bool in = i < len;
  const uint32_t v = in ? __ldg(a.tokens + b + i) : 0u;
  bad |= static_cast<uint32_t>(v >= a.vocab);
  return in ? min(v, a.vocab - 1) : kInf;
}
__device__ __forceinline__ void flag_bad(const CountArgs& a, uint32_t bad) {
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.err, 1u);
}

// One warp per document of up to P = 32*IPT tokens (IPT 2 / 8 / 16). One
// work item per warp and no grid-stride loop: with warp-uniform control flow
// that the compiler can see, the shuffles need no collective fallback paths
// (which doubled the code size of the unrolled network).
template <int IPT>
__global__ void __launch_bounds__(256, IPT <= 8 ? 6 : 4) count_warp_kernel(CountArgs a,
                                                                           const uint32_t* __restrict__ docs,
                                                                           uint32_t n_docs) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= n_docs) return;
  const uint32_t d = docs[q];
  const uint64_t b = a.doc_off[d];
  const uint32_t len = static_cast<uint32_t>(a.doc_off[d + 1] - b);
  uint32_t v[IPT], bad = 0;
#pragma unroll
  for (int k = 0; k < IPT; ++k) v[k] = load_key(a, b, k * 32 + lane, len, bad);  // coalesced; any order sorts
  bitonic_regs<IPT>(v, lane);
  flag_bad(a, bad);
  const uint32_t n = rle_regs<IPT, 1>(v, lane, len, a.ent + b, a, nullptr);
  if (lane == 0) a.nnz[d] = n;
}

template <int THREADS>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* scratch, uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = warp_inclusive_scan(v, lane);
  if (lane == 31) scratch[wid] = inc;
  __syncthreads();
  uint32_t wsum = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < THREADS / 32; ++w) {
    uint32_t x = scratch[w];
    wsum += (w < wid) ? x : 0u;
    tot += x;
  }
  *total = tot;
  __syncthreads();
  return wsum + inc - v;
}

// Group pass: one CTA of W warps per document of up to 512*W tokens, sorted
// as 512*W keys (IPT 16) in registers/shuffles/shared memory and run-length
// encoded straight into the final rows (no chunk scratch, no merge).
template <int W, int IPT>
__global__ void __launch_bounds__(32 * W) group_sort_kernel(CountArgs a, const uint32_t* __restrict__ docs,
                                                           uint32_t n_docs) {
  constexpr int T = 32 * W;
  __shared__ uint32_t sm[IPT * T];
  __shared__ uint32_t rle_sm[3 * W + 2];
  const uint32_t t = threadIdx.x;
  const uint32_t d = docs[blockIdx.x];
  const uint64_t b = a.doc_off[d];
  const uint32_t len = static_cast<uint32_t>(a.doc_off[d + 1] - b);
  uint32_t v[IPT], bad = 0;
  // warp w loads tokens [w*32*IPT, (w+1)*32*IPT), lane-strided (coalesced):
  // any order sorts, and warps past the end hold only padding
  const uint32_t wbase = (t & ~31u) * IPT, lane = t & 31;
#pragma unroll
  for (int k = 0; k < IPT; ++k) v[k] = load_key(a, b, wbase + k * 32 + lane, len, bad);
  gbitonic_sort_skip<IPT, T>(v, t, sm, wbase < len);
  flag_bad(a, bad);
  const uint32_t n = rle_regs<IPT, W>(v, t, len, a.ent + b, a, rle_sm);
  if (t == 0) a.nnz[d] = n;
}

// Split pass: documents of (P/2, P] tokens, P = 256 W, without the pow2 padding
// of the whole document (~30% of the keys at configs[1]): the first M = P/2
// tokens are sorted by warps [0, W/2) (M keys, no padding), the other r =
// len - M by the first R/256 warps of [W/2, W) as R = pow2(r) keys (at least
// 64: IPT 2 / 4 for one warp), each half with its own named barrier; then one
// merge path over the two sorted runs in shared memory gives every thread its
// 8 consecutive keys of the document, which are run-length encoded as in
// group_sort_kernel.
template <int IPT, int WR, int BAR>
__device__ __forceinline__ void split_rest_sort(const CountArgs& a, uint64_t b, uint32_t M, uint32_t len,
                                                uint32_t tr, uint32_t* scratch, uint32_t* B, uint32_t& bad) {
  constexpr int TR = 32 * WR;
  if (tr >= static_cast<uint32_t>(TR)) return;
  uint32_t v[IPT];
  const uint32_t wbase = (tr & ~31u) * IPT, lane = tr & 31;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const uint32_t i = M + wbase + k * 32 + lane;
    v[k] = load_key(a, b, i, len, bad);
  }
  if constexpr (WR == 1) {
    bitonic_regs<IPT>(v, lane);
  } else {
    gbitonic_sort<IPT, TR, BAR>(v, tr, scratch);
    group_barrier<BAR, TR>();  // B aliases the scratch the last exchange stage read
  }
#pragma unroll
  for (int q = 0; q < IPT; ++q) B[tr * IPT + q] = v[q];
}

template <int W>
__global__ void __launch_bounds__(32 * W) group_split_kernel(CountArgs a, const uint32_t* __restrict__ docs,
                                                            uint32_t n_docs) {
  constexpr int T = 32 * W, WM = W / 2, TM = 32 * WM;
  constexpr uint32_t M = 256u * WM;             // main run: exactly M tokens (len > M)
  // sort exchanges: main [0, 8 TM), rest [8 TM, 8 T); afterwards the sorted runs A (M = 8 TM words)
  // and B (<= M) in the same two regions
  __shared__ uint32_t scratch[8 * T];
  uint32_t* const A = scratch;
  uint32_t* const B = scratch + 8 * TM;
  __shared__ uint32_t rle_sm[3 * W + 2];
  const uint32_t t = threadIdx.x, lane = t & 31;
  const uint32_t d = docs[blockIdx.x];
  const uint64_t b = a.doc_off[d];
  const uint32_t len = static_cast<uint32_t>(a.doc_off[d + 1] - b);
  const uint32_t r = len - M;
  const uint32_t R = max(64u, next_pow2(r));
  uint32_t bad = 0;
  if (t < static_cast<uint32_t>(TM)) {  // main: tokens [0, M)
    uint32_t v[8];
    const uint32_t wbase = (t & ~31u) * 8;
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = load_key(a, b, wbase + k * 32 + lane, len, bad);
    if constexpr (WM == 1) {
      bitonic_regs<8>(v, lane);
    } else {
      gbitonic_sort<8, TM, 1>(v, t, scratch);
      group_barrier<1, TM>();  // A aliases the scratch the last exchange stage read
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) A[t * 8 + q] = v[q];
  } else {  // rest: tokens [M, len) as R keys
    const uint32_t tr = t - TM;
    uint32_t* sc = B;
    if (R == 64) {
      split_rest_sort<2, 1, 2>(a, b, M, len, tr, sc, B, bad);
    } else if (R == 128) {
      split_rest_sort<4, 1, 2>(a, b, M, len, tr, sc, B, bad);
    } else if (R == 256) {
      split_rest_sort<8, 1, 2>(a, b, M, len, tr, sc, B, bad);
    } else if (R == 512) {
      if constexpr (WM >= 2) split_rest_sort<8, 2, 2>(a, b, M, len, tr, sc, B, bad);
    } else if (R == 1024) {
      if constexpr (WM >= 4) split_rest_sort<8, 4, 2>(a, b, M, len, tr, sc, B, bad);
    } else if (R == 2048) {
      if constexpr (WM >= 8) split_rest_sort<8, 8, 2>(a, b, M, len, tr, sc, B, bad);
    } else {
      if constexpr (WM >= 16) split_rest_sort<8, 16, 2>(a, b, M, len, tr, sc, B, bad);
    }
  }
  flag_bad(a, bad);
  __syncthreads();
  // merge path: thread t takes outputs [8t, 8t + 8) of merge(A[0, M), B[0, R)); B's padding is kInf
  uint32_t v[8];
  const uint32_t diag = 8 * t;
  if (diag >= M + R) {
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = kInf;
  } else {
    uint32_t lo = diag > R ? diag - R : 0u, hi = min(diag, M);
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (A[mid] <= B[diag - mid - 1]) lo = mid + 1; else hi = mid;
    }
    uint32_t i = lo, j = diag - lo;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t x = i < M ? A[i] : kInf, y = j < R ? B[j] : kInf;
      const bool ta = x <= y;
      v[q] = ta ? x : y;
      i += ta;
      j += !ta;
    }
  }
  const uint32_t n = rle_regs<8, W>(v, t, len, a.ent + b, a, rle_sm);
  if (t == 0) a.nnz[d] = n;
}

// ---------------------------------------------------------------------------
// Documents longer than 8192 tokens: bitonic sort in a global scratch region
// (next_pow2(len) keys each), then a chunked block-wide RLE.
template <int THREADS>
__device__ __forceinline__ void bitonic_sort_mem(uint32_t* s, uint32_t P) {
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t idx = threadIdx.x; idx < (P >> 1); idx += THREADS) {
        uint32_t i = ((idx & ~(j - 1)) << 1) | (idx & (j - 1));
        uint32_t l = i + j;
        uint32_t x = s[i], y = s[l];
        bool up = (i & k) == 0;
        if ((x > y) == up) {
          s[i] = y;
          s[l] = x;
        }
      }
      __syncthreads();
    }
  }
}

template <int THREADS, int IPT>
__device__ __forceinline__ uint32_t rle_mem(const uint32_t* s, uint32_t len, uint2* ent, const CountArgs& ca,
                                            uint32_t* scan_scratch) {
  uint32_t base = 0;
  uint32_t* const dfr = df_replica(ca);
  for (uint32_t c0 = 0; c0 < len; c0 += THREADS * IPT) {
    const uint32_t lo = c0 + threadIdx.x * IPT;
    uint32_t heads = 0;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      uint32_t i = lo + q;
      if (i < len && (i == 0 || s[i] != s[i - 1])) ++heads;
    }
    uint32_t total;
    uint32_t pos = base + block_exclusive_scan<THREADS>(heads, scan_scratch, &total);
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      uint32_t i = lo + q;
      if (i < len && (i == 0 || s[i] != s[i - 1])) {
        const uint32_t key = s[i];
        uint32_t e = i + 1;
        while (e < len && s[e] == key) ++e;
        ent[pos] = make_uint2(key, e - i);
        atomicAdd(dfr + key, 1u);
        ++pos;
      }
    }
    base += total;
  }
  return base;
}

__global__ void __launch_bounds__(1024) count_large_kernel(CountArgs a, const uint32_t* __restrict__ long_docs,
                                                           const uint64_t* __restrict__ scratch_off,
                                                           uint32_t n_long, uint32_t* scratch) {
  __shared__ uint32_t scan_scratch[32];
  for (uint32_t q = blockIdx.x; q < n_long; q += gridDim.x) {
    const uint32_t d = long_docs[q];
    const uint64_t b = a.doc_off[d];
    const uint32_t len = static_cast<uint32_t>(a.doc_off[d + 1] - b);
    const uint32_t P = next_pow2(len);
    uint32_t* s = scratch + scratch_off[q];
    uint32_t bad = 0;
    for (uint32_t i = threadIdx.x; i < P; i += 1024) s[i] = load_key(a, b, i, len, bad);
    flag_bad(a, bad);  // P >= 16384: every thread runs the same trip count
    __syncthreads();
    bitonic_sort_mem<1024>(s, P);
    uint32_t n = rle_mem<1024, 8>(s, len, a.ent + b, a, scan_scratch);
    if (threadIdx.x == 0) a.nnz[d] = n;
    __syncthreads();
  }
}

__global__ void idf_kernel(const uint32_t* __restrict__ df_rep, uint32_t reps, uint32_t vocab, uint32_t n_docs,
                           int weight_mode, uint32_t* __restrict__ df, TermInfo* __restrict__ info) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < vocab; t += gridDim.x * blockDim.x) {
    uint32_t c = 0;
    for (uint32_t r = 0; r < reps; ++r) c += df_rep[static_cast<size_t>(r) * vocab + t];
    df[t] = c;
    float idf = 1.0f;
    if (weight_mode == 1) idf = static_cast<float>(log((1.0 + n_docs) / (1.0 + df[t])) + 1.0);
    info[t] = TermInfo{idf, -1};
  }
}

// idf from an externally reduced df (multi-GPU: each rank counts its shard of
// documents, df is all-reduced, then every rank recomputes the same table).
__global__ void idf_from_df_kernel(const uint32_t* __restrict__ df, uint32_t vocab, uint32_t n_docs, int weight_mode,
                                   TermInfo* __restrict__ info) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < vocab; t += gridDim.x * blockDim.x) {
    float idf = 1.0f;
    if (weight_mode == 1) idf = static_cast<float>(log((1.0 + n_docs) / (1.0 + df[t])) + 1.0);
    info[t] = TermInfo{idf, -1};
  }
}

// corpus_freq (SPEC.md FrequencyTable): cf[t] += count of every (doc, t) row,
// 64-bit atomics into R replicas (replica = warp index mod R: Zipf-head terms
// are in every document), then summed by cf_sum_kernel. Integer sums: exact.
__global__ void __launch_bounds__(256) cf_rows_kernel(const uint2* __restrict__ ent, const uint64_t* __restrict__ doc_off,
                                                      const uint32_t* __restrict__ nnz, uint32_t n_docs, uint32_t vocab,
                                                      uint32_t reps, unsigned long long* __restrict__ cf_rep) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (d >= n_docs) return;
  unsigned long long* rep = cf_rep + static_cast<size_t>(d % reps) * vocab;
  const uint2* e = ent + doc_off[d];
  for (uint32_t i = lane; i < nnz[d]; i += 32) {
    const uint2 x = e[i];
    atomicAdd(rep + x.x, static_cast<unsigned long long>(x.y));
  }
}

__global__ void cf_sum_kernel(const unsigned long long* __restrict__ cf_rep, uint32_t reps, uint32_t vocab,
                              uint64_t* __restrict__ cf) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < vocab; t += gridDim.x * blockDim.x) {
    unsigned long long c = 0;
    for (uint32_t r = 0; r < reps; ++r) c += cf_rep[static_cast<size_t>(r) * vocab + t];
    cf[t] = c;
  }
}

// Warp per doc.
__global__ void compact_csr_kernel(const uint2* __restrict__ ent, const uint64_t* __restrict__ doc_off,
                                   const uint32_t* __restrict__ nnz, const uint64_t* __restrict__ rowptr,
                                   uint32_t n_docs, uint32_t* __restrict__ ids, uint32_t* __restrict__ counts) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); d < n_docs; d += warps) {
    const uint2* src = ent + doc_off[d];
    const uint64_t dst = rowptr[d];
    const uint32_t n = nnz[d];
    for (uint32_t i = lane; i < n; i += 32) {
      uint2 e = src[i];
      ids[dst + i] = e.x;
      counts[dst + i] = e.y;
    }
  }
}

__global__ void inv_norm_kernel(const uint2* __restrict__ ent, const uint64_t* __restrict__ doc_off,
                                const uint32_t* __restrict__ nnz, const TermInfo* __restrict__ info,
                                uint32_t n_docs, float* __restrict__ inv_norm) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); d < n_docs; d += warps) {
    const uint2* src = ent + doc_off[d];
    const uint32_t n = nnz[d];
    float sq = 0.0f;
    for (uint32_t i = lane; i < n; i += 32) {
      uint2 e = src[i];
      float w = static_cast<float>(e.y) * info[e.x].idf;
      sq = fmaf(w, w, sq);
    }
    sq = warp_sum(sq);
    if (lane == 0) inv_norm[d] = sq > 0.0f ? 1.0f / sqrtf(sq) : 0.0f;
  }
}

int grid_for(uint64_t n, int per_sm) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  uint64_t g = static_cast<uint64_t>(sms) * per_sm;
  if (g > n) g = n;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

void launch_count_warp(int ipt, const CountArgs& a, const uint32_t* docs, uint32_t n, cudaStream_t s) {
  if (n == 0) return;
  const unsigned blocks = static_cast<unsigned>(ceil_div(n, 8));  // one warp per doc
  if (ipt == 2)
    count_warp_kernel<2><<<blocks, 256, 0, s>>>(a, docs, n);
  else if (ipt == 4)
    count_warp_kernel<4><<<blocks, 256, 0, s>>>(a, docs, n);
  else
    count_warp_kernel<8><<<blocks, 256, 0, s>>>(a, docs, n);
  note_launch();
}

void launch_count_group(int cls, const CountArgs& a, const uint32_t* docs, uint32_t n, cudaStream_t s) {
  if (n == 0) return;
  // split pass (group_split_kernel) for the classes in the mask (bit cls + 1); REFSIG_K1_SPLIT overrides
  static const uint32_t split_mask = [] {
    const char* m = std::getenv("REFSIG_K1_SPLIT");
    return m ? static_cast<uint32_t>(std::strtoul(m, nullptr, 0)) : 0x1Cu;  // classes 1-3 (>= 1025 tokens): measured A/B per class
  }();
  if ((split_mask >> (cls + 1)) & 1u) {
    switch (cls) {
      case -1: group_split_kernel<2><<<n, 64, 0, s>>>(a, docs, n); break;
      case 0: group_split_kernel<4><<<n, 128, 0, s>>>(a, docs, n); break;
      case 1: group_split_kernel<8><<<n, 256, 0, s>>>(a, docs, n); break;
      case 2: group_split_kernel<16><<<n, 512, 0, s>>>(a, docs, n); break;
      default: group_split_kernel<32><<<n, 1024, 0, s>>>(a, docs, n); break;
    }
    note_launch();
    return;
  }
  // 8 keys per thread: twice the threads of 16-key groups, half the serial
  // compare-exchange chain per thread (measured faster for every class)
  switch (cls) {
    case -1:  // 257..512 tokens
      group_sort_kernel<2, 8><<<n, 64, 0, s>>>(a, docs, n);
      break;
    case 0:
      group_sort_kernel<4, 8><<<n, 128, 0, s>>>(a, docs, n);
      break;
    case 1:
      group_sort_kernel<8, 8><<<n, 256, 0, s>>>(a, docs, n);
      break;
    case 2:
      group_sort_kernel<16, 8><<<n, 512, 0, s>>>(a, docs, n);
      break;
    default:
      group_sort_kernel<32, 8><<<n, 1024, 0, s>>>(a, docs, n);
      break;
  }
  note_launch();
}

void launch_count_large(const CountArgs& a, const uint32_t* long_docs, const uint64_t* scratch_off, uint32_t n_long,
                        uint32_t* scratch, cudaStream_t s) {
  if (n_long == 0) return;
  count_large_kernel<<<grid_for(n_long, 1), 1024, 0, s>>>(a, long_docs, scratch_off, n_long, scratch);
  note_launch();
}

void launch_idf(const uint32_t* df_rep, uint32_t reps, uint32_t vocab, uint32_t n_docs, int weight_mode, uint32_t* df,
                TermInfo* info, cudaStream_t s) {
  idf_kernel<<<grid_for((vocab + 255) / 256, 8), 256, 0, s>>>(df_rep, reps, vocab, n_docs, weight_mode, df, info);
  note_launch();
}

void launch_idf_from_df(const uint32_t* df, uint32_t vocab, uint32_t n_docs, int weight_mode, TermInfo* info,
                        cudaStream_t s) {
  idf_from_df_kernel<<<grid_for((vocab + 255) / 256, 8), 256, 0, s>>>(df, vocab, n_docs, weight_mode, info);
  note_launch();
}

void launch_corpus_freq(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, uint32_t n_docs,
                        uint32_t vocab, uint32_t reps, unsigned long long* cf_rep, uint64_t* cf, cudaStream_t s) {
  cudaMemsetAsync(cf_rep, 0, sizeof(unsigned long long) * static_cast<size_t>(reps) * vocab, s);
  if (n_docs)
    cf_rows_kernel<<<static_cast<unsigned>(ceil_div(n_docs, 8)), 256, 0, s>>>(ent, doc_off, nnz, n_docs, vocab, reps,
                                                                             cf_rep);
  cf_sum_kernel<<<grid_for((vocab + 255) / 256, 8), 256, 0, s>>>(cf_rep, reps, vocab, cf);
  note_launch();
  note_launch();
}

void launch_compact_csr(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, const uint64_t* rowptr,
                        uint32_t n_docs, uint32_t* ids, uint32_t* counts, cudaStream_t s) {
  if (n_docs == 0) return;
  compact_csr_kernel<<<grid_for((n_docs + 7) / 8, 16), 256, 0, s>>>(ent, doc_off, nnz, rowptr, n_docs, ids, counts);
  note_launch();
}

void launch_inv_norm(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, const TermInfo* info,
                     uint32_t n_docs, float* inv_norm, cudaStream_t s) {
  if (n_docs == 0) return;
  inv_norm_kernel<<<grid_for((n_docs + 7) / 8, 16), 256, 0, s>>>(ent, doc_off, nnz, info, n_docs, inv_norm);
  note_launch();
}

}  // namespace refsig_gpu
