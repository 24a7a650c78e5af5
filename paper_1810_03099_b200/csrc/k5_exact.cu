// k5_exact.cu — K5: exact sparse cosine verifier.
//
// Reference: cosine (ngram.hpp:184-202) = dot/(|a||b|) over the sorted sparse
// vectors, 0 for an empty vector, clamped to 1. Here over the weighted
// (TF or TF-IDF) corpus vectors, x = w/||w||, in fp32.
//
// Head / tail split with exact bounds. The H terms of highest df (the Zipf
// head: at configs[1] the top 64 terms carry 77% of the sum of df*(df-1)/2
// multiply-adds but, being frequent, little TF-IDF weight; selected on the
// device by a stable descending sort of df) are kept as dense rows A[d][H]
// with their norm hn[d]; every term's postings are doc-sorted (a stable radix
// sort of the CSR slots by term id) and entpos gives each entry's position in
// its term's list. One CTA (32 warps) per row i (column panels of up to
// kExactPanel docs in shared memory):
//   1. tail: for each tail term of doc i, exactly the postings after doc i
//      (j > i) add round(x_i * x_j * 2^30) to acc[j] with a shared-memory
//      integer atomic — fixed-point sums are exact, so the result does not
//      depend on the order the atomics land in. The kept lists are walked as
//      one flat index space split evenly over the warps (32 postings per warp
//      step, two steps at once inside one term), so lanes stay busy whatever
//      the list lengths;
//   2. scan j > i: tail = acc[j] * 2^-30; since head_ij <= hn_i * hn_j
//      (Cauchy-Schwarz), only pairs with tail + hn_i*hn_j >= tau - 1e-5 can
//      match; for those the head dot A_i . A_j (H fused multiply-adds in a
//      fixed order) is added and cos = min(tail + head, 1) >= tau sets the
//      pair's bit (shared pair bitmap, common emitter).
// Deterministic; the work is the tail's sum of df(df-1)/2 (424 M postings at
// configs[1]) plus a dense scan of the triangle. Fixed-point error <= 2^-31
// per product (< 1e-7 per pair for < 200 shared tail terms), far inside the
// 1e-5 border band of the parity tests.
//
// pair_cosines: warp per pair; lanes walk doc i's rows, binary-search doc j's
// sorted ids, warp-tree sum.

#include <algorithm>

#include <cub/device/device_radix_sort.cuh>

#include "kernels.cuh"

namespace refsig_gpu {
namespace {

__global__ void unit_weights_kernel(const uint2* __restrict__ ent, const uint64_t* __restrict__ doc_off,
                                    const uint32_t* __restrict__ nnz, const TermInfo* __restrict__ info,
                                    const float* __restrict__ inv_norm, uint32_t n_docs, float* __restrict__ x) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); d < n_docs; d += nw) {
    const uint64_t b = doc_off[d];
    const uint32_t n = nnz[d];
    const float inv = inv_norm[d];
    for (uint32_t i = lane; i < n; i += 32) {
      const uint2 e = ent[b + i];
      x[b + i] = static_cast<float>(e.y) * info[e.x].idf * inv;
    }
  }
}

// Dense head rows A[d][H] (zeroed by the caller) and hn[d] = ||head part||.
__global__ void head_rows_kernel(const uint2* __restrict__ ent, const uint64_t* __restrict__ doc_off,
                                 const uint32_t* __restrict__ nnz, const float* __restrict__ x,
                                 const int32_t* __restrict__ head_col, uint32_t n_docs, uint32_t H,
                                 float* __restrict__ A, float* __restrict__ hn) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (d >= n_docs) return;
  const uint64_t b = doc_off[d];
  const uint32_t n = nnz[d];
  float sq = 0.0f;
  for (uint32_t i = lane; i < n; i += 32) {
    const int32_t c = head_col[ent[b + i].x];
    if (c >= 0) {
      const float v = x[b + i];
      A[static_cast<size_t>(d) * H + c] = v;
      sq = fmaf(v, v, sq);
    }
  }
  sq = warp_sum(sq);
  if (lane == 0) hn[d] = sqrtf(sq);
}

constexpr float kFix = 1073741824.0f;  // 2^30
constexpr uint32_t kTailBatch = 1024;    // doc-i terms per batch (one per thread)

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint2 lds_u2(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint2 ldg_u2(const uint2* p) {
  uint2 v;
  asm("ld.global.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void reds_add(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Block-wide exclusive scan of v over the kTailBatch threads (warp scans + warp totals).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* part, uint32_t& total) {
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t inc = warp_inclusive_scan(v, static_cast<int>(lane));
  if (lane == 31) part[wid] = inc;
  __syncthreads();
  const uint32_t x = part[lane];  // kTailBatch / 32 == 32 warp totals
  const uint32_t xi = warp_inclusive_scan(x, static_cast<int>(lane));
  const uint32_t off = __shfl_sync(0xffffffffu, xi - x, wid);
  total = __shfl_sync(0xffffffffu, xi, 31);
  __syncthreads();  // part is reused by the next scan
  return off + inc - v;
}

// Row i per CTA (32 warps). Tail terms of doc i in batches of 1024: each keeps
// the part of its doc-sorted posting list after doc i — [entpos(i, t) + 1,
// end of t) — and the kept lists are walked as ONE flat index space split
// evenly over the warps: 32 consecutive postings per warp step, lane l's term
// found from the starts inside the 32-wide window (one OR-reduction +
// popcount), so every lane does a posting per step whatever the list lengths.
__global__ void __launch_bounds__(kTailBatch) exact_tail_kernel(ExactArgs a, uint32_t row_lo) {
  extern __shared__ uint4 acc4[];  // [panel/4] fixed-point tail sums, then H floats of A_i
  uint32_t* acc = reinterpret_cast<uint32_t*>(acc4);
  __shared__ uint32_t red[32];
  __shared__ uint32_t s_start[kTailBatch];  // flat start of kept term k
  __shared__ uint2 s_rec[kTailBatch];       // (first posting after doc i, x_i bits) of kept term k
  const uint32_t i = row_lo + blockIdx.x;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const uint64_t b = a.doc_off[i];
  const uint32_t n = a.nnz[i];
  float* ai = reinterpret_cast<float*>(acc + (a.panel + 3) / 4 * 4);
  for (uint32_t k = threadIdx.x; k < a.H; k += blockDim.x) ai[k] = a.A[static_cast<size_t>(i) * a.H + k];
  const float hni = a.hn[i];
  uint32_t cnt = 0;
  uint32_t* rowbits = a.bitmap + static_cast<size_t>(i) * a.words_per_row;
  for (uint32_t c0 = (i + 1) / a.panel * a.panel; c0 < a.n_docs; c0 += a.panel) {
    const uint32_t c1 = min(a.n_docs, c0 + a.panel);
    const uint32_t jlo = max(c0, i + 1);
    for (uint32_t k = threadIdx.x; k < (c1 - c0 + 3) / 4; k += blockDim.x) acc4[k] = make_uint4(0u, 0u, 0u, 0u);
    // 1. tail products x_i * x_j of every shared tail term, j > i, into acc[j - c0]
    for (uint32_t p0 = 0; p0 < n; p0 += kTailBatch) {
      const uint32_t p = p0 + threadIdx.x;
      uint32_t len = 0, q = 0;
      float xi = 0.0f;
      if (p < n) {
        const uint32_t t = a.ent[b + p].x;
        if (a.head_col[t] < 0) {
          q = a.entpos[b + p] + 1u;
          len = static_cast<uint32_t>(a.post_off[t + 1]) - q;
          xi = a.x[b + p];
        }
      }
      uint32_t n_kept, M;
      const uint32_t k = block_excl_scan(len ? 1u : 0u, red, n_kept);
      const uint32_t f = block_excl_scan(len, red, M);
      if (len) {
        s_start[k] = f;
        s_rec[k] = make_uint2(q - f, __float_as_uint(xi));  // posting of flat index idx: q - f + idx
      }
      __syncthreads();
      const uint32_t per = (M + nwarp - 1) / nwarp;
      const uint32_t f0 = min(M, wid * per), f1 = min(M, f0 + per);
      if (f0 < f1) {
        // cur = last kept term starting before f0 (-1 if none)
        int lo = 0, hi = static_cast<int>(n_kept);
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (s_start[mid] < f0) lo = mid + 1; else hi = mid;
        }
        int cur = lo - 1;
        // shared-window addresses computed once (the compiler otherwise rebuilds them every step)
        uint32_t start_a = static_cast<uint32_t>(__cvta_generic_to_shared(s_start));
        uint32_t rec_a = static_cast<uint32_t>(__cvta_generic_to_shared(s_rec));
        uint32_t acc_a = static_cast<uint32_t>(__cvta_generic_to_shared(acc));
        const uint2* posts = a.posts;
        asm volatile("" : "+r"(start_a), "+r"(rec_a), "+r"(acc_a), "+l"(posts));  // opaque: kept in registers
        const uint32_t le = (2u << lane) - 1u, span = c1 - c0;
        const int nk = static_cast<int>(n_kept);
        // the term containing the window start and where the next one starts
        uint2 rec = cur >= 0 ? lds_u2(rec_a + 8u * cur) : make_uint2(0u, 0u);
        uint32_t next = cur + 1 < nk ? lds_u32(start_a + 4u * (cur + 1)) : 0xFFFFFFFFu;
        uint32_t base = f0;
        while (base < f1) {
          if (next >= base + 64u && base + 32u < f1) {  // two whole windows inside the current term
            const uint32_t idx = base + lane;
            const uint2 p0 = ldg_u2(posts + rec.x + idx);
            const bool in2 = idx + 32u < f1;
            const uint2 p1 = in2 ? ldg_u2(posts + rec.x + idx + 32u) : make_uint2(0xFFFFFFFFu, 0u);
            const float xr = __uint_as_float(rec.y) * kFix;
            const uint32_t j0 = p0.x - c0, j1 = p1.x - c0;
            if (j0 < span) reds_add(acc_a + 4u * j0, __float2uint_rn(xr * __uint_as_float(p0.y)));
            if (j1 < span) reds_add(acc_a + 4u * j1, __float2uint_rn(xr * __uint_as_float(p1.y)));
            base += 64u;
            continue;
          }
          const uint32_t idx = base + lane;
          uint2 r = rec;
          if (next < base + 32u) {  // a term starts inside the window: per-lane terms
            const int m = cur + 1 + static_cast<int>(lane);
            const uint32_t sm = m < nk ? lds_u32(start_a + 4u * m) : 0xFFFFFFFFu;
            const uint32_t bits = __reduce_or_sync(0xffffffffu, sm < base + 32u ? 1u << (sm - base) : 0u);
            const int term = cur + __popc(bits & le);
            if (term != cur) r = lds_u2(rec_a + 8u * term);
            cur += __popc(bits);
            rec = lds_u2(rec_a + 8u * cur);
            next = cur + 1 < nk ? lds_u32(start_a + 4u * (cur + 1)) : 0xFFFFFFFFu;
          }
          if (idx < f1) {
            const uint2 pj = ldg_u2(posts + r.x + idx);
            const uint32_t jj = pj.x - c0;
            if (jj < span) reds_add(acc_a + 4u * jj, __float2uint_rn(__uint_as_float(r.y) * kFix * __uint_as_float(pj.y)));
          }
          base += 32u;
        }
      }
      __syncthreads();
    }
    if (a.tail_out) {  // evaluation mode: hand the exact tail sums to the tile pass
      uint32_t* dst = a.tail_out + static_cast<size_t>(blockIdx.x) * a.tail_ld;
      for (uint32_t j = jlo + threadIdx.x; j < c1; j += blockDim.x) dst[j] = acc[j - c0];
      __syncthreads();
      continue;
    }
    // 2. bound, head dot, threshold
    for (uint32_t j = jlo + threadIdx.x; j < c1; j += blockDim.x) {
      const float tail = static_cast<float>(acc[j - c0]) * (1.0f / kFix);
      const float hnj = a.hn[j];
      if (tail + hni * hnj >= a.tau - 1e-5f) {
        const float4* aj = reinterpret_cast<const float4*>(a.A + static_cast<size_t>(j) * a.H);
        float head = 0.0f;
        for (uint32_t k = 0; k < a.H / 4; ++k) {
          const float4 v = __ldg(aj + k);
          head = fmaf(ai[4 * k + 0], v.x, head);
          head = fmaf(ai[4 * k + 1], v.y, head);
          head = fmaf(ai[4 * k + 2], v.z, head);
          head = fmaf(ai[4 * k + 3], v.w, head);
        }
        if (fminf(tail + head, 1.0f) >= a.tau) {
          atomicOr(rowbits + (j >> 5), 1u << (j & 31));
          ++cnt;
        }
      }
    }
    __syncthreads();
  }
  cnt = warp_sum_u32(cnt);
  if (lane == 0) red[wid] = cnt;
  __syncthreads();
  if (threadIdx.x == 0 && !a.tail_out) {
    uint32_t s = 0;
    for (uint32_t w = 0; w < nwarp; ++w) s += red[w];
    a.rowcnt[i] = s;
  }
}

// Doc-sorted postings (CSC) of every term: a STABLE radix sort of the padded
// CSR slots — already in document order — by term id alone (padding slots get
// the key V, after every term), so each term's list comes out in document
// order; posting q = (doc of the slot, x[slot]) and entpos[slot] = q — the
// position of entry (d, t) inside t's list, so row i's walk starts right
// after itself.
__global__ void csc_keys_kernel(const uint2* __restrict__ ent, const uint64_t* __restrict__ doc_off,
                                const uint32_t* __restrict__ nnz, uint32_t n_docs, uint32_t vocab,
                                uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                uint32_t* __restrict__ slot_doc) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); d < n_docs; d += nw) {
    const uint64_t b = doc_off[d], e = doc_off[d + 1];
    const uint32_t n = nnz[d];
    for (uint64_t s = b + lane; s < e; s += 32) {
      keys[s] = s - b < n ? ent[s].x : vocab;
      vals[s] = static_cast<uint32_t>(s);
      slot_doc[s] = d;
    }
  }
}

__global__ void csc_fill_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t n_slots,
                                uint32_t vocab, const uint32_t* __restrict__ slot_doc, const float* __restrict__ x,
                                uint2* __restrict__ posts, uint32_t* __restrict__ entpos) {
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < n_slots;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (keys[q] >= vocab) break;  // padding sorts last
    const uint32_t s = vals[q];
    posts[q] = make_uint2(slot_doc[s], __float_as_uint(x[s]));
    entpos[s] = static_cast<uint32_t>(q);
  }
}

// ---- fused evaluation tiles (Eq. 2/3 of the paper, SPEC.md eval) ----------
// 64 x 128 pair tiles of the triangle, contiguous tile ranges per CTA; thread
// (ty, tx) owns rows ty*4..+3 and columns tx*8..+7 (32 pairs). Per tile: the
// head dot (H k-steps) and the MRC dot (K k-steps) from k-major panels staged
// in shared memory, the tail sums T (exact fixed point), the fingerprints;
// per pair the two errors against the exact cosine go into per-thread double
// sums (n, sum e, sum e^2, sum |e|) that are reduced in a fixed order.
constexpr int kEvR = 64, kEvC = 128;

// Tile t of row blocks br0.. (64 rows each): row block r has the col blocks
// r/2 .. nbc-1 (128 columns each, the ones holding some j > i).
__device__ __forceinline__ void eval_tile_coords(uint32_t t, uint32_t br0, uint32_t br1, uint32_t nbc, uint32_t& bi,
                                                 uint32_t& bj) {
  uint32_t r = br0;
  while (r < br1) {
    const uint32_t cnt = nbc - r / 2;
    if (t < cnt) break;
    t -= cnt;
    ++r;
  }
  bi = r;
  bj = r / 2 + t;
}

template <bool HEAD>
__device__ __forceinline__ void eval_dot(const float* __restrict__ src, uint32_t KK, uint32_t ld, uint32_t r0,
                                         uint32_t cb, float* P, float* Q, uint32_t tid, uint32_t tx, uint32_t ty,
                                         float (&acc)[4][8]) {
  for (uint32_t k0 = 0; k0 < KK; k0 += 32) {
    const uint32_t kc = min(32u, KK - k0);
    __syncthreads();
    for (uint32_t idx = tid; idx < kc * kEvR; idx += 256) {
      const uint32_t k = idx / kEvR, rr = idx % kEvR;
      P[k * kEvR + rr] = src[static_cast<size_t>(k0 + k) * ld + r0 + rr];
    }
    for (uint32_t idx = tid; idx < kc * kEvC; idx += 256) {
      const uint32_t k = idx / kEvC, cc = idx % kEvC;
      Q[k * kEvC + cc] = src[static_cast<size_t>(k0 + k) * ld + cb + cc];
    }
    __syncthreads();
    for (uint32_t k = 0; k < kc; ++k) {
      const float4 pa = *reinterpret_cast<const float4*>(P + k * kEvR + ty * 4);
      const float4 q0 = *reinterpret_cast<const float4*>(Q + k * kEvC + tx * 8);
      const float4 q1 = *reinterpret_cast<const float4*>(Q + k * kEvC + tx * 8 + 4);
      const float av[4] = {pa.x, pa.y, pa.z, pa.w};
      const float bv[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
    }
  }
}

__global__ void __launch_bounds__(256) eval_tiles_kernel(EvalArgs a, uint32_t nbr, uint32_t nbc, uint32_t br0,
                                                         uint64_t n_tiles) {
  extern __shared__ __align__(16) float esm[];  // A rows [kk][64] | A cols [kk][128], kk <= 32 per chunk
  __shared__ double red[8][8];
  const uint32_t tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const uint64_t t0 = n_tiles * blockIdx.x / gridDim.x, t1 = n_tiles * (blockIdx.x + 1) / gridDim.x;
  double sm_e = 0, sm_q = 0, sm_a = 0, ss_e = 0, ss_q = 0, ss_a = 0;
  uint64_t cnt = 0;
  float* P = esm;               // rows panel [32][64]
  float* Q = esm + 32 * kEvR;   // cols panel [32][128]
  for (uint64_t t = t0; t < t1; ++t) {
    uint32_t bi, bj;
    eval_tile_coords(static_cast<uint32_t>(t), br0, br0 + nbr, nbc, bi, bj);
    const uint32_t r0 = bi * kEvR, cb = bj * kEvC;
    float hd[4][8], md[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) hd[r][c] = md[r][c] = 0.0f;
    eval_dot<true>(a.AT, a.H, a.ld, r0, cb, P, Q, tid, tx, ty, hd);   // head dot (exact cosine part)
    eval_dot<false>(a.ST, a.K, a.ld, r0, cb, P, Q, tid, tx, ty, md);  // MRC compare
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t i = r0 + ty * 4 + r;
      if (i < a.row_lo || i >= a.row_hi) continue;
      const uint32_t* trow = a.T + static_cast<size_t>(i - a.row_lo) * a.ldT;
      const uint64_t fi = a.fp ? a.fp[i] : 0ull;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint32_t j = cb + tx * 8 + c;
        if (j <= i || j >= a.n_docs) continue;
        const float ex = fminf(hd[r][c] + static_cast<float>(trow[j]) * (1.0f / 1073741824.0f), 1.0f);
        const double em = static_cast<double>(fminf(md[r][c], 1.0f)) - static_cast<double>(ex);
        sm_e += em;
        sm_q = fma(em, em, sm_q);
        sm_a += fabs(em);
        if (a.fp) {
          const double es = (1.0 - __popcll(fi ^ a.fp[j]) / 64.0) - static_cast<double>(ex);
          ss_e += es;
          ss_q = fma(es, es, ss_q);
          ss_a += fabs(es);
        }
        ++cnt;
      }
    }
  }
  // fixed-order reduction: warp tree, then warps in order
  double v[7] = {static_cast<double>(cnt), sm_e, sm_q, sm_a, ss_e, ss_q, ss_a};
#pragma unroll
  for (int q = 0; q < 7; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  if ((tid & 31) == 0)
#pragma unroll
    for (int q = 0; q < 7; ++q) red[tid >> 5][q] = v[q];
  __syncthreads();
  if (tid < 7) {
    double x = 0;
    for (int w = 0; w < 8; ++w) x += red[w][tid];
    a.out[blockIdx.x * 8 + tid] = x;
  }
  if (tid == 7) a.out[blockIdx.x * 8 + 7] = 0.0;
}

__global__ void transpose_head_kernel(const float* __restrict__ A, uint32_t n, uint32_t H, uint32_t ld,
                                      float* __restrict__ AT) {
  __shared__ float tile[32][33];
  const uint32_t d0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (uint32_t r = threadIdx.y; r < 32; r += blockDim.y) {
    const uint32_t d = d0 + r, c = c0 + threadIdx.x;
    tile[r][threadIdx.x] = (d < n && c < H) ? A[static_cast<size_t>(d) * H + c] : 0.0f;
  }
  __syncthreads();
  for (uint32_t r = threadIdx.y; r < 32; r += blockDim.y) {
    const uint32_t c = c0 + r, d = d0 + threadIdx.x;
    if (c < H && d < ld) AT[static_cast<size_t>(c) * ld + d] = tile[threadIdx.x][r];
  }
}

__device__ __forceinline__ int lower_bound_ids(const uint2* e, uint32_t n, uint32_t key) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (e[mid].x < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return static_cast<int>(lo);
}

__global__ void pair_cosines_kernel(const uint2* __restrict__ ent, const uint64_t* __restrict__ doc_off,
                                    const uint32_t* __restrict__ nnz, const float* __restrict__ x,
                                    const uint64_t* __restrict__ keys, uint64_t n_keys, float* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < n_keys; q += nw) {
    uint32_t i = static_cast<uint32_t>(keys[q] >> 32), j = static_cast<uint32_t>(keys[q]);
    uint32_t ni = nnz[i], nj = nnz[j];
    if (ni > nj) {  // walk the shorter vector
      uint32_t t = i; i = j; j = t;
      t = ni; ni = nj; nj = t;
    }
    const uint2* ei = ent + doc_off[i];
    const uint2* ej = ent + doc_off[j];
    const float* xi = x + doc_off[i];
    const float* xj = x + doc_off[j];
    float dot = 0.0f;
    for (uint32_t p = lane; p < ni; p += 32) {
      const uint32_t t = ei[p].x;
      const int k = lower_bound_ids(ej, nj, t);
      if (k < static_cast<int>(nj) && ej[k].x == t) dot = fmaf(xi[p], xj[k], dot);
    }
    dot = warp_sum(dot);
    if (lane == 0) out[q] = (ni == 0 || nj == 0) ? 0.0f : fminf(dot, 1.0f);
  }
}

int sm_count() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

}  // namespace

void launch_unit_weights(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, const TermInfo* info,
                         const float* inv_norm, uint32_t n_docs, float* x, cudaStream_t s) {
  if (!n_docs) return;
  unsigned g = static_cast<unsigned>(std::min<uint64_t>(ceil_div(n_docs, 8), sm_count() * 16ull));
  unit_weights_kernel<<<g, 256, 0, s>>>(ent, doc_off, nnz, info, inv_norm, n_docs, x);
  note_launch();
}

static int bit_length(uint64_t v) { return v ? 64 - __builtin_clzll(v) : 1; }

size_t csc_sort_temp_bytes(uint64_t n_slots, uint32_t vocab) {
  size_t bytes = 0;
  cub::DoubleBuffer<uint32_t> k(nullptr, nullptr);
  cub::DoubleBuffer<uint32_t> v(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, v, static_cast<int64_t>(n_slots), 0, bit_length(vocab));
  return bytes;
}

void build_csc_postings(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, uint32_t n_docs,
                        uint32_t vocab, uint64_t n_slots, const float* x, uint32_t* keys_a, uint32_t* keys_b,
                        uint32_t* vals_a, uint32_t* vals_b, uint32_t* slot_doc, void* tmp, size_t tmp_bytes,
                        uint2* posts, uint32_t* entpos, cudaStream_t s) {
  if (!n_slots) return;
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>(ceil_div(n_docs, 8), sm_count() * 16ull));
  csc_keys_kernel<<<g, 256, 0, s>>>(ent, doc_off, nnz, n_docs, vocab, keys_a, vals_a, slot_doc);
  note_launch();
  cub::DoubleBuffer<uint32_t> k(keys_a, keys_b);
  cub::DoubleBuffer<uint32_t> v(vals_a, vals_b);
  size_t bytes = tmp_bytes;
  cub::DeviceRadixSort::SortPairs(tmp, bytes, k, v, static_cast<int64_t>(n_slots), 0, bit_length(vocab), s);  // stable
  note_launch();
  const unsigned g2 = static_cast<unsigned>(std::min<uint64_t>(ceil_div(n_slots, 256), sm_count() * 8ull));
  csc_fill_kernel<<<g2, 256, 0, s>>>(k.Current(), v.Current(), n_slots, vocab, slot_doc, x, posts, entpos);
  note_launch();
}

// Head terms on the device: a stable descending radix sort of (df, id) —
// equal df keep ascending ids — and head_col[id_k] = k for the first H.
__global__ void head_keys_kernel(const uint32_t* __restrict__ df, uint32_t vocab, uint32_t* __restrict__ keys,
                                 uint32_t* __restrict__ ids, int32_t* __restrict__ head_col) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < vocab; t += gridDim.x * blockDim.x) {
    keys[t] = df[t];
    ids[t] = t;
    head_col[t] = -1;
  }
}
__global__ void head_col_kernel(const uint32_t* __restrict__ ids, uint32_t H, int32_t* __restrict__ head_col) {
  for (uint32_t k = threadIdx.x; k < H; k += blockDim.x) head_col[ids[k]] = static_cast<int32_t>(k);
}

size_t head_select_temp_bytes(uint32_t vocab) {
  size_t bytes = 0;
  cub::DoubleBuffer<uint32_t> k(nullptr, nullptr);
  cub::DoubleBuffer<uint32_t> v(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, k, v, static_cast<int64_t>(vocab));
  return bytes;
}

void launch_head_select(const uint32_t* df, uint32_t vocab, uint32_t H, uint32_t* keys_a, uint32_t* keys_b,
                        uint32_t* ids_a, uint32_t* ids_b, void* tmp, size_t tmp_bytes, int32_t* head_col,
                        cudaStream_t s) {
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>(ceil_div(vocab, 256), sm_count() * 8ull));
  head_keys_kernel<<<g, 256, 0, s>>>(df, vocab, keys_a, ids_a, head_col);
  note_launch();
  cub::DoubleBuffer<uint32_t> k(keys_a, keys_b);
  cub::DoubleBuffer<uint32_t> v(ids_a, ids_b);
  size_t bytes = tmp_bytes;
  cub::DeviceRadixSort::SortPairsDescending(tmp, bytes, k, v, static_cast<int64_t>(vocab), 0, 32, s);  // stable
  note_launch();
  head_col_kernel<<<1, 256, 0, s>>>(v.Current(), std::min(H, vocab), head_col);
  note_launch();
}

void launch_head_rows(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, const float* x,
                      const int32_t* head_col, uint32_t n_docs, uint32_t H, float* A, float* hn, cudaStream_t s) {
  if (!n_docs) return;
  head_rows_kernel<<<static_cast<unsigned>(ceil_div(n_docs, 8)), 256, 0, s>>>(ent, doc_off, nnz, x, head_col, n_docs,
                                                                              H, A, hn);
  note_launch();
}

void launch_exact_tail(const ExactArgs& a, uint32_t row_lo, uint32_t row_hi, cudaStream_t s) {
  if (row_hi <= row_lo) return;
  const size_t smem = sizeof(uint32_t) * ((a.panel + 3) / 4 * 4 + a.H);
  ensure_smem(exact_tail_kernel, smem);
  exact_tail_kernel<<<row_hi - row_lo, kTailBatch, smem, s>>>(a, row_lo);
  note_launch();
}

uint32_t eval_grid() { return static_cast<uint32_t>(sm_count()) * 2; }

void launch_eval_tiles(const EvalArgs& a, cudaStream_t s) {
  if (a.row_hi <= a.row_lo) return;
  const uint32_t br0 = a.row_lo / kEvR, br1 = static_cast<uint32_t>(ceil_div(a.row_hi, kEvR));
  const uint32_t nbc = static_cast<uint32_t>(ceil_div(a.n_docs, kEvC));
  // tiles of row blocks [br0, br1): block r has col blocks r/2 .. nbc-1 (global r)
  uint64_t n_tiles = 0;
  for (uint32_t r = br0; r < br1; ++r) n_tiles += nbc - r / 2;
  // eval_tile_coords enumerates from row block br0 with the same rule: shift by br0 (even, panels
  // start at multiples of 128 rows = 2 row blocks) so r/2 stays the global value
  const size_t smem = sizeof(float) * 32 * (kEvR + kEvC);
  eval_tiles_kernel<<<eval_grid(), 256, smem, s>>>(a, br1 - br0, nbc, br0, n_tiles);
  note_launch();
}

void launch_transpose_head(const float* A, uint32_t n_docs, uint32_t H, uint32_t ld, float* AT, cudaStream_t s) {
  dim3 g(static_cast<unsigned>(ceil_div(ld, 32)), static_cast<unsigned>(ceil_div(H, 32)));
  transpose_head_kernel<<<g, dim3(32, 8), 0, s>>>(A, n_docs, H, ld, AT);
  note_launch();
}

void launch_pair_cosines(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, const float* x,
                         const uint64_t* keys, uint64_t n_keys, float* out, cudaStream_t s) {
  if (!n_keys) return;
  unsigned g = static_cast<unsigned>(std::min<uint64_t>(ceil_div(n_keys, 8), sm_count() * 16ull));
  pair_cosines_kernel<<<g, 256, 0, s>>>(ent, doc_off, nnz, x, keys, n_keys, out);
  note_launch();
}

}  // namespace refsig_gpu
