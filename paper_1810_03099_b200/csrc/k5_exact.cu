// k5_exact.cu — K5: exact sparse cosine verifier.
//
// Reference: cosine (ngram.hpp:184-202) = dot/(|a||b|) over the sorted sparse
// vectors, 0 for an empty vector, clamped to 1. Here over the weighted
// (TF or TF-IDF) corpus vectors, x = w/||w||, in fp32.
//
// v2: head / tail split with exact bounds. The H terms of highest df (the
// Zipf head: at configs[1] the top 64 terms carry 77% of the sum of
// df*(df-1)/2 multiply-adds but, being frequent, little TF-IDF weight) are
// kept as dense rows A[d][H] with their norm hn[d]; the other terms (tail) go
// to postings lists. One CTA per row i (column panels of up to kExactPanel
// docs in shared memory):
//   1. tail: for each tail term of doc i, every posting j > i adds
//      round(x_i * x_j * 2^30) to acc[j] with a shared-memory integer atomic —
//      fixed-point sums are exact, so the result is independent of the order
//      the atomics land in (no barrier per term);
//   2. scan j > i: tail = acc[j] * 2^-30; since head_ij <= hn_i * hn_j
//      (Cauchy-Schwarz), only pairs with tail + hn_i*hn_j >= tau - 1e-5 can
//      match; for those the head dot A_i . A_j (H fused multiply-adds in a
//      fixed order) is added and cos = min(tail + head, 1) >= tau sets the
//      pair's bit (shared pair bitmap, common emitter).
// Deterministic; the work is the tail's sum of df^2 (23% of the total at
// configs[1]) plus a dense scan of the triangle. Fixed-point error <= 2^-31
// per product (< 1e-7 per pair for < 200 shared tail terms), far inside the
// 1e-5 border band of the parity tests.
//
// pair_cosines: warp per pair; lanes walk doc i's rows, binary-search doc j's
// sorted ids, warp-tree sum.

#include <algorithm>

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

__global__ void postings_fill_kernel(const uint2* __restrict__ ent, const uint64_t* __restrict__ doc_off,
                                     const uint32_t* __restrict__ nnz, const float* __restrict__ x,
                                     const int32_t* __restrict__ head_col, uint32_t n_docs,
                                     uint64_t* __restrict__ fill, uint2* __restrict__ posts) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); d < n_docs; d += nw) {
    const uint64_t b = doc_off[d];
    const uint32_t n = nnz[d];
    for (uint32_t i = lane; i < n; i += 32) {
      const uint32_t t = ent[b + i].x;
      if (head_col && head_col[t] >= 0) continue;  // head terms live in the dense rows
      const uint64_t q = atomicAdd(reinterpret_cast<unsigned long long*>(fill + t), 1ull);
      posts[q] = make_uint2(d, __float_as_uint(x[b + i]));
    }
  }
}

// tdf[t] = df[t] for tail terms, 0 for head terms.
__global__ void tail_df_kernel(const uint32_t* __restrict__ df, const int32_t* __restrict__ head_col,
                               uint32_t vocab, uint32_t* __restrict__ tdf) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < vocab; t += gridDim.x * blockDim.x)
    tdf[t] = head_col[t] >= 0 ? 0u : df[t];
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

__global__ void __launch_bounds__(512) exact_tail_kernel(ExactArgs a, uint32_t row_lo) {
  extern __shared__ uint32_t acc[];  // [panel] fixed-point tail sums, then H floats of A_i
  __shared__ uint32_t red[16];
  const uint32_t i = row_lo + blockIdx.x;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const uint64_t b = a.doc_off[i];
  const uint32_t n = a.nnz[i];
  float* ai = reinterpret_cast<float*>(acc + a.panel);
  for (uint32_t k = threadIdx.x; k < a.H; k += blockDim.x) ai[k] = a.A[static_cast<size_t>(i) * a.H + k];
  const float hni = a.hn[i];
  uint32_t cnt = 0;
  uint32_t* rowbits = a.bitmap + static_cast<size_t>(i) * a.words_per_row;
  for (uint32_t c0 = (i + 1) / a.panel * a.panel; c0 < a.n_docs; c0 += a.panel) {
    const uint32_t c1 = min(a.n_docs, c0 + a.panel);
    const uint32_t jlo = max(c0, i + 1);
    for (uint32_t k = threadIdx.x; k < c1 - c0; k += blockDim.x) acc[k] = 0u;
    __syncthreads();
    // 1. tail terms of doc i: warp per term, lanes over its postings
    for (uint32_t p = wid; p < n; p += nwarp) {
      const uint32_t t = a.ent[b + p].x;
      if (a.head_col[t] >= 0) continue;
      const float xi = a.x[b + p];
      const uint64_t q1 = a.post_off[t + 1];
      for (uint64_t q = a.post_off[t] + lane; q < q1; q += 32) {
        const uint2 pj = a.posts[q];
        if (pj.x >= jlo && pj.x < c1) atomicAdd(&acc[pj.x - c0], __float2uint_rn(xi * __uint_as_float(pj.y) * kFix));
      }
    }
    __syncthreads();
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

void launch_postings_fill(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, const float* x,
                          const int32_t* head_col, uint32_t n_docs, uint64_t* fill, uint2* posts, cudaStream_t s) {
  if (!n_docs) return;
  unsigned g = static_cast<unsigned>(std::min<uint64_t>(ceil_div(n_docs, 8), sm_count() * 16ull));
  postings_fill_kernel<<<g, 256, 0, s>>>(ent, doc_off, nnz, x, head_col, n_docs, fill, posts);
  note_launch();
}

void launch_tail_df(const uint32_t* df, const int32_t* head_col, uint32_t vocab, uint32_t* tdf, cudaStream_t s) {
  unsigned g = static_cast<unsigned>(std::min<uint64_t>(ceil_div(vocab, 256), sm_count() * 8ull));
  tail_df_kernel<<<g, 256, 0, s>>>(df, head_col, vocab, tdf);
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
  const size_t smem = sizeof(uint32_t) * (a.panel + a.H);
  ensure_smem(exact_tail_kernel, smem);
  exact_tail_kernel<<<row_hi - row_lo, 512, smem, s>>>(a, row_lo);
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
