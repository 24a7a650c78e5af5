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
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (uint32_t w = 0; w < nwarp; ++w) s += red[w];
    a.rowcnt[i] = s;
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
  static size_t configured = 0;
  if (smem > configured) {
    cudaFuncSetAttribute(exact_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured = smem;
  }
  exact_tail_kernel<<<row_hi - row_lo, 512, smem, s>>>(a, row_lo);
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
