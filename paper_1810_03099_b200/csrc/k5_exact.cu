// k5_exact.cu — K5: exact sparse cosine verifier.
//
// Reference: cosine (ngram.hpp:184-202) = dot/(|a||b|) over the sorted sparse
// vectors, 0 for an empty vector, clamped to 1. Here over the weighted
// (TF or TF-IDF) corpus vectors, x = w/||w||, in fp32.
//
// v1 (this file): inverted-index accumulation. Postings (doc, x) per term are
// built on the device from the padded CSR (offsets = exclusive scan of df).
// One CTA owns a row i at a time and a private dense accumulator of n_docs
// floats: for each term of doc i in ascending id it adds x_i*x_j to acc[j]
// for every posting j > i (one __syncthreads per term, so each acc[j]
// receives its products in ascending term order — the merge-join order —
// and results are launch-configuration independent). A second pass over the
// same postings tests acc[j] >= tau into the shared pair bitmap and clears
// the accumulator. Pair keys are then emitted by the common emitter.
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
                                     uint32_t n_docs, uint64_t* __restrict__ fill, uint2* __restrict__ posts) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); d < n_docs; d += nw) {
    const uint64_t b = doc_off[d];
    const uint32_t n = nnz[d];
    for (uint32_t i = lane; i < n; i += 32) {
      const uint32_t t = ent[b + i].x;
      const uint64_t q = atomicAdd(reinterpret_cast<unsigned long long*>(fill + t), 1ull);
      posts[q] = make_uint2(d, __float_as_uint(x[b + i]));
    }
  }
}

__global__ void __launch_bounds__(256) exact_rows_kernel(ExactArgs a, uint32_t row_lo, uint32_t row_hi) {
  __shared__ uint32_t red[8];
  float* acc = a.acc_pool + static_cast<size_t>(blockIdx.x) * a.n_docs;
  for (uint32_t i = row_lo + blockIdx.x; i < row_hi; i += gridDim.x) {
    const uint64_t b = a.doc_off[i];
    const uint32_t n = a.nnz[i];
    for (uint32_t p = 0; p < n; ++p) {
      const uint32_t t = a.ent[b + p].x;
      const float xi = a.x[b + p];
      const uint64_t q1 = a.post_off[t + 1];
      for (uint64_t q = a.post_off[t] + threadIdx.x; q < q1; q += blockDim.x) {
        const uint2 pj = a.posts[q];
        if (pj.x > i) acc[pj.x] = fmaf(xi, __uint_as_float(pj.y), acc[pj.x]);
      }
      __syncthreads();
    }
    uint32_t cnt = 0;
    uint32_t* rowbits = a.bitmap + static_cast<size_t>(i) * a.words_per_row;
    for (uint32_t p = 0; p < n; ++p) {
      const uint32_t t = a.ent[b + p].x;
      const uint64_t q1 = a.post_off[t + 1];
      for (uint64_t q = a.post_off[t] + threadIdx.x; q < q1; q += blockDim.x) {
        const uint32_t j = a.posts[q].x;
        if (j > i) {
          const float v = acc[j];
          if (v != 0.0f) {
            acc[j] = 0.0f;
            if (fminf(v, 1.0f) >= a.tau) {
              atomicOr(rowbits + (j >> 5), 1u << (j & 31));
              ++cnt;
            }
          }
        }
      }
      __syncthreads();
    }
    cnt = warp_sum_u32(cnt);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t s = 0;
      for (int w = 0; w < 8; ++w) s += red[w];
      a.rowcnt[i] = s;
    }
    __syncthreads();
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

uint32_t exact_pool_ctas() { return static_cast<uint32_t>(sm_count()) * 8; }

void launch_unit_weights(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, const TermInfo* info,
                         const float* inv_norm, uint32_t n_docs, float* x, cudaStream_t s) {
  if (!n_docs) return;
  unsigned g = static_cast<unsigned>(std::min<uint64_t>(ceil_div(n_docs, 8), sm_count() * 16ull));
  unit_weights_kernel<<<g, 256, 0, s>>>(ent, doc_off, nnz, info, inv_norm, n_docs, x);
  note_launch();
}

void launch_postings_fill(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, const float* x,
                          uint32_t n_docs, uint64_t* fill, uint2* posts, cudaStream_t s) {
  if (!n_docs) return;
  unsigned g = static_cast<unsigned>(std::min<uint64_t>(ceil_div(n_docs, 8), sm_count() * 16ull));
  postings_fill_kernel<<<g, 256, 0, s>>>(ent, doc_off, nnz, x, n_docs, fill, posts);
  note_launch();
}

void launch_exact_rows(const ExactArgs& a, uint32_t row_lo, uint32_t row_hi, cudaStream_t s) {
  if (row_hi <= row_lo) return;
  unsigned g = std::min<uint32_t>(row_hi - row_lo, exact_pool_ctas());
  exact_rows_kernel<<<g, 256, 0, s>>>(a, row_lo, row_hi);
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
