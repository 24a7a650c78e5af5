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
// Dispatch: docs are binned by length on the host (at upload). Each bin runs a
// CTA-per-doc shared-memory bitonic sort sized to the bin, grid-strided over
// the bin's docs; docs > 8192 tokens sort in a global scratch region.

#include <cmath>

#include "kernels.cuh"

namespace refsig_gpu {
namespace {

__device__ __forceinline__ uint32_t next_pow2(uint32_t x) {
  return x <= 1 ? 1u : (1u << (32 - __clz(x - 1)));
}

// Block-wide exclusive scan of one value per thread; returns the block total
// through *total. `scratch` holds THREADS/32 words.
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
  __syncthreads();  // scratch reusable after return
  return wsum + inc - v;
}

// Bitonic sort (ascending) of P keys (P a power of two) held in `s`
// (shared or global memory, visible block-wide after __syncthreads).
template <int THREADS>
__device__ __forceinline__ void bitonic_sort(uint32_t* s, uint32_t P) {
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t idx = threadIdx.x; idx < (P >> 1); idx += THREADS) {
        uint32_t i = ((idx & ~(j - 1)) << 1) | (idx & (j - 1));
        uint32_t l = i + j;
        uint32_t a = s[i], b = s[l];
        bool up = (i & k) == 0;
        if ((a > b) == up) {
          s[i] = b;
          s[l] = a;
        }
      }
      __syncthreads();
    }
  }
}

// Run-length encode sorted keys s[0..len) into ent[base..]; df += 1 per run.
// IPT consecutive keys per thread per chunk; runs may cross chunk borders
// (a run head walks to its end).
template <int THREADS, int IPT>
__device__ __forceinline__ uint32_t rle_emit(const uint32_t* s, uint32_t len, uint2* ent, uint32_t* df,
                                             uint32_t* scan_scratch) {
  uint32_t base = 0;
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
        atomicAdd(df + key, 1u);
        ++pos;
      }
    }
    base += total;
  }
  return base;
}

template <int CAP, int THREADS>
__global__ void __launch_bounds__(THREADS) count_smem_kernel(CountArgs a, const uint32_t* __restrict__ bin_docs,
                                                             uint32_t n_bin) {
  __shared__ uint32_t keys[CAP];
  __shared__ uint32_t scan_scratch[THREADS / 32];
  for (uint32_t q = blockIdx.x; q < n_bin; q += gridDim.x) {
    const uint32_t d = bin_docs[q];
    const uint64_t b = a.doc_off[d];
    const uint32_t len = static_cast<uint32_t>(a.doc_off[d + 1] - b);
    const uint32_t P = next_pow2(len);
    for (uint32_t i = threadIdx.x; i < P; i += THREADS) {
      uint32_t v = kPadKey;
      if (i < len) {
        v = __ldg(a.tokens + b + i);
        if (v >= a.vocab) {
          atomicOr(a.err, 1u);
          v = a.vocab - 1;
        }
      }
      keys[i] = v;
    }
    __syncthreads();
    bitonic_sort<THREADS>(keys, P);
    uint32_t n = rle_emit<THREADS, CAP / THREADS>(keys, len, a.ent + b, a.df, scan_scratch);
    if (threadIdx.x == 0) a.nnz[d] = n;
    __syncthreads();
  }
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
    for (uint32_t i = threadIdx.x; i < P; i += 1024) {
      uint32_t v = kPadKey;
      if (i < len) {
        v = a.tokens[b + i];
        if (v >= a.vocab) {
          atomicOr(a.err, 1u);
          v = a.vocab - 1;
        }
      }
      s[i] = v;
    }
    __syncthreads();
    bitonic_sort<1024>(s, P);
    uint32_t n = rle_emit<1024, 8>(s, len, a.ent + b, a.df, scan_scratch);
    if (threadIdx.x == 0) a.nnz[d] = n;
    __syncthreads();
  }
}

__global__ void idf_kernel(const uint32_t* __restrict__ df, uint32_t vocab, uint32_t n_docs, int weight_mode,
                           TermInfo* __restrict__ info) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < vocab; t += gridDim.x * blockDim.x) {
    float idf = 1.0f;
    if (weight_mode == 1) idf = static_cast<float>(log((1.0 + n_docs) / (1.0 + df[t])) + 1.0);
    info[t] = TermInfo{idf, -1};
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

int grid_for(uint32_t n, int per_sm) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t g = static_cast<uint64_t>(sms) * per_sm;
  if (g > n) g = n;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

void launch_count_bin(int bin, const CountArgs& a, const uint32_t* bin_docs, uint32_t n_bin, cudaStream_t s) {
  if (n_bin == 0) return;
  switch (bin) {
    case 0:
      count_smem_kernel<256, 128><<<grid_for(n_bin, 16), 128, 0, s>>>(a, bin_docs, n_bin);
      note_launch();
      break;
    case 1:
      count_smem_kernel<1024, 256><<<grid_for(n_bin, 8), 256, 0, s>>>(a, bin_docs, n_bin);
      note_launch();
      break;
    case 2:
      count_smem_kernel<4096, 512><<<grid_for(n_bin, 4), 512, 0, s>>>(a, bin_docs, n_bin);
      note_launch();
      break;
    default:
      count_smem_kernel<8192, 1024><<<grid_for(n_bin, 2), 1024, 0, s>>>(a, bin_docs, n_bin);
      note_launch();
      break;
  }
}

void launch_count_large(const CountArgs& a, const uint32_t* long_docs, const uint64_t* scratch_off, uint32_t n_long,
                        uint32_t* scratch, cudaStream_t s) {
  if (n_long == 0) return;
  count_large_kernel<<<grid_for(n_long, 1), 1024, 0, s>>>(a, long_docs, scratch_off, n_long, scratch);
  note_launch();
}

void launch_idf(const uint32_t* df, uint32_t vocab, uint32_t n_docs, int weight_mode, TermInfo* info,
                cudaStream_t s) {
  idf_kernel<<<grid_for((vocab + 255) / 256, 8), 256, 0, s>>>(df, vocab, n_docs, weight_mode, info);
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
