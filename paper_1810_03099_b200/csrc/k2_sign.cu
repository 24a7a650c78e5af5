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
// document nonzero). The kernel is warp-per-document: lanes read 32 (id,count)
// rows per step (256 B coalesced), gather TermInfo, accumulate ||w||^2, and
// the warp ballots the nonzeros that hit U; each hit is broadcast and the
// lanes (one per reference column) FMA the coalesced R row. Accumulation order
// is ascending term id for every column, so results do not depend on the
// launch configuration. The norm is fused (warp-shuffle tree) and the unit
// signature for the compare kernel is written in the same pass.
//
// Algorithmic bytes per signature: 8*nnz_d (CSR rows) + 4*K (S row) + 4
// (inv_norm); the transposed unit copy for K3, TermInfo and R gathers are
// L2 traffic. R rows are padded to Kp = roundup(K,4) floats.

#include "kernels.cuh"

namespace refsig_gpu {
namespace {

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

__device__ __forceinline__ void ref_range(const RefArgs& r, uint32_t k, const uint2*& e, uint32_t& n) {
  if (r.docs) {
    const uint32_t d = r.docs[k];
    e = r.ent + r.doc_off[d];
    n = r.nnz[d];
  } else {
    e = r.ent + r.start[k];
    n = r.n[k];
  }
}

__global__ void ref_reset_kernel(TermInfo* __restrict__ info, uint32_t vocab) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < vocab; t += gridDim.x * blockDim.x)
    info[t].ref_row = -1;
}

__global__ void ref_claim_kernel(RefArgs r, TermInfo* __restrict__ info, uint32_t* __restrict__ counter) {
  for (uint32_t k = blockIdx.x; k < r.K; k += gridDim.x) {
    const uint2* e;
    uint32_t n;
    ref_range(r, k, e, n);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      int* slot = &info[e[i].x].ref_row;
      if (atomicCAS(slot, -1, -2) == -1) *slot = static_cast<int>(atomicAdd(counter, 1u));
    }
  }
}

// One CTA per reference vector: block-tree norm, then scatter unit weights.
__global__ void __launch_bounds__(256) ref_fill_kernel(RefArgs r, const TermInfo* __restrict__ info,
                                                       float* __restrict__ R) {
  __shared__ float red[8];
  for (uint32_t k = blockIdx.x; k < r.K; k += gridDim.x) {
    const uint2* e;
    uint32_t n;
    ref_range(r, k, e, n);
    float sq = 0.0f;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      uint2 x = e[i];
      float w = r.explicit_w ? __uint_as_float(x.y) : static_cast<float>(x.y) * info[x.x].idf;
      sq = fmaf(w, w, sq);
    }
    sq = warp_sum(sq);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    float tot = 0.0f;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += red[w];
    const float inv = tot > 0.0f ? 1.0f / sqrtf(tot) : 0.0f;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      uint2 x = e[i];
      float w = r.explicit_w ? __uint_as_float(x.y) : static_cast<float>(x.y) * info[x.x].idf;
      R[static_cast<size_t>(info[x.x].ref_row) * r.Kp + k] = w * inv;
    }
    __syncthreads();
  }
}

// Warp per document, documents in longest-first order (a.order) so the
// longest ones do not form the tail. Per 32-column slab of the signature:
//   1. lanes stream the doc's (id,count) rows 32 at a time (coalesced, next
//      chunk prefetched), gather TermInfo, accumulate ||w||^2, and append the
//      rows that hit the reference union to a per-warp hit queue in shared
//      memory (ballot + prefix popcount);
//   2. every 32 queued hits, each lane takes one hit and adds w*R[row][k0..]
//      for the slab's columns into its own 32 accumulators (float4 gathers of
//      the L2-resident table), so all lanes do useful work;
//   3. the 32x32 partial sums are transposed through shared memory and lane k
//      sums column k over the lanes in a fixed order (deterministic).
constexpr int kSignWarps = 8;

__global__ void __launch_bounds__(256) sign_kernel(SignArgs a) {
  __shared__ float part[kSignWarps][32][33];
  __shared__ int2 queue[kSignWarps][64];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t K = a.K, Kp = a.Kp;
  const uint32_t lt = (1u << lane) - 1u;
  // one document per warp (no grid-stride loop: keeps the shuffles free of
  // collective fallback code); blocks start in launch order, so `order`
  // (longest first) still front-loads the long documents
  const uint32_t q = blockIdx.x * (blockDim.x >> 5) + wid;
  if (q >= a.n_docs) return;
  {
    const uint32_t d = a.order[q];
    const uint2* __restrict__ e = a.ent + a.doc_off[d];
    const uint32_t n = a.nnz[d];
    float inv = 0.0f;
    float ss = 0.0f;  // lane k: squared signature values of its columns
    for (uint32_t k0 = 0; k0 < K; k0 += 32) {
      const uint32_t kc = min(32u, K - k0);
      float acc[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) acc[k] = 0.0f;
      float sq = 0.0f;
      uint32_t qn = 0;  // queued hits (warp-uniform)
      auto drain = [&](uint32_t cnt) {
        if (lane < cnt) {
          const int2 h = queue[wid][lane];
          const float w = __int_as_float(h.y);
          const float4* __restrict__ R4 = reinterpret_cast<const float4*>(a.R + static_cast<size_t>(h.x) * Kp + k0);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (4 * j < static_cast<int>(kc)) {
              const float4 r = __ldg(R4 + j);
              acc[4 * j + 0] = fmaf(w, r.x, acc[4 * j + 0]);
              acc[4 * j + 1] = fmaf(w, r.y, acc[4 * j + 1]);
              acc[4 * j + 2] = fmaf(w, r.z, acc[4 * j + 2]);
              acc[4 * j + 3] = fmaf(w, r.w, acc[4 * j + 3]);
            }
          }
        }
      };
      // U chunks of 32 rows per step: U coalesced loads, then U TermInfo
      // gathers in flight together (memory-level parallelism per warp)
      constexpr int U = 4;
      for (uint32_t c = 0; c < n; c += 32 * U) {
        uint2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t i = c + 32 * u + lane;
          x[u] = i < n ? __ldg(e + i) : make_uint2(0u, 0u);
        }
        TermInfo ti[U];
#pragma unroll
        for (int u = 0; u < U; ++u) ti[u] = (c + 32 * u + lane < n) ? a.info[x[u].x] : TermInfo{0.0f, -1};
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float w = static_cast<float>(x[u].y) * ti[u].idf;
          const int32_t row = ti[u].ref_row;
          sq = fmaf(w, w, sq);
          const uint32_t hits = __ballot_sync(0xffffffffu, row >= 0);
          if (row >= 0) queue[wid][qn + __popc(hits & lt)] = make_int2(row, __float_as_int(w));
          qn += __popc(hits);
          __syncwarp();
          if (qn >= 32) {
            drain(32);
            __syncwarp();
            if (lane < qn - 32) queue[wid][lane] = queue[wid][32 + lane];
            qn -= 32;
            __syncwarp();
          }
        }
      }
      drain(qn);
      if (k0 == 0) {
        sq = warp_sum(sq);
        inv = sq > 0.0f ? 1.0f / sqrtf(sq) : 0.0f;
        if (lane == 0) a.inv_norm[d] = inv;
      }
      // transpose-reduce: lane k sums column k over the 32 lanes
#pragma unroll
      for (int k = 0; k < 32; ++k) part[wid][lane][k] = acc[k];
      __syncwarp();
      float sum = 0.0f;
#pragma unroll 8
      for (int l = 0; l < 32; ++l) sum += part[wid][l][lane];
      __syncwarp();
      if (lane < kc) {
        const float s = fminf(sum * inv, 1.0f);  // ngram.hpp:201 clamp
        a.S[static_cast<size_t>(d) * K + k0 + lane] = s;
        ss = fmaf(s, s, ss);
      }
    }
    ss = warp_sum(ss);
    const float inv_s = ss > 0.0f ? 1.0f / sqrtf(ss) : 0.0f;  // SPEC.md:372 all-zero -> 0
    for (uint32_t k = lane; k < K; k += 32)
      a.ST[static_cast<size_t>(k) * a.ld + d] = a.S[static_cast<size_t>(d) * K + k] * inv_s;  // own write
  }
}

}  // namespace

void launch_ref_reset(TermInfo* info, uint32_t vocab, cudaStream_t s) {
  uint32_t g = (vocab + 255) / 256;
  if (g > 4096) g = 4096;
  ref_reset_kernel<<<g, 256, 0, s>>>(info, vocab);
  note_launch();
}

void launch_ref_claim(const RefArgs& r, TermInfo* info, uint32_t* counter, cudaStream_t s) {
  ref_claim_kernel<<<r.K < 1024 ? r.K : 1024, 256, 0, s>>>(r, info, counter);
  note_launch();
}

void launch_ref_fill(const RefArgs& r, const TermInfo* info, float* R, cudaStream_t s) {
  ref_fill_kernel<<<r.K < 1024 ? r.K : 1024, 256, 0, s>>>(r, info, R);
  note_launch();
}

void launch_sign(const SignArgs& a, cudaStream_t s) {
  if (a.n_docs == 0) return;
  const uint64_t blocks = ceil_div(a.n_docs, kSignWarps);
  sign_kernel<<<static_cast<unsigned>(blocks), 32 * kSignWarps, 0, s>>>(a);
  note_launch();
}

}  // namespace refsig_gpu
