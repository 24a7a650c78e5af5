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
// Algorithmic bytes per signature: 8*nnz_d (CSR rows) + 8*K (S and Sn rows)
// + 4 (inv_norm); TermInfo/R gathers are L2 traffic.

#include "kernels.cuh"

namespace refsig_gpu {
namespace {

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

__global__ void ref_doc_ranges_kernel(const uint64_t* __restrict__ doc_off, const uint32_t* __restrict__ nnz,
                                      const uint32_t* __restrict__ ref_docs, uint32_t K, uint64_t* start,
                                      uint32_t* n) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) {
    uint32_t d = ref_docs[k];
    start[k] = doc_off[d];
    n[k] = nnz[d];
  }
}

__global__ void ref_mark_kernel(RefArgs r, uint32_t* __restrict__ flags) {
  for (uint32_t k = blockIdx.x; k < r.K; k += gridDim.x) {
    const uint2* e = r.ent + r.start[k];
    const uint32_t n = r.n[k];
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) flags[e[i].x] = 1u;
  }
}

__global__ void ref_remap_kernel(const uint32_t* __restrict__ flags, const uint64_t* __restrict__ prefix,
                                 uint32_t vocab, TermInfo* __restrict__ info) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < vocab; t += gridDim.x * blockDim.x)
    info[t].ref_row = flags[t] ? static_cast<int32_t>(prefix[t]) : -1;
}

// One CTA per reference vector: block-tree norm, then scatter unit weights.
__global__ void __launch_bounds__(256) ref_fill_kernel(RefArgs r, const TermInfo* __restrict__ info,
                                                       float* __restrict__ R) {
  __shared__ float red[8];
  for (uint32_t k = blockIdx.x; k < r.K; k += gridDim.x) {
    const uint2* e = r.ent + r.start[k];
    const uint32_t n = r.n[k];
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
      R[static_cast<size_t>(info[x.x].ref_row) * r.K + k] = w * inv;
    }
    __syncthreads();
  }
}

// KPL = reference columns per lane per pass (K chunk = 32*KPL).
template <int KPL>
__global__ void __launch_bounds__(256) sign_kernel(SignArgs a) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  const uint32_t K = a.K;
  for (uint32_t d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); d < a.n_docs; d += nwarps) {
    const uint2* __restrict__ e = a.ent + a.doc_off[d];
    const uint32_t n = a.nnz[d];
    float inv = 0.0f;
    float ss = 0.0f;  // sum of squared (clamped) signature values, per lane
    for (uint32_t k0 = 0; k0 < K; k0 += 32 * KPL) {
      float acc[KPL];
#pragma unroll
      for (int q = 0; q < KPL; ++q) acc[q] = 0.0f;
      float sq = 0.0f;
      // software pipeline: the next chunk's rows are in flight while the
      // current chunk's hits are gathered
      uint2 xn = lane < n ? __ldg(e + lane) : make_uint2(0u, 0u);
      for (uint32_t c = 0; c < n; c += 32) {
        const uint32_t i = c + lane;
        const uint2 x = xn;
        if (i + 32 < n) xn = __ldg(e + i + 32);
        float w = 0.0f;
        int32_t row = -1;
        if (i < n) {
          const TermInfo ti = a.info[x.x];
          w = static_cast<float>(x.y) * ti.idf;
          row = ti.ref_row;
        }
        sq = fmaf(w, w, sq);
        uint32_t hits = __ballot_sync(0xffffffffu, row >= 0);
        // hits in ascending term order, 8 reference rows in flight per batch;
        // FMAs stay in hit order, so every column sums in the same order.
        while (hits) {
          constexpr int B = 8;
          int32_t rr[B];
          float ww[B];
#pragma unroll
          for (int u = 0; u < B; ++u) {
            const int src = hits ? __ffs(hits) - 1 : 0;
            const bool ok = hits != 0;
            hits &= hits - 1;
            rr[u] = __shfl_sync(0xffffffffu, row, src);
            ww[u] = __shfl_sync(0xffffffffu, w, src);
            if (!ok) rr[u] = -1;
          }
          float val[B][KPL];
#pragma unroll
          for (int u = 0; u < B; ++u) {
            const float* __restrict__ Rr = a.R + static_cast<size_t>(rr[u] < 0 ? 0 : rr[u]) * K + k0;
#pragma unroll
            for (int q = 0; q < KPL; ++q) {
              const uint32_t k = lane + 32 * q;
              val[u][q] = (rr[u] >= 0 && k0 + k < K) ? __ldg(Rr + k) : 0.0f;
            }
          }
#pragma unroll
          for (int u = 0; u < B; ++u)
#pragma unroll
            for (int q = 0; q < KPL; ++q)
              if (rr[u] >= 0) acc[q] = fmaf(ww[u], val[u][q], acc[q]);
        }
      }
      if (k0 == 0) {
        sq = warp_sum(sq);
        inv = sq > 0.0f ? 1.0f / sqrtf(sq) : 0.0f;
        if (lane == 0) a.inv_norm[d] = inv;
      }
#pragma unroll
      for (int q = 0; q < KPL; ++q) {
        const uint32_t k = k0 + lane + 32 * q;
        if (k < K) {
          const float s = fminf(acc[q] * inv, 1.0f);  // ngram.hpp:201 clamp
          a.S[static_cast<size_t>(d) * K + k] = s;
          ss = fmaf(s, s, ss);
        }
      }
    }
    ss = warp_sum(ss);
    const float inv_s = ss > 0.0f ? 1.0f / sqrtf(ss) : 0.0f;  // SPEC.md:372 all-zero -> 0
    for (uint32_t k = lane; k < K; k += 32)
      a.ST[static_cast<size_t>(k) * a.ld + d] = a.S[static_cast<size_t>(d) * K + k] * inv_s;  // own write
  }
}

}  // namespace

void launch_ref_doc_ranges(const uint64_t* doc_off, const uint32_t* nnz, const uint32_t* ref_docs, uint32_t K,
                           uint64_t* start, uint32_t* n, cudaStream_t s) {
  ref_doc_ranges_kernel<<<(K + 127) / 128, 128, 0, s>>>(doc_off, nnz, ref_docs, K, start, n);
  note_launch();
}

void launch_ref_mark(const RefArgs& r, uint32_t* flags, cudaStream_t s) {
  ref_mark_kernel<<<r.K < 1024 ? r.K : 1024, 256, 0, s>>>(r, flags);
  note_launch();
}

void launch_ref_remap(const uint32_t* flags, const uint64_t* prefix, uint32_t vocab, TermInfo* info,
                      cudaStream_t s) {
  uint32_t g = (vocab + 255) / 256;
  if (g > 4096) g = 4096;
  ref_remap_kernel<<<g, 256, 0, s>>>(flags, prefix, vocab, info);
  note_launch();
}

void launch_ref_fill(const RefArgs& r, const TermInfo* info, float* R, cudaStream_t s) {
  ref_fill_kernel<<<r.K < 1024 ? r.K : 1024, 256, 0, s>>>(r, info, R);
  note_launch();
}

void launch_sign(const SignArgs& a, cudaStream_t s) {
  if (a.n_docs == 0) return;
  const uint32_t warps_per_block = 8;
  uint64_t blocks = ceil_div(a.n_docs, warps_per_block);
  const uint64_t cap = static_cast<uint64_t>(sm_count()) * 8;  // 64 warps/SM resident
  if (blocks > cap) blocks = cap;
  if (a.K <= 32)
    sign_kernel<1><<<static_cast<unsigned>(blocks), 256, 0, s>>>(a);
  else if (a.K <= 64)
    sign_kernel<2><<<static_cast<unsigned>(blocks), 256, 0, s>>>(a);
  else
    sign_kernel<4><<<static_cast<unsigned>(blocks), 256, 0, s>>>(a);
  note_launch();
}

}  // namespace refsig_gpu
