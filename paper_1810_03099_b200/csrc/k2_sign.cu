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

// Warp per segment: a document's nonzeros are cut into segments of
// kSignSeg = 256 rows (8 per lane); one warp handles one segment, so the
// longest document is no longer the critical path (docs of 2,400 nonzeros
// used to keep one warp busy for the whole kernel) and every warp has 8
// independent 8-byte row loads and 8 TermInfo gathers in flight.
//   1. lanes load their 8 rows, gather TermInfo, accumulate ||w||^2, and the
//      rows that hit the reference union go to a per-warp hit queue in shared
//      memory (ballot + prefix popcount; queue order = ascending term id);
//   2. the warp splits into 4 groups of 8 lanes; group g takes hits g, g+4, ...
//      and lane j of a group accumulates columns 4j..4j+3 of the current
//      32-column slab with float4 gathers of the L2-resident table R; the 4
//      group sums are combined with two xor-shuffles (fixed order);
//   3. single-segment documents finish in place; a multi-segment document
//      writes per-segment partials, and the warp that arrives last (atomic
//      per-document counter, reset by that warp) adds the partials in segment
//      order and finishes. Every sum has a fixed order, so signatures do not
//      depend on the launch configuration or on scheduling.
constexpr int kSignWarps = 8;
constexpr uint32_t kSignSeg = kSignSegRows;

// Lanes 0..7 hold the 32 raw column sums of slab k0 as float4 (columns
// k0+4*lane..). Writes S = min(sum*inv, 1) and returns this lane's sum of S^2.
__device__ __forceinline__ float sign_finish_slab(const SignArgs& a, uint32_t d, uint32_t k0, uint32_t lane,
                                                  float4 v, float inv) {
  float ss = 0.0f;
  if (lane < 8) {
    const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t k = k0 + 4 * lane + j;
      if (k < a.K) {
        const float sv = fminf(x[j] * inv, 1.0f);  // ngram.hpp:201 clamp
        a.S[static_cast<size_t>(d) * a.K + k] = sv;
        ss = fmaf(sv, sv, ss);
      }
    }
  }
  return ss;
}

__global__ void __launch_bounds__(256, 5) sign_kernel(SignArgs a) {
  __shared__ int2 queue[kSignWarps][kSignSeg];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t q = blockIdx.x * kSignWarps + wid;
  if (q >= a.n_segs) return;
  const uint2 sg = a.segs[q];
  const uint32_t d = sg.x, s = sg.y;
  const uint32_t n = a.nnz[d];
  const uint32_t ns = n > kSignSeg ? (n + kSignSeg - 1) / kSignSeg : 1u;
  if (s >= ns) return;  // the plan sizes segments by tokens; nnz <= tokens
  const uint2* __restrict__ e = a.ent + a.doc_off[d] + s * kSignSeg;
  const uint32_t cnt = min(kSignSeg, n - min(n, s * kSignSeg));
  const uint32_t lt = (1u << lane) - 1u;
  int2* qw = queue[wid];

  uint2 x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const uint32_t i = 32 * u + lane;
    x[u] = i < cnt ? __ldg(e + i) : make_uint2(0u, 0u);
  }
  TermInfo ti[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) ti[u] = (32 * u + lane < cnt) ? a.info[x[u].x] : TermInfo{0.0f, -1};
  float sq = 0.0f;
  uint32_t qn = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const float w = static_cast<float>(x[u].y) * ti[u].idf;
    sq = fmaf(w, w, sq);
    const uint32_t hits = __ballot_sync(0xffffffffu, ti[u].ref_row >= 0);
    if (ti[u].ref_row >= 0) qw[qn + __popc(hits & lt)] = make_int2(ti[u].ref_row, __float_as_int(w));
    qn += __popc(hits);
  }
  sq = warp_sum(sq);
  __syncwarp();

  const uint32_t g = lane >> 3, sub = lane & 7;
  const bool multi = ns > 1;
  float ss = 0.0f;
  float inv = 0.0f;
  if (!multi) {
    inv = sq > 0.0f ? 1.0f / sqrtf(sq) : 0.0f;
    if (lane == 0) a.inv_norm[d] = inv;
  }
  for (uint32_t k0 = 0; k0 < a.K; k0 += 32) {
    const uint32_t col = k0 + 4 * sub;
    const bool on = col < a.Kp;  // R rows are zero-padded to Kp (multiple of 4)
    float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    for (uint32_t h0 = 0; h0 < qn; h0 += 32) {
      float4 r[8];
      float w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t h = h0 + 4 * j + g;
        w[j] = 0.0f;
        r[j] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (h < qn && on) {
          const int2 hv = qw[h];
          w[j] = __int_as_float(hv.y);
          r[j] = __ldg(reinterpret_cast<const float4*>(a.R + static_cast<size_t>(hv.x) * a.Kp + col));
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        acc.x = fmaf(w[j], r[j].x, acc.x);
        acc.y = fmaf(w[j], r[j].y, acc.y);
        acc.z = fmaf(w[j], r[j].z, acc.z);
        acc.w = fmaf(w[j], r[j].w, acc.w);
      }
    }
#pragma unroll
    for (int m = 8; m <= 16; m <<= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, m);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, m);
      acc.z += __shfl_xor_sync(0xffffffffu, acc.z, m);
      acc.w += __shfl_xor_sync(0xffffffffu, acc.w, m);
    }
    if (multi) {
      if (lane < 8 && on) *reinterpret_cast<float4*>(a.part + static_cast<size_t>(q) * a.Kp + col) = acc;
    } else {
      ss += sign_finish_slab(a, d, k0, lane, acc, inv);
    }
  }
  if (multi) {
    // publish this segment, then the last of the document's ns segments finishes it
    if (lane == 0) a.part_sq[q] = sq;
    __threadfence();
    uint32_t last = 0;
    if (lane == 0) last = atomicAdd(a.arrive + d, 1u) == ns - 1;
    if (!__shfl_sync(0xffffffffu, last, 0)) return;
    __threadfence();
    if (lane == 0) a.arrive[d] = 0;  // ready for the next launch
    const uint32_t q0 = q - s;
    float tot = 0.0f;
    for (uint32_t t = 0; t < ns; ++t) tot += __ldcg(a.part_sq + q0 + t);  // segment order
    inv = tot > 0.0f ? 1.0f / sqrtf(tot) : 0.0f;
    if (lane == 0) a.inv_norm[d] = inv;
    for (uint32_t k0 = 0; k0 < a.K; k0 += 32) {
      const uint32_t col = k0 + 4 * lane;
      float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      if (lane < 8 && col < a.Kp) {
        for (uint32_t t = 0; t < ns; ++t) {
          const float4 p4 = __ldcg(reinterpret_cast<const float4*>(a.part + static_cast<size_t>(q0 + t) * a.Kp + col));
          v.x += p4.x;
          v.y += p4.y;
          v.z += p4.z;
          v.w += p4.w;
        }
      }
      ss += sign_finish_slab(a, d, k0, lane, v, inv);
    }
  }
  ss = warp_sum(ss);
  const float inv_s = ss > 0.0f ? 1.0f / sqrtf(ss) : 0.0f;  // SPEC.md:372 all-zero -> 0
  __syncwarp();
  for (uint32_t k = lane; k < a.K; k += 32)
    a.ST[static_cast<size_t>(k) * a.ld + d] = a.S[static_cast<size_t>(d) * a.K + k] * inv_s;  // own warp's writes
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
  if (a.n_segs == 0) return;
  const uint64_t blocks = ceil_div(a.n_segs, kSignWarps);  // one warp per segment
  sign_kernel<<<static_cast<unsigned>(blocks), 32 * kSignWarps, 0, s>>>(a);
  note_launch();
}

}  // namespace refsig_gpu
