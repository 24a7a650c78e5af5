// k4_simhash.cu — K4a: 64-bit Simhash per document.
//
// Reference rule (simhash.hpp:35-45): for every bit column j, sum +w for a set
// hash bit and -w for a clear one; bit j = 1 iff the column sum is > 0 (tie
// -> 0); an empty doc gives 0. The reference sums +-1 per word occurrence,
// i.e. w = tf per unique term; configs[2] uses w = TF-IDF.
//
// Exactness: w = fl32(tf * idf32) >= 1 is a multiple of 2^-23, so W = w*2^23
// is an exact integer; column sums are exact integers (int8 tensor-core
// partial products, int64 totals), independent of order, and the fingerprint
// is bit-identical to the oracle's accumulation. (Raw-TF mode runs the same
// code with idf = 1, reproducing the reference's per-occurrence +-1 columns.)
// See simhash_kernel for the mapping.

#include "kernels.cuh"

namespace refsig_gpu {
namespace {

// 4x4 byte transpose: r[p] = {v0.byte p, v1.byte p, v2.byte p, v3.byte p}.
__device__ __forceinline__ void byte_transpose4(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3, uint32_t (&r)[4]) {
  const uint32_t t0 = __byte_perm(v0, v1, 0x5140), t1 = __byte_perm(v0, v1, 0x7362);
  const uint32_t t2 = __byte_perm(v2, v3, 0x5140), t3 = __byte_perm(v2, v3, 0x7362);
  r[0] = __byte_perm(t0, t2, 0x5410);
  r[1] = __byte_perm(t0, t2, 0x7632);
  r[2] = __byte_perm(t1, t3, 0x5410);
  r[3] = __byte_perm(t1, t3, 0x7632);
}

// D += A(16x32 u8) * B(32x8 u8), int32 accumulate (exact).
__device__ __forceinline__ void mma_u8(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Warp per document, 32 nonzeros per step, on the integer tensor cores:
// W = w * 2^23 is an exact integer (w = fl32(tf*idf32) >= 1 has ulp >= 2^-23),
// split into 8 byte planes. Per step the warp computes, for the 64 hash
// columns j and byte planes p, C[j][p] += sum_k bit_j(h_k) * byte_p(W_k) with
// four m16n8k32 u8 MMAs (A = hash bits, 16 columns x 32 nonzeros; B = weight
// bytes, 32 nonzeros x 8 planes), exact in int32 for < 2^23 nonzeros per
// document. S1_j = sum_p C[j][p] << 8p and S = sum_k W_k in int64; bit j = [2*S1_j > S]
// exactly as the reference's +-w columns (tie -> 0), for S < 2^63 (sum of
// weights < 2^40). Fragments: lane (g = lane/4, t = lane%4) needs bits
// g + 8p of hashes 4t..4t+3 and 16+4t..16+4t+3: (h >> g) & 0x0101..01 puts
// them in byte p, and 4x4 byte transposes turn bytes-per-hash into
// bytes-per-bit-row. ~4 warp instructions per nonzero instead of 64 scalar
// conditional adds spread over the lanes.
// Work split as in K2: documents in decreasing length (a.order); the first
// a.n_long (> kSignLongTokens tokens) get a CTA whose 8 warps take
// interleaved steps and add their integer partial sums through shared memory
// (exact, so any split gives the same fingerprint), the rest a warp each.
__global__ void __launch_bounds__(256) simhash_kernel(SimhashArgs a) {
  __shared__ __align__(16) uint64_t hs[8][32];
  __shared__ __align__(16) uint8_t wp[8][8][32];  // [warp][plane][nonzero]
  __shared__ int red[8][16][32];                  // CTA mode: per-warp accumulators
  __shared__ unsigned long long red_tot[8];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool cta = blockIdx.x < a.n_long;
  uint32_t q;
  if (cta) {
    q = blockIdx.x;
  } else {
    q = a.n_long + (blockIdx.x - a.n_long) * 8 + wid;
    if (q >= a.n_docs) return;
  }
  const uint32_t d = a.order[q];
  const uint32_t s0 = cta ? wid : 0u, stride = cta ? 8u : 1u;
  const uint2* __restrict__ e = a.ent + a.doc_off[d];
  const uint32_t n = a.nnz[d];
  const uint32_t g = lane >> 2, t = lane & 3;
  int acc[4][4] = {};
  uint64_t tot = 0;
  constexpr int U = 4;  // steps whose loads are issued together (memory-level parallelism)
  for (uint32_t c0 = s0 * 32 * U; c0 < n; c0 += stride * 32 * U) {
    uint64_t hv[U], Wv[U];
    uint2 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = c0 + 32 * u + lane;
      x[u] = i < n ? __ldg(e + i) : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = c0 + 32 * u + lane;
      hv[u] = 0;
      Wv[u] = 0;
      if (i < n) {
        const float idf = a.use_idf ? a.info[x[u].x].idf : 1.0f;
        const float wf = __fmul_rn(static_cast<float>(x[u].y), idf);  // fl32(tf*idf32)
        Wv[u] = __float2ull_rz(wf * 8388608.0f);                     // exact: wf * 2^23 is an integer
        hv[u] = a.term_hash ? __ldg(a.term_hash + x[u].x) : term_hash64(a.seed, x[u].x);
      }
      tot += Wv[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (c0 + 32 * u >= n) break;  // warp-uniform
      const uint64_t h = hv[u], W = Wv[u];
      hs[wid][lane] = h;
#pragma unroll
      for (int p = 0; p < 8; ++p) wp[wid][p][lane] = static_cast<uint8_t>(W >> (8 * p));
      __syncwarp();
      const uint32_t b0 = *reinterpret_cast<const uint32_t*>(&wp[wid][g][4 * t]);
      const uint32_t b1 = *reinterpret_cast<const uint32_t*>(&wp[wid][g][16 + 4 * t]);
      uint32_t lo[8], hi[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint64_t y = (hs[wid][(q < 4 ? 0 : 16) + 4 * t + (q & 3)] >> g) & 0x0101010101010101ull;
        lo[q] = static_cast<uint32_t>(y);        // bytes p = 0..3: bits g + 8p
        hi[q] = static_cast<uint32_t>(y >> 32);  // p = 4..7
      }
      __syncwarp();  // the next step restages
      uint32_t ra[4], rb[4], qa[4], qb[4];
      byte_transpose4(lo[0], lo[1], lo[2], lo[3], ra);  // ra[p]: bit g+8p of hashes 4t..4t+3
      byte_transpose4(hi[0], hi[1], hi[2], hi[3], rb);  //        bit g+8(p+4)
      byte_transpose4(lo[4], lo[5], lo[6], lo[7], qa);  // hashes 16+4t..16+4t+3
      byte_transpose4(hi[4], hi[5], hi[6], hi[7], qb);
      // MMA v covers hash columns 16v..16v+15: row g -> bit 16v+g, row g+8 -> bit 16v+g+8
      const uint32_t f0[4] = {ra[0], ra[1], qa[0], qa[1]};
      const uint32_t f1[4] = {ra[2], ra[3], qa[2], qa[3]};
      const uint32_t f2[4] = {rb[0], rb[1], qb[0], qb[1]};
      const uint32_t f3[4] = {rb[2], rb[3], qb[2], qb[3]};
      mma_u8(acc[0], f0, b0, b1);
      mma_u8(acc[1], f1, b0, b1);
      mma_u8(acc[2], f2, b0, b1);
      mma_u8(acc[3], f3, b0, b1);
    }
  }
  if (cta) {  // exact integer sums over the warps
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int r = 0; r < 4; ++r) red[wid][4 * u + r][lane] = acc[u][r];
    tot += __shfl_xor_sync(0xffffffffu, tot, 1);
    tot += __shfl_xor_sync(0xffffffffu, tot, 2);
    tot += __shfl_xor_sync(0xffffffffu, tot, 4);
    tot += __shfl_xor_sync(0xffffffffu, tot, 8);
    tot += __shfl_xor_sync(0xffffffffu, tot, 16);
    if (lane == 0) red_tot[wid] = tot;
    __syncthreads();
    if (wid != 0) return;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        int x = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) x += red[w][4 * u + r][lane];
        acc[u][r] = x;
      }
    tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += red_tot[w];
  } else {
    tot += __shfl_xor_sync(0xffffffffu, tot, 1);
    tot += __shfl_xor_sync(0xffffffffu, tot, 2);
    tot += __shfl_xor_sync(0xffffffffu, tot, 4);
    tot += __shfl_xor_sync(0xffffffffu, tot, 8);
    tot += __shfl_xor_sync(0xffffffffu, tot, 16);
  }
  // S1 of columns 16u+g (acc[u][0..1]: planes 2t, 2t+1) and 16u+g+8 (acc[u][2..3])
  uint64_t fp = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint64_t s1 = (static_cast<uint64_t>(static_cast<uint32_t>(acc[u][2 * half])) << (16 * t)) +
                    (static_cast<uint64_t>(static_cast<uint32_t>(acc[u][2 * half + 1])) << (16 * t + 8));
      s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
      s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
      if (s1 > tot - s1) fp |= 1ull << (16 * u + 8 * half + g);  // 2*S1 > S, tie -> 0
    }
  }
  const uint32_t flo = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(fp));
  const uint32_t fhi = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(fp >> 32));
  if (lane == 0) a.fp[d] = (static_cast<uint64_t>(fhi) << 32) | flo;
}

}  // namespace

void launch_simhash(const SimhashArgs& a, cudaStream_t s) {
  if (a.n_docs == 0) return;
  const uint64_t blocks = a.n_long + ceil_div(a.n_docs - a.n_long, 8);
  simhash_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(a);
  note_launch();
}

}  // namespace refsig_gpu
