// k4_simhash.cu — K4a: 64-bit Simhash per document.
//
// Reference rule (simhash.hpp:35-45): for every bit column j, sum +w for a set
// hash bit and -w for a clear one; bit j = 1 iff the column sum is > 0 (tie
// -> 0); an empty doc gives 0. The reference sums +-1 per word occurrence,
// i.e. w = tf per unique term; configs[2] uses w = TF-IDF.
//
// Exactness: w = fl32(tf * idf32) >= 1 is a multiple of 2^-23, so every
// partial sum of such weights below 2^30 is exact in fp64 and independent of
// order. col_j = 2*S1_j - S where S1_j sums the weights with bit j set and S
// sums all weights: the fingerprint is bit-identical to the oracle's int64
// accumulation for any thread mapping. (Raw-TF mode runs the same code with
// idf = 1, reproducing the reference's per-occurrence +-1 columns.)
//
// Mapping: warp per document. Phase 1 (lanes over nonzeros): 32 rows are
// loaded coalesced, hashed (splitmix64, Appendix A6, or a caller table such as
// the reference's MD5 word hashes) and weighted; staged as {h_lo,h_hi,w} in
// shared memory. Phase 2 (lanes over columns): lane l owns columns l and l+32
// and reads each staged entry by broadcast (one LDS.128), adding w under the
// bit predicate. The fingerprint is assembled with two ballots.

#include "kernels.cuh"

namespace refsig_gpu {
namespace {

// s += w when (h & bit) != 0: one LOP3 (predicate out) + one predicated DADD.
__device__ __forceinline__ void add_if_bit(double& s, double w, uint32_t h, uint32_t bit) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
      "and.b32 t, %2, %3;\n\t"
      "setp.ne.u32 p, t, 0;\n\t"
      "@p add.f64 %0, %0, %1;\n\t}"
      : "+d"(s)
      : "d"(w), "r"(h), "r"(bit));
}

struct __align__(16) Staged {
  uint32_t lo, hi;
  double w;
};

__global__ void __launch_bounds__(256) simhash_kernel(SimhashArgs a) {
  __shared__ Staged stage[8][32];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t d = blockIdx.x * (blockDim.x >> 5) + wid;  // one document per warp
  if (d >= a.n_docs) return;
  {
    const uint2* __restrict__ e = a.ent + a.doc_off[d];
    const uint32_t n = a.nnz[d];
    double s1a = 0.0, s1b = 0.0, tot = 0.0;
    const uint32_t bit = 1u << lane;
    for (uint32_t c = 0; c < n; c += 32) {
      const uint32_t i = c + lane;
      Staged st{0u, 0u, 0.0};
      if (i < n) {
        const uint2 x = __ldg(e + i);
        const float idf = a.use_idf ? a.info[x.x].idf : 1.0f;
        const float wf = __fmul_rn(static_cast<float>(x.y), idf);  // fl32(tf*idf32)
        const uint64_t h = a.term_hash ? __ldg(a.term_hash + x.x) : term_hash64(a.seed, x.x);
        st.lo = static_cast<uint32_t>(h);
        st.hi = static_cast<uint32_t>(h >> 32);
        st.w = static_cast<double>(wf);
      }
      tot += st.w;
      stage[wid][lane] = st;
      __syncwarp();
      const uint32_t m = min(32u, n - c);
#pragma unroll 8
      for (uint32_t q = 0; q < m; ++q) {
        const Staged v = stage[wid][q];
        add_if_bit(s1a, v.w, v.lo, bit);
        add_if_bit(s1b, v.w, v.hi, bit);
      }
      __syncwarp();
    }
    tot = warp_sum(tot);  // exact (multiples of 2^-23 below 2^30)
    const uint32_t lo = __ballot_sync(0xffffffffu, 2.0 * s1a > tot);
    const uint32_t hi = __ballot_sync(0xffffffffu, 2.0 * s1b > tot);
    if (lane == 0) a.fp[d] = (static_cast<uint64_t>(hi) << 32) | lo;
  }
}

}  // namespace

void launch_simhash(const SimhashArgs& a, cudaStream_t s) {
  if (a.n_docs == 0) return;
  const uint64_t blocks = ceil_div(a.n_docs, 8);
  simhash_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(a);
  note_launch();
}

}  // namespace refsig_gpu
