// f4 on-disk formats: MRCS signature records straight from HBM.
//
// SPEC.md:401 (signature module, External Interfaces): one signature file is
//   magic "MRCS" | version u32 LE = 1 | P u32 LE | ref_id u64 LE | P x f64 LE
// i.e. 20 header bytes then 8P payload bytes. The record size 20 + 8P is a
// multiple of 4, so the batch of n_docs records is written as 32-bit words,
// one thread per word, fully coalesced: words 0..4 are the header, word
// 5 + 2k (+1) the low (high) half of double(S[d][k]). fp32 -> f64 widening is
// exact, so decode(record) == double(sign(d)) bit for bit.
#include "kernels.cuh"

namespace refsig_gpu {
namespace {

__global__ void __launch_bounds__(256) mrcs_records_kernel(const float* __restrict__ S, uint32_t n_docs, uint32_t K,
                                                           uint64_t ref_id, uint32_t* __restrict__ out) {
  const uint32_t rw = 5 + 2 * K;  // words per record
  const uint64_t total = static_cast<uint64_t>(n_docs) * rw;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t d = i / rw;
    const uint32_t w = static_cast<uint32_t>(i - d * rw);
    uint32_t v;
    if (w >= 5) {
      const uint32_t k = (w - 5) >> 1;
      const double x = static_cast<double>(S[d * K + k]);
      const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
      v = (w - 5) & 1 ? static_cast<uint32_t>(b >> 32) : static_cast<uint32_t>(b);
    } else if (w == 0) {
      v = 0x5343524Du;  // "MRCS" little-endian
    } else if (w == 1) {
      v = 1u;
    } else if (w == 2) {
      v = K;
    } else if (w == 3) {
      v = static_cast<uint32_t>(ref_id);
    } else {
      v = static_cast<uint32_t>(ref_id >> 32);
    }
    out[i] = v;
  }
}

}  // namespace

void launch_mrcs_records(const float* S, uint32_t n_docs, uint32_t K, uint64_t ref_id, uint32_t* out,
                         cudaStream_t s) {
  const uint64_t total = static_cast<uint64_t>(n_docs) * (5 + 2 * K);
  if (!total) return;
  const uint64_t blocks = (total + 255) / 256;
  mrcs_records_kernel<<<static_cast<unsigned>(blocks < 148u * 16u ? blocks : 148u * 16u), 256, 0, s>>>(S, n_docs, K, ref_id, out);
  note_launch();
}

}  // namespace refsig_gpu
