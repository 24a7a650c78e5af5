// gpu_api_check.cpp — exercises the C++ host API (include/refsig/gpu.hpp) on
// the reference SPEC's known answers. Run by tests/test_gpu_cpp_api.py on a
// GPU box; exits non-zero on any mismatch.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "refsig/gpu.hpp"

#define EXPECT(c)                                                  \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      std::exit(1);                                                \
    }                                                              \
  } while (0)

int main() {
  using refsig::gpu::Context;
  using refsig::gpu::Weighting;
  // 3-gram ids (ngram.hpp:33-37): abc=28, bca=728, cab=1353, xyz=16197.
  // docs: "abcabc", the same again, and "xyz".
  std::vector<uint32_t> tokens = {28, 728, 1353, 28, 28, 728, 1353, 28, 16197};
  std::vector<uint64_t> off = {0, 4, 8, 9};
  Context ctx(0);
  ctx.load_corpus(tokens, off, 17576);
  ctx.count(Weighting::tf);
  auto m = ctx.counts();
  // "abcabc" -> {abc:2, bca:1, cab:1}
  EXPECT(m.rowptr[1] == 3 && m.ids[0] == 28 && m.counts[0] == 2 && m.ids[1] == 728 && m.counts[1] == 1);
  // partitions [{abc}], [{xyz}] -> [2/sqrt(6), 0]
  ctx.set_reference_partitions({{28}, {16197}});
  auto S = ctx.sign();
  EXPECT(std::fabs(S[0] - 2.0 / std::sqrt(6.0)) < 1e-6 && S[1] == 0.0f);
  EXPECT(S[4] == 0.0f && std::fabs(S[5] - 1.0f) < 1e-6);  // "xyz" vs {xyz}
  // compare: identical signatures -> 1; orthogonal -> 0 (:376)
  auto p = ctx.mrc_pairs(0.999f);
  EXPECT(p.size() == 1 && refsig::gpu::pair_first(p[0]) == 0 && refsig::gpu::pair_second(p[0]) == 1);
  // hamming(x,x) = 0
  auto fp = ctx.simhash(0, Weighting::tf);
  EXPECT(fp[0] == fp[1]);
  auto h = ctx.hamming_pairs(0);
  EXPECT(h.size() == 1 && h[0] == p[0]);
  // validation errors map to refsig::validation_error (error.hpp:8-14)
  bool threw = false;
  try {
    ctx.set_reference_docs({});
  } catch (const refsig::validation_error&) {
    threw = true;
  }
  EXPECT(threw);
  // pairs as CSR: row 0 -> {1}
  ctx.mrc_pairs(0.999f);
  auto csr = ctx.pairs_csr();
  EXPECT(csr.rowptr.size() == 4 && csr.rowptr[1] == 1 && csr.rowptr[3] == 1 && csr.cols.size() == 1 &&
         csr.cols[0] == 1);
  auto csr16 = ctx.pairs_csr16();
  EXPECT(csr16.rowptr == csr.rowptr && csr16.cols.size() == 1 && csr16.cols[0] == 1);
  // text front end: "abcabc" and "Abc-abc!" give the same 3-gram vector
  ctx.load_text("abcabcAbc-abc!", {0, 6, 14});
  ctx.count(Weighting::tf);
  auto t = ctx.counts();
  EXPECT(t.rowptr[1] == 3 && t.ids[0] == 28 && t.counts[0] == 2 && t.rowptr[2] == 4 && t.ids[3] == 28 &&
         t.counts[3] == 2);
  auto tf = ctx.simhash_text();  // one word "abcabc" vs two words "abc", "abc"
  EXPECT(tf.size() == 2 && tf[0] != 0 && tf[1] != 0);
  auto cf = ctx.corpus_freq();  // abc x2 in each doc
  EXPECT(cf.size() == 17576 && cf[28] == 4);
  ctx.set_reference_partitions({{28}});
  auto S1 = ctx.sign();
  auto rec = ctx.signature_records(0x1234);  // MRCS, 28 bytes per doc
  double v = 0;
  std::memcpy(&v, rec.data() + 28 + 20, 8);
  EXPECT(rec.size() == 56 && std::memcmp(rec.data(), "MRCS", 4) == 0 && rec[8] == 1 && rec[12] == 0x34 &&
         v == static_cast<double>(S1[1]));
  std::printf("gpu_api_check OK\n");
  return 0;
}
