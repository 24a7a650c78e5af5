// refsig/gpu.hpp — C++ host API over the C ABI (include/refsig_gpu.h).
//
// Keeps the reference's conventions (namespace refsig, value types owned by
// the caller, refsig::validation_error for caller-fixable input and
// std::runtime_error for everything else — reference error.hpp:8-14) and adds
// the batch operations the reference lacks. When the reference headers are on
// the include path, its own refsig::validation_error is used, so exceptions
// from this API are caught by the reference's existing handlers.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "refsig_gpu.h"

#if __has_include("refsig/error.hpp")
#include "refsig/error.hpp"
#else
namespace refsig {
// Same shape as the reference's (error.hpp:11-14).
class validation_error : public std::runtime_error {
 public:
  explicit validation_error(const std::string& what) : std::runtime_error(what) {}
};
}  // namespace refsig
#endif

namespace refsig::gpu {

// REFSIG_E_OVERFLOW: the exact pair count is kept so callers can resize.
class overflow_error : public std::runtime_error {
 public:
  overflow_error(const std::string& what, std::uint64_t count) : std::runtime_error(what), count_(count) {}
  std::uint64_t count() const { return count_; }

 private:
  std::uint64_t count_;
};

enum class Weighting : int { tf = REFSIG_WEIGHT_TF, tfidf = REFSIG_WEIGHT_TFIDF };

// Compact CSR of per-document sorted (id, count) rows — per document the same
// entries as refsig::NgramVector::entries() (ngram.hpp:57-109).
struct CountMatrix {
  std::vector<std::uint64_t> rowptr;
  std::vector<std::uint32_t> ids;
  std::vector<std::uint32_t> counts;
};

using PairKey = std::uint64_t;  // (i << 32) | j, i < j
inline std::uint32_t pair_first(PairKey k) { return static_cast<std::uint32_t>(k >> 32); }
inline std::uint32_t pair_second(PairKey k) { return static_cast<std::uint32_t>(k); }

class Context {
 public:
  explicit Context(int device = 0) {
    int rc = refsig_gpu_create(device, &ctx_);
    if (rc == REFSIG_E_VALIDATION) throw refsig::validation_error("refsig::gpu: bad device index");
    if (rc != REFSIG_OK) throw std::runtime_error("refsig::gpu: no usable CUDA device (sm_100a build)");
  }
  ~Context() { refsig_gpu_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  refsig_gpu_ctx* raw() const { return ctx_; }

  void load_corpus(const std::vector<std::uint32_t>& tokens, const std::vector<std::uint64_t>& doc_off,
                   std::uint32_t vocab) {
    if (doc_off.empty()) throw refsig::validation_error("doc_off must hold n_docs+1 offsets");
    check(refsig_gpu_load_corpus(ctx_, tokens.data(), doc_off.data(), static_cast<std::uint32_t>(doc_off.size() - 1),
                                 vocab));
    n_docs_ = static_cast<std::uint32_t>(doc_off.size() - 1);
    vocab_ = vocab;
  }
  void count(Weighting w = Weighting::tfidf) { check(refsig_gpu_count(ctx_, static_cast<int>(w))); }

  CountMatrix counts() {
    CountMatrix m;
    std::uint64_t nnz = 0;
    m.rowptr.resize(n_docs_hint() + 1);
    int rc = refsig_gpu_get_counts(ctx_, m.rowptr.data(), nullptr, nullptr, 0, &nnz);
    if (rc != REFSIG_E_OVERFLOW && rc != REFSIG_OK) check(rc);
    m.ids.resize(nnz);
    m.counts.resize(nnz);
    rc = refsig_gpu_get_counts(ctx_, m.rowptr.data(), m.ids.data(), m.counts.data(), nnz, &nnz);
    check(rc, nnz);
    return m;
  }

  // FrequencyTable corpus_freq per term id; doc_freq via refsig_gpu_get_df.
  std::vector<std::uint64_t> corpus_freq() {
    std::vector<std::uint64_t> cf(vocab_);
    check(refsig_gpu_get_corpus_freq(ctx_, cf.data()));
    return cf;
  }

  void set_reference_docs(const std::vector<std::uint32_t>& doc_ids) {
    check(refsig_gpu_set_reference_docs(ctx_, doc_ids.data(), static_cast<std::uint32_t>(doc_ids.size())));
    K_ = static_cast<std::uint32_t>(doc_ids.size());
  }
  // Partition vectors (reference SPEC.md:306-314): count-1 vectors.
  void set_reference_partitions(const std::vector<std::vector<std::uint32_t>>& parts) {
    std::vector<std::uint64_t> rowptr{0};
    std::vector<std::uint32_t> ids;
    for (const auto& p : parts) {
      ids.insert(ids.end(), p.begin(), p.end());
      rowptr.push_back(ids.size());
    }
    check(refsig_gpu_set_reference_vectors(ctx_, static_cast<std::uint32_t>(parts.size()), rowptr.data(), ids.data(),
                                           nullptr));
    K_ = static_cast<std::uint32_t>(parts.size());
  }

  // sign for every document: n_docs x K row-major.
  std::vector<float> sign() {
    check(refsig_gpu_sign(ctx_));
    std::vector<float> S(static_cast<size_t>(n_docs_hint()) * K_);
    check(refsig_gpu_get_signatures(ctx_, S.data()));
    return S;
  }

  // Multi-GPU building blocks (include/refsig_gpu.h).
  void set_global_df(std::uint32_t n_docs_global, const std::vector<std::uint32_t>* df_global = nullptr) {
    check(refsig_gpu_set_global_df(ctx_, df_global ? df_global->data() : nullptr, n_docs_global));
  }
  void set_reference_counts(const std::vector<std::uint64_t>& rowptr, const std::vector<std::uint32_t>& ids,
                            const std::vector<std::uint32_t>& counts) {
    if (rowptr.empty()) throw refsig::validation_error("rowptr must hold K+1 offsets");
    check(refsig_gpu_set_reference_counts(ctx_, static_cast<std::uint32_t>(rowptr.size() - 1), rowptr.data(),
                                          ids.data(), counts.data()));
    K_ = static_cast<std::uint32_t>(rowptr.size() - 1);
  }
  void set_signatures(const std::vector<float>& S, std::uint32_t n_docs, std::uint32_t K) {
    check(refsig_gpu_set_signatures(ctx_, n_docs, K, S.data(), 0));
    n_docs_ = n_docs;
    K_ = K;
  }

  // One MRCS signature file image per document, 20 + 8K bytes each, back to back.
  std::vector<std::uint8_t> signature_records(std::uint64_t ref_id) {
    std::vector<std::uint8_t> r(static_cast<size_t>(n_docs_hint()) * (20u + 8u * K_));
    check(refsig_gpu_get_signature_records(ctx_, ref_id, r.data(), r.size()));
    return r;
  }

  std::vector<PairKey> mrc_pairs(float tau) {
    return pairs([&](PairKey* out, std::uint64_t cap, std::uint64_t* n) {
      return refsig_gpu_mrc_pairs(ctx_, tau, out, cap, n);
    });
  }

  std::vector<std::uint64_t> simhash(std::uint64_t seed, Weighting w = Weighting::tfidf,
                                     const std::vector<std::uint64_t>* term_hash = nullptr) {
    check(refsig_gpu_simhash(ctx_, seed, static_cast<int>(w), term_hash ? term_hash->data() : nullptr));
    std::vector<std::uint64_t> fp(n_docs_hint());
    check(refsig_gpu_get_fingerprints(ctx_, fp.data()));
    return fp;
  }

  std::vector<PairKey> hamming_pairs(int max_dist) {
    return pairs([&](PairKey* out, std::uint64_t cap, std::uint64_t* n) {
      return refsig_gpu_hamming_pairs(ctx_, max_dist, out, cap, n);
    });
  }

  std::vector<PairKey> exact_pairs(float tau_cos) {
    return pairs([&](PairKey* out, std::uint64_t cap, std::uint64_t* n) {
      return refsig_gpu_exact_pairs(ctx_, tau_cos, out, cap, n);
    });
  }

  // Raw text documents text[byte_off[d] .. byte_off[d+1]): the corpus becomes
  // each document's 3-grams (normalize + extract_3grams, ngram.hpp:114-180),
  // vocabulary 17576; count() then yields extract_3grams' entries.
  void load_text(const std::string& text, const std::vector<std::uint64_t>& byte_off) {
    if (byte_off.size() < 2 || byte_off.back() > text.size())
      throw refsig::validation_error("refsig::gpu: byte_off must have n_docs+1 entries within the text");
    check(refsig_gpu_load_text(ctx_, reinterpret_cast<const std::uint8_t*>(text.data()), byte_off.data(),
                               static_cast<std::uint32_t>(byte_off.size() - 1)));
    n_docs_ = static_cast<std::uint32_t>(byte_off.size() - 1);
    vocab_ = 17576;
  }

  // simhash(extract_words(normalize(doc))) per document (simhash.hpp:35-45).
  std::vector<std::uint64_t> simhash_text() {
    check(refsig_gpu_simhash_text(ctx_));
    std::vector<std::uint64_t> fp(n_docs_hint());
    check(refsig_gpu_get_fingerprints(ctx_, fp.data()));
    return fp;
  }

  // The last pair call's pairs as CSR over all rows: rowptr[n_docs+1], cols.
  struct PairsCsr {
    std::vector<std::uint64_t> rowptr;
    std::vector<std::uint32_t> cols;
  };
  PairsCsr pairs_csr() {
    PairsCsr r;
    r.rowptr.resize(n_docs_hint() + 1);
    std::uint64_t n = 0;
    int rc = refsig_gpu_get_pairs_csr(ctx_, 0, n_docs_hint(), r.rowptr.data(), nullptr, 0, &n);
    if (rc != REFSIG_E_OVERFLOW) check(rc);
    r.cols.resize(n);
    rc = refsig_gpu_get_pairs_csr(ctx_, 0, n_docs_hint(), r.rowptr.data(), r.cols.data(), n, &n);
    check(rc, n);
    return r;
  }

  // The same with 16-bit column ids (n_docs <= 65536): half the bytes.
  struct PairsCsr16 {
    std::vector<std::uint64_t> rowptr;
    std::vector<std::uint16_t> cols;
  };
  PairsCsr16 pairs_csr16() {
    PairsCsr16 r;
    r.rowptr.resize(n_docs_hint() + 1);
    std::uint64_t n = 0;
    int rc = refsig_gpu_get_pairs_csr16(ctx_, 0, n_docs_hint(), r.rowptr.data(), nullptr, 0, &n);
    if (rc != REFSIG_E_OVERFLOW) check(rc);
    r.cols.resize(n);
    rc = refsig_gpu_get_pairs_csr16(ctx_, 0, n_docs_hint(), r.rowptr.data(), r.cols.data(), n, &n);
    check(rc, n);
    return r;
  }

  std::uint32_t n_docs_hint() const { return n_docs_; }

 private:
  template <class F>
  std::vector<PairKey> pairs(F&& f) {
    std::uint64_t n = 0;
    int rc = f(nullptr, 0, &n);  // count only; keys stay on the device
    check(rc, n);
    std::vector<PairKey> out(n);
    check(refsig_gpu_get_pairs(ctx_, out.data(), n));  // keys of the call above
    return out;
  }

  // count: the exact total an overflowing call returned through its out_count
  void check(int rc, std::uint64_t count = 0) const {
    if (rc == REFSIG_OK) return;
    std::string msg = std::string("refsig::gpu: ") + refsig_gpu_last_error(ctx_);
    if (rc == REFSIG_E_VALIDATION) throw refsig::validation_error(msg);
    if (rc == REFSIG_E_OVERFLOW) throw overflow_error(msg, count);
    throw std::runtime_error(msg);
  }

  refsig_gpu_ctx* ctx_ = nullptr;
  std::uint32_t K_ = 0;
  std::uint32_t n_docs_ = 0;
  std::uint32_t vocab_ = 0;
};

}  // namespace refsig::gpu
