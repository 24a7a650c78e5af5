// ref_shim.cpp — C-ABI shim over the REFERENCE's own headers
// (proj/include/refsig/{ngram,simhash}.hpp), compiled from where they lie under
// /root/reference by oracle/build_ref.sh into oracle/_ref/librefshim.so.
//
// TEST INFRASTRUCTURE ONLY: used to pin the oracle restatement and to produce
// tests/golden/ fixtures. No reference source is copied into this repo; this
// file only calls the reference's public functions.

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "refsig/ngram.hpp"
#include "refsig/simhash.hpp"

extern "C" {

// NgramVector::from_entries (ngram.hpp:62-75) over count-1 entries of ids.
// Writes sorted unique ids/counts; returns nnz. out arrays hold n entries.
uint64_t ref_from_entries(const uint32_t* ids, const uint32_t* counts, uint64_t n, uint32_t* out_ids,
                          uint32_t* out_counts, double* out_norm) {
  std::vector<refsig::GramCount> e(n);
  for (uint64_t i = 0; i < n; ++i) e[i] = {ids[i], counts ? counts[i] : 1u};
  refsig::NgramVector v = refsig::NgramVector::from_entries(std::move(e));
  const auto& r = v.entries();
  for (size_t i = 0; i < r.size(); ++i) {
    out_ids[i] = r[i].gram;
    out_counts[i] = r[i].count;
  }
  if (out_norm) *out_norm = v.norm();
  return r.size();
}

// refsig::cosine (ngram.hpp:184-202) over two count vectors given as entries.
double ref_cosine(const uint32_t* a_ids, const uint32_t* a_counts, uint64_t na, const uint32_t* b_ids,
                  const uint32_t* b_counts, uint64_t nb) {
  std::vector<refsig::GramCount> ea(na), eb(nb);
  for (uint64_t i = 0; i < na; ++i) ea[i] = {a_ids[i], a_counts[i]};
  for (uint64_t i = 0; i < nb; ++i) eb[i] = {b_ids[i], b_counts[i]};
  return refsig::cosine(refsig::NgramVector::from_entries(std::move(ea)),
                        refsig::NgramVector::from_entries(std::move(eb)));
}

// Text front end: normalize (ngram.hpp:114-129) + extract_3grams (:149-180).
uint64_t ref_extract_3grams(const char* text, uint64_t len, uint32_t* out_ids, uint32_t* out_counts,
                            uint64_t cap) {
  std::string norm = refsig::normalize(std::string_view(text, len));
  refsig::NgramVector v = refsig::extract_3grams(norm);
  const auto& r = v.entries();
  for (size_t i = 0; i < r.size() && i < cap; ++i) {
    out_ids[i] = r[i].gram;
    out_counts[i] = r[i].count;
  }
  return r.size();
}

uint64_t ref_normalize(const char* text, uint64_t len, char* out, uint64_t cap) {
  std::string norm = refsig::normalize(std::string_view(text, len));
  uint64_t n = norm.size() < cap ? norm.size() : cap;
  std::memcpy(out, norm.data(), n);
  return norm.size();
}

// word_hash64 (simhash.hpp:23-29): first 8 MD5 bytes big-endian. Returns 0 and
// sets *err=1 on refsig::validation_error (empty word).
uint64_t ref_word_hash64(const char* word, uint64_t len, int* err) {
  try {
    if (err) *err = 0;
    return refsig::word_hash64(std::string_view(word, len));
  } catch (const refsig::validation_error&) {
    if (err) *err = 1;
    return 0;
  }
}

// simhash (simhash.hpp:35-45) over n words packed back to back, lengths given.
uint64_t ref_simhash(const char* packed, const uint64_t* lens, uint64_t n) {
  std::vector<std::string> words;
  words.reserve(n);
  uint64_t off = 0;
  for (uint64_t i = 0; i < n; ++i) {
    words.emplace_back(packed + off, lens[i]);
    off += lens[i];
  }
  return refsig::simhash(words);
}

int ref_hamming(uint64_t a, uint64_t b) { return refsig::hamming(a, b); }

double ref_simhash_similarity(uint64_t a, uint64_t b) { return refsig::simhash_similarity(a, b); }

// pack_gram (ngram.hpp:33-37); returns -1 on validation_error.
int64_t ref_pack_gram(const char* g, uint64_t len) {
  try {
    return refsig::pack_gram(std::string_view(g, len));
  } catch (const refsig::validation_error&) {
    return -1;
  }
}

}  // extern "C"
