// oracle.cpp — CPU restatement of the reference MRC path (test infrastructure).
//
// TEST INFRASTRUCTURE ONLY: see oracle.h. Never linked into the product.
// Reference citations are file:line in the reference checkout.

#include "oracle.h"

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

namespace {

template <class F>
void parallel_rows(uint64_t lo, uint64_t hi, int threads, uint64_t chunk, F&& f) {
  int t = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  if (t < 1) t = 1;
  if (hi <= lo) return;
  if (t == 1) {
    for (uint64_t i = lo; i < hi; ++i) f(i, 0);
    return;
  }
  std::atomic<uint64_t> next{lo};
  std::vector<std::thread> th;
  for (int k = 0; k < t; ++k)
    th.emplace_back([&, k] {
      for (;;) {
        uint64_t b = next.fetch_add(chunk);
        if (b >= hi) break;
        uint64_t e = std::min(hi, b + chunk);
        for (uint64_t i = b; i < e; ++i) f(i, k);
      }
    });
  for (auto& x : th) x.join();
}

int nthreads(int threads) {
  int t = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  return t < 1 ? 1 : t;
}

// Row-partitioned pair collection with a deterministic merge: each row's
// matches are produced in ascending j, rows are concatenated in ascending i.
struct RowLists {
  std::vector<std::vector<uint64_t>> pairs, border;
  explicit RowLists(uint64_t rows) : pairs(rows), border(rows) {}
  void flatten(orc_pairs* out) {
    uint64_t np = 0, nb = 0;
    for (auto& v : pairs) np += v.size();
    for (auto& v : border) nb += v.size();
    out->n_pairs = np;
    out->n_border = nb;
    out->pairs = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (np ? np : 1)));
    out->border = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (nb ? nb : 1)));
    uint64_t p = 0, b = 0;
    for (auto& v : pairs) {
      if (!v.empty()) std::memcpy(out->pairs + p, v.data(), v.size() * 8);
      p += v.size();
    }
    for (auto& v : border) {
      if (!v.empty()) std::memcpy(out->border + b, v.data(), v.size() * 8);
      b += v.size();
    }
  }
};

inline uint64_t key(uint64_t i, uint64_t j) { return (i << 32) | j; }

inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

extern "C" {

// ngram.hpp:170-178 (std::sort, then run-length encode) — the same result as
// NgramVector::from_entries of count-1 entries (ngram.hpp:62-75).
uint64_t orc_count(const uint32_t* tokens, const uint64_t* doc_off, uint32_t n, uint64_t* rowptr, uint32_t* ids,
                   uint32_t* counts, int threads) {
  std::vector<uint64_t> nnz(n);
  // Write each doc's runs at its token offset, then compact.
  std::vector<uint32_t> tid(doc_off[n]), tcnt(doc_off[n]);
  parallel_rows(0, n, threads, 64, [&](uint64_t d, int) {
    uint64_t b = doc_off[d], e = doc_off[d + 1];
    std::vector<uint32_t> s(tokens + b, tokens + e);
    std::sort(s.begin(), s.end());
    uint64_t out = b;
    for (size_t k = 0; k < s.size();) {
      size_t run = k;
      while (run < s.size() && s[run] == s[k]) ++run;
      tid[out] = s[k];
      tcnt[out] = static_cast<uint32_t>(run - k);
      ++out;
      k = run;
    }
    nnz[d] = out - b;
  });
  rowptr[0] = 0;
  for (uint32_t d = 0; d < n; ++d) rowptr[d + 1] = rowptr[d] + nnz[d];
  parallel_rows(0, n, threads, 256, [&](uint64_t d, int) {
    std::memcpy(ids + rowptr[d], tid.data() + doc_off[d], nnz[d] * 4);
    std::memcpy(counts + rowptr[d], tcnt.data() + doc_off[d], nnz[d] * 4);
  });
  return rowptr[n];
}

// doc_freq = number of documents whose vector contains t.
void orc_df(const uint64_t* rowptr, const uint32_t* ids, uint32_t n, uint32_t vocab, uint32_t* df) {
  std::memset(df, 0, sizeof(uint32_t) * vocab);
  for (uint32_t d = 0; d < n; ++d)
    for (uint64_t p = rowptr[d]; p < rowptr[d + 1]; ++p) df[ids[p]]++;
}

// SURVEY.md Appendix A3 (no reference code: TF-IDF is future work in
// SPEC.md:13 / PAPER.md:243).
void orc_idf32(const uint32_t* df, uint32_t n_docs, uint32_t vocab, float* idf32) {
  for (uint32_t t = 0; t < vocab; ++t)
    idf32[t] = static_cast<float>(std::log((1.0 + n_docs) / (1.0 + df[t])) + 1.0);
}

// ngram.hpp:100-104: norm = sqrt(sum of squared weights), in double.
void orc_weights(const uint64_t* rowptr, const uint32_t* ids, const uint32_t* counts, uint32_t n,
                 const float* idf32, double* w, double* norm) {
  for (uint32_t d = 0; d < n; ++d) {
    double sq = 0.0;
    for (uint64_t p = rowptr[d]; p < rowptr[d + 1]; ++p) {
      double v = static_cast<double>(counts[p]);
      if (idf32) v *= static_cast<double>(idf32[ids[p]]);
      w[p] = v;
      sq += v * v;
    }
    norm[d] = std::sqrt(sq);
  }
}

// ngram.hpp:184-202: empty -> 0 (:185), merge-join dot (:190-200), clamp (:201).
double orc_cosine(const uint32_t* a_ids, const double* a_w, uint64_t na, double a_norm, const uint32_t* b_ids,
                  const double* b_w, uint64_t nb, double b_norm) {
  if (na == 0 || nb == 0) return 0.0;
  double dot = 0.0;
  uint64_t i = 0, j = 0;
  while (i < na && j < nb) {
    if (a_ids[i] == b_ids[j]) {
      dot += a_w[i] * b_w[j];
      ++i;
      ++j;
    } else if (a_ids[i] < b_ids[j]) {
      ++i;
    } else {
      ++j;
    }
  }
  return std::min(1.0, dot / (a_norm * b_norm));
}

// values[k] = cosine(doc, reference_k); empty doc -> zeros.
void orc_sign(const uint64_t* rowptr, const uint32_t* ids, const double* w, const double* norm, uint32_t n,
              const uint64_t* ref_rowptr, const uint32_t* ref_ids, const double* ref_w, const double* ref_norm,
              uint32_t K, double* S, int threads) {
  parallel_rows(0, n, threads, 64, [&](uint64_t d, int) {
    for (uint32_t k = 0; k < K; ++k)
      S[d * K + k] = orc_cosine(ids + rowptr[d], w + rowptr[d], rowptr[d + 1] - rowptr[d], norm[d],
                                ref_ids + ref_rowptr[k], ref_w + ref_rowptr[k], ref_rowptr[k + 1] - ref_rowptr[k],
                                ref_norm[k]);
  });
}

// cosine over the value vectors, all-zero -> 0.
double orc_compare(const double* a, const double* b, uint32_t K) {
  double dot = 0.0, na = 0.0, nb = 0.0;
  for (uint32_t k = 0; k < K; ++k) {
    dot += a[k] * b[k];
    na += a[k] * a[k];
    nb += b[k] * b[k];
  }
  if (na == 0.0 || nb == 0.0) return 0.0;
  return dot / (std::sqrt(na) * std::sqrt(nb));
}

void orc_pairs_free(orc_pairs* p) {
  if (!p) return;
  std::free(p->pairs);
  std::free(p->border);
  p->pairs = p->border = nullptr;
  p->n_pairs = p->n_border = 0;
}

// SPEC.md:426 (all i<j, lexicographic) with the compare rule above.
int orc_mrc_pairs(const double* S, uint32_t n, uint32_t K, double tau, double band, uint32_t row_lo, uint32_t row_hi,
                  orc_pairs* out, int threads) {
  if (row_hi > n) row_hi = n;
  if (row_lo > row_hi) row_lo = row_hi;
  // Pre-normalise once (the compare rule divides by both norms).
  std::vector<double> U(static_cast<size_t>(n) * K);
  std::vector<uint8_t> zero(n);
  for (uint32_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (uint32_t k = 0; k < K; ++k) s += S[(size_t)i * K + k] * S[(size_t)i * K + k];
    zero[i] = s == 0.0;
    double inv = zero[i] ? 0.0 : 1.0 / std::sqrt(s);
    for (uint32_t k = 0; k < K; ++k) U[(size_t)i * K + k] = S[(size_t)i * K + k] * inv;
  }
  RowLists rl(row_hi - row_lo);
  parallel_rows(row_lo, row_hi, threads, 16, [&](uint64_t i, int) {
    auto& P = rl.pairs[i - row_lo];
    auto& B = rl.border[i - row_lo];
    const double* a = U.data() + i * K;
    for (uint64_t j = i + 1; j < n; ++j) {
      double score = 0.0;
      if (!zero[i] && !zero[j]) {
        const double* b = U.data() + j * K;
        for (uint32_t k = 0; k < K; ++k) score += a[k] * b[k];
      }
      if (score >= tau) P.push_back(key(i, j));
      if (std::fabs(score - tau) <= band) B.push_back(key(i, j));
    }
  });
  rl.flatten(out);
  return 0;
}

int orc_mrc_query_pairs(const double* Sq, uint32_t nq, const double* Sd, uint32_t nd, uint32_t K, double tau,
                        double band, orc_pairs* out, int threads) {
  auto normed = [K](const double* S, uint32_t n, std::vector<double>& U, std::vector<uint8_t>& z) {
    U.resize(static_cast<size_t>(n) * K);
    z.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (uint32_t k = 0; k < K; ++k) s += S[(size_t)i * K + k] * S[(size_t)i * K + k];
      z[i] = s == 0.0;
      double inv = z[i] ? 0.0 : 1.0 / std::sqrt(s);
      for (uint32_t k = 0; k < K; ++k) U[(size_t)i * K + k] = S[(size_t)i * K + k] * inv;
    }
  };
  std::vector<double> Uq, Ud;
  std::vector<uint8_t> zq, zd;
  normed(Sq, nq, Uq, zq);
  normed(Sd, nd, Ud, zd);
  RowLists rl(nq);
  parallel_rows(0, nq, threads, 1, [&](uint64_t q, int) {
    const double* a = Uq.data() + q * K;
    for (uint64_t d = 0; d < nd; ++d) {
      double score = 0.0;
      if (!zq[q] && !zd[d]) {
        const double* b = Ud.data() + d * K;
        for (uint32_t k = 0; k < K; ++k) score += a[k] * b[k];
      }
      if (score >= tau) rl.pairs[q].push_back(key(q, d));
      if (std::fabs(score - tau) <= band) rl.border[q].push_back(key(q, d));
    }
  });
  rl.flatten(out);
  return 0;
}

// splitmix64 output for state seed + t*gamma.
uint64_t orc_term_hash(uint64_t seed, uint32_t term) {
  return mix64(seed + (static_cast<uint64_t>(term) + 1) * 0x9E3779B97F4A7C15ull);
}

// simhash.hpp:35-45 with per-unique-term weights (tf reproduces the
// per-occurrence +-1 loop of simhash.hpp:37-40 exactly).
void orc_simhash(const uint64_t* rowptr, const uint32_t* ids, const uint32_t* counts, uint32_t n,
                 const float* idf32, uint64_t seed, const uint64_t* term_hash, uint64_t* fp, int threads) {
  parallel_rows(0, n, threads, 64, [&](uint64_t d, int) {
    int64_t column[64] = {0};
    for (uint64_t p = rowptr[d]; p < rowptr[d + 1]; ++p) {
      uint32_t t = ids[p];
      uint64_t h = term_hash ? term_hash[t] : orc_term_hash(seed, t);
      int64_t wi;
      if (idf32) {
        float wf = static_cast<float>(counts[p]) * idf32[t];  // fl32(tf * idf32)
        wi = static_cast<int64_t>(static_cast<double>(wf) * 8388608.0);  // exact: wf >= 1
      } else {
        wi = counts[p];
      }
      for (int j = 0; j < 64; ++j) column[j] += ((h >> j) & 1u) ? wi : -wi;
    }
    uint64_t out = 0;
    for (int j = 0; j < 64; ++j)
      if (column[j] > 0) out |= uint64_t{1} << j;  // tie -> 0 (simhash.hpp:43)
    fp[d] = out;
  });
}

// simhash.hpp:47: hamming = popcount(a ^ b).
int orc_hamming_pairs(const uint64_t* fp, uint32_t n, int max_dist, uint32_t row_lo, uint32_t row_hi,
                      orc_pairs* out, int threads) {
  if (row_hi > n) row_hi = n;
  if (row_lo > row_hi) row_lo = row_hi;
  RowLists rl(row_hi - row_lo);
  parallel_rows(row_lo, row_hi, threads, 16, [&](uint64_t i, int) {
    auto& P = rl.pairs[i - row_lo];
    const uint64_t a = fp[i];
    for (uint64_t j = i + 1; j < n; ++j)
      if (__builtin_popcountll(a ^ fp[j]) <= max_dist) P.push_back(key(i, j));
  });
  rl.flatten(out);
  return 0;
}

int orc_hamming_query_pairs(const uint64_t* fq, uint32_t nq, const uint64_t* fd, uint32_t nd, int max_dist,
                            orc_pairs* out, int threads) {
  RowLists rl(nq);
  parallel_rows(0, nq, threads, 1, [&](uint64_t q, int) {
    const uint64_t a = fq[q];
    for (uint64_t d = 0; d < nd; ++d)
      if (__builtin_popcountll(a ^ fd[d]) <= max_dist) rl.pairs[q].push_back(key(q, d));
  });
  rl.flatten(out);
  return 0;
}

int orc_exact_pairs(const uint64_t* rowptr, const uint32_t* ids, const double* w, const double* norm, uint32_t n,
                    uint32_t vocab, double tau, double band, uint32_t row_lo, uint32_t row_hi, orc_pairs* out,
                    int threads) {
  if (row_hi > n) row_hi = n;
  if (row_lo > row_hi) row_lo = row_hi;
  // Postings per term, docs ascending.
  std::vector<uint64_t> tptr(static_cast<size_t>(vocab) + 1, 0);
  for (uint64_t p = 0; p < rowptr[n]; ++p) tptr[ids[p] + 1]++;
  for (uint32_t t = 0; t < vocab; ++t) tptr[t + 1] += tptr[t];
  std::vector<uint32_t> pdoc(rowptr[n]);
  std::vector<double> pw(rowptr[n]);
  {
    std::vector<uint64_t> fill(tptr.begin(), tptr.end() - 1);
    for (uint32_t d = 0; d < n; ++d)
      for (uint64_t p = rowptr[d]; p < rowptr[d + 1]; ++p) {
        uint64_t q = fill[ids[p]]++;
        pdoc[q] = d;
        pw[q] = w[p];
      }
  }
  const int T = nthreads(threads);
  std::vector<std::vector<double>> acc(T, std::vector<double>(n, 0.0));
  std::vector<std::vector<uint32_t>> touched(T);
  RowLists rl(row_hi - row_lo);
  parallel_rows(row_lo, row_hi, T, 4, [&](uint64_t i, int tid) {
    auto& A = acc[tid];
    auto& touch = touched[tid];
    touch.clear();
    if (rowptr[i + 1] == rowptr[i]) return;
    // Terms of doc i in ascending id: the merge-join visit order.
    for (uint64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      uint32_t t = ids[p];
      const double wi = w[p];
      // postings are doc-ascending: binary search the first doc > i
      const uint32_t* b = pdoc.data() + tptr[t];
      const uint32_t* e = pdoc.data() + tptr[t + 1];
      const uint32_t* s = std::upper_bound(b, e, static_cast<uint32_t>(i));
      for (const uint32_t* q = s; q < e; ++q) {
        uint32_t j = *q;
        if (A[j] == 0.0) touch.push_back(j);
        A[j] += wi * pw[q - pdoc.data()];
      }
    }
    std::sort(touch.begin(), touch.end());
    auto& P = rl.pairs[i - row_lo];
    auto& B = rl.border[i - row_lo];
    for (uint32_t j : touch) {
      double c = std::min(1.0, A[j] / (norm[i] * norm[j]));
      A[j] = 0.0;
      if (c >= tau) P.push_back(key(i, j));
      if (std::fabs(c - tau) <= band) B.push_back(key(i, j));
    }
  });
  rl.flatten(out);
  return 0;
}

void orc_cosine_pairs(const uint64_t* rowptr, const uint32_t* ids, const double* w, const double* norm,
                      const uint64_t* keys, uint64_t n_keys, double* out, int threads) {
  parallel_rows(0, n_keys, threads, 1024, [&](uint64_t q, int) {
    uint64_t i = keys[q] >> 32, j = keys[q] & 0xffffffffu;
    out[q] = orc_cosine(ids + rowptr[i], w + rowptr[i], rowptr[i + 1] - rowptr[i], norm[i], ids + rowptr[j],
                        w + rowptr[j], rowptr[j + 1] - rowptr[j], norm[j]);
  });
}


// ---- Text front end ----------------------------------
// normalize (ngram.hpp:114-129): ASCII letters lowercased, every maximal run
// of other bytes is a word break. A 3-gram is any window of three letters
// inside one word (ngram.hpp:149-166, id = ((c0*26)+c1)*26+c2 over 'a'..'z',
// ngram.hpp:33-37), so on the raw bytes: three consecutive letters.
static inline int orc_letter(uint8_t c) {
  if (c >= 'A' && c <= 'Z') return c - 'A';
  if (c >= 'a' && c <= 'z') return c - 'a';
  return -1;
}

// Per doc the 3-gram ids in document order (before sorting). gram_off[n+1].
// tokens may be NULL (counts only). Returns the total.
uint64_t orc_text_grams(const uint8_t* bytes, const uint64_t* off, uint32_t n, uint32_t* tokens, uint64_t* gram_off) {
  uint64_t k = 0;
  for (uint32_t d = 0; d < n; ++d) {
    gram_off[d] = k;
    for (uint64_t p = off[d]; p + 3 <= off[d + 1]; ++p) {
      int a = orc_letter(bytes[p]), b = orc_letter(bytes[p + 1]), c = orc_letter(bytes[p + 2]);
      if (a >= 0 && b >= 0 && c >= 0) {
        if (tokens) tokens[k] = static_cast<uint32_t>((a * 26 + b) * 26 + c);
        ++k;
      }
    }
  }
  gram_off[n] = k;
  return k;
}

// MD5 (RFC 1321), restated: 64-byte blocks, little-endian words, four rounds
// of 16 steps with the sine table T[i] = floor(2^32 |sin(i+1)|).
static void orc_md5(const uint8_t* msg, uint64_t len, uint8_t digest[16]) {
  static uint32_t T[64];
  static bool init = false;
  if (!init) {
    for (int i = 0; i < 64; ++i) T[i] = static_cast<uint32_t>(std::floor(std::fabs(std::sin(i + 1.0)) * 4294967296.0));
    init = true;
  }
  static const int R[4][4] = {{7, 12, 17, 22}, {5, 9, 14, 20}, {4, 11, 16, 23}, {6, 10, 15, 21}};
  uint32_t h0 = 0x67452301u, h1 = 0xefcdab89u, h2 = 0x98badcfeu, h3 = 0x10325476u;
  const uint64_t nblk = (len + 8) / 64 + 1;
  for (uint64_t blk = 0; blk < nblk; ++blk) {
    uint8_t buf[64];
    for (int i = 0; i < 64; ++i) {
      const uint64_t q = blk * 64 + i;
      uint8_t v = 0;
      if (q < len) v = msg[q];
      else if (q == len) v = 0x80;
      else if (q >= nblk * 64 - 8) v = static_cast<uint8_t>((len * 8) >> (8 * (q - (nblk * 64 - 8))));
      buf[i] = v;
    }
    uint32_t M[16];
    for (int i = 0; i < 16; ++i)
      M[i] = buf[4 * i] | (buf[4 * i + 1] << 8) | (buf[4 * i + 2] << 16) | (static_cast<uint32_t>(buf[4 * i + 3]) << 24);
    uint32_t a = h0, b = h1, c = h2, d = h3;
    for (int i = 0; i < 64; ++i) {
      uint32_t f;
      int g;
      if (i < 16) { f = (b & c) | (~b & d); g = i; }
      else if (i < 32) { f = (d & b) | (~d & c); g = (5 * i + 1) % 16; }
      else if (i < 48) { f = b ^ c ^ d; g = (3 * i + 5) % 16; }
      else { f = c ^ (b | ~d); g = (7 * i) % 16; }
      const uint32_t x = a + f + T[i] + M[g];
      const int r = R[i / 16][i % 4];
      a = d;
      d = c;
      c = b;
      b = b + ((x << r) | (x >> (32 - r)));
    }
    h0 += a; h1 += b; h2 += c; h3 += d;
  }
  const uint32_t h[4] = {h0, h1, h2, h3};
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) digest[4 * i + j] = static_cast<uint8_t>(h[i] >> (8 * j));
}

// word_hash64 (simhash.hpp:23-29): the first 8 digest bytes, big-endian.
uint64_t orc_word_hash64(const uint8_t* word, uint64_t len) {
  uint8_t dg[16];
  orc_md5(word, len, dg);
  uint64_t h = 0;
  for (int i = 0; i < 8; ++i) h = (h << 8) | dg[i];
  return h;
}

// simhash(extract_words(normalize(text))) per doc (simhash.hpp:35-45,
// ngram.hpp:132-145): words are the lowercased maximal letter runs, every
// occurrence votes +-1 per bit column, bit = column > 0, no words -> 0.
void orc_text_simhash(const uint8_t* bytes, const uint64_t* off, uint32_t n, uint64_t* fp, int threads) {
  parallel_rows(0, n, threads, 64, [&](uint64_t d, int) {
    int64_t col[64] = {0};
    std::vector<uint8_t> w;
    auto flush = [&]() {
      if (w.empty()) return;
      const uint64_t h = orc_word_hash64(w.data(), w.size());
      for (int j = 0; j < 64; ++j) col[j] += (h >> j & 1u) ? 1 : -1;
      w.clear();
    };
    for (uint64_t p = off[d]; p < off[d + 1]; ++p) {
      const int l = orc_letter(bytes[p]);
      if (l >= 0) w.push_back(static_cast<uint8_t>('a' + l));
      else flush();
    }
    flush();
    uint64_t out = 0;
    for (int j = 0; j < 64; ++j)
      if (col[j] > 0) out |= 1ull << j;
    fp[d] = out;
  });
}


// ---- evaluation (SPEC.md eval: evaluate, Eq. 2/3) ---------------------------
// Over all pairs i<j of rows [row_lo, row_hi): exact = cosine of the weighted
// vectors (merge-join, ngram.hpp:184-202), mrc = compare of the signatures
// (SPEC.md:369-377), sim = 1 - hd/64 (simhash.hpp:49-52); e = score - exact.
// out[0..6] = {pairs, sum e_mrc, sum e_mrc^2, sum |e_mrc|, sum e_sim,
// sum e_sim^2, sum |e_sim|} (fp may be NULL: Simhash sums 0).
void orc_evaluate(const uint64_t* rowptr, const uint32_t* ids, const double* w, const double* norm, uint32_t n,
                  const double* S, uint32_t K, const uint64_t* fp, uint32_t row_lo, uint32_t row_hi, double* out,
                  int threads) {
  const int T = threads > 0 ? threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  std::vector<std::array<double, 7>> acc(T);
  for (auto& a : acc) a.fill(0.0);
  parallel_rows(row_lo, row_hi, threads, 8, [&](uint64_t i, int tid) {
    auto& a = acc[tid];
    for (uint64_t j = i + 1; j < n; ++j) {
      const double ex = orc_cosine(ids + rowptr[i], w + rowptr[i], rowptr[i + 1] - rowptr[i], norm[i],
                                   ids + rowptr[j], w + rowptr[j], rowptr[j + 1] - rowptr[j], norm[j]);
      const double em = orc_compare(S + i * K, S + j * K, K) - ex;
      a[0] += 1;
      a[1] += em;
      a[2] += em * em;
      a[3] += std::fabs(em);
      if (fp) {
        const double es = (1.0 - __builtin_popcountll(fp[i] ^ fp[j]) / 64.0) - ex;
        a[4] += es;
        a[5] += es * es;
        a[6] += std::fabs(es);
      }
    }
  });
  for (int q = 0; q < 7; ++q) {
    out[q] = 0;
    for (int t = 0; t < T; ++t) out[q] += acc[t][q];
  }
}

}  // extern "C"
