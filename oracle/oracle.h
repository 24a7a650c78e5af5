/*
 * oracle.h — CPU restatement of the reference's MRC batch-similarity path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or as the timed CPU baseline. The product path
 * (paper_1810_03099_b200, librefsig_gpu.so) never calls it.
 *
 * Each function cites the reference file:line it restates. Paths are relative
 * to the reference checkout (proj/include/refsig/..., SPEC.md).
 *
 * Pinning: counts, raw-TF cosine, raw-TF signatures against
 * partition/doc references, the Simhash column rule and Hamming distance are
 * checked against the reference's own headers compiled into oracle/_ref
 * (tests/test_oracle_vs_ref.py, tests/golden/). TF-IDF weighting, the MRC
 * threshold and the splitmix64 term hash have no reference code: they are
 * restated from SURVEY.md Appendix A and pinned only through the TF-mode
 * equivalence (same code path with idf == NULL).
 */
#ifndef REFSIG_ORACLE_H
#define REFSIG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Per-doc counting: sort ids, run-length encode (ngram.hpp:170-178;
 * NgramVector::from_entries ngram.hpp:62-75). ids/counts must hold doc_off[n]
 * entries. Returns total nnz. */
uint64_t orc_count(const uint32_t* tokens, const uint64_t* doc_off, uint32_t n, uint64_t* rowptr,
                   uint32_t* ids, uint32_t* counts, int threads);

/* Document frequency (SPEC.md:214-222 doc_freq column). */
void orc_df(const uint64_t* rowptr, const uint32_t* ids, uint32_t n, uint32_t vocab, uint32_t* df);

/* Smoothed IDF: fl32(ln((1+N)/(1+df)) + 1). */
void orc_idf32(const uint32_t* df, uint32_t n_docs, uint32_t vocab, float* idf32);

/* Weights in double: w = count * idf32[id] (idf32 == NULL: raw TF counts, the
 * reference's GramCount.count, ngram.hpp:48-53); norm = sqrt(sum w^2)
 * (ngram.hpp:100-104). */
void orc_weights(const uint64_t* rowptr, const uint32_t* ids, const uint32_t* counts, uint32_t n,
                 const float* idf32, double* w, double* norm);

/* Exact cosine by merge-join (ngram.hpp:184-202): empty -> 0, clamp to 1. */
double orc_cosine(const uint32_t* a_ids, const double* a_w, uint64_t na, double a_norm,
                  const uint32_t* b_ids, const double* b_w, uint64_t nb, double b_norm);

/* sign: S[d*K+k] = cosine(doc_d, ref_k). */
void orc_sign(const uint64_t* rowptr, const uint32_t* ids, const double* w, const double* norm, uint32_t n,
              const uint64_t* ref_rowptr, const uint32_t* ref_ids, const double* ref_w, const double* ref_norm,
              uint32_t K, double* S, int threads);

/* compare: cosine of two signature vectors; 0 if either is
 * all-zero. */
double orc_compare(const double* a, const double* b, uint32_t K);

/* Result of an all-pairs sweep (SPEC.md:426 i<j enumeration). pairs are
 * sorted keys (i<<32 | j). border lists pairs with |score - tau| <= band. */
typedef struct orc_pairs {
  uint64_t* pairs;
  uint64_t n_pairs;
  uint64_t* border;
  uint64_t n_border;
} orc_pairs;
void orc_pairs_free(orc_pairs* p);

/* MRC all-pairs: match(i,j) <=> compare(S_i,S_j) >= tau, rows [row_lo,row_hi)
 * of the i<j triangle (row_hi = n for the whole triangle). */
int orc_mrc_pairs(const double* S, uint32_t n, uint32_t K, double tau, double band, uint32_t row_lo,
                  uint32_t row_hi, orc_pairs* out, int threads);

/* Query-vs-DB MRC: key (q<<32 | d), all q in [0,nq), d in [0,nd). */
int orc_mrc_query_pairs(const double* Sq, uint32_t nq, const double* Sd, uint32_t nd, uint32_t K, double tau,
                        double band, orc_pairs* out, int threads);

/* splitmix64 term hash, SURVEY.md Appendix A6 (replaces word_hash64,
 * simhash.hpp:23-29). */
uint64_t orc_term_hash(uint64_t seed, uint32_t term);

/* Simhash column rule (simhash.hpp:35-45: +w for a set bit, -w for a clear
 * bit, bit = column > 0, tie -> 0). idf32 == NULL: w = tf (the reference's
 * per-occurrence +-1 rule, exactly); else w = fl32(tf*idf32) scaled by 2^23 to
 * an exact int64. term_hash == NULL: splitmix64 of the
 * id with `seed`; else term_hash[id] (e.g. the reference's MD5 word hashes). */
void orc_simhash(const uint64_t* rowptr, const uint32_t* ids, const uint32_t* counts, uint32_t n,
                 const float* idf32, uint64_t seed, const uint64_t* term_hash, uint64_t* fp, int threads);

/* Hamming all-pairs (simhash.hpp:47): popcount(a^b) <= max_dist, i<j. */
int orc_hamming_pairs(const uint64_t* fp, uint32_t n, int max_dist, uint32_t row_lo, uint32_t row_hi,
                      orc_pairs* out, int threads);
int orc_hamming_query_pairs(const uint64_t* fq, uint32_t nq, const uint64_t* fd, uint32_t nd, int max_dist,
                            orc_pairs* out, int threads);

/* Exact all-pairs cosine >= tau over rows [row_lo,row_hi) x (i, n): an
 * inverted-index accumulation that adds the products of each pair in the same
 * (ascending term id) order as the merge-join of ngram.hpp:190-200, so every
 * score equals orc_cosine bit for bit. */
int orc_exact_pairs(const uint64_t* rowptr, const uint32_t* ids, const double* w, const double* norm, uint32_t n,
                    uint32_t vocab, double tau, double band, uint32_t row_lo, uint32_t row_hi, orc_pairs* out,
                    int threads);

/* Cosine for a list of pair keys (merge-join). */
void orc_cosine_pairs(const uint64_t* rowptr, const uint32_t* ids, const double* w, const double* norm,
                      const uint64_t* keys, uint64_t n_keys, double* out, int threads);

/* SPEC eval over pairs i<j of rows [row_lo,row_hi): out[7] = {pairs, sum e, sum e^2,
 * sum |e| for MRC, then the same for Simhash (fp NULL: zeros)}, e = score - exact. */
void orc_evaluate(const uint64_t* rowptr, const uint32_t* ids, const double* w, const double* norm, uint32_t n,
                  const double* S, uint32_t K, const uint64_t* fp, uint32_t row_lo, uint32_t row_hi, double* out,
                  int threads);
/* Text front end (ngram.hpp:114-180, simhash.hpp:23-45): per doc the 3-gram
 * ids in document order (tokens may be NULL), gram_off[n+1]; returns the total. */
uint64_t orc_text_grams(const uint8_t* bytes, const uint64_t* off, uint32_t n, uint32_t* tokens, uint64_t* gram_off);
/* word_hash64: first 8 bytes of MD5(word), big-endian (RFC 1321 restated). */
uint64_t orc_word_hash64(const uint8_t* word, uint64_t len);
/* simhash over each doc's normalized words, per occurrence +-1. */
void orc_text_simhash(const uint8_t* bytes, const uint64_t* off, uint32_t n, uint64_t* fp, int threads);

#ifdef __cplusplus
}
#endif
#endif
