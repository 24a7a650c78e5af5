/*
 * mrcgen.h — deterministic synthetic corpus generator (C ABI).
 *
 * The reference evaluates on NEWS20 (reference PAPER.md:219), which is not in
 * this build environment. BASELINE.json:configs[0..4] specify seeded synthetic
 * stand-ins (Zipf term ids, lognormal lengths, topic mixtures, planted
 * near-duplicates); this library produces them. Every random draw is a pure
 * function of (seed, stream tag, index) so any doc can be regenerated
 * independently and the output is identical for any thread count
 * (reference SPEC.md:548, "determinism under parallelism").
 *
 * Frozen definitions:
 *   - PRNG: splitmix64 streams, stream(seed,tag,idx).
 *   - Zipf(s) over ranks 0..V-1 (weight (r+1)^-s) sampled by a Vose alias table.
 *   - Lengths: lognormal via Box-Muller, llround, clipped to [len_min,len_max].
 *   - Topic c maps rank r to term (a_c*r + b_c) mod V, gcd(a_c,V)=1; the
 *     global distribution maps rank r to term r.
 *   - Each token: p=topic_mix from the doc's topic Zipf, else global Zipf.
 *   - Near-duplicates: round(dup_rate*N) positions chosen by partial
 *     Fisher-Yates; each copies an original source doc and resamples every
 *     token with probability rho (fixed, or uniform in [lo,hi] per dup).
 */
#ifndef MRCGEN_H
#define MRCGEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mrcgen_spec {
  uint64_t seed;
  uint32_t n_docs;
  uint32_t vocab;
  uint32_t n_topics;       /* 0 = no topic structure (global Zipf only) */
  uint32_t len_min;
  uint32_t len_max;
  uint32_t _pad;
  double zipf_global;      /* exponent s of the global Zipf */
  double zipf_topic;       /* exponent s of every topic Zipf */
  double topic_mix;        /* probability a token is drawn from the doc's topic */
  double len_median;
  double len_sigma;
  double dup_rate;         /* fraction of docs that are planted near-duplicates */
  double resample_lo;      /* per-dup resample fraction ~ U[lo,hi] (lo==hi: fixed) */
  double resample_hi;
} mrcgen_spec;

/* Status: 0 ok, 2 invalid argument (mirrors refsig::validation_error). */

/* Pass 1: doc_off[0..n_docs] (exclusive prefix of lengths). */
int mrcgen_offsets(const mrcgen_spec* spec, uint64_t* doc_off);

/* Pass 2: tokens[doc_off[n]] term ids and dup_src[n] (UINT32_MAX for an
 * original doc, else the source doc index). threads<=0 means hardware count. */
int mrcgen_fill(const mrcgen_spec* spec, const uint64_t* doc_off, uint32_t* tokens,
                uint32_t* dup_src, int threads);

/* Query batch for query-vs-database mode (configs[4]): q_spec describes the
 * queries (its seed must differ from the DB's; topics/vocab/Zipf as the DB).
 * Near-duplicate queries copy a DB doc. db_spec is used for the topic maps. */
int mrcgen_offsets_queries(const mrcgen_spec* q_spec, const mrcgen_spec* db_spec,
                           const uint64_t* db_off, uint64_t* q_off);
int mrcgen_fill_queries(const mrcgen_spec* q_spec, const mrcgen_spec* db_spec,
                        const uint64_t* db_off, const uint32_t* db_tokens,
                        const uint64_t* q_off, uint32_t* q_tokens, uint32_t* q_src,
                        int threads);

/* K distinct doc indices in [0,n) by partial Fisher-Yates on stream
 * (seed, tag=REF). Output in selection order. (SURVEY.md Appendix A4.) */
int mrcgen_sample_refs(uint64_t seed, uint32_t n, uint32_t k, uint32_t* out);

/* splitmix64 helpers exported so tests can pin the PRNG. */
uint64_t mrcgen_splitmix64_mix(uint64_t z);
uint64_t mrcgen_stream_seed(uint64_t seed, uint64_t tag, uint64_t idx);

#ifdef __cplusplus
}
#endif
#endif
