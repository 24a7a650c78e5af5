/*
 * refsig_gpu.h — C ABI of the B200-native MRC batch-similarity path.
 *
 * Drop-in boundary. The reference's API surface is the
 * header-only C++ in proj/include/refsig/ (pure functions over value types,
 * no batch API). This ABI adds the batch entry points the reference's callers
 * (SPEC eval/cli, absent in the reference) would bind, one per reference
 * operation it replaces:
 *
 *   refsig_gpu_count            NgramVector::from_entries / extract_3grams'
 *                               sort+RLE (ngram.hpp:62-75, :170-178) per doc,
 *                               + doc_freq + IDF (A3)
 *   refsig_gpu_set_reference_*  Reference.partition_vectors (SPEC.md:261-267,
 *                               :306-314) or K sampled reference docs
 *   refsig_gpu_sign             sign using cosine
 *                               (ngram.hpp:184-202)
 *   refsig_gpu_mrc_pairs        compare over all i<j
 *                               (sample_pairs "all")
 *   refsig_gpu_simhash          simhash (simhash.hpp:35-45) with word_hash64
 *                               (simhash.hpp:23-29) -> splitmix64 or a table
 *   refsig_gpu_hamming_pairs    hamming (simhash.hpp:47) over all i<j
 *   refsig_gpu_exact_pairs      cosine (ngram.hpp:184-202) over all i<j
 *   refsig_gpu_pair_cosines     cosine for a caller-given pair list
 *
 * Conventions
 *   - Status: 0 ok; 1 runtime failure (CUDA error, out of memory) — the
 *     reference's std::runtime_error, CLI exit 1; 2 validation failure (bad
 *     sizes, K = 0, id >= vocab, NULL pointers, call order) — the reference's
 *     refsig::validation_error (error.hpp:8-14), CLI exit 2; 3 candidate
 *     buffer overflow (runtime class): *out_count still holds the exact count
 *     and the first `capacity` pairs were written.
 *     refsig_gpu_last_error(ctx) describes the last non-zero status.
 *   - Ownership: the caller owns every host buffer; the ABI copies in and out.
 *     The context owns device memory; results stay device-resident between
 *     calls (corpus -> counts -> signatures -> pairs).
 *   - Threading: one context per host thread (no internal locking).
 *   - Ordering: calls that only produce device-resident state are enqueued on
 *     the context's stream and return without waiting; calls that write host
 *     buffers or return counts synchronise. Errors from enqueued work are
 *     reported by the next synchronising call.
 *   - Determinism: pair outputs are sorted keys (i << 32 | j), identical for
 *     any launch configuration.
 *   - No CPU fallback: every compute entry point runs CUDA kernels built for
 *     sm_100a; without a usable device refsig_gpu_create fails with 1.
 */
#ifndef REFSIG_GPU_H
#define REFSIG_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define REFSIG_OK 0
#define REFSIG_E_RUNTIME 1
#define REFSIG_E_VALIDATION 2
#define REFSIG_E_OVERFLOW 3

/* Term weighting for documents and reference docs. */
#define REFSIG_WEIGHT_TF 0    /* raw counts: the reference's GramCount.count (ngram.hpp:48-53) */
#define REFSIG_WEIGHT_TFIDF 1 /* count * fl32(ln((1+N)/(1+df))+1) */

typedef struct refsig_gpu_ctx refsig_gpu_ctx;

/* ---- lifetime ------------------------------------------------------------ */
int refsig_gpu_create(int device, refsig_gpu_ctx** out);
void refsig_gpu_destroy(refsig_gpu_ctx* ctx);
const char* refsig_gpu_last_error(const refsig_gpu_ctx* ctx);
const char* refsig_gpu_version(void);
/* Use an external cudaStream_t (e.g. the framework's current stream); NULL
 * restores the context-owned stream. */
int refsig_gpu_set_stream(refsig_gpu_ctx* ctx, void* cuda_stream);
void* refsig_gpu_get_stream(const refsig_gpu_ctx* ctx);
int refsig_gpu_synchronize(refsig_gpu_ctx* ctx);

/* ---- corpus (A14 input) ---------------------------------------------------
 * tokens[doc_off[n_docs]] term ids (< vocab) and doc_off[n_docs+1] (doc_off[0]
 * = 0, non-decreasing), both HOST pointers; copied to HBM (async when the
 * tokens are pinned). Resets counts, reference, signatures and fingerprints. */
int refsig_gpu_load_corpus(refsig_gpu_ctx* ctx, const uint32_t* tokens, const uint64_t* doc_off, uint32_t n_docs,
                           uint32_t vocab);
/* Same, with tokens already resident in device memory (borrowed, must stay
 * alive until the next load); doc_off is a host array (length metadata). */
int refsig_gpu_load_corpus_device(refsig_gpu_ctx* ctx, const uint32_t* d_tokens, const uint64_t* doc_off,
                                  uint32_t n_docs, uint32_t vocab);

/* ---- text front end -----------------------------------
 * Raw documents text[byte_off[d] .. byte_off[d+1]) (HOST pointers): the corpus
 * becomes each document's character 3-grams — normalize (ngram.hpp:114-129) +
 * extract_3grams (ngram.hpp:149-180), ids ((c0*26)+c1)*26+c2 < 17576 — in
 * document order, so count() yields exactly the reference's NgramVector
 * entries; vocab = 17576. The bytes stay resident for simhash_text. */
int refsig_gpu_load_text(refsig_gpu_ctx* ctx, const uint8_t* text, const uint64_t* byte_off, uint32_t n_docs);
/* Per-document simhash(extract_words(normalize(text))) (simhash.hpp:35-45,
 * word_hash64 = first 8 MD5 bytes big-endian, simhash.hpp:23-29) of the text
 * loaded by refsig_gpu_load_text; read with refsig_gpu_get_fingerprints. */
int refsig_gpu_simhash_text(refsig_gpu_ctx* ctx);

/* ---- K1: counts, df, idf (A2-A4) ------------------------------------------ */
int refsig_gpu_count(refsig_gpu_ctx* ctx, int weight_mode);
/* Compact CSR of the per-doc sorted (id,count) rows, exactly the reference's
 * NgramVector::entries() per doc. rowptr[n_docs+1]; ids/counts hold `cap`
 * entries; *nnz receives the total (REFSIG_E_OVERFLOW if nnz > cap). */
int refsig_gpu_get_counts(refsig_gpu_ctx* ctx, uint64_t* rowptr, uint32_t* ids, uint32_t* counts, uint64_t cap,
                          uint64_t* nnz);
/* df[vocab] and idf32[vocab] (either may be NULL). */
int refsig_gpu_get_df(refsig_gpu_ctx* ctx, uint32_t* df, float* idf32);
/* cf[vocab]: total occurrences of each term over the corpus (the corpus_freq
 * column of SPEC.md's FrequencyTable, build_frequency_table SPEC.md:214-222). */
int refsig_gpu_get_corpus_freq(refsig_gpu_ctx* ctx, uint64_t* cf);
/* 1/||w_d|| per doc (0 for an empty doc). */
int refsig_gpu_get_inv_norm(refsig_gpu_ctx* ctx, float* inv_norm);

/* ---- A5: reference vectors ------------------------------------------------- */
/* K corpus docs (indices < n_docs) as references, weighted like the corpus.
 * 1 <= K <= 256 (validation error otherwise). */
int refsig_gpu_set_reference_docs(refsig_gpu_ctx* ctx, const uint32_t* ref_doc_ids, uint32_t K);
/* K explicit reference vectors (host CSR): vector k = term_ids[rowptr[k] ..
 * rowptr[k+1]) with weights (NULL: all 1.0, the reference's count-1 partition
 * vectors). Ids must be unique within a vector and < vocab; 1 <= K <= 256. */
int refsig_gpu_set_reference_vectors(refsig_gpu_ctx* ctx, uint32_t K, const uint64_t* rowptr, const uint32_t* term_ids,
                                     const float* weights);
/* Size of the compact reference table (terms in the union U). */
int refsig_gpu_reference_union(refsig_gpu_ctx* ctx, uint32_t* out_u);

/* ---- K2: signatures (A6) ---------------------------------------------------- */
int refsig_gpu_sign(refsig_gpu_ctx* ctx);
/* S[n_docs*K] row-major: S[d*K+k] = cosine(doc d, reference k). */
int refsig_gpu_get_signatures(refsig_gpu_ctx* ctx, float* S);

/* f4: one MRCS signature file image per document: magic "MRCS",
 * u32 version 1, u32 P=K, u64 ref_id, K float64 (exact widening of the fp32
 * signatures), little-endian, 20 + 8K bytes each, records back to back in
 * document order. out_bytes >= n_docs * (20 + 8K). */
int refsig_gpu_get_signature_records(refsig_gpu_ctx* ctx, uint64_t ref_id, uint8_t* out, uint64_t out_bytes);

/* ---- K3: MRC all-pairs (A7) -------------------------------------------------
 * All i<j with compare(S_i,S_j) >= tau. out_pairs: host buffer of `capacity`
 * keys or NULL (keys stay on the device; count only). */
int refsig_gpu_mrc_pairs(refsig_gpu_ctx* ctx, float tau, uint64_t* out_pairs, uint64_t capacity,
                         uint64_t* out_count);

/* Rows [row_lo, row_hi) of the same triangle (pairs i<j with row_lo <= i <
 * row_hi): the unit a rank owns when the triangle is sharded across GPUs.
 * Row ranges are aligned to the 128-row tile internally; keys are global. */
int refsig_gpu_mrc_pairs_rows(refsig_gpu_ctx* ctx, float tau, uint32_t row_lo, uint32_t row_hi, uint64_t* out_pairs,
                              uint64_t capacity, uint64_t* out_count);

/* The whole MRC step — count(weight_mode) -> set_reference_docs -> sign ->
 * pairs of rows [row_lo,row_hi) with compare >= tau — enqueued without any host
 * synchronisation. The first call for a given (corpus, weighting, references,
 * tau, rows, stream) runs eagerly and captures the sequence as a CUDA graph;
 * later identical calls replay the graph (one launch). Collect the result with
 * refsig_gpu_step_result before the next step. */
int refsig_gpu_mrc_step(refsig_gpu_ctx* ctx, int weight_mode, const uint32_t* ref_doc_ids, uint32_t K, float tau,
                        uint32_t row_lo, uint32_t row_hi);
/* Wait for the step; *out_count = pairs; copies min(count, capacity) sorted
 * keys to out_pairs (may be NULL: keys stay on the device, refsig_gpu_get_pairs). */
int refsig_gpu_step_result(refsig_gpu_ctx* ctx, uint64_t* out_pairs, uint64_t capacity, uint64_t* out_count);

/* ---- K4: Simhash + Hamming (A8-A10) -----------------------------------------
 * weight_mode as above (TF reproduces the reference's per-occurrence rule).
 * term_hash: optional HOST table of vocab 64-bit hashes (e.g. word_hash64 of
 * each term's word); NULL uses splitmix64(seed, id) (Appendix A6). */
int refsig_gpu_simhash(refsig_gpu_ctx* ctx, uint64_t seed, int weight_mode, const uint64_t* term_hash);
int refsig_gpu_get_fingerprints(refsig_gpu_ctx* ctx, uint64_t* fp);
int refsig_gpu_hamming_pairs(refsig_gpu_ctx* ctx, int max_dist, uint64_t* out_pairs, uint64_t capacity,
                             uint64_t* out_count);

/* ---- K5: exact cosine verifier (A12) ---------------------------------------- */
int refsig_gpu_exact_pairs(refsig_gpu_ctx* ctx, float tau_cos, uint64_t* out_pairs, uint64_t capacity,
                           uint64_t* out_count);
/* Exact cosine (fp32) of the corpus' weighted vectors for n pair keys. */
int refsig_gpu_pair_cosines(refsig_gpu_ctx* ctx, const uint64_t* keys, uint64_t n, float* out);

/* ---- evaluation (SPEC.md eval, Eq. 2/3) -----------------
 * Over all pairs i<j with row_lo <= i < row_hi (row_lo a multiple of 128):
 * e = score - exact cosine of the weighted vectors (the exact verifier's
 * definition; count(REFSIG_WEIGHT_TF) gives the reference's 3-gram-count
 * cosine); mae = mean |e|, mean_error = mean e, variance = mean (e -
 * mean_error)^2, for MRC (compare of the signatures) and, when fingerprints
 * exist, Simhash (1 - hd/64). Fused on the GPU: no pair list is materialised;
 * sums are accumulated in double in a fixed order (deterministic). */
typedef struct {
  uint64_t pairs;
  double mrc_mae, mrc_mean_error, mrc_variance;
  double simhash_mae, simhash_mean_error, simhash_variance; /* NaN without fingerprints */
} refsig_gpu_eval;
int refsig_gpu_evaluate(refsig_gpu_ctx* ctx, uint32_t row_lo, uint32_t row_hi, refsig_gpu_eval* out);

/* ---- multi-GPU building blocks -----------------------------
 * One rank per GPU holds a contiguous shard of the documents:
 *   1. refsig_gpu_count() on the shard; all-reduce the df table in place
 *      (refsig_gpu_device_buffer(REFSIG_BUF_DF), NCCL sum) or pass the global
 *      table from the host, then refsig_gpu_set_global_df(ctx, df|NULL, N):
 *      idf from the global df and N (bit-identical on every rank);
 *   2. the K reference documents' (id, count) rows (from their owners) via
 *      refsig_gpu_set_reference_counts: weighted count * idf on the device,
 *      exactly as refsig_gpu_set_reference_docs weights them;
 *   3. refsig_gpu_sign(); all-gather the shards' S (REFSIG_BUF_SIGNATURES) in
 *      rank order;
 *   4. on a pairs context: refsig_gpu_set_signatures(ctx, N, K, S_all, on_device)
 *      builds the unit transposed signatures (bit-identical to sign()'s), then
 *      refsig_gpu_mrc_pairs_rows() over this rank's row panel (shard.row_shards).
 * The resulting candidate lists concatenate, in rank order, into the
 * single-GPU list. */
int refsig_gpu_set_global_df(refsig_gpu_ctx* ctx, const uint32_t* df_global, uint32_t n_docs_global);
int refsig_gpu_set_reference_counts(refsig_gpu_ctx* ctx, uint32_t K, const uint64_t* rowptr, const uint32_t* term_ids,
                                    const uint32_t* counts);
int refsig_gpu_set_signatures(refsig_gpu_ctx* ctx, uint32_t n_docs, uint32_t K, const float* S, int on_device);

/* ---- streaming batches (configs[4] query batches) -----------------------------
 * refsig_gpu_stage_corpus starts the host->device copy of a LATER batch on
 * the context's copy stream (into staging buffers; up to two batches may be
 * staged ahead) and returns at once; pass pinned host memory for the copy to
 * overlap. refsig_gpu_swap_corpus makes the oldest staged batch the context's
 * corpus, exactly as load_corpus would (the compute stream waits for the copy
 * on the device; the host does not).
 * Typical loop: stage(b0); stage(b1); swap; count/sign/pairs(b0); stage(b2);
 * swap; count/sign/pairs(b1); ... — with two staged, the copy engine always
 * has the next upload queued behind the current one. */
int refsig_gpu_stage_corpus(refsig_gpu_ctx* ctx, const uint32_t* tokens, const uint64_t* doc_off, uint32_t n_docs,
                            uint32_t vocab);
int refsig_gpu_swap_corpus(refsig_gpu_ctx* ctx);

/* ---- query-vs-database mode (configs[4]) -------------------------------------
 * `db` holds the signed/fingerprinted database; `q` holds the query corpus,
 * counted with the database's IDF and signed against its reference. */
int refsig_gpu_attach_database(refsig_gpu_ctx* q, refsig_gpu_ctx* db);
int refsig_gpu_mrc_query_pairs(refsig_gpu_ctx* q, float tau, uint64_t* out_pairs, uint64_t capacity,
                               uint64_t* out_count);
int refsig_gpu_hamming_query_pairs(refsig_gpu_ctx* q, int max_dist, uint64_t* out_pairs, uint64_t capacity,
                                   uint64_t* out_count);

/* Copy the first min(capacity, count) keys of the last pair call (any of the
 * *_pairs functions) to a host buffer. */
int refsig_gpu_get_pairs(refsig_gpu_ctx* ctx, uint64_t* out_pairs, uint64_t capacity);
/* The same pairs as CSR over rows [row_lo, row_hi) of the last pair call:
 * rowptr[0..n] (n = row_hi-row_lo, rowptr[0] = 0) and the sorted column ids
 * of each row in cols (up to capacity). Half the bytes of the 64-bit keys. */
int refsig_gpu_get_pairs_csr(refsig_gpu_ctx* ctx, uint32_t row_lo, uint32_t row_hi, uint64_t* rowptr, uint32_t* cols,
                             uint64_t capacity, uint64_t* out_count);

/* The same, with 16-bit column ids (the grid's n_cols <= 65536): half the
 * device->host bytes of get_pairs_csr; narrowed on the device. */
int refsig_gpu_get_pairs_csr16(refsig_gpu_ctx* ctx, uint32_t row_lo, uint32_t row_hi, uint64_t* rowptr,
                               uint16_t* cols, uint64_t capacity, uint64_t* out_count);

/* Asynchronous get_pairs_csr16 over the last pair call's whole row range: the
 * rebased rowptr (n_rows + 1) and the first min(count, capacity) 16-bit
 * columns are copied to the (pinned) host buffers on a separate stream while
 * the caller moves on to the next batch; *out_count (exact) is returned at
 * once (3 on overflow, as get_pairs_csr16). The buffers are complete after
 * refsig_gpu_wait_fetch. Two fetches may be in flight. */
int refsig_gpu_get_pairs_csr16_async(refsig_gpu_ctx* ctx, uint64_t* rowptr, uint16_t* cols, uint64_t capacity,
                                     uint64_t* out_count);
int refsig_gpu_wait_fetch(refsig_gpu_ctx* ctx);

/* ---- device views (for frameworks / collectives; read-only) ------------------ */
#define REFSIG_BUF_PAIRS 0      /* uint64 keys of the last pair call */
#define REFSIG_BUF_SIGNATURES 1 /* float S[n_docs*K] */
#define REFSIG_BUF_DF 2         /* uint32 df[vocab] */
#define REFSIG_BUF_FINGERPRINTS 3
int refsig_gpu_device_buffer(refsig_gpu_ctx* ctx, int which, void** ptr, uint64_t* bytes);

/* ---- measurement -------------------------------------------------------------
 * With profiling on, every phase below is bracketed by CUDA events recorded on
 * the context's stream (the stream its kernels run on). phase_times syncs and
 * returns the summed device time (ms) and call count per phase since the last
 * set_profiling call. */
#define REFSIG_PHASE_COUNT 0      /* K1: sort + RLE + df + idf */
#define REFSIG_PHASE_REFERENCE 1  /* A5: union, remap, reference table */
#define REFSIG_PHASE_SIGN 2       /* K2 */
#define REFSIG_PHASE_PAIR_TILES 3 /* K3 / K4b / K5 tile kernel */
#define REFSIG_PHASE_PAIR_EMIT 4  /* row-count scan + sorted key emission */
#define REFSIG_PHASE_SIMHASH 5    /* K4a */
#define REFSIG_PHASE_H2D 6        /* corpus upload */
#define REFSIG_PHASE_D2H 7        /* result download */
#define REFSIG_N_PHASES 8
int refsig_gpu_set_profiling(refsig_gpu_ctx* ctx, int on);
int refsig_gpu_phase_times(refsig_gpu_ctx* ctx, double* ms, uint64_t* calls);
/* K3 compare path (testing / A-B measurement): 0 auto (tcgen05 when K <= 128
 * and |tau| is 0 or >= 2^-14, else FP32 CUDA cores), 1 FP32 CUDA cores,
 * 2 tcgen05 (validation error at the pair call if K / tau do not fit it).
 * Both paths apply the same compare rule. */
#define REFSIG_K3_AUTO 0
#define REFSIG_K3_FP32 1
#define REFSIG_K3_TENSOR 2
int refsig_gpu_set_k3_path(refsig_gpu_ctx* ctx, int path);
/* Debug: with REFSIG_CANARY=1 in the environment every device buffer carries
 * a guard region past its end; this synchronises and returns 1 (runtime)
 * naming any buffer whose guard a kernel overwrote. 0 when clean or off. */
int refsig_gpu_debug_check(refsig_gpu_ctx* ctx);
/* Kernels launched by this library in this process so far. */
uint64_t refsig_gpu_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
