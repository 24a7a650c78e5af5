// kernels.cuh — launcher declarations for the refsig B200 kernels.
//
// K1 count  : per-doc sort + run-length encode, df, idf      (ngram.hpp:62-75,170-178)
// K2 sign   : warp-per-doc gather against the compact reference table
// K3 pairs  : all-pairs signature compare -> pair bitmap -> sorted keys
// K4 simhash: exact column sums + ballot-free bit build; Hamming pairs (simhash.hpp:35-47)
// K5 exact  : exact sparse cosine verifier (ngram.hpp:184-202)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace refsig_gpu {

// ---- text front end (k0_text.cu) -------------------------------------------
// Per doc of raw bytes [off[d], off[d+1]): tokens == NULL -> cnt[d] = number of
// 3-grams; else the 3-gram ids (vocabulary 17576) at tokens[gram_off[d] ..).
void launch_text_grams(const uint8_t* text, const uint64_t* off, uint32_t n_docs, const uint64_t* gram_off,
                       uint32_t* cnt, uint32_t* tokens, cudaStream_t s);
// fp[d] = simhash of the doc's normalized words (MD5 word hashes, +-1 votes).
void launch_text_simhash(const uint8_t* text, const uint64_t* off, uint32_t n_docs, uint64_t* fp, cudaStream_t s);
constexpr uint32_t kGramSpace = 26u * 26u * 26u;  // ngram.hpp: 17576 3-grams

// ---- K1 -------------------------------------------------------------------
// Count work plan (k1_count.cu, built at upload): documents of <= 64 / 128 /
// 256 tokens are sorted by one warp each (that many keys in registers);
// 257..8192 tokens by one CTA of 2..32 warps (8 keys per thread; kGroupCap
// classes above 512); longer ones in a global scratch region.
constexpr uint32_t kTinyMax = 64;
constexpr int kGroupClasses = 4;
constexpr uint32_t kGroupCap[kGroupClasses] = {1024, 2048, 4096, 8192};
constexpr uint32_t kGroupMax = 8192;

struct CountArgs {
  const uint32_t* tokens;
  const uint64_t* doc_off;
  uint32_t vocab;
  uint2* ent;        // padded CSR: doc d's (id,count) rows at ent[doc_off[d] ..)
  uint32_t* nnz;     // [n_docs]
  uint32_t* df;      // [df_reps][vocab] replicas, zeroed by the caller
  uint32_t df_reps;
  uint32_t* err;     // bit 0: token id >= vocab
};

// One warp per doc, 32*ipt keys (ipt 2 / 4 / 8).
void launch_count_warp(int ipt, const CountArgs& a, const uint32_t* docs, uint32_t n, cudaStream_t s);
// One CTA per doc, 8 keys per thread: cls -1 = 257..512 tokens (2 warps),
// 0..3 = the kGroupCap classes (4/8/16/32 warps).
void launch_count_group(int cls, const CountArgs& a, const uint32_t* docs, uint32_t n, cudaStream_t s);
void launch_count_large(const CountArgs& a, const uint32_t* long_docs, const uint64_t* scratch_off,
                        uint32_t n_long, uint32_t* scratch, cudaStream_t s);
// df[t] = sum of the replicas; idf32[t] = fl32(ln((1+N)/(1+df))+1) (or 1 for
// raw-TF weighting); ref_row = -1.
void launch_idf(const uint32_t* df_rep, uint32_t reps, uint32_t vocab, uint32_t n_docs, int weight_mode, uint32_t* df,
                TermInfo* info, cudaStream_t s);
// MRCS signature records, 20 + 8K bytes per doc, as 32-bit words.
void launch_mrcs_records(const float* S, uint32_t n_docs, uint32_t K, uint64_t ref_id, uint32_t* out,
                         cudaStream_t s);
// info[t] = {idf(df[t], n_docs), -1} from a (globally reduced) df table.
void launch_idf_from_df(const uint32_t* df, uint32_t vocab, uint32_t n_docs, int weight_mode, TermInfo* info,
                        cudaStream_t s);
// ST[k][ld] = unit(S[d][.]) for externally supplied signatures (k2_sign.cu).
void launch_st_from_s(const float* S, uint32_t n_docs, uint32_t K, uint32_t ld, float* ST, cudaStream_t s);
// cf[t] = sum of the counts of term t over all documents (exact, 64-bit).
void launch_corpus_freq(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, uint32_t n_docs,
                        uint32_t vocab, uint32_t reps, unsigned long long* cf_rep, uint64_t* cf, cudaStream_t s);
// Compact padded CSR -> rowptr/ids/counts (rowptr from an exclusive scan of nnz).
void launch_compact_csr(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, const uint64_t* rowptr,
                        uint32_t n_docs, uint32_t* ids, uint32_t* counts, cudaStream_t s);
// inv_norm[d] = 1/||w_d|| (0 for an empty doc), w = count*idf.
void launch_inv_norm(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, const TermInfo* info,
                     uint32_t n_docs, float* inv_norm, cudaStream_t s);

// ---- scans ----------------------------------------------------------------
// out[0..n] = exclusive prefix of in[0..n) (out[n] = total). tmp >= scan_tmp_bytes(n).
size_t scan_tmp_bytes(uint64_t n);
// total_out (optional, e.g. mapped pinned memory): also receives out[n].
void launch_exclusive_scan_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t n, void* tmp, cudaStream_t s,
                                      uint64_t* total_out = nullptr);

// ---- A5 reference table ----------------------------------------------------
// K reference vectors. Docs mode (docs != NULL): vector k is corpus doc
// docs[k], rows ent[doc_off[d] ..+nnz[d]) with ent.y a count (w = count*idf).
// Explicit mode: vector k = ent[start[k] ..+n[k]) with ent.y the float bits of
// the raw weight (partition vectors use 1.0). Ids are unique
// within a vector.
struct RefArgs {
  uint32_t K;
  const uint64_t* start;
  const uint32_t* n;
  const uint2* ent;
  bool explicit_w;
  uint32_t Kp;  // row stride of R: roundup(K,4) for K <= 32, roundup(K,32) above (k2_sign.cu)
  const uint64_t* doc_off;  // with nnz and ids: reference k = document ids[k] of the corpus
  const uint32_t* nnz;
  uint32_t ids[256];  // by value (kernel parameter: no upload before the reference build); K <= 256
};
// info[t].ref_row = -1 for all t (only needed when a reference is replaced).
void launch_ref_reset(TermInfo* info, uint32_t vocab, cudaStream_t s);
// Compact rows for the union U (zeroed), then R[row*Kp + k] = w_k[t]/||w_k||;
// *counter = |U|. One launch when the K vectors hold at most n_entries_max <=
// 65536 entries (a bound: e.g. their token counts), else three (k2_sign.cu).
// info[].ref_row must be -1.
void launch_ref_build(const RefArgs& r, TermInfo* info, uint32_t vocab, uint32_t* counter, float* R,
                      uint64_t n_entries_max, cudaStream_t s);

// ---- K2 sign ----------------------------------------------------------------
struct SignArgs {
  const uint2* ent;
  const uint64_t* doc_off;
  const uint32_t* nnz;
  const TermInfo* info;
  const float* R;
  uint32_t n_docs;
  uint32_t K;
  uint32_t Kp;           // row stride of R
  const uint32_t* order;  // docs by decreasing length; the first n_long get a CTA each (k2_sign.cu)
  uint32_t n_long;
  uint32_t n_half;         // K <= 32: order[n_half..) (<= kSignHalfTokens tokens) go two per warp
  float* S;         // [n_docs*K] raw cosines, row-major (API output)
  float* ST;        // [K][ld] unit-normalised signatures, transposed (K3 operand; 0 if all-zero)
  uint32_t ld;      // leading dimension of ST (n_docs rounded up to 128; pad columns zero)
  float* inv_norm;  // [n_docs] 1/||w_d||
};
constexpr uint32_t kSignLongTokens = 2048;  // K2: longer documents get a CTA
constexpr uint32_t kSignHalfTokens = 1024;  // K2 (K <= 32): shorter documents go two per warp (768-1024 best)
constexpr uint32_t kMaxRefs = 256;          // K limit (K2 keeps a signature row in registers)
void launch_sign(const SignArgs& a, cudaStream_t s);

// ---- K3 / K4b pair bitmaps --------------------------------------------------
// bitmap: row-major, words_per_row = n_pad_cols/32. Bits (i,j) set iff pair
// matches; only tiles with col-tile >= row-tile are written (i<j triangle) for
// the self-join, all tiles for the query join. rowcnt[i] += matches in row i.
struct PairGrid {
  uint32_t n_rows;      // rows (queries for a join)
  uint32_t n_cols;      // columns (= n_rows for a self-join)
  uint32_t words_per_row;
  bool triangle;        // self-join: only j > i
  uint32_t row_begin;   // rows this call covers: [row_begin, row_end), row_begin % 128 == 0
  uint32_t row_end;
  uint32_t tile0;       // first tile index (set by the launcher)
};
void launch_mrc_bitmap(const float* ST_rows, uint32_t ld_rows, const float* ST_cols, uint32_t ld_cols, uint32_t K,
                       float tau, const PairGrid& g, uint32_t* bitmap, uint32_t* rowcnt, cudaStream_t s);
// K3 on tcgen05 (k3_tc.cu): split-fp16 operand forms of the unit signatures,
// then the tile kernel writing the same bitmap + row counts as launch_mrc_bitmap.
uint32_t mrc_tc_kp(uint32_t K);
bool mrc_tc_supported(uint32_t K, float tau);
size_t mrc_tc_form_bytes(uint32_t K, uint32_t n_docs);
// rowcnt != NULL: also zero rowcnt[0 .. n_rowcnt) (the tile kernel's row counts; n_rowcnt <= n_docs panels).
void launch_mrc_tc_forms(const float* ST, uint32_t ld, uint32_t n_docs, uint32_t K, float tau, void* rowf, void* colf,
                         uint32_t* rowcnt, uint32_t n_rowcnt, cudaStream_t s, bool col64 = false);
// CTA-pair (cta_group::2) K3 for the chunked query join; column forms in 64-document panels (col64).
bool mrc_tc2_applies(uint32_t K, const PairGrid& g);
// false: the TMA descriptor could not be built (cuTensorMapEncodeTiled unavailable / failed)
bool launch_mrc_tc2(const void* rowf, const void* colf, uint32_t K, const PairGrid& g, uint32_t* bitmap,
                    uint32_t* rowcnt, cudaStream_t s);
void launch_mrc_tc(const void* rowf, const void* colf, uint32_t K, const PairGrid& g, uint32_t* bitmap,
                   uint32_t* rowcnt, cudaStream_t s);
// Hamming join on the tensor cores (k3_tc.cu): +-1 int8 forms of the 64-bit
// fingerprints (row forms carry the threshold), then the tcgen05 tile kernel
// with kind::i8 into the same bitmap / row counts as launch_hamming_bitmap.
size_t ham_tc_form_bytes(uint32_t n);
void launch_ham_tc_forms(const uint64_t* fp, uint32_t n, int max_dist, void* rowf, void* colf, cudaStream_t s);
void launch_ham_tc(const void* rowf, const void* colf, const PairGrid& g, uint32_t* bitmap, uint32_t* rowcnt,
                   cudaStream_t s);
void launch_hamming_bitmap(const uint64_t* f_rows, const uint64_t* f_cols, int max_dist, const PairGrid& g,
                           uint32_t* bitmap, uint32_t* rowcnt, cudaStream_t s);
// keys[k] = (i<<32) | cols[k] for rows [row_begin, row_end) (CSR -> sorted keys).
void launch_cols_to_keys(const uint64_t* rowstart, uint32_t row_begin, uint32_t row_end, const uint32_t* cols,
                         uint64_t* keys, cudaStream_t s);
// Sorted CSR columns: row i's matches j ascending at cols[rowstart[i] ..);
// writes only below capacity.
// counter: two device words, zero at the first launch; the kernel leaves them zero.
void launch_emit_pairs(const uint32_t* bitmap, const PairGrid& g, const uint32_t* rowcnt, const uint64_t* rowstart,
                       uint32_t* out, uint64_t capacity, uint32_t* counter, cudaStream_t s);

// out[k] = (uint16) in[k] (column ids of a grid with n_cols <= 65536).
void launch_narrow_cols(const uint32_t* in, uint64_t n, uint16_t* out, cudaStream_t s);
// out[i] = in[i] - in[0] for i < n (a row range's CSR offsets rebased to 0).
void launch_rebase_rowptr(const uint64_t* in, uint64_t n, uint64_t* out, cudaStream_t s);
// n <= kParamWords host words to the device as kernel parameters (no copy engine).
constexpr uint32_t kParamWords = 256;
void launch_param_words(const uint32_t* host_src, uint32_t n, uint32_t* dst, cudaStream_t s);
// n words device -> device by a kernel (16-byte aligned pointers).
void launch_copy_words(const uint32_t* src, uint64_t n, uint32_t* dst, cudaStream_t s);
// n device words into mapped pinned host memory (device pointer of it) by a kernel.
void launch_words_to_host(const uint32_t* src, uint32_t n, uint32_t* mapped_dst, cudaStream_t s);

// ---- K4a simhash -------------------------------------------------------------
struct SimhashArgs {
  const uint2* ent;
  const uint64_t* doc_off;
  const uint32_t* nnz;
  const TermInfo* info;
  const uint64_t* term_hash;  // optional [vocab] table (NULL: splitmix64 with seed)
  uint64_t seed;
  uint32_t n_docs;
  bool use_idf;               // false: raw TF weights (the reference's +-1 per occurrence)
  uint64_t* fp;
  const uint32_t* order;      // docs by decreasing length; the first n_long get a CTA each
  uint32_t n_long;
};
void launch_simhash(const SimhashArgs& a, cudaStream_t s);

// ---- K5 exact cosine --------------------------------------------------------
constexpr uint32_t kExactHead = 64;     // dense head terms (highest df)
constexpr uint32_t kExactPanel = 49152;  // docs per shared-memory column panel (192 KB)
struct ExactArgs {
  const uint2* ent;
  const uint64_t* doc_off;
  const uint32_t* nnz;
  const float* x;            // unit weights aligned with ent (padded CSR)
  const int32_t* head_col;   // [vocab] column in A of a head term, -1 for tail terms
  const uint64_t* post_off;  // [vocab+1] postings offsets (exclusive scan of df)
  const uint2* posts;        // (doc, x bits) per posting, each term's list sorted by doc
  const uint32_t* entpos;    // [padded CSR slot] position of entry (d, t) in t's postings
  const float* A;            // [n_docs][H] dense head rows
  const float* hn;           // [n_docs] norm of the head part
  uint32_t H;                // multiple of 4
  uint32_t n_docs;
  uint32_t panel;            // column panel (docs)
  float tau;
  uint32_t* bitmap;          // zeroed rows, words_per_row words each
  uint32_t words_per_row;
  uint32_t* rowcnt;
  uint32_t* tail_out;        // evaluation mode: the fixed-point tail sums of rows [row_lo, row_hi) for
                             // j > i, row-major [row_hi-row_lo][tail_ld] (no threshold, no bitmap)
  uint32_t tail_ld;          // row stride of tail_out (>= n_docs; the tensor-core evaluation wants 128-multiples)
};
void launch_unit_weights(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, const TermInfo* info,
                         const float* inv_norm, uint32_t n_docs, float* x, cudaStream_t s);
// The H highest-df terms (ties: lower id first) -> head_col[t] = rank or -1.
size_t head_select_temp_bytes(uint32_t vocab);
void launch_head_select(const uint32_t* df, uint32_t vocab, uint32_t H, uint32_t* keys_a, uint32_t* keys_b,
                        uint32_t* ids_a, uint32_t* ids_b, void* tmp, size_t tmp_bytes, int32_t* head_col,
                        cudaStream_t s);
// Doc-sorted postings of every term (stable radix sort of the padded CSR slots
// by term id); keys/vals/slot_doc hold n_slots words, tmp is csc_sort_temp_bytes().
size_t csc_sort_temp_bytes(uint64_t n_slots, uint32_t vocab);
void build_csc_postings(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, uint32_t n_docs,
                        uint32_t vocab, uint64_t n_slots, const float* x, uint32_t* keys_a, uint32_t* keys_b,
                        uint32_t* vals_a, uint32_t* vals_b, uint32_t* slot_doc, void* tmp, size_t tmp_bytes,
                        uint2* posts, uint32_t* entpos, cudaStream_t s);
void launch_head_rows(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, const float* x,
                      const int32_t* head_col, uint32_t n_docs, uint32_t H, float* A, float* hn, cudaStream_t s);
// Rows [row_lo, row_hi): tail accumulation, bound, head dot, threshold into the bitmap.
void launch_exact_tail(const ExactArgs& a, uint32_t row_lo, uint32_t row_hi, cudaStream_t s);
// ---- fused evaluation -------------------------------------
// Per pair i<j of rows [row_lo, row_hi): exact = min(A_i.A_j + T_ij * 2^-30, 1)
// (dense head + fixed-point tail), mrc = min(S^_i.S^_j, 1), sim = 1 - hd/64;
// e = score - exact. out[cta*8 + {0..7}] = {n, sum e_mrc, sum e_mrc^2,
// sum |e_mrc|, sum e_sim, sum e_sim^2, sum |e_sim|, 0} (double, fixed order).
struct EvalArgs {
  const float* AT;   // [H][ld] head rows, k-major, zero-padded columns
  uint32_t H;        // multiple of 4
  const float* ST;   // [K][ld] unit signatures
  uint32_t K;
  uint32_t ld;
  const uint64_t* fp;  // [n_docs] fingerprints (NULL: no Simhash errors)
  const uint32_t* T;   // tail sums, row-major [row_hi-row_lo][ldT]
  uint32_t n_docs, row_lo, row_hi;
  double* out;         // [grid*8]
  uint32_t ldT;
};
uint32_t eval_grid();
void launch_eval_tiles(const EvalArgs& a, cudaStream_t s);
// The same evaluation with the head and MRC dots on tcgen05 (k5_tc.cu): split-
// fp16 operand forms of [head | MRC] per document, then one tile kernel
// (returns its grid: out holds grid x 8 doubles). T rows have stride ldT.
bool eval_tc_supported(uint32_t H, uint32_t K);
size_t eval_tc_form_bytes(uint32_t H, uint32_t K, uint32_t n_docs);
void launch_eval_tc_forms(const float* AT, uint32_t H, const float* ST, uint32_t K, uint32_t ld, uint32_t n_docs,
                          void* rowf, void* colf, cudaStream_t s);
uint32_t launch_eval_tc(const void* rowf, const void* colf, uint32_t H, uint32_t K, uint32_t n_docs, uint32_t row_lo,
                        uint32_t row_hi, const uint32_t* T, uint32_t ldT, const uint64_t* fp, double* out,
                        cudaStream_t s);
// AT[c*ld + d] = A[d*H + c] (ld >= n_docs, pad columns zero).
void launch_transpose_head(const float* A, uint32_t n_docs, uint32_t H, uint32_t ld, float* AT, cudaStream_t s);
void launch_pair_cosines(const uint2* ent, const uint64_t* doc_off, const uint32_t* nnz, const float* x,
                         const uint64_t* keys, uint64_t n_keys, float* out, cudaStream_t s);

}  // namespace refsig_gpu
