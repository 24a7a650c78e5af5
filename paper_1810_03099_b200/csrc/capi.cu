// capi.cu — the C ABI (include/refsig_gpu.h): context, device buffers,
// validation and the status <-> refsig::validation_error / runtime_error
// mapping (reference error.hpp:8-14). Every compute entry point enqueues CUDA
// kernels (kernels.cuh); there is no host compute path.

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "refsig_gpu.h"

using namespace refsig_gpu;

#include <atomic>
#include <map>
#include <mutex>
#include <utility>

namespace {
std::atomic<uint64_t> g_launches{0};
std::atomic<uint64_t> g_alloc_gen{0};  // bumped on every device (re)allocation: invalidates captured graphs
}  // namespace

namespace refsig_gpu {
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

bool pdl_enabled() {
  static const bool on = [] {
    const char* m = std::getenv("REFSIG_NO_PDL");
    return !(m && m[0] == '1');
  }();
  return on;
}

void ensure_smem_attr(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> set;  // (kernel, device) -> bytes already allowed
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  int& have = set[{func, dev}];
  if (have >= bytes) return;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess) have = bytes;
}
}  // namespace refsig_gpu

namespace {

struct Status {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Status{code, msg}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(REFSIG_E_RUNTIME, std::string(what) + ": " + cudaGetErrorString(e));
}

// (const char* overload: the message is only built on failure — require() runs
// per document in the upload validation loops)
void require(bool ok, const char* msg) {
  if (!ok) fail(REFSIG_E_VALIDATION, msg);
}

// Debug guard (REFSIG_CANARY=1): every device buffer gets kCanaryBytes of
// 0xA5 past its capacity; refsig_gpu_debug_check verifies them (a kernel that
// wrote past a buffer's end is reported by name). compute-sanitizer is closed
// on the GPU pool this was built on; this is the out-of-bounds-write check.
constexpr size_t kCanaryBytes = 4096;
bool canary_on() {
  static const bool on = [] {
    const char* m = std::getenv("REFSIG_CANARY");
    return m && m[0] == '1';
  }();
  return on;
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  // Grow-only; contents are not preserved. Returns true if (re)allocated.
  // A regrowth takes 1/8 headroom: streamed batches vary in size by a few
  // percent, and every reallocation's cudaFree waits for the whole device
  // (it would serialise the batch pipeline).
  bool ensure(size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (bytes <= cap) return false;
    if (p) {
      cudaFree(p);
      p = nullptr;
      cap = 0;
      bytes += bytes / 8;
    }
    const size_t extra = canary_on() ? kCanaryBytes : 0;
    ck(cudaMalloc(&p, bytes + extra), "cudaMalloc");
    if (extra) ck(cudaMemset(static_cast<char*>(p) + bytes, 0xA5, extra), "canary");
    cap = bytes;
    g_alloc_gen.fetch_add(1);
    return true;
  }
  // true if the canary past cap is intact (or canaries are off)
  bool canary_ok() const {
    if (!canary_on() || !p) return true;
    std::vector<unsigned char> h(kCanaryBytes);
    if (cudaMemcpy(h.data(), static_cast<const char*>(p) + cap, kCanaryBytes, cudaMemcpyDeviceToHost) != cudaSuccess)
      return false;
    for (unsigned char b : h)
      if (b != 0xA5) return false;
    return true;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace

constexpr int kPlanListCount = 10;  // refsig_gpu_ctx::kPlanLists
// Host side of a work plan (the K1/K2/K4a document lists) and where it sits in
// its pinned staging buffer: doc_off (u64), the u32 lists, then the u64
// scratch offsets of documents > 8192 tokens.
struct PlanInfo {
  uint32_t n_docs = 0, vocab = 0;
  uint64_t n_tokens = 0;
  uint32_t plan_off[kPlanListCount] = {}, plan_n[kPlanListCount] = {};
  uint32_t n_sign_long = 0, n_sign_half = 0;
  uint32_t n_loff = 0;
  uint64_t scratch = 0;  // words of K1 long-document scratch
  size_t off_bytes = 0, list_bytes = 0, loff_at = 0, bytes = 0;
};

struct refsig_gpu_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  // side streams + events for the fork/join inside count() (independent K1
  // work classes overlap instead of serialising their tails)
  cudaStream_t side[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join[3] = {nullptr, nullptr, nullptr};
  std::string err;
  uint64_t* h_pin = nullptr;  // mapped pinned scratch for small D2H reads (written by kernels)
  uint32_t* d_pin = nullptr;  // its device address

  // corpus
  bool loaded = false;
  uint32_t n_docs = 0, vocab = 0;
  uint64_t n_tokens = 0;
  std::vector<uint64_t> h_off;
  DevBuf tokens, doc_off;
  const uint32_t* tok = nullptr;
  // K1/K2/K4a work plan, one device buffer (plan), written from one pinned host
  // buffer (h_plan) by one copy: doc lists by work class, longest docs first.
  DevBuf plan;
  uint32_t* h_plan = nullptr;
  size_t h_plan_cap = 0;
  cudaEvent_t plan_done = nullptr;  // h_plan consumed by its copy
  enum { kPlanTiny, kPlanW4, kPlanW8, kPlanW16, kPlanG0, kPlanG1, kPlanG2, kPlanG3, kPlanLong, kPlanOrder, kPlanLists };
  uint32_t plan_off[kPlanLists] = {}, plan_n[kPlanLists] = {};
  static_assert(kPlanLists == kPlanListCount, "PlanInfo list count");
  const uint32_t* plan_list(int k) const { return plan.as<uint32_t>() + plan_off[k]; }
  DevBuf long_off, long_scratch;
  uint32_t n_sign_long = 0;  // order[0, n_sign_long): > kSignLongTokens tokens, one CTA each in K2/K4a
  uint32_t n_sign_half = 0;  // order[n_sign_half, N): <= kSignHalfTokens tokens, two per warp in K2

  // K1
  bool counted = false;
  int weight_mode = REFSIG_WEIGHT_TFIDF;
  DevBuf ent, nnz, df, df_rep, info, flags;
  DevBuf rowptr, c_ids, c_counts, inv_norm;
  bool have_inv_norm = false;

  // reference
  bool have_ref = false;
  uint32_t K = 0, Kp = 0;  // Kp: row stride of R
  DevBuf ref_start, ref_n, ref_ent, ref_count, R;
  std::vector<uint32_t> ref_ids;  // reference document ids (kernel parameters)
  bool ref_dirty = false;  // info[].ref_row holds a previous reference's rows

  // sign
  bool signed_ = false;
  DevBuf S, ST;
  uint32_t ld = 0;  // leading dimension of ST

  // pairs
  // pair output: sorted CSR columns (cand) over rowstart; the 64-bit keys
  // (keys) are materialised only when a caller asks for them
  DevBuf bitmap, rowcnt, rowstart, cand, scan_tmp, keys, emit_ctr;
  DevBuf cand16;  // 16-bit column copy for get_pairs_csr16
  const uint32_t* plan_tok = nullptr;  // token pointer the plan / step graph were built with
  uint64_t cand_count = 0;
  bool have_pairs = false;  // cand/rowstart/emit_grid hold the last pair computation
  bool keys_valid = false;

  // simhash
  bool have_fp = false;
  // text front end: the raw corpus stays resident for simhash_text
  DevBuf text, text_off, text_cnt;
  uint32_t text_docs = 0;
  bool have_text = false;
  DevBuf fp, term_hash;

  // exact
  bool have_x = false;
  DevBuf x, post_off, posts, head_col, headA, head_norm, entpos, csc_ka, csc_kb, csc_va, csc_vb, csc_doc, csc_tmp;  // K5
  DevBuf headAT, eval_tail, eval_part;                                         // evaluation
  DevBuf cf_rep, cf;                                                           // corpus frequencies
  DevBuf records;                                                              // MRCS records
  DevBuf tc_forms;                                                             // K3 tcgen05 operand forms
  DevBuf ham_forms;                                                            // Hamming int8 forms (tcgen05 kind::i8)

  // staged batches (refsig_gpu_stage_corpus / swap_corpus), up to kStageDepth
  // ahead in a ring: tokens and the work plan (built on the host at stage time)
  // copied on copy_stream into the slot's buffers while earlier batches
  // compute; a swap exchanges the slot's buffers with the live ones
  struct Staged {
    DevBuf tokens, doc_off, plan, long_off;
    cudaEvent_t ev_ready = nullptr;  // the slot's copies are done (copy stream)
    cudaEvent_t ev_plan = nullptr;   // its plan copies are done: h_plan reusable (copy stream)
    cudaEvent_t ev_free = nullptr;   // its buffers are no longer read by compute (compute stream)
    bool free_recorded = false;
    PlanInfo pi;
    std::vector<uint64_t> off;
  };
  static constexpr int kStageDepth = 2;
  Staged stg[kStageDepth];
  // pinned plan staging, a ring deeper than the slots: the buffer reused now was
  // read by plan copies issued kPlanRing stages ago (those can queue behind a
  // token upload on the copy engine, so one ring per slot was not enough)
  static constexpr int kPlanRing = 4;
  uint32_t* h_plans[kPlanRing] = {};
  size_t h_plans_cap[kPlanRing] = {};
  cudaEvent_t ev_hplan[kPlanRing] = {};
  bool hplan_recorded[kPlanRing] = {};
  int hplan_next = 0;
  int stg_head = 0, stg_count = 0;
  cudaStream_t copy_stream = nullptr;  // staged tokens, back to back
  cudaStream_t plan_stream = nullptr;  // staged plans: small copies that must not sit between two token uploads

  // asynchronous result fetch (refsig_gpu_get_pairs_csr16_async): two slots of
  // device staging (rebased rowptr, 16-bit columns) copied to the host on
  // d2h_stream while the next batch computes
  cudaStream_t d2h_stream = nullptr;
  cudaEvent_t ev_fetch_ready = nullptr, ev_fetched[2] = {nullptr, nullptr};
  DevBuf fetch_rowptr[2], fetch_cols[2];
  bool fetch_pending[2] = {false, false};
  int fetch_slot = 0;

  // tcgen05 column forms of this (database) context's signatures, cached for
  // query joins (they do not depend on tau); valid while sign_gen is unchanged
  DevBuf tc_colf;
  uint64_t sign_gen = 0, tc_colf_gen = ~0ull;
  bool tc_colf_col64 = false;  // tc_colf laid out as 64-document panels (CTA-pair kernel)

  // query mode
  refsig_gpu_ctx* db = nullptr;
  int k3_path = REFSIG_K3_AUTO;  // refsig_gpu_set_k3_path

  // emit in flight (enqueue_emit -> finish_emit)
  bool emit_pending = false;
  PairGrid emit_grid{};

  // captured MRC step (refsig_gpu_mrc_step)
  cudaGraphExec_t step_exec = nullptr;
  struct StepKey {
    uint64_t alloc_gen = ~0ull, load_gen = 0;
    int weight_mode = -1;
    std::vector<uint32_t> refs;
    float tau = 0.0f;
    uint32_t lo = 0, hi = 0;
    cudaStream_t stream = nullptr;
    bool operator==(const StepKey& o) const {
      return alloc_gen == o.alloc_gen && load_gen == o.load_gen && weight_mode == o.weight_mode && refs == o.refs &&
             tau == o.tau && lo == o.lo && hi == o.hi && stream == o.stream;
    }
  } step_key;
  uint64_t load_gen = 0;
  bool capturing = false;

  // profiling: event pairs per phase on `stream`, resolved lazily
  bool prof = false;
  struct Mark {
    int phase;
    cudaEvent_t a, b;
  };
  std::vector<Mark> marks;
  std::vector<cudaEvent_t> ev_free;

  // (name, buffer) of every device buffer, for refsig_gpu_debug_check
  std::vector<std::pair<const char*, const DevBuf*>> buffers() const {
    return {{"tokens", &tokens}, {"doc_off", &doc_off}, {"plan", &plan}, {"long_off", &long_off},
            {"stg0.tokens", &stg[0].tokens}, {"stg0.doc_off", &stg[0].doc_off}, {"stg0.plan", &stg[0].plan},
            {"stg0.long_off", &stg[0].long_off}, {"stg1.tokens", &stg[1].tokens}, {"stg1.doc_off", &stg[1].doc_off},
            {"stg1.plan", &stg[1].plan}, {"stg1.long_off", &stg[1].long_off},
            {"long_scratch", &long_scratch}, {"ent", &ent}, {"nnz", &nnz}, {"df", &df}, {"df_rep", &df_rep},
            {"info", &info}, {"flags", &flags}, {"rowptr", &rowptr}, {"c_ids", &c_ids}, {"c_counts", &c_counts},
            {"inv_norm", &inv_norm}, {"ref_start", &ref_start}, {"ref_n", &ref_n},
            {"ref_ent", &ref_ent}, {"ref_count", &ref_count}, {"R", &R}, {"S", &S}, {"ST", &ST}, {"bitmap", &bitmap},
            {"rowcnt", &rowcnt}, {"rowstart", &rowstart}, {"cand", &cand}, {"scan_tmp", &scan_tmp}, {"keys", &keys},
            {"emit_ctr", &emit_ctr}, {"cand16", &cand16}, {"text", &text}, {"text_off", &text_off},
            {"text_cnt", &text_cnt}, {"fp", &fp}, {"term_hash", &term_hash}, {"x", &x}, {"post_off", &post_off},
            {"posts", &posts}, {"head_col", &head_col}, {"headA", &headA},
            {"head_norm", &head_norm}, {"entpos", &entpos}, {"csc_ka", &csc_ka}, {"csc_kb", &csc_kb},
            {"ham_forms", &ham_forms}, {"csc_va", &csc_va}, {"csc_vb", &csc_vb}, {"csc_doc", &csc_doc}, {"csc_tmp", &csc_tmp}, {"headAT", &headAT}, {"eval_tail", &eval_tail},
            {"eval_part", &eval_part}, {"cf_rep", &cf_rep}, {"cf", &cf}, {"records", &records},
            {"tc_forms", &tc_forms}, {"fetch_rowptr0", &fetch_rowptr[0]}, {"fetch_rowptr1", &fetch_rowptr[1]},
            {"fetch_cols0", &fetch_cols[0]}, {"fetch_cols1", &fetch_cols[1]}};
  }
  ~refsig_gpu_ctx() {
    for (auto& m : marks) {
      cudaEventDestroy(m.a);
      cudaEventDestroy(m.b);
    }
    for (auto e : ev_free) cudaEventDestroy(e);
    if (h_plan) cudaFreeHost(h_plan);
    for (int k = 0; k < kPlanRing; ++k) {
      if (h_plans[k]) cudaFreeHost(h_plans[k]);
      if (ev_hplan[k]) cudaEventDestroy(ev_hplan[k]);
    }
    for (auto& g : stg) {
      if (g.ev_ready) cudaEventDestroy(g.ev_ready);
      if (g.ev_plan) cudaEventDestroy(g.ev_plan);
      if (g.ev_free) cudaEventDestroy(g.ev_free);
    }
    if (plan_done) cudaEventDestroy(plan_done);
    if (step_exec) cudaGraphExecDestroy(step_exec);
    if (ev_fetch_ready) cudaEventDestroy(ev_fetch_ready);
    for (auto e : ev_fetched)
      if (e) cudaEventDestroy(e);
  }
};

namespace {

template <class F>
int guard(refsig_gpu_ctx* ctx, F&& f) {
  if (!ctx) return REFSIG_E_VALIDATION;
  try {
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    f();
    ctx->err.clear();
    return REFSIG_OK;
  } catch (const Status& s) {
    ctx->err = s.msg;
    return s.code;
  } catch (const std::bad_alloc&) {
    ctx->err = "host out of memory";
    return REFSIG_E_RUNTIME;
  }
}

// Synchronise the stream and surface errors of enqueued work (CUDA faults,
// token ids >= vocab flagged by K1).
void sync(refsig_gpu_ctx* c) {
  if (c->flags.p) launch_words_to_host(c->flags.as<uint32_t>(), 1, c->d_pin + 14, c->stream);  // -> h_pin[7]
  ck(cudaStreamSynchronize(c->stream), "kernel execution");
  ck(cudaGetLastError(), "kernel launch");
  if (c->flags.p) {
    uint32_t f = static_cast<uint32_t>(c->h_pin[7]);
    if (f & 1u) {
      ck(cudaMemsetAsync(c->flags.p, 0, 4, c->stream), "memset");
      c->counted = false;
      fail(REFSIG_E_VALIDATION, "token id >= vocab in corpus");
    }
  }
}

void launched(const char* what) {
  // REFSIG_SYNC_DEBUG=1: synchronise after every phase so a fault is reported by the phase that caused it
  static const bool dbg = [] {
    const char* m = std::getenv("REFSIG_SYNC_DEBUG");
    return m && m[0] == '1';
  }();
  if (dbg) ck(cudaDeviceSynchronize(), what);
  ck(cudaGetLastError(), what);
}

cudaEvent_t take_event(refsig_gpu_ctx* c) {
  if (!c->ev_free.empty()) {
    cudaEvent_t e = c->ev_free.back();
    c->ev_free.pop_back();
    return e;
  }
  cudaEvent_t e;
  ck(cudaEventCreate(&e), "cudaEventCreate");
  return e;
}

// RAII: brackets the enqueued work of one phase with events on ctx->stream.
struct Phase {
  refsig_gpu_ctx* c;
  int id;
  cudaEvent_t a = nullptr;
  Phase(refsig_gpu_ctx* ctx, int phase) : c(ctx), id(phase) {
    if (!c->prof) return;
    a = take_event(c);
    ck(cudaEventRecord(a, c->stream), "cudaEventRecord");
  }
  ~Phase() {
    if (!a) return;
    cudaEvent_t b = nullptr;
    if (!c->ev_free.empty()) {
      b = c->ev_free.back();
      c->ev_free.pop_back();
    } else if (cudaEventCreate(&b) != cudaSuccess) {
      c->ev_free.push_back(a);
      return;
    }
    cudaEventRecord(b, c->stream);
    c->marks.push_back({id, a, b});
  }
};


void reset_downstream(refsig_gpu_ctx* c) {
  c->have_ref = c->signed_ = c->have_fp = c->have_x = c->have_inv_norm = false;
  c->cand_count = 0;
  c->have_pairs = false;
}

int sm_count_host() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

uint32_t words_per_row(uint32_t n_cols) { return static_cast<uint32_t>(ceil_div(n_cols, kTile) * 4); }

// The 64-bit keys (i<<32|j) of the last pair computation, built on demand
// from the CSR columns (rows outside the emit range have no pairs).
void materialize_keys(refsig_gpu_ctx* c) {
  if (c->keys_valid) return;
  c->keys.ensure(sizeof(uint64_t) * std::max<uint64_t>(c->cand_count, 1));
  const PairGrid& g = c->emit_grid;
  launch_cols_to_keys(c->rowstart.as<uint64_t>(), g.row_begin, g.row_end, c->cand.as<uint32_t>(),
                      c->keys.as<uint64_t>(), c->stream);
  c->keys_valid = true;
}

// Scan rowcnt and emit sorted CSR columns into ctx->cand with its capacity;
// the total is copied (async) to h_pin[0]. No host synchronisation.
void enqueue_emit(refsig_gpu_ctx* c, const PairGrid& g) {
  const uint64_t n = g.n_rows;
  c->rowstart.ensure(sizeof(uint64_t) * (n + 1));
  c->scan_tmp.ensure(scan_tmp_bytes(n));
  c->cand.ensure(sizeof(uint32_t) * (1u << 20));
  if (c->emit_ctr.ensure(2 * sizeof(uint32_t)))  // the emit kernel leaves its counters zero
    ck(cudaMemsetAsync(c->emit_ctr.p, 0, 2 * sizeof(uint32_t), c->stream), "memset");
  {
    Phase ph(c, REFSIG_PHASE_PAIR_EMIT);
    // the total also goes straight to h_pin[0] (mapped) from the scan: no readback node after the
    // emission (the host reads it only after synchronising the stream, i.e. after the emission too)
    launch_exclusive_scan_u32_to_u64(c->rowcnt.as<uint32_t>(), c->rowstart.as<uint64_t>(), n, c->scan_tmp.p,
                                     c->stream, reinterpret_cast<uint64_t*>(c->d_pin));
    launch_emit_pairs(c->bitmap.as<uint32_t>(), g, c->rowcnt.as<uint32_t>(), c->rowstart.as<uint64_t>(),
                      c->cand.as<uint32_t>(), c->cand.cap / sizeof(uint32_t), c->emit_ctr.as<uint32_t>(), c->stream);
    launched("emit");
  }
  c->emit_pending = true;
  c->have_pairs = false;
  c->keys_valid = false;
  c->emit_grid = g;
}

// Wait for the enqueued emission; if ctx->cand was too small, grow it and
// emit again (the bitmap is still valid); optionally copy to the caller.
int finish_emit(refsig_gpu_ctx* c, uint64_t* out, uint64_t capacity, uint64_t* out_count) {
  require(c->emit_pending, "no pair computation in flight");
  sync(c);
  c->emit_pending = false;
  const PairGrid& g = c->emit_grid;
  const uint64_t total = c->h_pin[0];
  if (total > c->cand.cap / sizeof(uint32_t)) {
    c->cand.ensure(sizeof(uint32_t) * (total + total / 4 + 1024));
    Phase ph(c, REFSIG_PHASE_PAIR_EMIT);
    launch_emit_pairs(c->bitmap.as<uint32_t>(), g, c->rowcnt.as<uint32_t>(), c->rowstart.as<uint64_t>(),
                      c->cand.as<uint32_t>(), c->cand.cap / sizeof(uint32_t), c->emit_ctr.as<uint32_t>(), c->stream);
    launched("emit");
  }
  c->cand_count = total;
  c->have_pairs = true;
  *out_count = total;
  if (out && capacity) {
    const uint64_t m = std::min(total, capacity);
    materialize_keys(c);
    Phase ph(c, REFSIG_PHASE_D2H);
    if (m) ck(cudaMemcpyAsync(out, c->keys.p, m * 8, cudaMemcpyDeviceToHost, c->stream), "D2H pairs");
  }
  sync(c);
  if (total > capacity && out) {
    c->err = "candidate buffer overflow: " + std::to_string(total) + " pairs > capacity " + std::to_string(capacity);
    return REFSIG_E_OVERFLOW;
  }
  return REFSIG_OK;
}

int run_emit(refsig_gpu_ctx* c, const PairGrid& g, uint64_t* out, uint64_t capacity, uint64_t* out_count) {
  enqueue_emit(c, g);
  return finish_emit(c, out, capacity, out_count);
}

// zero_rowcnt = false: the caller's first kernel zeroes the row counts (run_mrc_tiles)
void prepare_bitmap(refsig_gpu_ctx* c, const PairGrid& g, bool zero, bool zero_rowcnt = true) {
  c->bitmap.ensure(sizeof(uint32_t) * static_cast<size_t>(g.n_rows) * g.words_per_row);
  c->rowcnt.ensure(sizeof(uint32_t) * (g.n_rows ? g.n_rows : 1));
  if (zero_rowcnt) ck(cudaMemsetAsync(c->rowcnt.p, 0, sizeof(uint32_t) * g.n_rows, c->stream), "memset rowcnt");
  if (zero)
    ck(cudaMemsetAsync(c->bitmap.p, 0, sizeof(uint32_t) * static_cast<size_t>(g.n_rows) * g.words_per_row,
                       c->stream),
       "memset bitmap");
}

// K3: the tcgen05 kernel when K fits (3K+3 <= 128), else the CUDA-core tiles.
// REFSIG_K3=fp32 forces the CUDA-core kernel.
bool k3_use_tc(const refsig_gpu_ctx* c, uint32_t K, float tau) {
  static const bool off = [] {
    const char* m = std::getenv("REFSIG_K3");
    return m && std::strcmp(m, "fp32") == 0;
  }();
  if (c->k3_path == REFSIG_K3_FP32) return false;
  if (c->k3_path == REFSIG_K3_TENSOR) {
    require(mrc_tc_supported(K, tau), "tensor-core K3 needs K <= 234 and |tau| = 0 or >= 2^-14");
    return true;
  }
  return !off && mrc_tc_supported(K, tau);
}

void run_mrc_tiles(refsig_gpu_ctx* c, const float* STr, uint32_t ldr, uint32_t nr, const float* STc, uint32_t ldc,
                   uint32_t ncl, bool self, uint32_t K, float tau, const PairGrid& g) {
  // (prepare_bitmap left the row counts to this function: zeroed by the forms kernel on the tcgen05 path)
  if (!k3_use_tc(c, K, tau)) {
    ck(cudaMemsetAsync(c->rowcnt.p, 0, sizeof(uint32_t) * g.n_rows, c->stream), "memset rowcnt");
    launch_mrc_bitmap(STr, ldr, STc, ldc, K, tau, g, c->bitmap.as<uint32_t>(), c->rowcnt.as<uint32_t>(), c->stream);
    return;
  }
  const size_t rb = mrc_tc_form_bytes(K, nr), cb = mrc_tc_form_bytes(K, ncl);
  char* rowf;
  char* colf;
  if (self) {
    c->tc_forms.ensure(rb + cb);
    rowf = c->tc_forms.as<char>();
    colf = rowf + rb;
    const bool pair = mrc_tc2_applies(K, g);  // CTA-pair kernel: column forms in 64-document panels
    launch_mrc_tc_forms(STr, ldr, nr, K, tau, rowf, colf, c->rowcnt.as<uint32_t>(), g.n_rows, c->stream, pair);
    if (pair) {
      launched("tcgen05 operand forms");
      if (!launch_mrc_tc2(rowf, colf, K, g, c->bitmap.as<uint32_t>(), c->rowcnt.as<uint32_t>(), c->stream))
        fail(REFSIG_E_RUNTIME, "CTA-pair K3: TMA descriptor (cuTensorMapEncodeTiled) failed");
      return;
    }
  } else {
    // query join: the database's column forms do not depend on tau and stay
    // valid until it is signed again, so they are built once per database
    refsig_gpu_ctx* db = c->db;
    c->tc_forms.ensure(rb);
    rowf = c->tc_forms.as<char>();
    launch_mrc_tc_forms(STr, ldr, nr, K, tau, rowf, nullptr, c->rowcnt.as<uint32_t>(), g.n_rows, c->stream);
    static const bool no_cache = std::getenv("REFSIG_NO_FORM_CACHE") != nullptr;
    const bool pair = mrc_tc2_applies(K, g);  // CTA-pair kernel: column forms in 64-document panels
    if (no_cache || db->tc_colf_gen != db->sign_gen || db->tc_colf.cap < cb || db->tc_colf_col64 != pair) {
      db->tc_colf.ensure(cb);
      launch_mrc_tc_forms(STc, ldc, ncl, K, tau, nullptr, db->tc_colf.p, nullptr, 0, c->stream, pair);
      db->tc_colf_gen = db->sign_gen;
      db->tc_colf_col64 = pair;
    }
    colf = db->tc_colf.as<char>();
    launched("tcgen05 operand forms");
    if (pair) {
      if (!launch_mrc_tc2(rowf, colf, K, g, c->bitmap.as<uint32_t>(), c->rowcnt.as<uint32_t>(), c->stream))
        fail(REFSIG_E_RUNTIME, "CTA-pair K3: TMA descriptor (cuTensorMapEncodeTiled) failed");
      return;
    }
  }
  launched("tcgen05 operand forms");
  launch_mrc_tc(rowf, colf, K, g, c->bitmap.as<uint32_t>(), c->rowcnt.as<uint32_t>(), c->stream);
}

// A5: union, remap and the compact table from c->ref_{start,n} and `ent`.
void build_reference(refsig_gpu_ctx* c, const RefArgs& r, uint64_t n_entries) {
  const uint32_t V = c->vocab;
  // rows: one per reference entry (A5's canonical row of a term is its first entry's)
  const uint64_t u_cap = std::min<uint64_t>(n_entries, static_cast<uint64_t>(V) * r.K);
  // K2 addresses R rows by 32-bit element offsets (row * Kp)
  require(u_cap * r.Kp < (1ull << 32), "reference term union too large (|U| * K >= 2^32)");
  const size_t rbytes = sizeof(float) * std::max<uint64_t>(u_cap, 1) * r.Kp;
  c->R.ensure(rbytes);
  // [barrier arrivals, finished CTAs, |U|, |U| partial sums]; the kernel leaves [0], [1], [3] zero
  if (c->ref_count.ensure(4 * sizeof(uint32_t)))
    ck(cudaMemsetAsync(c->ref_count.p, 0, 4 * sizeof(uint32_t), c->stream), "memset");
  Phase ph(c, REFSIG_PHASE_REFERENCE);
  // info[].ref_row is -1 right after count(); a replaced reference resets it
  if (c->ref_dirty) launch_ref_reset(c->info.as<TermInfo>(), V, c->stream);
  launch_ref_build(r, c->info.as<TermInfo>(), V, c->ref_count.as<uint32_t>(), c->R.as<float>(), n_entries,
                   c->stream);
  launched("reference");
  c->K = r.K;
  c->Kp = r.Kp;
  c->have_ref = true;
  c->ref_dirty = true;
  c->signed_ = false;
}

void ensure_unit_weights(refsig_gpu_ctx* c) {
  if (c->have_x) return;
  c->inv_norm.ensure(sizeof(float) * c->n_docs);
  launch_inv_norm(c->ent.as<uint2>(), c->doc_off.as<uint64_t>(), c->nnz.as<uint32_t>(), c->info.as<TermInfo>(),
                  c->n_docs, c->inv_norm.as<float>(), c->stream);
  c->x.ensure(sizeof(float) * std::max<uint64_t>(c->n_tokens, 1));
  launch_unit_weights(c->ent.as<uint2>(), c->doc_off.as<uint64_t>(), c->nnz.as<uint32_t>(), c->info.as<TermInfo>(),
                      c->inv_norm.as<float>(), c->n_docs, c->x.as<float>(), c->stream);
  launched("unit weights");
  c->have_x = true;
  c->have_inv_norm = true;
}

struct HostProf {  // REFSIG_HOST_PROF=1: host time of load_common's sections (stderr)
  const char* name;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  static bool on() {
    static const bool v = std::getenv("REFSIG_HOST_PROF") != nullptr;
    return v;
  }
  void lap(const char* what) {
    if (!on()) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "%s %s %.1f us\n", name, what, std::chrono::duration<double, std::micro>(t - t0).count());
    t0 = t;
  }
};

static_assert(kMaxRefs <= kParamWords, "reference ids travel as kernel parameters");

void validate_doc_off(const uint64_t* doc_off, uint32_t n_docs, uint32_t vocab) {
  require(doc_off != nullptr, "doc_off is NULL");
  require(n_docs >= 1, "empty corpus");
  require(vocab >= 1 && vocab < 0x7fffffffu, "vocab out of range");
  require(doc_off[0] == 0, "doc_off[0] must be 0");
}

// Validate doc_off and build the plan into the pinned buffer *h (grown as
// needed; the caller guarantees no copy still reads it).
void plan_build(const uint64_t* doc_off, uint32_t n_docs, uint32_t vocab, PlanInfo& pi, uint32_t*& h, size_t& h_cap,
                HostProf& hp) {
  uint64_t max_len = 0;
  for (uint32_t d = 0; d < n_docs; ++d) {
    require(doc_off[d + 1] >= doc_off[d], "doc_off must be non-decreasing");
    max_len = std::max<uint64_t>(max_len, doc_off[d + 1] - doc_off[d]);
  }
  require(max_len < (1ull << 31), "document longer than 2^31 tokens");
  hp.lap("validate");
  pi = PlanInfo{};
  pi.n_docs = n_docs;
  pi.vocab = vocab;
  pi.n_tokens = doc_off[n_docs];
  // Work plan: documents in decreasing length (counting sort on the length
  // for the usual corpora, a key sort otherwise; ties by id), then split by
  // work class, each list keeping that order (longest first = fewest tails).
  std::vector<uint32_t> order(n_docs);
  auto len = [&](uint32_t d) { return doc_off[d + 1] - doc_off[d]; };
  if (max_len <= (1u << 20)) {
    std::vector<uint32_t> cnt(max_len + 2, 0);
    for (uint32_t d = 0; d < n_docs; ++d) ++cnt[max_len - len(d) + 1];
    for (size_t i = 1; i < cnt.size(); ++i) cnt[i] += cnt[i - 1];
    for (uint32_t d = 0; d < n_docs; ++d) order[cnt[max_len - len(d)]++] = d;
  } else {
    std::vector<uint64_t> key(n_docs);
    for (uint32_t d = 0; d < n_docs; ++d) key[d] = ((max_len - len(d)) << 32) | d;
    std::sort(key.begin(), key.end());
    for (uint32_t d = 0; d < n_docs; ++d) order[d] = static_cast<uint32_t>(key[d]);
  }
  hp.lap("order");
  uint32_t n_class[refsig_gpu_ctx::kPlanLists] = {};
  // work class by ceil(log2(length)): <= 64 tiny, 128 / 256 / 512 warp sorts, 1024..8192 the
  // group classes (kGroupCap), longer the global path — one table lookup per document
  static_assert(kTinyMax == 64 && kGroupCap[0] == 1024 && kGroupCap[3] == 8192 && kGroupMax == 8192,
                "class table below assumes these bounds");
  static constexpr uint8_t kClassOfLog[15] = {
      refsig_gpu_ctx::kPlanTiny, refsig_gpu_ctx::kPlanTiny, refsig_gpu_ctx::kPlanTiny, refsig_gpu_ctx::kPlanTiny,
      refsig_gpu_ctx::kPlanTiny, refsig_gpu_ctx::kPlanTiny, refsig_gpu_ctx::kPlanTiny, refsig_gpu_ctx::kPlanW4,
      refsig_gpu_ctx::kPlanW8,   refsig_gpu_ctx::kPlanW16,  refsig_gpu_ctx::kPlanG0,   refsig_gpu_ctx::kPlanG0 + 1,
      refsig_gpu_ctx::kPlanG0 + 2, refsig_gpu_ctx::kPlanG0 + 3, refsig_gpu_ctx::kPlanLong};
  auto cls_of = [](uint64_t l) -> int {
    const int b = l <= 1 ? 0 : 64 - __builtin_clzll(l - 1);  // ceil(log2(l))
    return kClassOfLog[b < 14 ? b : 14];
  };
  std::vector<uint8_t> cls(n_docs);
  for (uint32_t d = 0; d < n_docs; ++d) {
    cls[d] = static_cast<uint8_t>(cls_of(doc_off[d + 1] - doc_off[d]));
    ++n_class[cls[d]];
  }
  n_class[refsig_gpu_ctx::kPlanOrder] = n_docs;
  uint32_t off = 0;
  for (int k = 0; k < refsig_gpu_ctx::kPlanLists; ++k) {
    pi.plan_off[k] = off;
    pi.plan_n[k] = n_class[k];
    off += n_class[k];
  }
  pi.off_bytes = sizeof(uint64_t) * (n_docs + 1);
  pi.list_bytes = sizeof(uint32_t) * std::max(off, 1u);
  pi.loff_at = (pi.off_bytes + pi.list_bytes + 7) & ~size_t{7};
  pi.bytes = pi.loff_at + sizeof(uint64_t) * n_class[refsig_gpu_ctx::kPlanLong];
  hp.lap("classes");
  if (pi.bytes > h_cap) {
    if (h) cudaFreeHost(h);
    h = nullptr;
    h_cap = 0;
    ck(cudaMallocHost(reinterpret_cast<void**>(&h), pi.bytes), "cudaMallocHost");
    h_cap = pi.bytes;
  }
  std::memcpy(h, doc_off, pi.off_bytes);
  uint32_t* lists = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(h) + pi.off_bytes);
  uint32_t fill[refsig_gpu_ctx::kPlanLists];
  for (int k = 0; k < refsig_gpu_ctx::kPlanLists; ++k) fill[k] = pi.plan_off[k];
  uint64_t* loff = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(h) + pi.loff_at);
  for (uint32_t i = 0; i < n_docs; ++i) {
    const uint32_t d = order[i];
    lists[fill[refsig_gpu_ctx::kPlanOrder]++] = d;
    const int k = cls[d];
    lists[fill[k]++] = d;
    if (k == refsig_gpu_ctx::kPlanLong) {
      loff[pi.n_loff++] = pi.scratch;
      uint64_t p = 1;
      while (p < len(d)) p <<= 1;
      pi.scratch += p;
    }
  }
  while (pi.n_sign_long < n_docs && len(order[pi.n_sign_long]) > kSignLongTokens) ++pi.n_sign_long;
  pi.n_sign_half = pi.n_sign_long;
  while (pi.n_sign_half < n_docs && len(order[pi.n_sign_half]) > kSignHalfTokens) ++pi.n_sign_half;
  hp.lap("lists");
}

// The plan's three device copies on stream s (ordered after earlier work on s
// that may still read the destinations).
void plan_copy(const PlanInfo& pi, const uint32_t* h, DevBuf& doc_off_dst, DevBuf& plan_dst, DevBuf& long_off_dst,
               cudaStream_t s) {
  doc_off_dst.ensure(pi.off_bytes);
  plan_dst.ensure(pi.list_bytes);
  ck(cudaMemcpyAsync(doc_off_dst.p, h, pi.off_bytes, cudaMemcpyHostToDevice, s), "H2D doc_off");
  ck(cudaMemcpyAsync(plan_dst.p, reinterpret_cast<const char*>(h) + pi.off_bytes, pi.list_bytes,
                     cudaMemcpyHostToDevice, s),
     "H2D plan");
  if (pi.n_loff) {
    long_off_dst.ensure(8ull * pi.n_loff);
    ck(cudaMemcpyAsync(long_off_dst.p, reinterpret_cast<const char*>(h) + pi.loff_at, 8ull * pi.n_loff,
                       cudaMemcpyHostToDevice, s),
       "H2D long offsets");
  }
}

// Make the plan the context's current one (host fields and state).
void plan_apply(refsig_gpu_ctx* c, const PlanInfo& pi, const uint64_t* doc_off) {
  c->h_off.assign(doc_off, doc_off + pi.n_docs + 1);
  c->have_text = false;  // refsig_gpu_load_text sets it after this
  c->n_docs = pi.n_docs;
  c->vocab = pi.vocab;
  c->n_tokens = pi.n_tokens;
  std::memcpy(c->plan_off, pi.plan_off, sizeof(pi.plan_off));
  std::memcpy(c->plan_n, pi.plan_n, sizeof(pi.plan_n));
  c->n_sign_long = pi.n_sign_long;
  c->n_sign_half = pi.n_sign_half;
  // (a reallocation here frees the old buffer: cudaFree waits for the device)
  if (pi.n_loff) c->long_scratch.ensure(sizeof(uint32_t) * pi.scratch);
  c->loaded = true;
  c->counted = false;
  c->plan_tok = c->tok;
  ++c->load_gen;
  reset_downstream(c);
}

void load_common(refsig_gpu_ctx* c, const uint64_t* doc_off, uint32_t n_docs, uint32_t vocab) {
  HostProf hp{"load_common"};
  validate_doc_off(doc_off, n_docs, vocab);
  // Same document layout as the loaded corpus (a new batch of the same shape,
  // or the same batch re-uploaded): the work plan is a function of doc_off
  // only, so it and the device copy of doc_off stay valid, and so does a
  // captured step graph (it reads the token buffer, which was just rewritten).
  if (c->loaded && c->plan_tok == c->tok && n_docs == c->n_docs && vocab == c->vocab &&
      c->h_off.size() == static_cast<size_t>(n_docs) + 1 &&
      std::memcmp(c->h_off.data(), doc_off, sizeof(uint64_t) * (n_docs + 1)) == 0) {
    c->have_text = false;
    c->counted = false;
    reset_downstream(c);
    return;
  }
  if (!c->plan_done) ck(cudaEventCreateWithFlags(&c->plan_done, cudaEventDisableTiming), "event");
  ck(cudaEventSynchronize(c->plan_done), "plan staging");  // the previous copy consumed h_plan
  hp.lap("plan_done sync");
  PlanInfo pi;
  plan_build(doc_off, n_docs, vocab, pi, c->h_plan, c->h_plan_cap, hp);
  // ordered on ctx->stream after earlier work that may still read the previous plan (K1's side
  // streams fork from and join back into ctx->stream)
  plan_copy(pi, c->h_plan, c->doc_off, c->plan, c->long_off, c->stream);
  ck(cudaEventRecord(c->plan_done, c->stream), "event");  // h_plan consumed
  hp.lap("copies");
  plan_apply(c, pi, doc_off);
}

// R row stride: K <= 32 -> roundup(K,4) (float4 rows, lane-per-hit K2);
// K > 32 -> roundup(K,32) (column-owner K2 reads lane-indexed columns).
uint32_t ref_row_stride(uint32_t K) { return K <= 32 ? (K + 3) & ~3u : (K + 31) & ~31u; }

PairGrid self_grid(const refsig_gpu_ctx* c) {
  return PairGrid{c->n_docs, c->n_docs, words_per_row(c->n_docs), true, 0, c->n_docs, 0};
}

}  // namespace

// Column panel of the K5 tail accumulator: kExactPanel docs of shared memory;
// REFSIG_EXACT_PANEL (a multiple of 4) forces smaller panels (tests: the
// multi-panel walk on a small corpus).
static uint32_t exact_panel(uint32_t N) {
  static const uint32_t env = [] {
    const char* m = std::getenv("REFSIG_EXACT_PANEL");
    return m ? static_cast<uint32_t>(std::atoi(m)) : 0u;
  }();
  const uint32_t p = env ? std::max<uint32_t>(4u, env & ~3u) : kExactPanel;
  return std::min<uint32_t>(N, std::min<uint32_t>(p, kExactPanel));
}

// K5 inputs (exact verifier and evaluation): unit weights, the kExactHead
// highest-df terms as dense rows + norms, and the tail postings. Returns H.
uint32_t prepare_exact(refsig_gpu_ctx* ctx) {
  const uint32_t N = ctx->n_docs, V = ctx->vocab;
  require(ctx->n_tokens < (1ull << 32), "exact verifier: more than 2^32 postings");  // 32-bit posting offsets
  ensure_unit_weights(ctx);
  // head terms: the kExactHead highest df (ties by id), selected on the device
  const uint32_t H = std::min<uint32_t>(kExactHead, (V + 3) & ~3u);
  const uint64_t T = std::max<uint64_t>(ctx->n_tokens, 1);
  const uint64_t W = std::max<uint64_t>(T, V);  // sort scratch: slots or terms
  ctx->csc_ka.ensure(4ull * W);
  ctx->csc_kb.ensure(4ull * W);
  ctx->csc_va.ensure(4ull * W);
  ctx->csc_vb.ensure(4ull * W);
  ctx->csc_tmp.ensure(std::max(csc_sort_temp_bytes(ctx->n_tokens, V), head_select_temp_bytes(V)));
  ctx->head_col.ensure(4ull * V);
  launch_head_select(ctx->df.as<uint32_t>(), V, H, ctx->csc_ka.as<uint32_t>(), ctx->csc_kb.as<uint32_t>(),
                     ctx->csc_va.as<uint32_t>(), ctx->csc_vb.as<uint32_t>(), ctx->csc_tmp.p, ctx->csc_tmp.cap,
                     ctx->head_col.as<int32_t>(), ctx->stream);
  // dense head rows + their norms
  ctx->headA.ensure(sizeof(float) * static_cast<size_t>(N) * H);
  ctx->head_norm.ensure(sizeof(float) * N);
  ck(cudaMemsetAsync(ctx->headA.p, 0, sizeof(float) * static_cast<size_t>(N) * H, ctx->stream), "memset A");
  launch_head_rows(ctx->ent.as<uint2>(), ctx->doc_off.as<uint64_t>(), ctx->nnz.as<uint32_t>(), ctx->x.as<float>(),
                   ctx->head_col.as<int32_t>(), N, H, ctx->headA.as<float>(), ctx->head_norm.as<float>(),
                   ctx->stream);
  // doc-sorted postings of every term: offsets = exclusive scan of df, lists by a stable radix sort by term
  ctx->post_off.ensure(8ull * (V + 1));
  ctx->posts.ensure(sizeof(uint2) * T);
  ctx->entpos.ensure(4ull * T);
  ctx->csc_doc.ensure(4ull * T);
  ctx->scan_tmp.ensure(scan_tmp_bytes(std::max(N, V)));
  launch_exclusive_scan_u32_to_u64(ctx->df.as<uint32_t>(), ctx->post_off.as<uint64_t>(), V, ctx->scan_tmp.p,
                                   ctx->stream);
  build_csc_postings(ctx->ent.as<uint2>(), ctx->doc_off.as<uint64_t>(), ctx->nnz.as<uint32_t>(), N, V, ctx->n_tokens,
                     ctx->x.as<float>(), ctx->csc_ka.as<uint32_t>(), ctx->csc_kb.as<uint32_t>(),
                     ctx->csc_va.as<uint32_t>(), ctx->csc_vb.as<uint32_t>(), ctx->csc_doc.as<uint32_t>(),
                     ctx->csc_tmp.p, ctx->csc_tmp.cap, ctx->posts.as<uint2>(), ctx->entpos.as<uint32_t>(), ctx->stream);
  return H;
}

extern "C" {

const char* refsig_gpu_version(void) { return "refsig-b200 0.1 (sm_100a)"; }

int refsig_gpu_create(int device, refsig_gpu_ctx** out) {
  if (!out) return REFSIG_E_VALIDATION;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return REFSIG_E_RUNTIME;
  }
  if (device < 0 || device >= n) return REFSIG_E_VALIDATION;
  refsig_gpu_ctx* c = new (std::nothrow) refsig_gpu_ctx();
  if (!c) return REFSIG_E_RUNTIME;
  c->device = device;
  bool ok = cudaSetDevice(device) == cudaSuccess &&
            cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaHostAlloc(&c->h_pin, 64, cudaHostAllocMapped) == cudaSuccess &&
            cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->d_pin), c->h_pin, 0) == cudaSuccess &&
            cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) == cudaSuccess;
  for (int k = 0; ok && k < 3; ++k)
    ok = cudaStreamCreateWithFlags(&c->side[k], cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&c->ev_join[k], cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    delete c;
    return REFSIG_E_RUNTIME;
  }
  c->stream = c->own_stream;
  *out = c;
  return REFSIG_OK;
}

void refsig_gpu_destroy(refsig_gpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (int k = 0; k < 3; ++k) {
    if (ctx->side[k]) {
      cudaStreamSynchronize(ctx->side[k]);
      cudaStreamDestroy(ctx->side[k]);
    }
    if (ctx->ev_join[k]) cudaEventDestroy(ctx->ev_join[k]);
  }
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->plan_stream) {
    cudaStreamSynchronize(ctx->plan_stream);
    cudaStreamDestroy(ctx->plan_stream);
  }
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  if (ctx->d2h_stream) {
    cudaStreamSynchronize(ctx->d2h_stream);
    cudaStreamDestroy(ctx->d2h_stream);
  }
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  if (ctx->h_pin) cudaFreeHost(ctx->h_pin);
  delete ctx;
}

const char* refsig_gpu_last_error(const refsig_gpu_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int refsig_gpu_set_stream(refsig_gpu_ctx* ctx, void* s) {
  return guard(ctx, [&] {
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
  });
}

void* refsig_gpu_get_stream(const refsig_gpu_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

int refsig_gpu_synchronize(refsig_gpu_ctx* ctx) {
  return guard(ctx, [&] { sync(ctx); });
}

int refsig_gpu_load_corpus(refsig_gpu_ctx* ctx, const uint32_t* tokens, const uint64_t* doc_off, uint32_t n_docs,
                           uint32_t vocab) {
  return guard(ctx, [&] {
    require(doc_off != nullptr, "doc_off is NULL");
    require(n_docs >= 1, "empty corpus");
    require(tokens != nullptr || doc_off[n_docs] == 0, "tokens is NULL");
    const uint64_t T = doc_off[n_docs];
    ctx->tokens.ensure(sizeof(uint32_t) * std::max<uint64_t>(T, 1));
    if (T) {
      Phase ph(ctx, REFSIG_PHASE_H2D);
      ck(cudaMemcpyAsync(ctx->tokens.p, tokens, sizeof(uint32_t) * T, cudaMemcpyHostToDevice, ctx->stream),
         "H2D tokens");
    }
    ctx->tok = ctx->tokens.as<uint32_t>();
    load_common(ctx, doc_off, n_docs, vocab);
  });
}

int refsig_gpu_load_corpus_device(refsig_gpu_ctx* ctx, const uint32_t* d_tokens, const uint64_t* doc_off,
                                  uint32_t n_docs, uint32_t vocab) {
  return guard(ctx, [&] {
    require(doc_off != nullptr, "doc_off is NULL");
    require(n_docs >= 1, "empty corpus");
    require(d_tokens != nullptr || doc_off[n_docs] == 0, "tokens is NULL");
    ctx->tok = d_tokens;
    load_common(ctx, doc_off, n_docs, vocab);
  });
}

int refsig_gpu_stage_corpus(refsig_gpu_ctx* ctx, const uint32_t* tokens, const uint64_t* doc_off, uint32_t n_docs,
                            uint32_t vocab) {
  return guard(ctx, [&] {
    validate_doc_off(doc_off, n_docs, vocab);
    const uint64_t T = doc_off[n_docs];
    require(tokens != nullptr || T == 0, "tokens is NULL");
    require(ctx->stg_count < refsig_gpu_ctx::kStageDepth,
            "two staged corpora are waiting for refsig_gpu_swap_corpus");
    if (!ctx->copy_stream) {
      ck(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "copy stream");
      ck(cudaStreamCreateWithFlags(&ctx->plan_stream, cudaStreamNonBlocking), "plan stream");
    }
    auto& g = ctx->stg[(ctx->stg_head + ctx->stg_count) % refsig_gpu_ctx::kStageDepth];
    if (!g.ev_ready) {
      ck(cudaEventCreateWithFlags(&g.ev_ready, cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&g.ev_plan, cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&g.ev_free, cudaEventDisableTiming), "event");
    }
    HostProf hp{"stage_corpus"};
    const int hk = ctx->hplan_next;
    ctx->hplan_next = (hk + 1) % refsig_gpu_ctx::kPlanRing;
    if (!ctx->ev_hplan[hk]) ck(cudaEventCreateWithFlags(&ctx->ev_hplan[hk], cudaEventDisableTiming), "event");
    if (ctx->hplan_recorded[hk]) ck(cudaEventSynchronize(ctx->ev_hplan[hk]), "staged plan copies");
    hp.lap("plan ring sync");
    plan_build(doc_off, n_docs, vocab, g.pi, ctx->h_plans[hk], ctx->h_plans_cap[hk], hp);
    // the slot's device buffers may still be read by work enqueued before they were swapped out
    if (g.free_recorded) {
      ck(cudaStreamWaitEvent(ctx->copy_stream, g.ev_free, 0), "wait");
      ck(cudaStreamWaitEvent(ctx->plan_stream, g.ev_free, 0), "wait");
    }
    // the small plan copies on their own stream: they run beside the previous batch's token
    // upload instead of delaying the next one (a small copy next to a large D2H takes ~60 us)
    plan_copy(g.pi, ctx->h_plans[hk], g.doc_off, g.plan, g.long_off, ctx->plan_stream);
    ck(cudaEventRecord(g.ev_plan, ctx->plan_stream), "event");
    ck(cudaEventRecord(ctx->ev_hplan[hk], ctx->plan_stream), "event");
    ctx->hplan_recorded[hk] = true;
    hp.lap("plan copies");
    g.tokens.ensure(sizeof(uint32_t) * std::max<uint64_t>(T, 1));
    if (T)
      ck(cudaMemcpyAsync(g.tokens.p, tokens, sizeof(uint32_t) * T, cudaMemcpyHostToDevice, ctx->copy_stream),
         "H2D staged tokens");
    ck(cudaEventRecord(g.ev_ready, ctx->copy_stream), "event");
    hp.lap("token copy");
    g.off.assign(doc_off, doc_off + n_docs + 1);
    ++ctx->stg_count;
  });
}

static void swap_buf(DevBuf& a, DevBuf& b) {
  std::swap(a.p, b.p);
  std::swap(a.cap, b.cap);
}

int refsig_gpu_swap_corpus(refsig_gpu_ctx* ctx) {
  return guard(ctx, [&] {
    require(ctx->stg_count > 0, "no staged corpus (refsig_gpu_stage_corpus)");
    auto& g = ctx->stg[ctx->stg_head];
    // compute waits for the slot's copies on the device, not the host
    ck(cudaStreamWaitEvent(ctx->stream, g.ev_plan, 0), "wait staged plan");
    ck(cudaStreamWaitEvent(ctx->stream, g.ev_ready, 0), "wait staged");
    swap_buf(ctx->tokens, g.tokens);
    swap_buf(ctx->doc_off, g.doc_off);
    swap_buf(ctx->plan, g.plan);
    swap_buf(ctx->long_off, g.long_off);
    // the previous batch's buffers now sit in the slot: free once the work
    // already enqueued on the compute stream is done with them
    ck(cudaEventRecord(g.ev_free, ctx->stream), "event");
    g.free_recorded = true;
    ctx->stg_head = (ctx->stg_head + 1) % refsig_gpu_ctx::kStageDepth;
    --ctx->stg_count;
    ctx->tok = ctx->tokens.as<uint32_t>();
    g_alloc_gen.fetch_add(1);  // captured step graphs read the old buffers
    plan_apply(ctx, g.pi, g.off.data());
  });
}

static void do_count(refsig_gpu_ctx* ctx, int weight_mode) {
  require(ctx->loaded, "no corpus loaded");
  require(weight_mode == REFSIG_WEIGHT_TF || weight_mode == REFSIG_WEIGHT_TFIDF, "bad weight mode");
  refsig_gpu_ctx* db = ctx->db;
  if (db) {
    require(db->counted, "attached database not counted");
    require(db->vocab == ctx->vocab, "query vocab differs from database vocab");
  }
  const uint32_t N = ctx->n_docs, V = ctx->vocab;
  ctx->ent.ensure(sizeof(uint2) * std::max<uint64_t>(ctx->n_tokens, 1));
  ctx->nnz.ensure(sizeof(uint32_t) * N);
  ctx->df.ensure(sizeof(uint32_t) * V);
  ctx->info.ensure(sizeof(TermInfo) * V);
  if (ctx->flags.ensure(16)) ck(cudaMemsetAsync(ctx->flags.p, 0, 16, ctx->stream), "memset");
  Phase ph(ctx, REFSIG_PHASE_COUNT);
  // df replicas (k1_count.cu df_replica): Zipf-head terms are in nearly every document, so one
  // array would serialise their atomics; R copies divide that contention. REFSIG_DF_REPS overrides
  // (measurement).
  static const uint32_t reps_env = [] {
    const char* m = std::getenv("REFSIG_DF_REPS");
    return m ? static_cast<uint32_t>(std::atoi(m)) : 0u;
  }();
  // ~32 MB of replicas, 1..32 copies: 32 at configs[1] (measured: 1 copy 283 us, 2: 165, 4: 113, 16: 98,
  // 32: 95.5, 64: 97 us for K1), 16 at configs[3], 8 at configs[4]
  const uint32_t reps = reps_env ? reps_env : std::max<uint32_t>(1u, std::min<uint32_t>(32u, (8u << 20) / V));
  // zeroed right before K1 (measured: zeroing them in the idf kernel of the previous count
  // instead left the lines cold in L2 — K1's atomics then missed, count 90 -> 125 us)
  ctx->df_rep.ensure(sizeof(uint32_t) * static_cast<size_t>(V) * reps);
  ck(cudaMemsetAsync(ctx->df_rep.p, 0, sizeof(uint32_t) * static_cast<size_t>(V) * reps, ctx->stream), "memset df");
  CountArgs a{ctx->tok, ctx->doc_off.as<uint64_t>(), V, ctx->ent.as<uint2>(), ctx->nnz.as<uint32_t>(),
              ctx->df_rep.as<uint32_t>(), reps, ctx->flags.as<uint32_t>()};
  // fork: the two longest group classes on side[1] / side[2] (one CTA per
  // doc: latency-bound, so they start first), the other two and the 512-key
  // warp sorts on the main stream, tiny / 256-key / > 8192-token docs on
  // side[0]; joined before the idf kernel.
  using P = refsig_gpu_ctx;
  cudaStream_t m0 = ctx->stream;
  ck(cudaEventRecord(ctx->ev_fork, m0), "fork");
  for (int k = 0; k < 3; ++k) ck(cudaStreamWaitEvent(ctx->side[k], ctx->ev_fork, 0), "fork");
  launch_count_group(3, a, ctx->plan_list(P::kPlanG3), ctx->plan_n[P::kPlanG3], ctx->side[1]);
  launch_count_group(2, a, ctx->plan_list(P::kPlanG2), ctx->plan_n[P::kPlanG2], ctx->side[2]);
  launch_count_group(1, a, ctx->plan_list(P::kPlanG1), ctx->plan_n[P::kPlanG1], m0);
  launch_count_group(0, a, ctx->plan_list(P::kPlanG0), ctx->plan_n[P::kPlanG0], m0);
  launch_count_group(-1, a, ctx->plan_list(P::kPlanW16), ctx->plan_n[P::kPlanW16], ctx->side[1]);
#ifdef REFSIG_K1_WARP_BIG_FIRST
  launch_count_warp(8, a, ctx->plan_list(P::kPlanW8), ctx->plan_n[P::kPlanW8], ctx->side[0]);
  launch_count_warp(4, a, ctx->plan_list(P::kPlanW4), ctx->plan_n[P::kPlanW4], ctx->side[0]);
  launch_count_warp(2, a, ctx->plan_list(P::kPlanTiny), ctx->plan_n[P::kPlanTiny], ctx->side[0]);
#else
  launch_count_warp(2, a, ctx->plan_list(P::kPlanTiny), ctx->plan_n[P::kPlanTiny], ctx->side[0]);
  launch_count_warp(4, a, ctx->plan_list(P::kPlanW4), ctx->plan_n[P::kPlanW4], ctx->side[0]);
  launch_count_warp(8, a, ctx->plan_list(P::kPlanW8), ctx->plan_n[P::kPlanW8], ctx->side[0]);
#endif
  launch_count_large(a, ctx->plan_list(P::kPlanLong), ctx->long_off.as<uint64_t>(), ctx->plan_n[P::kPlanLong],
                     ctx->long_scratch.as<uint32_t>(), ctx->side[0]);
  for (int k = 0; k < 3; ++k) {  // join
    ck(cudaEventRecord(ctx->ev_join[k], ctx->side[k]), "join");
    ck(cudaStreamWaitEvent(m0, ctx->ev_join[k], 0), "join");
  }
  launch_idf(ctx->df_rep.as<uint32_t>(), reps, V, N, weight_mode, ctx->df.as<uint32_t>(), ctx->info.as<TermInfo>(),
             ctx->stream);
  ctx->ref_dirty = false;  // idf_kernel resets info[].ref_row
  ctx->weight_mode = weight_mode;
  if (db) {
    // Query mode: the database's IDF and reference rows (configs[4]); the
    // query batch keeps its own df.
    ck(cudaStreamSynchronize(db->stream), "sync database");
    launch_copy_words(db->info.as<uint32_t>(), 2ull * V, ctx->info.as<uint32_t>(), ctx->stream);  // TermInfo = 2 words
    ctx->weight_mode = db->weight_mode;
  }
  launched("count");
  ctx->counted = true;
  reset_downstream(ctx);
}

int refsig_gpu_count(refsig_gpu_ctx* ctx, int weight_mode) {
  return guard(ctx, [&] { do_count(ctx, weight_mode); });
}

int refsig_gpu_get_counts(refsig_gpu_ctx* ctx, uint64_t* rowptr, uint32_t* ids, uint32_t* counts, uint64_t cap,
                          uint64_t* nnz_out) {
  int overflow = 0;
  int rc = guard(ctx, [&] {
    require(ctx->counted, "count() not called");
    require(rowptr && nnz_out, "NULL output");
    require(cap == 0 || (ids && counts), "NULL output");
    const uint32_t N = ctx->n_docs;
    ctx->rowptr.ensure(sizeof(uint64_t) * (N + 1));
    ctx->scan_tmp.ensure(scan_tmp_bytes(N));
    launch_exclusive_scan_u32_to_u64(ctx->nnz.as<uint32_t>(), ctx->rowptr.as<uint64_t>(), N, ctx->scan_tmp.p,
                                     ctx->stream);
    ck(cudaMemcpyAsync(rowptr, ctx->rowptr.p, sizeof(uint64_t) * (N + 1), cudaMemcpyDeviceToHost, ctx->stream),
       "D2H rowptr");
    sync(ctx);
    const uint64_t total = rowptr[N];
    *nnz_out = total;
    if (total > cap) {
      overflow = 1;
      return;
    }
    ctx->c_ids.ensure(sizeof(uint32_t) * std::max<uint64_t>(total, 1));
    ctx->c_counts.ensure(sizeof(uint32_t) * std::max<uint64_t>(total, 1));
    launch_compact_csr(ctx->ent.as<uint2>(), ctx->doc_off.as<uint64_t>(), ctx->nnz.as<uint32_t>(),
                       ctx->rowptr.as<uint64_t>(), N, ctx->c_ids.as<uint32_t>(), ctx->c_counts.as<uint32_t>(),
                       ctx->stream);
    launched("compact");
    if (total) {
      ck(cudaMemcpyAsync(ids, ctx->c_ids.p, 4 * total, cudaMemcpyDeviceToHost, ctx->stream), "D2H ids");
      ck(cudaMemcpyAsync(counts, ctx->c_counts.p, 4 * total, cudaMemcpyDeviceToHost, ctx->stream), "D2H counts");
    }
    sync(ctx);
  });
  if (rc == REFSIG_OK && overflow) {
    ctx->err = "counts buffer overflow";
    return REFSIG_E_OVERFLOW;
  }
  return rc;
}

int refsig_gpu_get_df(refsig_gpu_ctx* ctx, uint32_t* df, float* idf32) {
  return guard(ctx, [&] {
    require(ctx->counted, "count() not called");
    const uint32_t V = ctx->vocab;
    std::vector<TermInfo> info;
    if (df) ck(cudaMemcpyAsync(df, ctx->df.p, 4ull * V, cudaMemcpyDeviceToHost, ctx->stream), "D2H df");
    if (idf32) {
      info.resize(V);
      ck(cudaMemcpyAsync(info.data(), ctx->info.p, sizeof(TermInfo) * V, cudaMemcpyDeviceToHost, ctx->stream),
         "D2H idf");
    }
    sync(ctx);
    if (idf32)
      for (uint32_t t = 0; t < V; ++t) idf32[t] = info[t].idf;
  });
}

int refsig_gpu_get_corpus_freq(refsig_gpu_ctx* ctx, uint64_t* cf) {
  return guard(ctx, [&] {
    require(ctx->counted, "count() not called");
    require(cf != nullptr, "NULL output");
    const uint32_t V = ctx->vocab;
    const uint32_t reps = std::max<uint32_t>(1u, std::min<uint32_t>(8u, (1u << 20) / V));
    ctx->cf_rep.ensure(sizeof(unsigned long long) * static_cast<size_t>(reps) * V);
    ctx->cf.ensure(sizeof(uint64_t) * V);
    launch_corpus_freq(ctx->ent.as<uint2>(), ctx->doc_off.as<uint64_t>(), ctx->nnz.as<uint32_t>(), ctx->n_docs, V, reps,
                       ctx->cf_rep.as<unsigned long long>(), ctx->cf.as<uint64_t>(), ctx->stream);
    ck(cudaMemcpyAsync(cf, ctx->cf.p, 8ull * V, cudaMemcpyDeviceToHost, ctx->stream), "D2H cf");
    sync(ctx);
  });
}

int refsig_gpu_get_inv_norm(refsig_gpu_ctx* ctx, float* inv_norm) {
  return guard(ctx, [&] {
    require(ctx->counted, "count() not called");
    require(inv_norm != nullptr, "NULL output");
    ctx->inv_norm.ensure(sizeof(float) * ctx->n_docs);
    launch_inv_norm(ctx->ent.as<uint2>(), ctx->doc_off.as<uint64_t>(), ctx->nnz.as<uint32_t>(),
                    ctx->info.as<TermInfo>(), ctx->n_docs, ctx->inv_norm.as<float>(), ctx->stream);
    launched("inv_norm");
    ck(cudaMemcpyAsync(inv_norm, ctx->inv_norm.p, 4ull * ctx->n_docs, cudaMemcpyDeviceToHost, ctx->stream),
       "D2H inv_norm");
    sync(ctx);
  });
}

// Validate the reference doc ids and upload them (returns the |U| bound: their token counts).
static uint64_t stage_reference_docs(refsig_gpu_ctx* ctx, const uint32_t* ref_doc_ids, uint32_t K) {
  require(ctx->loaded, "no corpus loaded");
  require(!ctx->db, "query context uses the attached database's reference");
  require(ref_doc_ids != nullptr, "ref_doc_ids is NULL");
  require(K >= 1 && K <= kMaxRefs, "K must be in 1..256");
  uint64_t u_cap = 0;
  for (uint32_t k = 0; k < K; ++k) {
    require(ref_doc_ids[k] < ctx->n_docs, "reference doc id >= n_docs");
    u_cap += ctx->h_off[ref_doc_ids[k] + 1] - ctx->h_off[ref_doc_ids[k]];
  }
  ctx->ref_ids.assign(ref_doc_ids, ref_doc_ids + K);  // kernel parameters of the reference build
  return u_cap;
}

static void build_reference_docs(refsig_gpu_ctx* ctx, uint32_t K, uint64_t u_cap) {
  require(ctx->counted, "count() not called");
  RefArgs r{K, nullptr, nullptr, ctx->ent.as<uint2>(), false, ref_row_stride(K), ctx->doc_off.as<uint64_t>(),
            ctx->nnz.as<uint32_t>(), {}};
  std::copy(ctx->ref_ids.begin(), ctx->ref_ids.end(), r.ids);
  build_reference(ctx, r, u_cap);
}

static void do_set_reference_docs(refsig_gpu_ctx* ctx, const uint32_t* ref_doc_ids, uint32_t K) {
  require(ctx->counted, "count() not called");
  build_reference_docs(ctx, K, stage_reference_docs(ctx, ref_doc_ids, K));
}

int refsig_gpu_set_reference_docs(refsig_gpu_ctx* ctx, const uint32_t* ref_doc_ids, uint32_t K) {
  return guard(ctx, [&] { do_set_reference_docs(ctx, ref_doc_ids, K); });
}

// Explicit reference vectors: weights as given (explicit_w) or counts weighted
// on the device with this context's idf (count * idf, like reference docs).
static void do_set_reference_table(refsig_gpu_ctx* ctx, uint32_t K, const uint64_t* rowptr, const uint32_t* term_ids,
                                   const float* weights, bool from_counts, const uint32_t* counts) {
  require(ctx->counted, "count() not called");
  require(!ctx->db, "query context uses the attached database's reference");
  require(K >= 1 && K <= kMaxRefs, "K must be in 1..256");
  require(rowptr != nullptr, "rowptr is NULL");
  require(rowptr[0] == 0, "rowptr[0] must be 0");
  for (uint32_t k = 0; k < K; ++k) require(rowptr[k + 1] >= rowptr[k], "rowptr must be non-decreasing");
  const uint64_t n = rowptr[K];
  require(n == 0 || term_ids != nullptr, "term_ids is NULL");
  require(!from_counts || n == 0 || counts != nullptr, "counts is NULL");
  std::vector<uint2> h(n);
  std::vector<uint64_t> start(K);
  std::vector<uint32_t> cnt(K);
  for (uint32_t k = 0; k < K; ++k) {
    start[k] = rowptr[k];
    cnt[k] = static_cast<uint32_t>(rowptr[k + 1] - rowptr[k]);
    std::vector<uint32_t> ids(term_ids + rowptr[k], term_ids + rowptr[k + 1]);
    std::sort(ids.begin(), ids.end());
    for (size_t i = 0; i < ids.size(); ++i) {
      require(ids[i] < ctx->vocab, "reference term id >= vocab");
      require(i == 0 || ids[i] != ids[i - 1], "duplicate term in a reference vector");
    }
    for (uint64_t p = rowptr[k]; p < rowptr[k + 1]; ++p) {
      uint32_t bits;
      if (from_counts) {
        bits = counts[p];
      } else {
        const float w = weights ? weights[p] : 1.0f;
        require(std::isfinite(w) && w >= 0.0f, "reference weights must be finite and >= 0");
        std::memcpy(&bits, &w, 4);
      }
      h[p] = make_uint2(term_ids[p], bits);
    }
  }
  ctx->ref_ent.ensure(sizeof(uint2) * std::max<uint64_t>(n, 1));
  ctx->ref_start.ensure(8ull * K);
  ctx->ref_n.ensure(4ull * K);
  if (n) ck(cudaMemcpyAsync(ctx->ref_ent.p, h.data(), sizeof(uint2) * n, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  ck(cudaMemcpyAsync(ctx->ref_start.p, start.data(), 8ull * K, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  ck(cudaMemcpyAsync(ctx->ref_n.p, cnt.data(), 4ull * K, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  RefArgs r{K, ctx->ref_start.as<uint64_t>(), ctx->ref_n.as<uint32_t>(), ctx->ref_ent.as<uint2>(), !from_counts,
            ref_row_stride(K), nullptr, nullptr, {}};
  build_reference(ctx, r, n);
  ck(cudaStreamSynchronize(ctx->stream), "reference");
}

int refsig_gpu_set_reference_vectors(refsig_gpu_ctx* ctx, uint32_t K, const uint64_t* rowptr, const uint32_t* term_ids,
                                     const float* weights) {
  return guard(ctx, [&] { do_set_reference_table(ctx, K, rowptr, term_ids, weights, false, nullptr); });
}

int refsig_gpu_set_reference_counts(refsig_gpu_ctx* ctx, uint32_t K, const uint64_t* rowptr, const uint32_t* term_ids,
                                    const uint32_t* counts) {
  return guard(ctx, [&] { do_set_reference_table(ctx, K, rowptr, term_ids, nullptr, true, counts); });
}

int refsig_gpu_set_global_df(refsig_gpu_ctx* ctx, const uint32_t* df_global, uint32_t n_docs_global) {
  return guard(ctx, [&] {
    require(ctx->counted, "count() not called");
    require(!ctx->db, "query contexts use the attached database's idf");
    require(n_docs_global >= ctx->n_docs, "n_docs_global is smaller than this shard");
    if (df_global)
      ck(cudaMemcpyAsync(ctx->df.p, df_global, 4ull * ctx->vocab, cudaMemcpyHostToDevice, ctx->stream), "H2D df");
    launch_idf_from_df(ctx->df.as<uint32_t>(), ctx->vocab, n_docs_global, ctx->weight_mode, ctx->info.as<TermInfo>(),
                       ctx->stream);
    launched("global idf");
    ctx->ref_dirty = false;  // idf_from_df resets info[].ref_row
    reset_downstream(ctx);
    sync(ctx);
  });
}

int refsig_gpu_set_signatures(refsig_gpu_ctx* ctx, uint32_t n_docs, uint32_t K, const float* S, int on_device) {
  return guard(ctx, [&] {
    require(K >= 1 && K <= kMaxRefs, "K must be in 1..256");
    require(S != nullptr || n_docs == 0, "S is NULL");
    require(!ctx->emit_pending, "pair computation in flight");
    const uint32_t ld = static_cast<uint32_t>(ceil_div(n_docs, kTile) * kTile);
    ctx->S.ensure(sizeof(float) * static_cast<size_t>(n_docs) * K);
    ctx->ST.ensure(sizeof(float) * static_cast<size_t>(std::max<uint32_t>(ld, 1)) * K);
    if (n_docs)
      ck(cudaMemcpyAsync(ctx->S.p, S, sizeof(float) * static_cast<size_t>(n_docs) * K,
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ctx->stream),
         "copy signatures");
    if (ld > n_docs)
      ck(cudaMemset2DAsync(ctx->ST.as<float>() + n_docs, sizeof(float) * ld, 0, sizeof(float) * (ld - n_docs), K,
                           ctx->stream),
         "memset ST pad");
    launch_st_from_s(ctx->S.as<float>(), n_docs, K, ld, ctx->ST.as<float>(), ctx->stream);
    launched("signatures");
    reset_downstream(ctx);
    ctx->n_docs = n_docs;
    ctx->K = K;
    ctx->ld = ld;
    ctx->signed_ = true;
    ++ctx->sign_gen;
    ctx->counted = ctx->loaded = false;  // a pairs-only context until the next load
    sync(ctx);
  });
}

int refsig_gpu_reference_union(refsig_gpu_ctx* ctx, uint32_t* out_u) {
  return guard(ctx, [&] {
    require(ctx->have_ref, "no reference set");
    require(out_u != nullptr, "NULL output");
    ck(cudaMemcpyAsync(ctx->h_pin, ctx->ref_count.as<uint32_t>() + 2, 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    sync(ctx);
    *out_u = static_cast<uint32_t>(ctx->h_pin[0] & 0xffffffffu);
  });
}

static void do_sign(refsig_gpu_ctx* ctx) {
  require(ctx->counted, "count() not called");
  const refsig_gpu_ctx* refc = ctx->db ? ctx->db : ctx;
  require(refc->have_ref, "no reference set");
  const uint32_t N = ctx->n_docs, K = refc->K;
  ctx->S.ensure(sizeof(float) * static_cast<size_t>(N) * K);
  const uint32_t ld = static_cast<uint32_t>(ceil_div(N, kTile) * kTile);
  ctx->ST.ensure(sizeof(float) * static_cast<size_t>(ld) * K);
  ctx->ld = ld;  // (the sign kernel zeroes the pad columns [N, ld) of ST)
  ctx->inv_norm.ensure(sizeof(float) * N);
  if (ctx->db) ck(cudaStreamSynchronize(ctx->db->stream), "sync database");
  SignArgs a{ctx->ent.as<uint2>(), ctx->doc_off.as<uint64_t>(), ctx->nnz.as<uint32_t>(), ctx->info.as<TermInfo>(),
             refc->R.as<float>(), N, K, refc->Kp, ctx->plan_list(refsig_gpu_ctx::kPlanOrder), ctx->n_sign_long,
             ctx->n_sign_half,
             ctx->S.as<float>(), ctx->ST.as<float>(), ld, ctx->inv_norm.as<float>()};
  {
    Phase ph(ctx, REFSIG_PHASE_SIGN);
    launch_sign(a, ctx->stream);
    launched("sign");
  }
  ctx->K = K;
  ctx->signed_ = true;
  ctx->have_inv_norm = true;
  ++ctx->sign_gen;
}

int refsig_gpu_sign(refsig_gpu_ctx* ctx) {
  return guard(ctx, [&] { do_sign(ctx); });
}

int refsig_gpu_get_signatures(refsig_gpu_ctx* ctx, float* S) {
  return guard(ctx, [&] {
    require(ctx->signed_, "sign() not called");
    require(S != nullptr, "NULL output");
    ck(cudaMemcpyAsync(S, ctx->S.p, sizeof(float) * static_cast<size_t>(ctx->n_docs) * ctx->K,
                       cudaMemcpyDeviceToHost, ctx->stream),
       "D2H signatures");
    sync(ctx);
  });
}

int refsig_gpu_get_signature_records(refsig_gpu_ctx* ctx, uint64_t ref_id, uint8_t* out, uint64_t out_bytes) {
  return guard(ctx, [&] {
    require(ctx->signed_, "sign() not called");
    require(out != nullptr, "NULL output");
    const uint64_t bytes = static_cast<uint64_t>(ctx->n_docs) * (20ull + 8ull * ctx->K);
    require(out_bytes >= bytes, "output buffer smaller than n_docs * (20 + 8K) bytes");
    if (!bytes) return;
    ctx->records.ensure(bytes);
    launch_mrcs_records(ctx->S.as<float>(), ctx->n_docs, ctx->K, ref_id, ctx->records.as<uint32_t>(), ctx->stream);
    launched("mrcs records");
    ck(cudaMemcpyAsync(out, ctx->records.p, bytes, cudaMemcpyDeviceToHost, ctx->stream), "D2H records");
    sync(ctx);
  });
}

int refsig_gpu_mrc_pairs(refsig_gpu_ctx* ctx, float tau, uint64_t* out_pairs, uint64_t capacity,
                         uint64_t* out_count) {
  int rc2 = REFSIG_OK;
  int rc = guard(ctx, [&] {
    require(ctx->signed_, "sign() not called");
    require(out_count != nullptr, "out_count is NULL");
    require(!std::isnan(tau), "tau is NaN");
    require(capacity == 0 || out_pairs != nullptr, "out_pairs is NULL");
    const PairGrid g = self_grid(ctx);
    {
      Phase ph_tiles(ctx, REFSIG_PHASE_PAIR_TILES);
      prepare_bitmap(ctx, g, false, false);
      run_mrc_tiles(ctx, ctx->ST.as<float>(), ctx->ld, ctx->n_docs, ctx->ST.as<float>(), ctx->ld, ctx->n_docs, true,
                    ctx->K, tau, g);
      launched("mrc bitmap");
    }
    rc2 = run_emit(ctx, g, out_pairs, capacity, out_count);
  });
  return rc != REFSIG_OK ? rc : rc2;
}

int refsig_gpu_simhash(refsig_gpu_ctx* ctx, uint64_t seed, int weight_mode, const uint64_t* term_hash) {
  return guard(ctx, [&] {
    require(ctx->counted, "count() not called");
    require(weight_mode == REFSIG_WEIGHT_TF || weight_mode == REFSIG_WEIGHT_TFIDF, "bad weight mode");
    require(weight_mode == REFSIG_WEIGHT_TF || ctx->weight_mode == REFSIG_WEIGHT_TFIDF,
            "TF-IDF simhash needs count(REFSIG_WEIGHT_TFIDF)");
    const uint64_t* th = nullptr;
    if (term_hash) {
      ctx->term_hash.ensure(8ull * ctx->vocab);
      ck(cudaMemcpyAsync(ctx->term_hash.p, term_hash, 8ull * ctx->vocab, cudaMemcpyHostToDevice, ctx->stream),
         "H2D term hash");
      th = ctx->term_hash.as<uint64_t>();
    }
    ctx->fp.ensure(8ull * ctx->n_docs);
    SimhashArgs a{ctx->ent.as<uint2>(), ctx->doc_off.as<uint64_t>(), ctx->nnz.as<uint32_t>(), ctx->info.as<TermInfo>(),
                  th, seed, ctx->n_docs, weight_mode == REFSIG_WEIGHT_TFIDF, ctx->fp.as<uint64_t>(),
                  ctx->plan_list(refsig_gpu_ctx::kPlanOrder), ctx->n_sign_long};
    {
      Phase ph(ctx, REFSIG_PHASE_SIMHASH);
      launch_simhash(a, ctx->stream);
      launched("simhash");
    }
    if (term_hash) ck(cudaStreamSynchronize(ctx->stream), "simhash");
    ctx->have_fp = true;
  });
}

int refsig_gpu_load_text(refsig_gpu_ctx* ctx, const uint8_t* text, const uint64_t* byte_off, uint32_t n_docs) {
  return guard(ctx, [&] {
    require(byte_off != nullptr, "byte_off is NULL");
    require(n_docs >= 1, "empty corpus");
    require(byte_off[0] == 0, "byte_off[0] must be 0");
    for (uint32_t d = 0; d < n_docs; ++d) require(byte_off[d + 1] >= byte_off[d], "byte_off must be non-decreasing");
    const uint64_t B = byte_off[n_docs];
    require(text != nullptr || B == 0, "text is NULL");
    ctx->text.ensure(B + 16);  // padded: 32-bit loads may read up to 8 bytes past the end
    ck(cudaMemsetAsync(static_cast<uint8_t*>(ctx->text.p) + B, 0, 16, ctx->stream), "memset text pad");
    ctx->text_off.ensure(8ull * (n_docs + 1));
    ctx->text_cnt.ensure(4ull * n_docs);
    {
      Phase ph(ctx, REFSIG_PHASE_H2D);
      if (B) ck(cudaMemcpyAsync(ctx->text.p, text, B, cudaMemcpyHostToDevice, ctx->stream), "H2D text");
      ck(cudaMemcpyAsync(ctx->text_off.p, byte_off, 8ull * (n_docs + 1), cudaMemcpyHostToDevice, ctx->stream),
         "H2D text offsets");
    }
    // pass 1: 3-grams per doc -> host offsets (the K1 plan needs them)
    launch_text_grams(ctx->text.as<uint8_t>(), ctx->text_off.as<uint64_t>(), n_docs, nullptr,
                      ctx->text_cnt.as<uint32_t>(), nullptr, ctx->stream);
    std::vector<uint32_t> cnt(n_docs);
    ck(cudaMemcpyAsync(cnt.data(), ctx->text_cnt.p, 4ull * n_docs, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    sync(ctx);
    std::vector<uint64_t> goff(n_docs + 1, 0);
    for (uint32_t d = 0; d < n_docs; ++d) goff[d + 1] = goff[d] + cnt[d];
    ctx->tokens.ensure(sizeof(uint32_t) * std::max<uint64_t>(goff[n_docs], 1));
    ctx->tok = ctx->tokens.as<uint32_t>();
    load_common(ctx, goff.data(), n_docs, kGramSpace);  // uploads the gram offsets to ctx->doc_off
    // pass 2: the 3-gram ids in document order
    launch_text_grams(ctx->text.as<uint8_t>(), ctx->text_off.as<uint64_t>(), n_docs, ctx->doc_off.as<uint64_t>(),
                      nullptr, ctx->tokens.as<uint32_t>(), ctx->stream);
    launched("text grams");
    ctx->text_docs = n_docs;
    ctx->have_text = true;
  });
}

int refsig_gpu_simhash_text(refsig_gpu_ctx* ctx) {
  return guard(ctx, [&] {
    require(ctx->have_text && ctx->loaded && ctx->text_docs == ctx->n_docs, "load_text() not called");
    ctx->fp.ensure(8ull * ctx->n_docs);
    {
      Phase ph(ctx, REFSIG_PHASE_SIMHASH);
      launch_text_simhash(ctx->text.as<uint8_t>(), ctx->text_off.as<uint64_t>(), ctx->n_docs, ctx->fp.as<uint64_t>(),
                          ctx->stream);
      launched("text simhash");
    }
    ctx->have_fp = true;
  });
}

int refsig_gpu_get_fingerprints(refsig_gpu_ctx* ctx, uint64_t* fp) {
  return guard(ctx, [&] {
    require(ctx->have_fp, "simhash() not called");
    require(fp != nullptr, "NULL output");
    ck(cudaMemcpyAsync(fp, ctx->fp.p, 8ull * ctx->n_docs, cudaMemcpyDeviceToHost, ctx->stream), "D2H fp");
    sync(ctx);
  });
}

// Hamming tiles into ctx's bitmap / row counts: on the tensor cores (int8 +-1
// forms, kind::i8) unless REFSIG_HAMMING=cuda selects the POPC kernel.
static void hamming_tiles(refsig_gpu_ctx* c, const uint64_t* f_rows, uint32_t n_rows, const uint64_t* f_cols,
                          uint32_t n_cols, int max_dist, const PairGrid& g) {
  static const bool cuda_cores = [] {
    const char* m = std::getenv("REFSIG_HAMMING");
    return m && std::strcmp(m, "cuda") == 0;
  }();
  if (cuda_cores) {
    launch_hamming_bitmap(f_rows, f_cols, max_dist, g, c->bitmap.as<uint32_t>(), c->rowcnt.as<uint32_t>(), c->stream);
    return;
  }
  const size_t rb = ham_tc_form_bytes(n_rows), cb = ham_tc_form_bytes(n_cols);
  c->ham_forms.ensure(rb + cb);
  void* rowf = c->ham_forms.p;
  void* colf = c->ham_forms.as<char>() + rb;
  if (f_rows == f_cols) {  // self join: both forms in one pass (they differ in the threshold byte)
    launch_ham_tc_forms(f_rows, n_rows, max_dist, rowf, colf, c->stream);
  } else {
    launch_ham_tc_forms(f_rows, n_rows, max_dist, rowf, nullptr, c->stream);
    launch_ham_tc_forms(f_cols, n_cols, max_dist, nullptr, colf, c->stream);
  }
  launch_ham_tc(rowf, colf, g, c->bitmap.as<uint32_t>(), c->rowcnt.as<uint32_t>(), c->stream);
}

int refsig_gpu_hamming_pairs(refsig_gpu_ctx* ctx, int max_dist, uint64_t* out_pairs, uint64_t capacity,
                             uint64_t* out_count) {
  int rc2 = REFSIG_OK;
  int rc = guard(ctx, [&] {
    require(ctx->have_fp, "simhash() not called");
    require(out_count != nullptr, "out_count is NULL");
    require(max_dist >= 0 && max_dist <= 64, "max_dist must be in [0, 64]");
    require(capacity == 0 || out_pairs != nullptr, "out_pairs is NULL");
    const PairGrid g = self_grid(ctx);
    {
      Phase ph_tiles(ctx, REFSIG_PHASE_PAIR_TILES);
      prepare_bitmap(ctx, g, false);
      hamming_tiles(ctx, ctx->fp.as<uint64_t>(), ctx->n_docs, ctx->fp.as<uint64_t>(), ctx->n_docs, max_dist, g);
      launched("hamming bitmap");
    }
    rc2 = run_emit(ctx, g, out_pairs, capacity, out_count);
  });
  return rc != REFSIG_OK ? rc : rc2;
}

int refsig_gpu_exact_pairs(refsig_gpu_ctx* ctx, float tau_cos, uint64_t* out_pairs, uint64_t capacity,
                           uint64_t* out_count) {
  int rc2 = REFSIG_OK;
  int rc = guard(ctx, [&] {
    require(ctx->counted, "count() not called");
    require(out_count != nullptr, "out_count is NULL");
    require(tau_cos > 0.0f && tau_cos <= 1.0f, "tau_cos must be in (0, 1]");
    require(capacity == 0 || out_pairs != nullptr, "out_pairs is NULL");
    const uint32_t N = ctx->n_docs;
    const uint32_t H = prepare_exact(ctx);
    const PairGrid g = self_grid(ctx);
    {
      Phase ph_tiles(ctx, REFSIG_PHASE_PAIR_TILES);
      prepare_bitmap(ctx, g, true);
      ExactArgs a{ctx->ent.as<uint2>(),        ctx->doc_off.as<uint64_t>(), ctx->nnz.as<uint32_t>(),
                  ctx->x.as<float>(),          ctx->head_col.as<int32_t>(), ctx->post_off.as<uint64_t>(),
                  ctx->posts.as<uint2>(),      ctx->entpos.as<uint32_t>(),  ctx->headA.as<float>(),      ctx->head_norm.as<float>(),
                  H,                           N,                           exact_panel(N),
                  tau_cos,                     ctx->bitmap.as<uint32_t>(),  g.words_per_row,
                  ctx->rowcnt.as<uint32_t>(),  nullptr,                     0};
      launch_exact_tail(a, 0, N, ctx->stream);
      launched("exact");
    }
    rc2 = run_emit(ctx, g, out_pairs, capacity, out_count);
  });
  return rc != REFSIG_OK ? rc : rc2;
}

int refsig_gpu_evaluate(refsig_gpu_ctx* ctx, uint32_t row_lo, uint32_t row_hi, refsig_gpu_eval* out) {
  return guard(ctx, [&] {
    require(ctx->counted && ctx->signed_, "count() and sign() first");
    require(out != nullptr, "NULL output");
    const uint32_t N = ctx->n_docs;
    require(row_lo <= row_hi && row_hi <= N, "bad row range");
    require(row_lo % 128 == 0, "row_lo must be a multiple of 128");
    require(ctx->emit_pending == false, "pair computation in flight");
    const uint32_t H = prepare_exact(ctx);
    const uint32_t ld = ctx->ld;
    ctx->headAT.ensure(sizeof(float) * static_cast<size_t>(H) * ld);
    launch_transpose_head(ctx->headA.as<float>(), N, H, ld, ctx->headAT.as<float>(), ctx->stream);
    // the head and MRC dots on tcgen05 when the operands fit (every config: H = 64, K <= 128),
    // else the FP32 tiles; REFSIG_EVAL=fp32 forces the latter
    static const bool eval_fp32 = [] {
      const char* m = std::getenv("REFSIG_EVAL");
      return m && std::strcmp(m, "fp32") == 0;
    }();
    const bool tc = !eval_fp32 && eval_tc_supported(H, ctx->K);
    if (tc) {
      const size_t fb = eval_tc_form_bytes(H, ctx->K, N);
      ctx->tc_forms.ensure(2 * fb);
      launch_eval_tc_forms(ctx->headAT.as<float>(), H, ctx->ST.as<float>(), ctx->K, ld, N, ctx->tc_forms.p,
                           ctx->tc_forms.as<char>() + fb, ctx->stream);
      launched("evaluation forms");
    }
    // row panels (multiples of 128 rows) whose fixed-point tail sums fit ~2 GB
    uint64_t panel = std::max<uint64_t>(128, ((2ull << 30) / (4ull * ld)) / 128 * 128);
    const uint32_t grid = tc ? static_cast<uint32_t>(sm_count_host()) : eval_grid();
    ctx->eval_part.ensure(sizeof(double) * 8 * grid);
    std::vector<double> part(8 * grid);
    double sum[7] = {0, 0, 0, 0, 0, 0, 0};
    for (uint64_t p0 = row_lo; p0 < row_hi; p0 += panel) {
      const uint32_t p1 = static_cast<uint32_t>(std::min<uint64_t>(row_hi, p0 + panel));
      ctx->eval_tail.ensure(4ull * (p1 - p0) * ld);
      uint32_t used = grid;
      {
        Phase ph(ctx, REFSIG_PHASE_PAIR_TILES);
        ExactArgs a{ctx->ent.as<uint2>(),        ctx->doc_off.as<uint64_t>(), ctx->nnz.as<uint32_t>(),
                    ctx->x.as<float>(),          ctx->head_col.as<int32_t>(), ctx->post_off.as<uint64_t>(),
                    ctx->posts.as<uint2>(),      ctx->entpos.as<uint32_t>(),  ctx->headA.as<float>(),      ctx->head_norm.as<float>(),
                    H,                           N,                           exact_panel(N),
                    0.0f,                        nullptr,                     0,
                    nullptr,                     ctx->eval_tail.as<uint32_t>(), ld};
        launch_exact_tail(a, static_cast<uint32_t>(p0), p1, ctx->stream);
        const uint64_t* fp = ctx->have_fp ? ctx->fp.as<uint64_t>() : nullptr;
        if (tc) {
          const size_t fb = eval_tc_form_bytes(H, ctx->K, N);
          used = launch_eval_tc(ctx->tc_forms.p, ctx->tc_forms.as<char>() + fb, H, ctx->K, N,
                                static_cast<uint32_t>(p0), p1, ctx->eval_tail.as<uint32_t>(), ld, fp,
                                ctx->eval_part.as<double>(), ctx->stream);
        } else {
          EvalArgs e{ctx->headAT.as<float>(), H, ctx->ST.as<float>(), ctx->K, ld, fp, ctx->eval_tail.as<uint32_t>(),
                     N, static_cast<uint32_t>(p0), p1, ctx->eval_part.as<double>(), ld};
          launch_eval_tiles(e, ctx->stream);
        }
        launched("evaluate");
      }
      ck(cudaMemcpyAsync(part.data(), ctx->eval_part.p, sizeof(double) * 8 * used, cudaMemcpyDeviceToHost,
                         ctx->stream),
         "D2H eval");
      sync(ctx);
      for (uint32_t b = 0; b < used; ++b)  // CTA order: deterministic
        for (int q = 0; q < 7; ++q) sum[q] += part[8 * b + q];
    }
    const double n = sum[0];
    out->pairs = static_cast<uint64_t>(n);
    const double nan = std::nan("");
    auto fill = [&](double se, double sq, double sa, double* mae, double* me, double* var) {
      if (n <= 0) {
        *mae = *me = *var = nan;
        return;
      }
      *mae = sa / n;
      *me = se / n;
      *var = std::max(0.0, sq / n - (*me) * (*me));
    };
    fill(sum[1], sum[2], sum[3], &out->mrc_mae, &out->mrc_mean_error, &out->mrc_variance);
    if (ctx->have_fp)
      fill(sum[4], sum[5], sum[6], &out->simhash_mae, &out->simhash_mean_error, &out->simhash_variance);
    else
      out->simhash_mae = out->simhash_mean_error = out->simhash_variance = nan;
  });
}

int refsig_gpu_pair_cosines(refsig_gpu_ctx* ctx, const uint64_t* keys, uint64_t n, float* out) {
  return guard(ctx, [&] {
    require(ctx->counted, "count() not called");
    require(n == 0 || (keys && out), "NULL argument");
    for (uint64_t q = 0; q < n; ++q)
      require((keys[q] >> 32) < ctx->n_docs && (keys[q] & 0xffffffffu) < ctx->n_docs, "pair index >= n_docs");
    if (!n) return;
    ensure_unit_weights(ctx);
    DevBuf dk, dout;
    dk.ensure(8 * n);
    dout.ensure(4 * n);
    ck(cudaMemcpyAsync(dk.p, keys, 8 * n, cudaMemcpyHostToDevice, ctx->stream), "H2D keys");
    launch_pair_cosines(ctx->ent.as<uint2>(), ctx->doc_off.as<uint64_t>(), ctx->nnz.as<uint32_t>(), ctx->x.as<float>(),
                        dk.as<uint64_t>(), n, dout.as<float>(), ctx->stream);
    launched("pair cosines");
    ck(cudaMemcpyAsync(out, dout.p, 4 * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    sync(ctx);
  });
}

int refsig_gpu_attach_database(refsig_gpu_ctx* q, refsig_gpu_ctx* db) {
  return guard(q, [&] {
    require(db != nullptr && db != q, "bad database context");
    require(db->device == q->device, "database on another device");
    require(db->counted && db->have_ref, "database must be counted and have a reference");
    q->db = db;
    q->counted = false;
    reset_downstream(q);
  });
}

int refsig_gpu_mrc_query_pairs(refsig_gpu_ctx* q, float tau, uint64_t* out_pairs, uint64_t capacity,
                               uint64_t* out_count) {
  int rc2 = REFSIG_OK;
  int rc = guard(q, [&] {
    refsig_gpu_ctx* db = q->db;
    require(db != nullptr, "no database attached");
    require(q->signed_ && db->signed_, "sign() the queries and the database first");
    require(q->K == db->K, "queries and database signed with different references");
    require(out_count != nullptr, "out_count is NULL");
    require(!std::isnan(tau), "tau is NaN");
    require(capacity == 0 || out_pairs != nullptr, "out_pairs is NULL");
    ck(cudaStreamSynchronize(db->stream), "sync database");
    const PairGrid g{q->n_docs, db->n_docs, words_per_row(db->n_docs), false, 0, q->n_docs, 0};
    {
      Phase ph_tiles(q, REFSIG_PHASE_PAIR_TILES);
      prepare_bitmap(q, g, false, false);
      run_mrc_tiles(q, q->ST.as<float>(), q->ld, q->n_docs, db->ST.as<float>(), db->ld, db->n_docs, false, q->K, tau,
                    g);
      launched("mrc query bitmap");
    }
    rc2 = run_emit(q, g, out_pairs, capacity, out_count);
  });
  return rc != REFSIG_OK ? rc : rc2;
}

int refsig_gpu_hamming_query_pairs(refsig_gpu_ctx* q, int max_dist, uint64_t* out_pairs, uint64_t capacity,
                                   uint64_t* out_count) {
  int rc2 = REFSIG_OK;
  int rc = guard(q, [&] {
    refsig_gpu_ctx* db = q->db;
    require(db != nullptr, "no database attached");
    require(q->have_fp && db->have_fp, "simhash() the queries and the database first");
    require(out_count != nullptr, "out_count is NULL");
    require(max_dist >= 0 && max_dist <= 64, "max_dist must be in [0, 64]");
    require(capacity == 0 || out_pairs != nullptr, "out_pairs is NULL");
    ck(cudaStreamSynchronize(db->stream), "sync database");
    const PairGrid g{q->n_docs, db->n_docs, words_per_row(db->n_docs), false, 0, q->n_docs, 0};
    {
      Phase ph_tiles(q, REFSIG_PHASE_PAIR_TILES);
      prepare_bitmap(q, g, false);
      hamming_tiles(q, q->fp.as<uint64_t>(), q->n_docs, db->fp.as<uint64_t>(), db->n_docs, max_dist, g);
      launched("hamming query bitmap");
    }
    rc2 = run_emit(q, g, out_pairs, capacity, out_count);
  });
  return rc != REFSIG_OK ? rc : rc2;
}

int refsig_gpu_mrc_pairs_rows(refsig_gpu_ctx* ctx, float tau, uint32_t row_lo, uint32_t row_hi, uint64_t* out_pairs,
                              uint64_t capacity, uint64_t* out_count) {
  int rc2 = REFSIG_OK;
  int rc = guard(ctx, [&] {
    require(ctx->signed_, "sign() not called");
    require(out_count != nullptr, "out_count is NULL");
    require(!std::isnan(tau), "tau is NaN");
    require(capacity == 0 || out_pairs != nullptr, "out_pairs is NULL");
    require(row_lo <= row_hi && row_hi <= ctx->n_docs, "bad row range");
    require(row_lo == row_hi || (row_lo % kTile == 0 && (row_hi % kTile == 0 || row_hi == ctx->n_docs)),
            "row range must be aligned to 128-row tiles");
    PairGrid g = self_grid(ctx);
    g.row_begin = row_lo;
    g.row_end = row_hi;
    {
      Phase ph_tiles(ctx, REFSIG_PHASE_PAIR_TILES);
      prepare_bitmap(ctx, g, false, false);
      run_mrc_tiles(ctx, ctx->ST.as<float>(), ctx->ld, ctx->n_docs, ctx->ST.as<float>(), ctx->ld, ctx->n_docs, true,
                    ctx->K, tau, g);
      launched("mrc bitmap");
    }
    rc2 = run_emit(ctx, g, out_pairs, capacity, out_count);
  });
  return rc != REFSIG_OK ? rc : rc2;
}

// The hot path as one enqueue: count -> reference docs -> sign -> tiles ->
// scan -> emit (rows [lo, hi)), no host synchronisation.
static void enqueue_step(refsig_gpu_ctx* ctx, int weight_mode, const uint32_t* refs, uint32_t K, float tau,
                         uint32_t lo, uint32_t hi) {
  // the reference ids' H2D goes first, so that count's idf kernel -> reference build -> sign -> operand
  // forms -> tiles -> scan -> emission is a chain of programmatic-dependent launches with no copy or memset
  // node in between
  const uint64_t u_cap = stage_reference_docs(ctx, refs, K);
  do_count(ctx, weight_mode);
  build_reference_docs(ctx, K, u_cap);
  do_sign(ctx);
  PairGrid g = self_grid(ctx);
  g.row_begin = lo;
  g.row_end = hi;
  {
    Phase ph_tiles(ctx, REFSIG_PHASE_PAIR_TILES);
    prepare_bitmap(ctx, g, false, false);
    run_mrc_tiles(ctx, ctx->ST.as<float>(), ctx->ld, ctx->n_docs, ctx->ST.as<float>(), ctx->ld, ctx->n_docs, true,
                  ctx->K, tau, g);
    launched("mrc bitmap");
  }
  enqueue_emit(ctx, g);
}

int refsig_gpu_mrc_step(refsig_gpu_ctx* ctx, int weight_mode, const uint32_t* ref_doc_ids, uint32_t K, float tau,
                        uint32_t row_lo, uint32_t row_hi) {
  return guard(ctx, [&] {
    require(ctx->loaded, "no corpus loaded");
    require(!ctx->db, "query contexts use the attached database's reference");
    require(!ctx->emit_pending, "previous step not collected (refsig_gpu_step_result)");
    require(ref_doc_ids != nullptr && K >= 1 && K <= kMaxRefs, "reference docs required (K in 1..256)");
    require(!std::isnan(tau), "tau is NaN");
    require(row_lo <= row_hi && row_hi <= ctx->n_docs, "bad row range");
    require(row_lo == row_hi || (row_lo % kTile == 0 && (row_hi % kTile == 0 || row_hi == ctx->n_docs)),
            "row range must be aligned to 128-row tiles");
    refsig_gpu_ctx::StepKey key;
    key.load_gen = ctx->load_gen;
    key.weight_mode = weight_mode;
    key.refs.assign(ref_doc_ids, ref_doc_ids + K);
    key.tau = tau;
    key.lo = row_lo;
    key.hi = row_hi;
    key.stream = ctx->stream;
    key.alloc_gen = g_alloc_gen.load();
    if (ctx->step_exec && key == ctx->step_key) {
      // replay: every buffer and the candidate capacity are exactly as
      // captured; the reference ids are kernel parameters of the graph (the
      // key includes them)
      ck(cudaGraphLaunch(ctx->step_exec, ctx->stream), "cudaGraphLaunch");
      ctx->emit_pending = true;
      ctx->have_pairs = ctx->keys_valid = false;
      ctx->emit_grid = self_grid(ctx);
      ctx->emit_grid.row_begin = row_lo;
      ctx->emit_grid.row_end = row_hi;
      ctx->counted = ctx->have_ref = ctx->signed_ = true;
      ctx->have_fp = ctx->have_x = false;
      return;
    }
    // First run for this key: eager (sizes every buffer, results are valid),
    // then capture the same enqueue sequence for later calls.
    if (ctx->step_exec) {
      cudaGraphExecDestroy(ctx->step_exec);
      ctx->step_exec = nullptr;
    }
    enqueue_step(ctx, weight_mode, ref_doc_ids, K, tau, row_lo, row_hi);
    uint64_t total = 0;
    const int rc = finish_emit(ctx, nullptr, 0, &total);  // grows ctx->cand if needed
    (void)rc;
    const uint64_t keep_count = total;
    key.alloc_gen = g_alloc_gen.load();
    const bool prof = ctx->prof;
    ctx->prof = false;
    ctx->capturing = true;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) {
      try {
        enqueue_step(ctx, weight_mode, ref_doc_ids, K, tau, row_lo, row_hi);
      } catch (...) {
        cudaStreamEndCapture(ctx->stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        ctx->capturing = false;
        ctx->prof = prof;
        throw;
      }
      e = cudaStreamEndCapture(ctx->stream, &graph);
    }
    ctx->capturing = false;
    ctx->prof = prof;
    ck(e, "stream capture");
    e = cudaGraphInstantiate(&ctx->step_exec, graph, 0);
    cudaGraphDestroy(graph);
    ck(e, "cudaGraphInstantiate");
    ctx->step_key = key;
    if (key.alloc_gen != g_alloc_gen.load()) {  // capture allocated: do not trust the graph
      cudaGraphExecDestroy(ctx->step_exec);
      ctx->step_exec = nullptr;
    }
    // the eager results stand: report them through step_result
    ctx->h_pin[0] = keep_count;
    ctx->emit_pending = true;
    ctx->have_pairs = ctx->keys_valid = false;
    ctx->emit_grid = self_grid(ctx);
    ctx->emit_grid.row_begin = row_lo;
    ctx->emit_grid.row_end = row_hi;
  });
}

int refsig_gpu_step_result(refsig_gpu_ctx* ctx, uint64_t* out_pairs, uint64_t capacity, uint64_t* out_count) {
  int rc2 = REFSIG_OK;
  int rc = guard(ctx, [&] {
    require(out_count != nullptr, "out_count is NULL");
    require(capacity == 0 || out_pairs != nullptr, "out_pairs is NULL");
    rc2 = finish_emit(ctx, out_pairs, capacity, out_count);
  });
  return rc != REFSIG_OK ? rc : rc2;
}

int refsig_gpu_set_profiling(refsig_gpu_ctx* ctx, int on) {
  return guard(ctx, [&] {
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    for (auto& m : ctx->marks) {
      ctx->ev_free.push_back(m.a);
      ctx->ev_free.push_back(m.b);
    }
    ctx->marks.clear();
    ctx->prof = on != 0;
  });
}

int refsig_gpu_phase_times(refsig_gpu_ctx* ctx, double* ms, uint64_t* calls) {
  return guard(ctx, [&] {
    require(ms != nullptr, "NULL output");
    sync(ctx);
    for (int p = 0; p < REFSIG_N_PHASES; ++p) {
      ms[p] = 0.0;
      if (calls) calls[p] = 0;
    }
    for (auto& m : ctx->marks) {
      float t = 0.0f;
      ck(cudaEventElapsedTime(&t, m.a, m.b), "cudaEventElapsedTime");
      ms[m.phase] += t;
      if (calls) calls[m.phase] += 1;
    }
  });
}

uint64_t refsig_gpu_launch_count(void) { return g_launches.load(); }

int refsig_gpu_debug_check(refsig_gpu_ctx* ctx) {
  return guard(ctx, [&] {
    sync(ctx);
    ck(cudaDeviceSynchronize(), "device sync");
    std::string bad;
    for (auto& nb : ctx->buffers())
      if (!nb.second->canary_ok()) bad += std::string(bad.empty() ? "" : ", ") + nb.first;
    if (!bad.empty()) fail(REFSIG_E_RUNTIME, "write past the end of device buffer(s): " + bad);
  });
}

int refsig_gpu_set_k3_path(refsig_gpu_ctx* ctx, int path) {
  return guard(ctx, [&] {
    require(path == REFSIG_K3_AUTO || path == REFSIG_K3_FP32 || path == REFSIG_K3_TENSOR, "bad K3 path");
    if (path != ctx->k3_path && ctx->step_exec) {  // a captured step bakes in the path
      cudaGraphExecDestroy(ctx->step_exec);
      ctx->step_exec = nullptr;
    }
    ctx->k3_path = path;
  });
}

int refsig_gpu_get_pairs(refsig_gpu_ctx* ctx, uint64_t* out_pairs, uint64_t capacity) {
  return guard(ctx, [&] {
    require(capacity == 0 || out_pairs != nullptr, "out_pairs is NULL");
    const uint64_t m = std::min(capacity, ctx->cand_count);
    if (m) {
      require(ctx->have_pairs && !ctx->emit_pending, "no finished pair computation to fetch");
      materialize_keys(ctx);
      ck(cudaMemcpyAsync(out_pairs, ctx->keys.p, 8 * m, cudaMemcpyDeviceToHost, ctx->stream), "D2H pairs");
    }
    sync(ctx);
  });
}

int refsig_gpu_get_pairs_csr(refsig_gpu_ctx* ctx, uint32_t row_lo, uint32_t row_hi, uint64_t* rowptr, uint32_t* cols,
                             uint64_t capacity, uint64_t* out_count) {
  int rc2 = REFSIG_OK;
  int rc = guard(ctx, [&] {
    require(ctx->have_pairs && !ctx->emit_pending, "no finished pair computation to fetch");
    require(rowptr != nullptr && out_count != nullptr, "NULL output");
    require(capacity == 0 || cols != nullptr, "cols is NULL");
    const PairGrid& g = ctx->emit_grid;
    require(row_lo <= row_hi && row_hi <= g.n_rows, "bad row range");
    const uint64_t n_rows = row_hi - row_lo;
    ck(cudaMemcpyAsync(rowptr, ctx->rowstart.as<uint64_t>() + row_lo, 8 * (n_rows + 1), cudaMemcpyDeviceToHost,
                       ctx->stream),
       "D2H rowptr");
    sync(ctx);
    const uint64_t base = rowptr[0], total = rowptr[n_rows] - base;
    for (uint64_t r = 0; r <= n_rows; ++r) rowptr[r] -= base;
    *out_count = total;
    const uint64_t m = std::min(total, capacity);
    if (m) {
      Phase ph(ctx, REFSIG_PHASE_D2H);
      ck(cudaMemcpyAsync(cols, ctx->cand.as<uint32_t>() + base, 4 * m, cudaMemcpyDeviceToHost, ctx->stream),
         "D2H cols");
    }
    sync(ctx);
    if (total > capacity) {
      ctx->err = "candidate buffer overflow: " + std::to_string(total) + " pairs > capacity " + std::to_string(capacity);
      rc2 = REFSIG_E_OVERFLOW;
    }
  });
  return rc != REFSIG_OK ? rc : rc2;
}

int refsig_gpu_get_pairs_csr16(refsig_gpu_ctx* ctx, uint32_t row_lo, uint32_t row_hi, uint64_t* rowptr,
                               uint16_t* cols, uint64_t capacity, uint64_t* out_count) {
  int rc2 = REFSIG_OK;
  int rc = guard(ctx, [&] {
    require(ctx->have_pairs && !ctx->emit_pending, "no finished pair computation to fetch");
    require(rowptr != nullptr && out_count != nullptr, "NULL output");
    require(capacity == 0 || cols != nullptr, "cols is NULL");
    const PairGrid& g = ctx->emit_grid;
    require(g.n_cols <= 65536u, "16-bit columns need n_cols <= 65536 (use get_pairs_csr)");
    require(row_lo <= row_hi && row_hi <= g.n_rows, "bad row range");
    const uint64_t n_rows = row_hi - row_lo;
    ck(cudaMemcpyAsync(rowptr, ctx->rowstart.as<uint64_t>() + row_lo, 8 * (n_rows + 1), cudaMemcpyDeviceToHost,
                       ctx->stream),
       "D2H rowptr");
    sync(ctx);
    const uint64_t base = rowptr[0], total = rowptr[n_rows] - base;
    for (uint64_t r = 0; r <= n_rows; ++r) rowptr[r] -= base;
    *out_count = total;
    const uint64_t m = std::min(total, capacity);
    if (m) {
      ctx->cand16.ensure(2 * m + 16);
      launch_narrow_cols(ctx->cand.as<uint32_t>() + base, m, ctx->cand16.as<uint16_t>(), ctx->stream);
      launched("narrow");
      Phase ph(ctx, REFSIG_PHASE_D2H);
      ck(cudaMemcpyAsync(cols, ctx->cand16.p, 2 * m, cudaMemcpyDeviceToHost, ctx->stream), "D2H cols");
    }
    sync(ctx);
    if (total > capacity) {
      ctx->err = "candidate buffer overflow: " + std::to_string(total) + " pairs > capacity " + std::to_string(capacity);
      rc2 = REFSIG_E_OVERFLOW;
    }
  });
  return rc != REFSIG_OK ? rc : rc2;
}

int refsig_gpu_get_pairs_csr16_async(refsig_gpu_ctx* ctx, uint64_t* rowptr, uint16_t* cols, uint64_t capacity,
                                     uint64_t* out_count) {
  int rc2 = REFSIG_OK;
  int rc = guard(ctx, [&] {
    require(ctx->have_pairs && !ctx->emit_pending, "no finished pair computation to fetch");
    require(rowptr != nullptr && out_count != nullptr, "NULL output");
    require(capacity == 0 || cols != nullptr, "cols is NULL");
    const PairGrid& g = ctx->emit_grid;
    require(g.n_cols <= 65536u, "16-bit columns need n_cols <= 65536 (use get_pairs_csr)");
    if (!ctx->d2h_stream) {
      ck(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking), "d2h stream");
      ck(cudaEventCreateWithFlags(&ctx->ev_fetch_ready, cudaEventDisableTiming), "event");
      for (auto& e : ctx->ev_fetched) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    }
    const int slot = ctx->fetch_slot;
    ctx->fetch_slot ^= 1;
    // the slot's previous copy must have left its staging buffers
    if (ctx->fetch_pending[slot]) ck(cudaStreamWaitEvent(ctx->stream, ctx->ev_fetched[slot], 0), "wait fetch");
    const uint64_t n_rows = g.row_end - g.row_begin, total = ctx->cand_count;
    const uint64_t m = std::min(total, capacity);
    ctx->fetch_rowptr[slot].ensure(8 * (n_rows + 1));
    ctx->fetch_cols[slot].ensure(2 * m + 16);
    launch_rebase_rowptr(ctx->rowstart.as<uint64_t>() + g.row_begin, n_rows + 1, ctx->fetch_rowptr[slot].as<uint64_t>(),
                         ctx->stream);
    if (m) launch_narrow_cols(ctx->cand.as<uint32_t>(), m, ctx->fetch_cols[slot].as<uint16_t>(), ctx->stream);
    launched("fetch");
    ck(cudaEventRecord(ctx->ev_fetch_ready, ctx->stream), "event");
    ck(cudaStreamWaitEvent(ctx->d2h_stream, ctx->ev_fetch_ready, 0), "wait");
    ck(cudaMemcpyAsync(rowptr, ctx->fetch_rowptr[slot].p, 8 * (n_rows + 1), cudaMemcpyDeviceToHost, ctx->d2h_stream),
       "D2H rowptr");
    if (m) ck(cudaMemcpyAsync(cols, ctx->fetch_cols[slot].p, 2 * m, cudaMemcpyDeviceToHost, ctx->d2h_stream), "D2H cols");
    ck(cudaEventRecord(ctx->ev_fetched[slot], ctx->d2h_stream), "event");
    ctx->fetch_pending[slot] = true;
    *out_count = total;
    if (total > capacity) {
      ctx->err = "candidate buffer overflow: " + std::to_string(total) + " pairs > capacity " + std::to_string(capacity);
      rc2 = REFSIG_E_OVERFLOW;
    }
  });
  return rc != REFSIG_OK ? rc : rc2;
}

int refsig_gpu_wait_fetch(refsig_gpu_ctx* ctx) {
  return guard(ctx, [&] {
    for (int k = 0; k < 2; ++k)
      if (ctx->fetch_pending[k]) {
        ck(cudaEventSynchronize(ctx->ev_fetched[k]), "fetch");
        ctx->fetch_pending[k] = false;
      }
  });
}

int refsig_gpu_device_buffer(refsig_gpu_ctx* ctx, int which, void** ptr, uint64_t* bytes) {
  return guard(ctx, [&] {
    require(ptr && bytes, "NULL output");
    switch (which) {
      case REFSIG_BUF_PAIRS:
        require(ctx->have_pairs && !ctx->emit_pending, "no finished pair computation");
        materialize_keys(ctx);
        sync(ctx);
        *ptr = ctx->keys.p;
        *bytes = ctx->cand_count * 8;
        break;
      case REFSIG_BUF_SIGNATURES:
        require(ctx->signed_, "sign() not called");
        *ptr = ctx->S.p;
        *bytes = 4ull * ctx->n_docs * ctx->K;
        break;
      case REFSIG_BUF_DF:
        require(ctx->counted, "count() not called");
        *ptr = ctx->df.p;
        *bytes = 4ull * ctx->vocab;
        break;
      case REFSIG_BUF_FINGERPRINTS:
        require(ctx->have_fp, "simhash() not called");
        *ptr = ctx->fp.p;
        *bytes = 8ull * ctx->n_docs;
        break;
      default:
        fail(REFSIG_E_VALIDATION, "unknown buffer");
    }
  });
}

}  // extern "C"
