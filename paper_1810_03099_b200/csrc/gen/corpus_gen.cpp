// corpus_gen.cpp — deterministic synthetic corpora for BASELINE.json:configs[0..4].
//
// Input generation only (not the hot path, not the oracle). The reference's
// own corpus is NEWS20 read from disk (reference SPEC.md:183-250,
// PAPER.md:219); it is absent here, so these seeded generators stand in for it
// with the shapes BASELINE.json names. See include/mrcgen.h for the frozen
// definitions.

#include "mrcgen.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

enum Tag : uint64_t {
  kTagLen = 1,
  kTagTopic = 2,
  kTagTok = 3,
  kTagDupSel = 4,
  kTagDupSrc = 5,
  kTagResample = 6,
  kTagRef = 7,
  kTagTopicPerm = 8,
};

inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Rng {
  uint64_t s;
  uint64_t next() {
    s += kGamma;
    return mix64(s);
  }
  // uniform in [0,1) with 53 bits
  double u01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  // uniform in (0,1]
  double u01_open0() { return static_cast<double>((next() >> 11) + 1) * 0x1.0p-53; }
  // uniform integer in [0,n) (multiply-high; n < 2^32 here)
  uint64_t below(uint64_t n) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(next()) * n) >> 64);
  }
};

inline uint64_t stream_seed(uint64_t seed, uint64_t tag, uint64_t idx) {
  return mix64(seed ^ mix64(tag * kGamma + 0x632BE59BD9B4E019ull)) ^ mix64(idx + 0xD1B54A32D192ED03ull);
}

inline Rng stream(uint64_t seed, uint64_t tag, uint64_t idx) { return Rng{stream_seed(seed, tag, idx)}; }

// Vose alias table for Zipf(s) over ranks 0..V-1, weight (r+1)^-s.
struct Alias {
  std::vector<double> prob;
  std::vector<uint32_t> alias;
  uint32_t n = 0;
  void build(uint32_t v, double s) {
    n = v;
    std::vector<double> w(v);
    double total = 0.0;
    for (uint32_t r = 0; r < v; ++r) {
      w[r] = std::pow(static_cast<double>(r) + 1.0, -s);
      total += w[r];
    }
    prob.assign(v, 0.0);
    alias.assign(v, 0);
    std::vector<double> scaled(v);
    std::vector<uint32_t> small, large;
    small.reserve(v);
    large.reserve(v);
    for (uint32_t r = 0; r < v; ++r) {
      scaled[r] = w[r] * v / total;
      if (scaled[r] < 1.0)
        small.push_back(r);
      else
        large.push_back(r);
    }
    while (!small.empty() && !large.empty()) {
      uint32_t l = small.back();
      small.pop_back();
      uint32_t g = large.back();
      large.pop_back();
      prob[l] = scaled[l];
      alias[l] = g;
      scaled[g] = (scaled[g] + scaled[l]) - 1.0;
      if (scaled[g] < 1.0)
        small.push_back(g);
      else
        large.push_back(g);
    }
    for (uint32_t g : large) { prob[g] = 1.0; alias[g] = g; }
    for (uint32_t l : small) { prob[l] = 1.0; alias[l] = l; }
  }
  uint32_t sample(Rng& rng) const {
    uint32_t i = static_cast<uint32_t>(rng.below(n));
    return rng.u01() < prob[i] ? i : alias[i];
  }
};

struct TopicMap {
  uint64_t a, b;
};

struct Model {
  mrcgen_spec spec;
  Alias global, topic;
  std::vector<TopicMap> maps;
  bool has_topic_alias = false;
};

bool valid(const mrcgen_spec* s) {
  if (!s) return false;
  if (s->n_docs == 0 || s->vocab == 0) return false;
  if (s->len_min > s->len_max) return false;
  if (!(s->len_median > 0.0) || !(s->len_sigma >= 0.0)) return false;
  if (!(s->topic_mix >= 0.0 && s->topic_mix <= 1.0)) return false;
  if (!(s->dup_rate >= 0.0 && s->dup_rate < 1.0)) return false;
  if (!(s->resample_lo >= 0.0 && s->resample_hi <= 1.0 && s->resample_lo <= s->resample_hi)) return false;
  if (!(s->zipf_global > 0.0)) return false;
  if (s->n_topics > 0 && !(s->zipf_topic > 0.0)) return false;
  return true;
}

// Topic maps derive from the spec that owns the vocabulary (the DB in query mode).
std::vector<TopicMap> make_maps(const mrcgen_spec& s) {
  std::vector<TopicMap> m(s.n_topics);
  for (uint32_t c = 0; c < s.n_topics; ++c) {
    Rng r = stream(s.seed, kTagTopicPerm, c);
    uint64_t a;
    do {
      a = 1 + r.below(s.vocab > 1 ? s.vocab - 1 : 1);
    } while (std::gcd<uint64_t, uint64_t>(a, s.vocab) != 1);
    m[c] = TopicMap{a, r.below(s.vocab)};
  }
  return m;
}

// Shared alias tables are cached per (V, s): configs reuse them across calls.
std::mutex g_cache_mu;
std::unordered_map<std::string, std::shared_ptr<Alias>> g_cache;

std::shared_ptr<Alias> cached_alias(uint32_t v, double s) {
  std::string key = std::to_string(v) + ":" + std::to_string(s);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_cache.find(key);
  if (it != g_cache.end()) return it->second;
  auto a = std::make_shared<Alias>();
  a->build(v, s);
  g_cache[key] = a;
  return a;
}

uint32_t draw_len(const mrcgen_spec& s, uint64_t d) {
  Rng r = stream(s.seed, kTagLen, d);
  double u1 = r.u01_open0();
  double u2 = r.u01();
  double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  double x = std::exp(std::log(s.len_median) + s.len_sigma * z);
  long long L = std::llround(x);
  if (L < static_cast<long long>(s.len_min)) L = s.len_min;
  if (L > static_cast<long long>(s.len_max)) L = s.len_max;
  return static_cast<uint32_t>(L);
}

// Dup positions: first round(rate*n) entries of a partial Fisher-Yates.
// Sources: uniform over originals (rejection), or over an external DB.
void dup_plan(const mrcgen_spec& s, uint64_t n_src_pool, bool external_pool,
              std::vector<uint32_t>& dup_src) {
  const uint32_t n = s.n_docs;
  dup_src.assign(n, UINT32_MAX);
  uint64_t n_dup = static_cast<uint64_t>(std::llround(s.dup_rate * n));
  if (n_dup == 0) return;
  if (!external_pool && n_dup >= n) n_dup = n - 1;
  std::vector<uint32_t> perm(n);
  std::iota(perm.begin(), perm.end(), 0u);
  Rng r = stream(s.seed, kTagDupSel, 0);
  for (uint64_t i = 0; i < n_dup; ++i) {
    uint64_t j = i + r.below(n - i);
    std::swap(perm[i], perm[j]);
  }
  std::vector<uint8_t> is_dup(n, 0);
  for (uint64_t i = 0; i < n_dup; ++i) is_dup[perm[i]] = 1;
  Rng rs = stream(s.seed, kTagDupSrc, 0);
  // Assign sources in increasing dup-position order for determinism.
  std::vector<uint32_t> pos(perm.begin(), perm.begin() + n_dup);
  std::sort(pos.begin(), pos.end());
  for (uint32_t p : pos) {
    uint32_t src;
    if (external_pool) {
      src = static_cast<uint32_t>(rs.below(n_src_pool));
    } else {
      do {
        src = static_cast<uint32_t>(rs.below(n));
      } while (is_dup[src]);
    }
    dup_src[p] = src;
  }
}

inline uint32_t topic_of(const mrcgen_spec& s, uint64_t d) {
  if (s.n_topics == 0) return 0;
  Rng r = stream(s.seed, kTagTopic, d);
  return static_cast<uint32_t>(r.below(s.n_topics));
}

struct Sampler {
  const mrcgen_spec* s;
  const Alias* global;
  const Alias* topic;
  const std::vector<TopicMap>* maps;
  uint32_t draw(Rng& r, uint32_t topic_id) const {
    if (s->n_topics > 0) {
      double u = r.u01();
      if (u < s->topic_mix) {
        uint64_t rank = topic->sample(r);
        const TopicMap& m = (*maps)[topic_id];
        return static_cast<uint32_t>((m.a * rank + m.b) % s->vocab);
      }
    }
    return global->sample(r);
  }
};

template <class F>
void parallel_for(uint64_t n, int threads, F&& f) {
  int t = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  if (t < 1) t = 1;
  if (static_cast<uint64_t>(t) > n) t = static_cast<int>(n ? n : 1);
  if (t == 1) {
    for (uint64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  const uint64_t chunk = 64;
  std::atomic<uint64_t> next{0};
  for (int k = 0; k < t; ++k)
    th.emplace_back([&] {
      for (;;) {
        uint64_t b = next.fetch_add(chunk);
        if (b >= n) break;
        uint64_t e = std::min(n, b + chunk);
        for (uint64_t i = b; i < e; ++i) f(i);
      }
    });
  for (auto& x : th) x.join();
}

double resample_frac(const mrcgen_spec& s, Rng& r) {
  if (s.resample_hi <= s.resample_lo) return s.resample_lo;
  return s.resample_lo + (s.resample_hi - s.resample_lo) * r.u01();
}

}  // namespace

extern "C" {

uint64_t mrcgen_splitmix64_mix(uint64_t z) { return mix64(z); }
uint64_t mrcgen_stream_seed(uint64_t seed, uint64_t tag, uint64_t idx) { return stream_seed(seed, tag, idx); }

int mrcgen_offsets(const mrcgen_spec* spec, uint64_t* doc_off) {
  if (!valid(spec) || !doc_off) return 2;
  const mrcgen_spec& s = *spec;
  std::vector<uint32_t> dup_src;
  dup_plan(s, 0, false, dup_src);
  std::vector<uint32_t> len(s.n_docs);
  for (uint32_t d = 0; d < s.n_docs; ++d) len[d] = draw_len(s, d);
  doc_off[0] = 0;
  for (uint32_t d = 0; d < s.n_docs; ++d) {
    uint32_t L = dup_src[d] == UINT32_MAX ? len[d] : len[dup_src[d]];
    doc_off[d + 1] = doc_off[d] + L;
  }
  return 0;
}

int mrcgen_fill(const mrcgen_spec* spec, const uint64_t* doc_off, uint32_t* tokens, uint32_t* dup_src_out,
                int threads) {
  if (!valid(spec) || !doc_off || !tokens) return 2;
  const mrcgen_spec& s = *spec;
  auto g = cached_alias(s.vocab, s.zipf_global);
  std::shared_ptr<Alias> t;
  if (s.n_topics > 0) t = cached_alias(s.vocab, s.zipf_topic);
  std::vector<TopicMap> maps = make_maps(s);
  Sampler smp{&s, g.get(), t.get(), &maps};
  std::vector<uint32_t> dup_src;
  dup_plan(s, 0, false, dup_src);
  // originals
  parallel_for(s.n_docs, threads, [&](uint64_t d) {
    if (dup_src[d] != UINT32_MAX) return;
    uint32_t topic = topic_of(s, d);
    Rng r = stream(s.seed, kTagTok, d);
    for (uint64_t p = doc_off[d]; p < doc_off[d + 1]; ++p) tokens[p] = smp.draw(r, topic);
  });
  // near-duplicates (sources are originals, already filled)
  parallel_for(s.n_docs, threads, [&](uint64_t d) {
    uint32_t src = dup_src[d];
    if (src == UINT32_MAX) return;
    uint32_t topic = topic_of(s, src);
    Rng r = stream(s.seed, kTagResample, d);
    double rho = resample_frac(s, r);
    uint64_t so = doc_off[src];
    uint64_t n = doc_off[d + 1] - doc_off[d];
    for (uint64_t k = 0; k < n; ++k) {
      uint32_t tok = tokens[so + k];
      if (r.u01() < rho) tok = smp.draw(r, topic);
      tokens[doc_off[d] + k] = tok;
    }
  });
  if (dup_src_out) std::memcpy(dup_src_out, dup_src.data(), sizeof(uint32_t) * s.n_docs);
  return 0;
}

int mrcgen_offsets_queries(const mrcgen_spec* q, const mrcgen_spec* db, const uint64_t* db_off, uint64_t* q_off) {
  if (!valid(q) || !valid(db) || !db_off || !q_off) return 2;
  if (q->vocab != db->vocab || q->n_topics != db->n_topics) return 2;
  std::vector<uint32_t> dup_src;
  dup_plan(*q, db->n_docs, true, dup_src);
  q_off[0] = 0;
  for (uint32_t d = 0; d < q->n_docs; ++d) {
    uint64_t L = dup_src[d] == UINT32_MAX ? draw_len(*q, d) : db_off[dup_src[d] + 1] - db_off[dup_src[d]];
    q_off[d + 1] = q_off[d] + L;
  }
  return 0;
}

int mrcgen_fill_queries(const mrcgen_spec* q, const mrcgen_spec* db, const uint64_t* db_off,
                        const uint32_t* db_tokens, const uint64_t* q_off, uint32_t* q_tokens, uint32_t* q_src,
                        int threads) {
  if (!valid(q) || !valid(db) || !db_off || !db_tokens || !q_off || !q_tokens) return 2;
  if (q->vocab != db->vocab || q->n_topics != db->n_topics) return 2;
  const mrcgen_spec& s = *q;
  auto g = cached_alias(s.vocab, s.zipf_global);
  std::shared_ptr<Alias> t;
  if (s.n_topics > 0) t = cached_alias(s.vocab, s.zipf_topic);
  std::vector<TopicMap> maps = make_maps(*db);  // topics shared with the database
  Sampler smp{&s, g.get(), t.get(), &maps};
  std::vector<uint32_t> dup_src;
  dup_plan(s, db->n_docs, true, dup_src);
  parallel_for(s.n_docs, threads, [&](uint64_t d) {
    uint32_t src = dup_src[d];
    if (src == UINT32_MAX) {
      uint32_t topic = topic_of(s, d);
      Rng r = stream(s.seed, kTagTok, d);
      for (uint64_t p = q_off[d]; p < q_off[d + 1]; ++p) q_tokens[p] = smp.draw(r, topic);
    } else {
      uint32_t topic = topic_of(*db, src);
      Rng r = stream(s.seed, kTagResample, d);
      double rho = resample_frac(s, r);
      uint64_t so = db_off[src];
      uint64_t n = q_off[d + 1] - q_off[d];
      for (uint64_t k = 0; k < n; ++k) {
        uint32_t tok = db_tokens[so + k];
        if (r.u01() < rho) tok = smp.draw(r, topic);
        q_tokens[q_off[d] + k] = tok;
      }
    }
  });
  if (q_src) std::memcpy(q_src, dup_src.data(), sizeof(uint32_t) * s.n_docs);
  return 0;
}

int mrcgen_sample_refs(uint64_t seed, uint32_t n, uint32_t k, uint32_t* out) {
  if (!out || k == 0 || k > n) return 2;
  // Sparse partial Fisher-Yates: O(k) memory even for n = 1e6.
  std::unordered_map<uint32_t, uint32_t> swapped;
  auto at = [&](uint32_t i) {
    auto it = swapped.find(i);
    return it == swapped.end() ? i : it->second;
  };
  Rng r = stream(seed, kTagRef, 0);
  for (uint32_t i = 0; i < k; ++i) {
    uint32_t j = i + static_cast<uint32_t>(r.below(n - i));
    uint32_t vi = at(i), vj = at(j);
    swapped[i] = vj;
    swapped[j] = vi;
    out[i] = vj;
  }
  return 0;
}

}  // extern "C"
