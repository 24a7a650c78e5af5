// k0_text.cu — text front end: raw document bytes ->
// 3-gram id stream (the K1 input) and per-occurrence word Simhash.
//
// Reference semantics:
//   normalize (ngram.hpp:114-129): ASCII letters lowercased; every maximal run
//     of other bytes (digits, punctuation, whitespace, bytes >= 0x80) is one
//     word break;
//   extract_3grams (ngram.hpp:149-180): sliding 3-letter windows inside each
//     word, id = ((c0*26)+c1)*26+c2 (pack_gram, ngram.hpp:33-37) — on the raw
//     bytes that is every window of three consecutive letters;
//   extract_words (ngram.hpp:132-145) + word_hash64 (simhash.hpp:23-29: first
//     8 bytes of the word's MD5, big-endian) + simhash (simhash.hpp:35-45: per
//     occurrence +-1 per bit column, bit = column > 0, no words -> 0).
//
// Mapping: warp per document, 32 bytes per step (lane = byte; the next two
// bytes via SHFL). Grams: ballot + prefix popcount place each id; a first
// pass only counts (the host needs the per-doc gram counts to plan K1).
// Words: word starts/ends per step come from two ballots; completed words
// (start, length) are queued in shared memory and hashed 32 at a time, one
// word per lane (MD5 over 64-byte blocks, RFC 1321); the bit columns are
// counted with 64 ballots + popcounts per 32 words.

#include "kernels.cuh"

namespace refsig_gpu {
namespace {

__constant__ uint32_t c_md5_t[64];

__device__ __forceinline__ uint32_t lower_letter(uint32_t b) { return (b | 32u) - 'a'; }  // < 26 iff a letter

// Bytes of doc [p, end): this lane's byte and the next two (0 past the end).
__device__ __forceinline__ void load3(const uint8_t* __restrict__ text, uint64_t p, uint64_t end, uint32_t lane,
                                      uint32_t& b0, uint32_t& b1, uint32_t& b2) {
  b0 = p + lane < end ? text[p + lane] : 0u;
  b1 = __shfl_down_sync(0xffffffffu, b0, 1);
  b2 = __shfl_down_sync(0xffffffffu, b0, 2);
  if (lane >= 30) {
    const uint64_t q1 = p + lane + 1, q2 = p + lane + 2;
    if (lane == 31) b1 = q1 < end ? text[q1] : 0u;
    b2 = q2 < end ? text[q2] : 0u;
  }
}

__global__ void __launch_bounds__(256) text_grams_kernel(const uint8_t* __restrict__ text,
                                                         const uint64_t* __restrict__ off, uint32_t n_docs,
                                                         const uint64_t* __restrict__ gram_off,
                                                         uint32_t* __restrict__ cnt, uint32_t* __restrict__ tokens) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (d >= n_docs) return;
  const uint64_t beg = off[d], end = off[d + 1];
  uint64_t out = tokens ? gram_off[d] : 0;
  uint32_t total = 0;
  for (uint64_t p = beg; p < end; p += 32) {
    uint32_t b0, b1, b2;
    load3(text, p, end, lane, b0, b1, b2);
    const uint32_t l0 = lower_letter(b0), l1 = lower_letter(b1), l2 = lower_letter(b2);
    const bool g = l0 < 26 && l1 < 26 && l2 < 26 && p + lane + 2 < end;
    const uint32_t m = __ballot_sync(0xffffffffu, g);
    if (tokens && g) tokens[out + __popc(m & ((1u << lane) - 1u))] = (l0 * 26 + l1) * 26 + l2;
    out += __popc(m);
    total += __popc(m);
  }
  if (cnt && lane == 0) cnt[d] = total;
}

// MD5 of the lowercased letters text[s, s+len) (RFC 1321); the first 8 digest
// bytes big-endian.
__device__ uint64_t word_md5_64(const uint8_t* __restrict__ text, uint64_t s, uint32_t len) {
  uint32_t h0 = 0x67452301u, h1 = 0xefcdab89u, h2 = 0x98badcfeu, h3 = 0x10325476u;
  const uint32_t nblk = (len + 8) / 64 + 1;
  for (uint32_t blk = 0; blk < nblk; ++blk) {
    uint32_t M[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      uint32_t w = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t q = blk * 64 + 4 * i + k;
        uint32_t v = 0;
        if (q < len)
          v = text[s + q] | 32u;  // letters only: lowercase
        else if (q == len)
          v = 0x80u;
        w |= v << (8 * k);
      }
      M[i] = w;
    }
    if (blk + 1 == nblk) {  // length in bits, little-endian, in the last 8 bytes
      const uint64_t bits = static_cast<uint64_t>(len) * 8;
      M[14] = static_cast<uint32_t>(bits);
      M[15] = static_cast<uint32_t>(bits >> 32);
    }
    uint32_t a = h0, b = h1, c = h2, d = h3;
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      uint32_t f;
      int g, r;
      if (i < 16) {
        f = (b & c) | (~b & d);
        g = i;
        r = (i & 3) == 0 ? 7 : (i & 3) == 1 ? 12 : (i & 3) == 2 ? 17 : 22;
      } else if (i < 32) {
        f = (d & b) | (~d & c);
        g = (5 * i + 1) & 15;
        r = (i & 3) == 0 ? 5 : (i & 3) == 1 ? 9 : (i & 3) == 2 ? 14 : 20;
      } else if (i < 48) {
        f = b ^ c ^ d;
        g = (3 * i + 5) & 15;
        r = (i & 3) == 0 ? 4 : (i & 3) == 1 ? 11 : (i & 3) == 2 ? 16 : 23;
      } else {
        f = c ^ (b | ~d);
        g = (7 * i) & 15;
        r = (i & 3) == 0 ? 6 : (i & 3) == 1 ? 10 : (i & 3) == 2 ? 15 : 21;
      }
      const uint32_t x = a + f + c_md5_t[i] + M[g];
      a = d;
      d = c;
      c = b;
      b = b + __funnelshift_l(x, x, r);
    }
    h0 += a;
    h1 += b;
    h2 += c;
    h3 += d;
  }
  // digest bytes 0..7 = h0, h1 little-endian; read big-endian
  return (static_cast<uint64_t>(__byte_perm(h0, 0, 0x0123)) << 32) | __byte_perm(h1, 0, 0x0123);
}

constexpr int kWordQ = 64;  // per-warp queue of completed words

__global__ void __launch_bounds__(256) text_simhash_kernel(const uint8_t* __restrict__ text,
                                                           const uint64_t* __restrict__ off, uint32_t n_docs,
                                                           uint64_t* __restrict__ fp) {
  __shared__ uint2 q[8][kWordQ];  // {start - doc begin, length}
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t d = blockIdx.x * (blockDim.x >> 5) + wid;
  if (d >= n_docs) return;
  const uint64_t beg = off[d], end = off[d + 1];
  uint32_t c0 = 0, c1 = 0, nw = 0;  // lane: votes of columns lane and lane+32; words seen
  uint32_t qn = 0;                  // queued words (warp-uniform)
  int64_t open = -1;                // start of a word still running at the step boundary
  auto hash_batch = [&](uint32_t m) {
    const bool v = lane < m;
    uint64_t h = 0;
    if (v) {
      const uint2 w = q[wid][lane];
      h = word_md5_64(text, beg + w.x, w.y);
    }
    const uint32_t lo = static_cast<uint32_t>(h), hi = static_cast<uint32_t>(h >> 32);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint32_t bl = __ballot_sync(0xffffffffu, v && ((lo >> j) & 1u));
      const uint32_t bh = __ballot_sync(0xffffffffu, v && ((hi >> j) & 1u));
      if (lane == static_cast<uint32_t>(j)) {
        c0 += __popc(bl);
        c1 += __popc(bh);
      }
    }
    nw += m;
  };
  for (uint64_t p = beg; p < end; p += 32) {
    uint32_t b0, b1, b2;
    load3(text, p, end, lane, b0, b1, b2);
    (void)b2;
    const uint64_t pos = p + lane;
    const bool in = pos < end;
    const bool let = in && lower_letter(b0) < 26;
    const uint32_t prev = __shfl_up_sync(0xffffffffu, b0, 1);
    const bool prev_let = lane == 0 ? (p > beg && lower_letter(text[p - 1]) < 26) : lower_letter(prev) < 26;
    const bool next_let = pos + 1 < end && lower_letter(b1) < 26;
    const uint32_t S = __ballot_sync(0xffffffffu, let && !prev_let);  // word starts
    const uint32_t E = __ballot_sync(0xffffffffu, let && !next_let);  // last letter of a word
    // pair ends with starts in order: an open word takes the first end
    uint32_t s_rem = S, e_rem = E;
    while (e_rem) {
      const int e = __ffs(e_rem) - 1;
      e_rem &= e_rem - 1;
      uint64_t st;
      if (open >= 0) {
        st = static_cast<uint64_t>(open);
        open = -1;
      } else {
        const int s = __ffs(s_rem) - 1;
        s_rem &= s_rem - 1;
        st = p + s;
      }
      if (lane == 0) q[wid][qn] = make_uint2(static_cast<uint32_t>(st - beg), static_cast<uint32_t>(p + e + 1 - st));
      ++qn;
    }
    if (s_rem) open = static_cast<int64_t>(p + (31 - __clz(s_rem)));  // a start without its end yet
    __syncwarp();
    if (qn >= 32) {
      hash_batch(32);
      __syncwarp();
      if (lane < qn - 32) q[wid][lane] = q[wid][32 + lane];
      qn -= 32;
      __syncwarp();
    }
  }
  if (qn) hash_batch(qn);
  // bit j = votes_j > words - votes_j (2*votes > words; tie -> 0)
  const uint32_t lo = __ballot_sync(0xffffffffu, 2 * c0 > nw);
  const uint32_t hi = __ballot_sync(0xffffffffu, 2 * c1 > nw);
  if (lane == 0) fp[d] = (static_cast<uint64_t>(hi) << 32) | lo;
}

}  // namespace

void text_init_tables() {
  static bool done = false;
  if (done) return;
  uint32_t t[64];
  for (int i = 0; i < 64; ++i) t[i] = static_cast<uint32_t>(std::floor(std::fabs(std::sin(i + 1.0)) * 4294967296.0));
  cudaMemcpyToSymbol(c_md5_t, t, sizeof(t));
  done = true;
}

void launch_text_grams(const uint8_t* text, const uint64_t* off, uint32_t n_docs, const uint64_t* gram_off,
                       uint32_t* cnt, uint32_t* tokens, cudaStream_t s) {
  if (!n_docs) return;
  text_grams_kernel<<<static_cast<unsigned>(ceil_div(n_docs, 8)), 256, 0, s>>>(text, off, n_docs, gram_off, cnt,
                                                                               tokens);
  note_launch();
}

void launch_text_simhash(const uint8_t* text, const uint64_t* off, uint32_t n_docs, uint64_t* fp, cudaStream_t s) {
  if (!n_docs) return;
  text_init_tables();
  text_simhash_kernel<<<static_cast<unsigned>(ceil_div(n_docs, 8)), 256, 0, s>>>(text, off, n_docs, fp);
  note_launch();
}

}  // namespace refsig_gpu
