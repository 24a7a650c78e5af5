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
// Mapping: warp per document, 128 bytes per step (4 per lane, read by
// aligned 32-bit loads; neighbour bytes via SHFL). Grams: a warp scan of the
// per-lane counts places each id; a first pass only counts (the host needs
// the per-doc gram counts to plan K1). Words: each lane finds word starts and
// ends in its 4 bytes, the start of a word ending in a lane comes from a warp
// max-scan of the last start per lane (or a word left open by the previous
// step); completed words (start, length) are queued in shared memory and
// hashed 32 at a time, one word per lane (MD5 over 64-byte blocks, RFC 1321);
// the bit columns are counted by a 32x32 warp bit transpose + popcount.

#include <atomic>
#include <cmath>

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

// 4 bytes at an arbitrary byte address from aligned 32-bit loads (the text
// buffer is padded by 8 bytes so the second load never leaves it).
__device__ __forceinline__ uint32_t load4u(const uint8_t* __restrict__ text, uint64_t q) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(text + (q & ~3ull));
  return __funnelshift_r(__ldg(w), __ldg(w + 1), static_cast<uint32_t>(q & 3) * 8);
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
  // 128 bytes per step, 4 per lane (the two bytes after a lane's four come
  // from the next lane); four steps' loads are issued together
  constexpr int U = 4;
  for (uint64_t p0 = beg; p0 < end; p0 += 128 * U) {
    uint32_t wv[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t q = p0 + 128 * u + 4 * lane;
      wv[u] = q < end ? load4u(text, q) : 0u;
      xv[u] = (lane == 31 && q + 4 < end) ? load4u(text, q + 4) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
    const uint64_t p = p0 + 128 * u;
    if (p >= end) break;  // warp-uniform
    const uint64_t q = p + 4 * lane;
    const uint32_t w = wv[u];
    uint32_t nx = __shfl_down_sync(0xffffffffu, w, 1);
    if (lane == 31) nx = xv[u];
    uint32_t l[6];
#pragma unroll
    for (int k = 0; k < 4; ++k) l[k] = lower_letter((w >> (8 * k)) & 0xffu);
    l[4] = lower_letter(nx & 0xffu);
    l[5] = lower_letter((nx >> 8) & 0xffu);
    uint32_t gm = 0;  // bit k: a gram starts at q+k
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (l[k] < 26 && l[k + 1] < 26 && l[k + 2] < 26 && q + k + 2 < end) gm |= 1u << k;
    const uint32_t c = __popc(gm);
    const uint32_t inc = warp_inclusive_scan(c, lane);
    if (tokens) {
      uint64_t o = out + inc - c;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (gm & (1u << k)) tokens[o++] = (l[k] * 26 + l[k + 1]) * 26 + l[k + 2];
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
    out += tot;
    total += tot;
    }
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
      const uint32_t q = blk * 64 + 4 * i;  // message bytes q .. q+3
      uint32_t w = 0;
      if (q < len) {
        w = load4u(text, s + q) | 0x20202020u;  // letters only: lowercase
        if (len - q < 4) w &= (1u << (8 * (len - q))) - 1u;
      }
      if (q <= len && len < q + 4) w |= 0x80u << (8 * (len - q));
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

constexpr int kWordQ = 128;  // per-warp queue of completed words (<= 64 per step + < 32 carried)

// 32x32 bit transpose across the warp (row = lane): returns in lane l the
// bits of column 31-l of all lanes' rows (bit b of the result = row 31-b).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, uint32_t lane) {
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) {
    const uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu : j == 2 ? 0x33333333u
                                                                                                  : 0x55555555u;
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
    const bool up = lane & j;
    const uint32_t t = ((up ? y : x) ^ ((up ? x : y) >> j)) & m;
    x ^= up ? (t << j) : t;
  }
  return x;
}

__global__ void __launch_bounds__(256) text_simhash_kernel(const uint8_t* __restrict__ text,
                                                           const uint64_t* __restrict__ off, uint32_t n_docs,
                                                           uint64_t* __restrict__ fp) {
  __shared__ uint2 q[8][kWordQ];  // {start - doc begin, length}
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t d = blockIdx.x * (blockDim.x >> 5) + wid;
  if (d >= n_docs) return;
  const uint64_t beg = off[d], end = off[d + 1];
  uint32_t c_lo = 0, c_hi = 0, nw = 0;  // lane l: votes of columns 31-l and 63-l; words seen
  uint32_t qn = 0;                      // queued words (warp-uniform)
  int64_t open = -1;                    // start of a word still running at the step boundary
  auto hash_batch = [&](uint32_t m) {
    uint64_t h = 0;
    if (lane < m) {
      const uint2 w = q[wid][lane];
      h = word_md5_64(text, beg + w.x, w.y);
    }
    // column votes: transpose the 32 hashes' bits, popcount per column
    c_lo += __popc(warp_transpose32(static_cast<uint32_t>(h), lane));
    c_hi += __popc(warp_transpose32(static_cast<uint32_t>(h >> 32), lane));
    nw += m;
  };
  // 128 bytes per step, 4 per lane; neighbour bytes via SHFL
  for (uint64_t p = beg; p < end; p += 128) {
    const uint64_t q0 = p + 4 * lane;
    const uint32_t w = q0 < end ? load4u(text, q0) : 0u;
    uint32_t prev = __shfl_up_sync(0xffffffffu, w, 1) >> 24;   // byte q0-1
    uint32_t next = __shfl_down_sync(0xffffffffu, w, 1) & 0xffu;  // byte q0+4
    if (lane == 0) prev = p > beg ? text[p - 1] : 0u;
    if (lane == 31) next = q0 + 4 < end ? text[q0 + 4] : 0u;
    uint32_t let = 0;  // bit k: byte q0+k is a letter of this doc
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (q0 + k < end && lower_letter((w >> (8 * k)) & 0xffu) < 26) let |= 1u << k;
    const uint32_t lp = (let << 1) | (lower_letter(prev) < 26 ? 1u : 0u);         // bit k: byte q0+k-1
    const uint32_t ln = (let >> 1) | ((q0 + 4 < end && lower_letter(next) < 26) ? 8u : 0u);  // bit k: q0+k+1
    const uint32_t sm = let & ~lp & 0xfu;  // word starts
    const uint32_t em = let & ~ln & 0xfu;  // last letters of words
    // latest start before this lane's bytes: max-scan of "last start" over lanes
    int64_t ls = sm ? static_cast<int64_t>(q0 + 31 - __clz(sm)) : -1;
    int64_t run = ls;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, run, o);
      if (lane >= static_cast<uint32_t>(o)) run = max(run, y);
    }
    int64_t before = __shfl_up_sync(0xffffffffu, run, 1);
    if (lane == 0) before = -1;
    if (before < 0) before = open;
    const uint32_t ne = __popc(em);
    const uint32_t inc = warp_inclusive_scan(ne, lane);
    uint32_t slot = qn + inc - ne;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (em & (1u << k)) {
        const uint32_t sk = sm & ((2u << k) - 1u);  // starts at or before byte k in this lane
        const uint64_t st = sk ? q0 + 31 - __clz(sk) : static_cast<uint64_t>(before);
        q[wid][slot++] = make_uint2(static_cast<uint32_t>(st - beg), static_cast<uint32_t>(q0 + k + 1 - st));
      }
    qn += __shfl_sync(0xffffffffu, inc, 31);
    // a word left open at the end of the step: the last start after the last end
    const int64_t last_s = __shfl_sync(0xffffffffu, run, 31);
    const int64_t le = em ? static_cast<int64_t>(q0 + 31 - __clz(em)) : -1;
    int64_t lem = le;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lem = max(lem, __shfl_xor_sync(0xffffffffu, lem, o));
    if (last_s > lem) open = last_s;
    else if (lem >= 0) open = -1;
    __syncwarp();
    while (qn >= 32) {
      hash_batch(32);
      __syncwarp();
      for (uint32_t i = lane; i + 32 < qn; i += 32) q[wid][i] = q[wid][i + 32];
      qn -= 32;
      __syncwarp();
    }
  }
  if (qn) hash_batch(qn);
  // bit j = 2*votes_j > words (tie -> 0); lane l holds columns 31-l / 63-l
  const uint32_t lo = __brev(__ballot_sync(0xffffffffu, 2 * c_lo > nw));
  const uint32_t hi = __brev(__ballot_sync(0xffffffffu, 2 * c_hi > nw));
  if (lane == 0) fp[d] = (static_cast<uint64_t>(hi) << 32) | lo;
}

}  // namespace

void text_init_tables() {
  // __constant__ memory is per device context: one upload per device ordinal
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load() & bit) return;
  uint32_t t[64];
  for (int i = 0; i < 64; ++i) t[i] = static_cast<uint32_t>(std::floor(std::fabs(std::sin(i + 1.0)) * 4294967296.0));
  cudaMemcpyToSymbol(c_md5_t, t, sizeof(t));
  done.fetch_or(bit);
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
