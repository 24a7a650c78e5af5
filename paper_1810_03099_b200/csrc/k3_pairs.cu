// k3_pairs.cu — all-pairs kernels: MRC signature compare (K3), Hamming
// compare (K4b), and the deterministic emitter shared by both.
//
// Reference semantics:
//   compare(a,b) = cosine of the signature vectors, 0 if either is all-zero
//                  (SPEC.md:369-377); match <=> score >= tau.
//   hamming(a,b) = popcount(a ^ b) (simhash.hpp:47); match <=> hd <= max_dist.
//   pairs are i<j in lexicographic order.
//
// Design: a compare kernel evaluates 128x128 pair tiles of the upper triangle
// (all tiles for a query-vs-DB join) and writes one bit per pair into a
// row-major pair bitmap (words_per_row = ceil(cols/128)*4), plus per-row match
// counts. An exclusive scan of the counts gives each row's output offset and
// the emitter turns set bits into sorted keys (i<<32 | j). No atomics decide
// output positions, so the candidate list is sorted and identical for every
// launch configuration without a device sort.
//
// MRC tile: 256 threads, 8x8 register micro-tile per thread over the two
// halves of the tile (conflict-free float4 LDS), K-chunks of 32 staged in
// shared memory. Inner loop: 4 LDS.128 per 64 FFMA. Epilogue: per row a
// nibble per half, OR-combined across the 8 lanes that share a 32-bit word.

#include "kernels.cuh"

namespace refsig_gpu {
namespace {

constexpr int kKC = 32;  // K chunk staged in shared memory

// Tile t -> (bi, bj): triangle (bi <= bj, row-major) or rectangle.
__device__ __forceinline__ void tile_coords(uint32_t t, uint32_t nbr, uint32_t nbc, bool triangle, uint32_t& bi,
                                            uint32_t& bj) {
  if (!triangle) {
    bi = t / nbc;
    bj = t - bi * nbc;
    return;
  }
  const double nb = nbc;
  double x = (nb + 0.5) - sqrt((nb + 0.5) * (nb + 0.5) - 2.0 * t);
  int64_t b = static_cast<int64_t>(x);
  auto S = [&](int64_t r) { return r * static_cast<int64_t>(nbc) - r * (r - 1) / 2; };
  if (b < 0) b = 0;
  while (b + 1 <= static_cast<int64_t>(nbc) && S(b + 1) <= static_cast<int64_t>(t)) ++b;
  while (b > 0 && S(b) > static_cast<int64_t>(t)) --b;
  bi = static_cast<uint32_t>(b);
  bj = bi + static_cast<uint32_t>(t - S(b));
}

// Valid-column mask for the 32 columns starting at lo in row i.
__device__ __forceinline__ uint32_t col_mask(uint32_t lo, uint32_t i, const PairGrid& g) {
  uint32_t m = 0xffffffffu;
  if (lo >= g.n_cols) return 0u;
  if (lo + 32 > g.n_cols) m >>= (lo + 32 - g.n_cols);
  if (g.triangle && lo <= i) {
    const uint32_t first = i + 1 - lo;  // first valid bit
    m = first >= 32 ? 0u : (m & (0xffffffffu << first));
  }
  return m;
}

__global__ void __launch_bounds__(256, 2) mrc_bitmap_kernel(const float* __restrict__ Sr,
                                                            const float* __restrict__ Sc, uint32_t K, float tau,
                                                            PairGrid g, uint32_t nbr, uint32_t nbc,
                                                            uint32_t* __restrict__ bitmap,
                                                            uint32_t* __restrict__ rowcnt) {
  __shared__ __align__(16) float As[kKC][kTile];
  __shared__ __align__(16) float Bs[kKC][kTile];
  uint32_t bi, bj;
  tile_coords(blockIdx.x + g.tile0, nbr, nbc, g.triangle, bi, bj);
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const uint32_t row0 = bi * kTile, col0 = bj * kTile;

  float acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.0f;

  for (uint32_t k0 = 0; k0 < K; k0 += kKC) {
    const uint32_t kc = min(static_cast<uint32_t>(kKC), K - k0);
    // Stage the row and column panels (row-major Sn -> [k][row] in smem).
    for (uint32_t idx = tid; idx < kTile * kc; idx += 256) {
      const uint32_t r = idx / kc, k = idx - r * kc;
      const uint32_t gi = row0 + r, gj = col0 + r;
      As[k][r] = gi < g.n_rows ? __ldg(Sr + static_cast<size_t>(gi) * K + k0 + k) : 0.0f;
      Bs[k][r] = gj < g.n_cols ? __ldg(Sc + static_cast<size_t>(gj) * K + k0 + k) : 0.0f;
    }
    __syncthreads();
#pragma unroll 4
    for (uint32_t k = 0; k < kc; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[k][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[k][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
    }
    __syncthreads();
  }

  // Epilogue: bit (r,c) = acc >= tau; assemble 32-bit words across 8 lanes.
  const int sh = (tx & 7) * 4;
  uint32_t my_w0 = 0, my_w1 = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    uint32_t n0 = 0, n1 = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      n0 |= (acc[r][c] >= tau ? 1u : 0u) << c;
      n1 |= (acc[r][c + 4] >= tau ? 1u : 0u) << c;
    }
    uint32_t w0 = n0 << sh, w1 = n1 << sh;
    w0 |= __shfl_xor_sync(0xffffffffu, w0, 1);
    w1 |= __shfl_xor_sync(0xffffffffu, w1, 1);
    w0 |= __shfl_xor_sync(0xffffffffu, w0, 2);
    w1 |= __shfl_xor_sync(0xffffffffu, w1, 2);
    w0 |= __shfl_xor_sync(0xffffffffu, w0, 4);
    w1 |= __shfl_xor_sync(0xffffffffu, w1, 4);
    if ((tx & 7) == r) {
      my_w0 = w0;
      my_w1 = w1;
    }
  }
  const int r = tx & 7;
  const uint32_t lr = r < 4 ? ty * 4 + r : 64 + ty * 4 + (r - 4);
  const uint32_t i = row0 + lr;
  const uint32_t grp = tx >> 3;  // word 0/1 of each 64-column half
  uint32_t cnt = 0;
  if (i < g.n_rows) {
    const uint32_t wa = grp, wb = 2 + grp;
    const uint32_t va = my_w0 & col_mask(col0 + wa * 32, i, g);
    const uint32_t vb = my_w1 & col_mask(col0 + wb * 32, i, g);
    uint32_t* rowp = bitmap + static_cast<size_t>(i) * g.words_per_row + bj * 4;
    rowp[wa] = va;
    rowp[wb] = vb;
    cnt = __popc(va) + __popc(vb);
  }
  cnt += __shfl_xor_sync(0xffffffffu, cnt, 8);
  if (grp == 0 && cnt && i < g.n_rows) atomicAdd(rowcnt + i, cnt);
}

// Hamming tile: warp w handles rows (w&3)*32+lane and words (w>>2)*2..+1.
__global__ void __launch_bounds__(256) hamming_bitmap_kernel(const uint64_t* __restrict__ fr,
                                                             const uint64_t* __restrict__ fc, int max_dist,
                                                             PairGrid g, uint32_t nbr, uint32_t nbc,
                                                             uint32_t* __restrict__ bitmap,
                                                             uint32_t* __restrict__ rowcnt) {
  __shared__ __align__(16) uint2 Fc[kTile];
  uint32_t bi, bj;
  tile_coords(blockIdx.x + g.tile0, nbr, nbc, g.triangle, bi, bj);
  const uint32_t row0 = bi * kTile, col0 = bj * kTile;
  if (threadIdx.x < kTile) {
    const uint32_t j = col0 + threadIdx.x;
    const uint64_t v = j < g.n_cols ? fc[j] : 0ull;
    Fc[threadIdx.x] = make_uint2(static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t i = row0 + (w & 3) * 32 + lane;
  const uint64_t x64 = i < g.n_rows ? fr[i] : 0ull;
  const uint32_t xl = static_cast<uint32_t>(x64), xh = static_cast<uint32_t>(x64 >> 32);
  const int thr = max_dist + 1;
  uint32_t cnt = 0;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int wi = (w >> 2) * 2 + q;
    uint32_t bits = 0;
    // Columns 31..0 of this word: shift in the sign of (hd - thr) so column b
    // ends at bit b (one funnel shift per pair).
#pragma unroll
    for (int b = 31; b >= 0; b -= 2) {
      const uint4 y = *reinterpret_cast<const uint4*>(&Fc[wi * 32 + b - 1]);  // cols b-1, b
      const int d1 = __popc(xl ^ y.z) + __popc(xh ^ y.w) - thr;
      bits = __funnelshift_l(static_cast<uint32_t>(d1), bits, 1);
      const int d0 = __popc(xl ^ y.x) + __popc(xh ^ y.y) - thr;
      bits = __funnelshift_l(static_cast<uint32_t>(d0), bits, 1);
    }
    if (i < g.n_rows) {
      const uint32_t v = bits & col_mask(col0 + wi * 32, i, g);
      bitmap[static_cast<size_t>(i) * g.words_per_row + bj * 4 + wi] = v;
      cnt += __popc(v);
    }
  }
  if (cnt) atomicAdd(rowcnt + i, cnt);
}

// Warp per row: scan the row's words from its first written tile, write keys.
__global__ void __launch_bounds__(256) emit_kernel(const uint32_t* __restrict__ bitmap, PairGrid g,
                                                   const uint32_t* __restrict__ rowcnt,
                                                   const uint64_t* __restrict__ rowstart, uint64_t* __restrict__ out,
                                                   uint64_t capacity) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t i = g.row_begin + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < g.row_end; i += nwarps) {
    uint32_t remaining = rowcnt[i];
    if (remaining == 0) continue;
    uint64_t base = rowstart[i];
    const uint32_t* row = bitmap + static_cast<size_t>(i) * g.words_per_row;
    const uint32_t wbeg = g.triangle ? (i / kTile) * 4 : 0;
    for (uint32_t c = wbeg; c < g.words_per_row && remaining; c += 32) {
      const uint32_t wi = c + lane;
      uint32_t word = wi < g.words_per_row ? row[wi] : 0u;
      const uint32_t n = __popc(word);
      const uint32_t inc = warp_inclusive_scan(n, lane);
      const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
      uint64_t pos = base + inc - n;
      const uint64_t hi = static_cast<uint64_t>(i) << 32;
      while (word) {
        const int b = __ffs(word) - 1;
        word &= word - 1;
        if (pos < capacity) out[pos] = hi | (wi * 32u + b);
        ++pos;
      }
      base += tot;
      remaining -= tot;
    }
  }
}

int sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// Tiles of row panels [row_begin/128, ceil(row_end/128)); sets g.tile0.
uint64_t n_tiles(PairGrid& g, uint32_t& nbr, uint32_t& nbc) {
  nbr = static_cast<uint32_t>(ceil_div(g.n_rows, kTile));
  nbc = static_cast<uint32_t>(ceil_div(g.n_cols, kTile));
  const uint64_t p0 = g.row_begin / kTile, p1 = ceil_div(g.row_end, kTile);
  if (p1 <= p0) return 0;
  if (g.triangle) {
    auto S = [&](uint64_t r) { return r * nbc - r * (r - 1) / 2; };
    g.tile0 = static_cast<uint32_t>(S(p0));
    return S(p1) - S(p0);
  }
  g.tile0 = static_cast<uint32_t>(p0 * nbc);
  return (p1 - p0) * nbc;
}

}  // namespace

void launch_mrc_bitmap(const float* Sn_rows, const float* Sn_cols, uint32_t K, float tau, const PairGrid& g_in,
                       uint32_t* bitmap, uint32_t* rowcnt, cudaStream_t s) {
  PairGrid g = g_in;
  uint32_t nbr, nbc;
  const uint64_t t = n_tiles(g, nbr, nbc);
  if (t == 0) return;
  mrc_bitmap_kernel<<<static_cast<unsigned>(t), 256, 0, s>>>(Sn_rows, Sn_cols, K, tau, g, nbr, nbc, bitmap, rowcnt);
  note_launch();
}

void launch_hamming_bitmap(const uint64_t* f_rows, const uint64_t* f_cols, int max_dist, const PairGrid& g_in,
                           uint32_t* bitmap, uint32_t* rowcnt, cudaStream_t s) {
  PairGrid g = g_in;
  uint32_t nbr, nbc;
  const uint64_t t = n_tiles(g, nbr, nbc);
  if (t == 0) return;
  hamming_bitmap_kernel<<<static_cast<unsigned>(t), 256, 0, s>>>(f_rows, f_cols, max_dist, g, nbr, nbc, bitmap,
                                                                 rowcnt);
  note_launch();
}

void launch_emit_pairs(const uint32_t* bitmap, const PairGrid& g, const uint32_t* rowcnt, const uint64_t* rowstart,
                       uint64_t* out, uint64_t capacity, cudaStream_t s) {
  if (g.row_end <= g.row_begin) return;
  uint64_t blocks = ceil_div(g.row_end - g.row_begin, 8);
  const uint64_t cap = static_cast<uint64_t>(sms()) * 8;
  if (blocks > cap) blocks = cap;
  emit_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(bitmap, g, rowcnt, rowstart, out, capacity);
  note_launch();
}

}  // namespace refsig_gpu
