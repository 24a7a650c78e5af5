// k3_tc.cu — K3 on the 5th-generation tensor cores: the all-pairs MRC compare
// (SPEC.md:369-377 over i<j) as a tcgen05 kernel whose fp32
// accumulators live in TMEM, with the threshold folded into the MMA.
//
// Exactness. compare() needs fp32-class dot products (the parity bar puts
// every pair farther than 1e-5 from tau on the oracle's side), so a plain
// fp16 MMA (11-bit operands) is not enough. Each unit signature value v is
// split into fp16 hi = rn(v) and lo = rn(v - hi) (v - hi is exact in fp32),
// and the operands are laid out so that ONE K-chain computes
//     a.b ~= sum_k a_hi b_hi + a_hi b_lo + a_lo b_hi  -  tau
// (the a_lo b_lo term is < 2^-22 |a||b|): the row form of a document is
// [hi | hi | lo | -tau_0 -tau_1 -tau_2 | 0..], the column form
// [hi | lo | hi | 1 1 1 | 0..], K' = roundup16(3K + 3) fp16 values, where
// tau = tau_0 + tau_1 + tau_2 exactly in fp16 pieces. The accumulator is then
// dot - tau and its sign bit is the match bit (match <=> dot >= tau), so the
// epilogue is one funnel shift per pair. Error against the fp64 dot: a few
// 1e-7 (DESIGN.md §5 K3-TC; tests/test_gpu_parity.py border checks).
//
// Layout. Both forms are stored as 128-document panels in the canonical
// K-major no-swizzle UMMA layout: panel p = [K'/8 chunks][128 docs][8 fp16],
// so a panel is one contiguous 256*K'-byte block: one cp.async.bulk per
// operand panel, and the smem descriptor has LBO = 2048 B (next 8-wide K
// chunk) and SBO = 128 B (next 8-row group).
//
// Kernel. Persistent, one CTA per SM, 608 threads (19 warps): warp 0 =
// bulk-copy producer (A panels resident per row group, B panels through an
// 8-stage ring), warps 1..2 = MMA issuers (even / odd tiles; warp-converged
// issue with an elected lane), warps 3..18 = two 8-warp epilogue groups, one
// per TMEM accumulator. Tile = 256 rows (two 128-row blocks, one 128x128x16
// MMA each per K step) x 128 columns; on the triangle the column walk starts
// at the row group, so no tile lies below the diagonal. Accumulators are
// double-buffered in TMEM (2 x 256 of the 512 columns) so the epilogue of
// tile t overlaps the MMAs of tile t+1. Epilogue warp w reads TMEM lanes
// 32*(w%4).. (its hardware lane quarter) of row block ((w-3)>>2)&1 with
// tcgen05.ld.32x32b.x32, sign bits -> four 32-bit words = the row's 128 bits
// of one bitmap block, written as one 16-byte store in the same
// bitmap/rowcnt format as the CUDA-core kernel (k3_pairs.cu), so the scan
// and emitter are shared.

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace refsig_gpu {
namespace {

constexpr uint32_t kTcThreads = 608;  // producer warp, 2 MMA warps, 16 epilogue warps
// Timing experiments (build with -DREFSIG_TC_TRACE; tools/tc_trace_run.py):
// REFSIG_TC_DEBUG bits 1 no epilogue math, 2 no B refill, 4 no MMA, 8 record
// per-tile clock64 events of CTA 0 (16: the last CTA) and print them.
#ifdef REFSIG_TC_TRACE
__device__ long long g_tc_trace[12][64];
__device__ __forceinline__ void tc_trace(const uint32_t dbg, int ev, uint32_t it) {
  if ((dbg & 8) && blockIdx.x == ((dbg & 16) ? gridDim.x - 1 : 0) && it < 64) g_tc_trace[ev][it] = clock64();
}
#define TC_DBG(a) ((a).dbg)
#else
__device__ __forceinline__ void tc_trace(uint32_t, int, uint32_t) {}
#define TC_DBG(a) 0u
#endif
// K' > 128: B streamed in chunks of kTcChunkK halves (16 KB per 128-doc
// panel) through up to kTcMaxStages stages.
constexpr uint32_t kTcChunkK = 64;
constexpr uint32_t kTcMaxStages = 16;
constexpr uint32_t kTcSmallKP = 128;  // tc_forms_kernel (shared-memory staging) up to K' = 128 (K <= 41)

// (b << 1) | (v >> 31) on the FMA pipe: mul.hi(v, 2) = v >> 31, then b*2 + that.
// `two` is a runtime 2 (kernel argument) so ptxas keeps IMADs instead of
// turning them into ALU shifts.
__device__ __forceinline__ uint32_t fma_pipe_shift_in(uint32_t b, uint32_t v, uint32_t two) {
  uint32_t s, r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(s) : "r"(v), "r"(two));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(two), "r"(s));
  return r;
}

// Valid-column mask for the 32 columns starting at lo in row i (k3_pairs.cu col_mask).
__device__ __forceinline__ uint32_t tc_col_mask(uint32_t lo, uint32_t i, const PairGrid& g) {
  uint32_t m = 0xffffffffu;
  if (lo >= g.n_cols) return 0u;
  if (lo + 32 > g.n_cols) m >>= (lo + 32 - g.n_cols);
  if (g.triangle && lo <= i) {
    const uint32_t first = i + 1 - lo;
    m = first >= 32 ? 0u : (m & (0xffffffffu << first));
  }
  return m;
}

struct TcArgs {
  const __half* Ar;  // row-form panels
  const __half* Bc;  // column-form panels
  uint32_t KP;       // K' (multiple of 16)
  uint32_t nch;      // K chunks per tile: kTcChunkK wide (4 MMA k-steps), the last one 1..4 k-steps
  uint32_t last_steps;
  uint32_t CB;       // bytes of one B chunk stage (128 docs x min(K', 64) halves)
  uint32_t rb;       // row blocks per row group: 2, or 1 when two A panels and a ring do not fit
  uint32_t abufs;    // A buffers: 2 (the next group's A loads during the current group) or 1
  PairGrid g;
  uint32_t nbr, nbc;     // 128-row / 128-column blocks
  uint32_t rb0, rb1;     // row blocks [rb0, rb1) of this call
  uint64_t n_tiles;
  uint32_t stages;
  uint32_t* bitmap;
  uint32_t* rowcnt;
  uint32_t two;  // 2, as data (see fma_pipe_shift_in)
  uint32_t dbg;  // timing experiments only (REFSIG_TC_DEBUG): 1 no epilogue math, 2 no B refill, 4 no MMA
  // rectangle (query x database) only: stripe-major walk. Item i = (column
  // stripe i / n_groups of `stripe` column blocks, row group i % n_groups);
  // CTA b takes items b, b + grid, ... so at any time the CTAs work on one or
  // two stripes and each B panel comes from DRAM about once (with contiguous
  // tile ranges per CTA every row group re-read the whole database from DRAM).
  uint32_t stripe;    // column blocks per stripe; 0 = contiguous tile ranges
  uint32_t n_groups;  // row groups of this call
};

// Row group p = row blocks rb0 + rb*p (.. + rb - 1): A resident in smem while
// the CTA walks the group's column blocks. Column blocks of group p: from its
// first row block on the triangle, all of them for a rectangle. (FS > 0: rb = 2
// at compile time, see mrc_tc_kernel.)
template <uint32_t FS>
__device__ __forceinline__ uint32_t tc_rb(const TcArgs& a) { return FS ? 2u : a.rb; }
template <uint32_t FS>
__device__ __forceinline__ uint32_t tc_r0(const TcArgs& a, uint32_t p) { return a.rb0 + tc_rb<FS>(a) * p; }
template <uint32_t FS>
__device__ __forceinline__ uint32_t tc_cs(const TcArgs& a, uint32_t p) { return a.g.triangle ? tc_r0<FS>(a, p) : 0u; }
template <uint32_t FS>
__device__ __forceinline__ uint32_t tc_ct(const TcArgs& a, uint32_t p) { return a.nbc - tc_cs<FS>(a, p); }
// row block r0 + h exists in this call
template <uint32_t FS>
__device__ __forceinline__ bool tc_rvalid(const TcArgs& a, uint32_t p, uint32_t h) {
  return h < tc_rb<FS>(a) && tc_r0<FS>(a, p) + h < a.rb1;
}

template <uint32_t FS, bool MC = false>
struct TileWalk {
  uint32_t p, c;        // row group, column block relative to tc_cs (absolute for a rectangle)
  uint32_t item, cend;  // stripe-major walk: current item, end column of its stripe
  bool ghost = false;   // MC: this CTA's half of the pair's item has no row group (odd count)
  // MC (CTA pairs sharing each B chunk by multicast): items are (stripe, pair of
  // row groups), walked by the cluster; rank r takes row group 2 gp + r
  __device__ void set_item(const TcArgs& a) {
    if constexpr (MC) {
      const uint32_t ngp = (a.n_groups + 1) / 2;
      const uint32_t st = item / ngp, gp = item % ngp;
      p = 2 * gp + (blockIdx.x & 1u);
      ghost = p >= a.n_groups;
      if (ghost) p = 2 * gp;  // valid operands, results discarded
      c = st * a.stripe;
    } else {
      const uint32_t st = item / a.n_groups;
      p = item % a.n_groups;
      c = st * a.stripe;
    }
    cend = min(c + a.stripe, a.nbc);
  }
  __device__ void start(const TcArgs& a, uint64_t t) {
    if (a.stripe) {
      item = MC ? blockIdx.x >> 1 : blockIdx.x;
      set_item(a);
      return;
    }
    p = 0;
    while (t >= tc_ct<FS>(a, p)) {
      t -= tc_ct<FS>(a, p);
      ++p;
    }
    c = static_cast<uint32_t>(t);
  }
  // returns true when the next tile starts a new row group (stripe-major: a new item)
  __device__ bool next(const TcArgs& a) {
    if (a.stripe) {
      if (++c == cend) {
        item += MC ? gridDim.x >> 1 : gridDim.x;
        set_item(a);
        return true;
      }
      return false;
    }
    if (++c == tc_ct<FS>(a, p)) {
      c = 0;
      ++p;
      return true;
    }
    return false;
  }
};

// Tiles of this CTA in the stripe-major walk (MC: of its pair).
template <bool MC = false>
__device__ __forceinline__ uint32_t tc_striped_tiles(const TcArgs& a) {
  const uint32_t ns = (a.nbc + a.stripe - 1) / a.stripe;
  const uint32_t ng = MC ? (a.n_groups + 1) / 2 : a.n_groups;
  const uint32_t i0 = MC ? blockIdx.x >> 1 : blockIdx.x, di = MC ? gridDim.x >> 1 : gridDim.x;
  uint32_t n = 0;
  for (uint32_t i = i0; i < ng * ns; i += di) {
    const uint32_t c0 = (i / ng) * a.stripe;
    n += min(a.stripe, a.nbc - c0);
  }
  return n;
}

// Tile = rb*128 rows (row group: A panels resident) x 128 columns (one B
// panel per tile, streamed through S stages in 64-wide K chunks, so
// K' is not bounded by the ring: K' = 208 at K = 64 is four chunks, K' = 400
// at K = 128 seven). Per K step: one N=128 MMA per valid row block into that
// block's 128 accumulator columns. FS > 0: K' = 16*FS <= 128 as ONE chunk
// (whole panel per stage), two row blocks and two A buffers, all compile-time
// (the MMA issue loop fully unrolled: at K = 20 the issuing thread's latency
// per MMA is on the critical path).
template <uint32_t FS, bool I8 = false, bool MC = false>
__global__ void __launch_bounds__(kTcThreads, 1) mrc_tc_kernel(TcArgs a) {
  static_assert(!MC || FS == 0, "B multicast is built for the chunked (K' > 128, single issuer) path");
  extern __shared__ __align__(1024) uint8_t tsm[];
  __shared__ __align__(8) uint64_t full_bar[kTcMaxStages], empty_bar[kTcMaxStages], afull_bar[2], aempty_bar[2], tfull_bar[2],
      tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  // warp index broadcast from lane 0: lets ptxas prove it warp-uniform, so the
  // MMA issuers keep descriptors and counters in uniform registers
  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
  const uint64_t t0 = a.n_tiles * blockIdx.x / gridDim.x, t1 = a.n_tiles * (blockIdx.x + 1) / gridDim.x;
  const uint32_t n_it = a.stripe ? tc_striped_tiles<MC>(a) : static_cast<uint32_t>(t1 - t0);
  const uint32_t crank = MC ? cluster_rank() : 0u;
  const uint32_t PB = 256u * a.KP;  // bytes per operand panel
  // B ring(s): every ring has ONE consumer taking its fills in order (with two
  // consumers of a shared ring, one could wait on a stage's fill k while fill
  // k-1 — the other's — was still in flight, and a parity wait then passes a
  // phase early). FS > 0: two issuers (even / odd tiles), stages [0, S0) and
  // [S0, S). FS == 0 (K' > 128, >= 13 MMAs per row block and tile): issuer 0
  // alone issues every tile from the whole ring; the MMAs themselves, not
  // the issue latency, bound the tile there.
  // (FS == 0 with two issuers and split rings measured 1-2% slower at c3 and
  // 16% slower at c4 once the issue path ran on uniform registers)
  constexpr bool kTwoIssuers = FS != 0;
  const uint32_t S = a.stages, S0 = kTwoIssuers ? (S + 1) / 2 : S, S1 = S - S0;
  const uint32_t NCH = FS ? 1u : a.nch, CB = FS ? PB : a.CB;
  const uint32_t ABUFS = FS ? 2u : a.abufs, RB = FS ? 2u : a.rb, LAST = FS ? FS : a.last_steps;
  constexpr uint32_t kStepsMax = FS ? FS : kTcChunkK / 16;  // k-steps per chunk
  uint8_t* sAbase = tsm;                      // ABUFS buffers x RB panels
  uint8_t* sBbase = tsm + ABUFS * RB * PB;    // S stages x one chunk
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mb_init(&full_bar[s], 1);
      mb_init(&empty_bar[s], MC ? 2 : 1);  // MC: both CTAs' MMA commits free a stage
    }
    for (int s = 0; s < 2; ++s) {
      mb_init(&afull_bar[s], 1);
      mb_init(&aempty_bar[s], 2);
      mb_init(&tfull_bar[s], 1);
      mb_init(&tempty_bar[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  if constexpr (MC) cluster_sync_all();  // the peer's barriers are initialised before any multicast
  pdl_wait();  // setup above overlaps the operand-forms kernel's tail

  if (warp == 0) {
    if (lane == 0 && n_it) {  // producer
      TileWalk<FS, MC> w;
      w.start(a, t0);
      uint32_t g = 0;  // row groups started by this CTA
      uint32_t qm[2] = {0, 0};  // B chunks issued into issuer m's ring
      bool new_group = true;
      for (uint32_t it = 0; it < n_it; ++it) {
        if (new_group) {  // A panels of the group into buffer g % abufs
          const uint32_t ab = g % ABUFS;
          if (g >= ABUFS) mb_wait(&aempty_bar[ab], ((g / ABUFS) - 1) & 1u);
          const uint32_t np = tc_rvalid<FS>(a, w.p, 1) ? 2u : 1u;
          mb_expect_tx(&afull_bar[ab], np * PB);
          bulk_g2s(sAbase + ab * RB * PB,
                   reinterpret_cast<const uint8_t*>(a.Ar) + static_cast<size_t>(tc_r0<FS>(a, w.p)) * PB, np * PB,
                   &afull_bar[ab]);
          ++g;
        }
        const uint32_t bj = tc_cs<FS>(a, w.p) + w.c;
        const uint8_t* src = reinterpret_cast<const uint8_t*>(a.Bc) + static_cast<size_t>(bj) * PB;
        const uint32_t m = kTwoIssuers ? (it & 1) : 0u, Sm = m ? S1 : S0, base = m ? S0 : 0u;
        uint32_t& q = qm[m];
        for (uint32_t ch = 0; ch < NCH; ++ch, ++q) {
          const uint32_t st = base + q % Sm;
          if (q >= Sm) mb_wait(&empty_bar[st], ((q / Sm) - 1) & 1u);
          const uint32_t bytes = ch + 1 < NCH ? CB : LAST * 4096u;
          if ((TC_DBG(a) & 2) && q >= Sm) {
            mb_arrive(&full_bar[st]);
          } else {
            mb_expect_tx(&full_bar[st], bytes);
            if constexpr (MC) {  // the leader's one copy fills both CTAs' stage
              if (crank == 0)
                bulk_g2s_mc(sBbase + static_cast<size_t>(st) * CB, src + static_cast<size_t>(ch) * CB, bytes,
                            &full_bar[st], 3);
            } else {
              bulk_g2s(sBbase + static_cast<size_t>(st) * CB, src + static_cast<size_t>(ch) * CB, bytes,
                       &full_bar[st]);
            }
          }
        }
        new_group = w.next(a);
      }
    }
    __syncwarp();
  } else if (warp == 1 || warp == 2) {
    // MMA issuers: warp 1 + m issues the tiles with it % 2 == m into
    // accumulator m (two threads in flight hide each one's issue latency;
    // FS == 0: warp 1 issues every tile, into accumulator it % 2); whole warp
    // converged, one elected lane issues
    const uint32_t m = warp - 1;
    if (n_it) {
      TileWalk<FS, MC> w;
      w.start(a, t0);
      const uint64_t dA0 = smem_desc(smem_u32(sAbase)), dB0 = smem_desc(smem_u32(sBbase));
      const uint64_t dPB = PB >> 4, dCB = CB >> 4;
      const uint32_t Sm = m ? S1 : S0, base = m ? S0 : 0u;  // this issuer's ring
      uint32_t g = 0, q = 0;
      bool new_group = true;
      for (uint32_t it = 0; it < n_it; ++it) {
        if (new_group) {
          mb_wait_warp(&afull_bar[g % ABUFS], (g / ABUFS) & 1u);
          ++g;
        }
        const uint32_t ab = (g - 1) % ABUFS;
        const uint32_t acc = it & 1;
        if (kTwoIssuers ? acc == m : m == 0) {
          const uint32_t bj = tc_cs<FS>(a, w.p) + w.c;
          const uint32_t r0 = tc_r0<FS>(a, w.p);
          const bool v1 = tc_rvalid<FS>(a, w.p, 1) && !(a.g.triangle && bj < r0 + 1);
          if (lane == 0 && m == 0) tc_trace(TC_DBG(a), 0, it);
          if (it >= 2) mb_wait_warp(&tempty_bar[acc], ((it >> 1) - 1) & 1u);
          if (lane == 0 && m == 0) tc_trace(TC_DBG(a), 2, it);
          const uint64_t dA = dA0 + ab * RB * dPB;
          const uint32_t d0 = tmem + acc * 256;
          for (uint32_t ch = 0; ch < NCH; ++ch, ++q) {
            const uint32_t st = base + q % Sm;
            mb_wait_warp(&full_bar[st], (q / Sm) & 1u);
            const uint32_t e = elect_one();
            if (lane == 0 && m == 0 && ch == 0) tc_trace(TC_DBG(a), 1, it);
            tc_fence_after();
            const uint32_t steps = ch + 1 < NCH ? kStepsMax : LAST;
            const uint64_t dB = dB0 + st * dCB, dAc = dA + ch * kStepsMax * 256u;
            if (!(TC_DBG(a) & 4)) {
#pragma unroll
              for (uint32_t j = 0; j < kStepsMax; ++j) {
                if (j < steps) {
                  if constexpr (I8) {  // Hamming: +-1 int8 operands, s32 accumulators (same bytes per step)
                    mma_i8_e(e, d0, dAc + j * 256, dB + j * 256, (ch | j) != 0);
                    if (v1) mma_i8_e(e, d0 + 128, dAc + dPB + j * 256, dB + j * 256, (ch | j) != 0);
                  } else {
                    mma_f16_e(e, d0, dAc + j * 256, dB + j * 256, (ch | j) != 0);
                    if (v1) mma_f16_e(e, d0 + 128, dAc + dPB + j * 256, dB + j * 256, (ch | j) != 0);
                  }
                }
              }
            }
            if constexpr (MC)
              mma_commit_mc_e(e, &empty_bar[st], 3);  // both CTAs' producers wait on this stage
            else
              mma_commit_e(e, &empty_bar[st]);
          }
          if (lane == 0 && m == 0) tc_trace(TC_DBG(a), 3, it);
          __syncwarp();
          mma_commit_e(elect_one(), &tfull_bar[acc]);
        }
        new_group = w.next(a);
        // both issuers release the group's A buffer (a commit with nothing
        // outstanding from this thread arrives at once)
        __syncwarp();
        if (new_group || it + 1 == n_it) mma_commit_e(elect_one(), &aempty_bar[ab]);
        __syncwarp();
      }
    }
    __syncwarp();
  } else {  // epilogue warps 3..18: group eg = tiles with it % 2 == eg (accumulator eg),
             // lane quarter q, row block h of the row group; all 128 columns in two halves
    const uint32_t ew = threadIdx.x >> 5;  // (not the uniform copy: the epilogue measured faster this way)
    const uint32_t q = ew & 3, eg = (ew - 3) >> 3, h = ((ew - 3) >> 2) & 1;
    const uint32_t wpr = a.g.words_per_row;
    const uint32_t two = a.two;
    TileWalk<FS, MC> w;
    if (n_it) w.start(a, t0);
    uint32_t cnt = 0;
    for (uint32_t it = 0; it < n_it; ++it) {
      const uint32_t acc = it & 1;
      const uint32_t p = w.p;
      const uint32_t r = tc_r0<FS>(a, p) + h;
      const uint32_t bj = tc_cs<FS>(a, p) + w.c;
      const uint32_t i = r * 128 + q * 32 + lane;
      if (acc == eg) {
        const uint32_t u = it >> 1;  // this group's use count of its accumulator
        if (warp == 3 && lane == 0) tc_trace(TC_DBG(a), 4, it);
        mb_wait_warp(&tfull_bar[acc], u & 1u);
        if (warp == 3 && lane == 0) tc_trace(TC_DBG(a), 5, it);
        tc_fence_after();
        const bool valid = tc_rvalid<FS>(a, p, h) && !(a.g.triangle && bj < r) && !w.ghost;
        const bool edge = (a.g.triangle && bj == r) || bj + 1 == a.nbc;
        uint32_t mw[4];
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t v0[32], v1[32];
          if (valid) {
            const uint32_t ta = tmem + ((q * 32u) << 16) + acc * 256 + h * 128 + half * 64;
            TC_LD32(ta, v0);
            TC_LD32(ta + 32, v1);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          }
          if (warp == 3 && lane == 0) tc_trace(TC_DBG(a), 8 + 2 * half, it);
          if (half == 1) {  // accumulator fully read: hand it back to the MMA issuer
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mb_arrive(&tempty_bar[acc]);
            if (warp == 3 && lane == 0) tc_trace(TC_DBG(a), 6, it);
          }
          if (valid && !(TC_DBG(a) & 1)) {
            // bit c = sign(dot - tau) of column c: eight independent 8-deep
            // chains (one per byte), then bytes -> words with PRMT. Bytes 0-2 of
            // each word use the ALU funnel shift (1 op per bit), byte 3 the FMA
            // pipe (IMAD.HI gives v >> 31, IMAD appends it: 2 ops per bit), so
            // the two 2-cycle pipes share the per-pair work ~48:32 instead of
            // 64:0 cycles per 32 pairs.
            uint32_t b[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) b[k] = 0;
#pragma unroll
            for (int c = 7; c >= 0; --c) {
#pragma unroll
              for (int k = 0; k < 3; ++k) {
                b[k] = __funnelshift_l(v0[8 * k + c], b[k], 1);
                b[4 + k] = __funnelshift_l(v1[8 * k + c], b[4 + k], 1);
              }
              b[3] = fma_pipe_shift_in(b[3], v0[24 + c], two);
              b[7] = fma_pipe_shift_in(b[7], v1[24 + c], two);
            }
            mw[2 * half] = ~__byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
            mw[2 * half + 1] = ~__byte_perm(__byte_perm(b[4], b[5], 0x0040), __byte_perm(b[6], b[7], 0x0040), 0x5410);
          }
          if (warp == 3 && lane == 0) tc_trace(TC_DBG(a), 9 + 2 * half, it);
        }
        if (valid && !(TC_DBG(a) & 1)) {
          if (edge) {
            const uint32_t c0 = bj * 128;
#pragma unroll
            for (int k = 0; k < 4; ++k) mw[k] &= tc_col_mask(c0 + 32 * k, i, a.g);
          }
          if (i < a.g.n_rows) {
            *reinterpret_cast<uint4*>(a.bitmap + static_cast<size_t>(i) * wpr + bj * 4) =
                make_uint4(mw[0], mw[1], mw[2], mw[3]);
            cnt += __popc(mw[0]) + __popc(mw[1]) + __popc(mw[2]) + __popc(mw[3]);
          }
        }
        if (warp == 3 && lane == 0) tc_trace(TC_DBG(a), 7, it);
      }
      if (w.next(a) || it + 1 == n_it) {
        if (cnt && i < a.g.n_rows) atomicAdd(a.rowcnt + i, cnt);
        cnt = 0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (MC) cluster_sync_all();  // no multicast copy or commit still targets this CTA
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// ---- K3 on CTA pairs (cta_group::2), chunked K' > 128, query rectangle ----
// The pair (cluster of 2 CTAs on one TPC) computes 256 rows x 128 columns per
// tile with ONE tcgen05.mma.cta_group::2 per K step (M = 256): each CTA holds
// its own 128-row A block (resident per item) and HALF of each B chunk — 64
// columns, from column forms laid out as 64-document panels — and its TMEM
// receives its 128 rows x all 128 columns (CUTLASS SM100_MMA_F16BF16_2x1SM_SS
// split). So every SM ingests half the B bytes per flop of the one-CTA rb = 1
// kernel (whose per-SM share of L2 bandwidth bounded the configs[4] join).
// The leader (rank 0) issues the MMAs; the peer's copies land in the peer's
// own barriers, so a forwarder thread of the peer re-arrives each completed
// fill on the leader's pair barriers (remote mbarrier arrive), and another
// forwards the peer epilogue's accumulator releases. Commits from the leader
// multicast to both CTAs (ring stages, A buffers, accumulators).
// Items: (column stripe, row-group pair) as in the stripe-major walk; rank r
// takes row block 2 gp + r (a ghost half without stores when the count is odd).
constexpr uint32_t kTc2ChunkK = 64;  // K halves per B stage: 8 KB of a 64-doc half panel (16 KB stages, 7 of
                                     // them, measured 7.40 vs 6.92 ms at configs[4])
constexpr uint32_t kTc2ChunkBytes = 64u * kTc2ChunkK * 2u;

struct Tc2Walk {
  uint32_t p, c, item, cend, gp;  // p: this CTA's row block (relative to rb0), c: absolute column block
  bool ghost;
  // rectangle: stripe-major items (stripe, row-block pair gp); triangle: the pair's contiguous range of
  // pair tiles, pair group gp = row blocks rb0 + 2 gp (+1), columns from rb0 + 2 gp (the lower block;
  // the upper block's tile on that column lies below the diagonal and is masked)
  __device__ uint32_t tri_cs(const TcArgs& a, uint32_t g) const { return a.rb0 + 2 * g; }
  __device__ void set_rows(const TcArgs& a) {
    p = 2 * gp + (blockIdx.x & 1u);
    ghost = a.rb0 + p >= a.rb1;
    if (ghost) p = 2 * gp;  // valid operands, results discarded
  }
  __device__ void set_item(const TcArgs& a) {
    const uint32_t ngp = (a.n_groups + 1) / 2;
    const uint32_t st = item / ngp;
    gp = item % ngp;
    set_rows(a);
    c = st * a.stripe;
    cend = min(c + a.stripe, a.nbc);
  }
  __device__ void start(const TcArgs& a, uint64_t t) {
    if (a.g.triangle) {
      gp = 0;
      while (t >= a.nbc - tri_cs(a, gp)) {
        t -= a.nbc - tri_cs(a, gp);
        ++gp;
      }
      set_rows(a);
      c = tri_cs(a, gp) + static_cast<uint32_t>(t);
      cend = a.nbc;
      return;
    }
    item = blockIdx.x >> 1;
    set_item(a);
  }
  __device__ bool next(const TcArgs& a) {
    if (++c == cend) {
      if (a.g.triangle) {
        ++gp;
        set_rows(a);
        c = tri_cs(a, gp);
      } else {
        item += gridDim.x >> 1;
        set_item(a);
      }
      return true;
    }
    return false;
  }
};

__global__ void __launch_bounds__(kTcThreads, 1) mrc_tc2_kernel(TcArgs a, const __grid_constant__ CUtensorMap bmap) {
  extern __shared__ __align__(1024) uint8_t tsm[];
  constexpr uint32_t NACC = 4;  // 4 x 128 TMEM columns: the MMAs run up to three tiles ahead of the epilogues
  __shared__ __align__(8) uint64_t full_bar[kTcMaxStages], empty_bar[kTcMaxStages], afull_bar[2],
      pafull_bar[2], aempty_bar[2], tfull_bar[NACC], tempty_bar[NACC], ptempty_bar[NACC];
  __shared__ uint32_t tmem_base_sh;
  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const uint32_t npairs = gridDim.x >> 1, pair = blockIdx.x >> 1;
  const uint64_t pt0 = a.n_tiles * pair / npairs, pt1 = a.n_tiles * (pair + 1) / npairs;  // triangle: pair tiles
  const uint32_t n_it = a.g.triangle ? static_cast<uint32_t>(pt1 - pt0) : tc_striped_tiles<true>(a);
  const uint32_t PB = 256u * a.KP;                    // bytes of one 128-row A panel
  const uint32_t S = a.stages, NCH = a.nch, ABUFS = a.abufs, LAST = a.last_steps;
  uint8_t* sAbase = tsm;                               // ABUFS A panels
  uint8_t* sBbase = tsm + ABUFS * PB;                  // S stages x 8 KB half chunks
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mb_init(&full_bar[s], 1);
      mb_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mb_init(&afull_bar[s], 1);
      mb_init(&pafull_bar[s], 1);
      mb_init(&aempty_bar[s], 1);
    }
    for (uint32_t s = 0; s < NACC; ++s) {
      mb_init(&tfull_bar[s], 1);
      mb_init(&tempty_bar[s], 8);
      mb_init(&ptempty_bar[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // the same warp in both CTAs (cta_group::2 allocation)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  pdl_wait();

  if (warp == 0) {
    if (lane == 0 && n_it) {  // producer (both CTAs): own A block, own B halves
      Tc2Walk w;
      w.start(a, pt0);
      uint32_t g = 0, q = 0;
      bool new_group = true;
      for (uint32_t it = 0; it < n_it; ++it) {
        if (new_group) {
          const uint32_t ab = g % ABUFS;
          if (g >= ABUFS) mb_wait_cluster(&aempty_bar[ab], ((g / ABUFS) - 1) & 1u);
          mb_expect_tx(&afull_bar[ab], PB);
          bulk_g2s(sAbase + ab * PB, reinterpret_cast<const uint8_t*>(a.Ar) + static_cast<size_t>(a.rb0 + w.p) * PB,
                   PB, &afull_bar[ab]);
          ++g;
        }
        // the 64-document half panel 2 bj + rank of the column forms, one 8 KB box per K chunk by
        // TMA with .cta_group::2: both CTAs' boxes complete the LEADER's stage barrier (peer bit
        // cleared), so no forwarding sits in the refill chain
        const uint32_t c_base = (2 * w.c + rank) * (a.KP / 8);
        const uint32_t bar_mask = 0xFEFFFFFFu;
        for (uint32_t ch = 0; ch < NCH; ++ch, ++q) {
          const uint32_t st = q % S;
          if (q >= S) mb_wait_cluster(&empty_bar[st], ((q / S) - 1) & 1u);
          if (rank == 0) mb_expect_tx(&full_bar[st], 2u * kTc2ChunkBytes);
          asm volatile(
              "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(sBbase + static_cast<size_t>(st) * kTc2ChunkBytes)),
              "l"(reinterpret_cast<uint64_t>(&bmap)), "r"(smem_u32(&full_bar[st]) & bar_mask), "r"(0),
              "r"((c_base + ch * (kTc2ChunkK / 8)) * 2u)  // 1 KB chunks = two 512-byte rows
              : "memory");
        }
        new_group = w.next(a);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (n_it && rank == 0) {  // leader: the MMA issuer
      Tc2Walk w;
      w.start(a, pt0);
      const uint64_t dA0 = smem_desc(smem_u32(sAbase));
      const uint64_t dB0 = smem_desc_lbo(smem_u32(sBbase), 1024u);
      const uint64_t dPB = PB >> 4, dCB = kTc2ChunkBytes >> 4;
      uint32_t g = 0, q = 0;
      bool new_group = true;
      for (uint32_t it = 0; it < n_it; ++it) {
        if (new_group) {
          mb_wait(&afull_bar[g % ABUFS], (g / ABUFS) & 1u);
          mb_wait_cluster(&pafull_bar[g % ABUFS], (g / ABUFS) & 1u);
          __syncwarp();
          ++g;
        }
        const uint32_t ab = (g - 1) % ABUFS;
        const uint32_t acc = it % NACC;
        if (it >= NACC) {
          mb_wait(&tempty_bar[acc], ((it / NACC) - 1) & 1u);
          mb_wait_cluster(&ptempty_bar[acc], ((it / NACC) - 1) & 1u);
          __syncwarp();
        }
        const uint64_t dA = dA0 + ab * dPB;
        const uint32_t d0 = tmem + acc * 128;
        for (uint32_t ch = 0; ch < NCH; ++ch, ++q) {
          const uint32_t st = q % S;
          mb_wait_cluster(&full_bar[st], (q / S) & 1u);  // both halves (the peer's box completes it too)
          __syncwarp();
          const uint32_t e = elect_one();
          tc_fence_after();
          const uint32_t steps = ch + 1 < NCH ? kTc2ChunkK / 16 : LAST;
          const uint64_t dB = dB0 + st * dCB, dAc = dA + ch * (kTc2ChunkK / 16) * 256u;
          if (!(a.dbg & 4)) {
#pragma unroll
            for (uint32_t j = 0; j < kTc2ChunkK / 16; ++j)
              if (j < steps) mma2_f16_e(e, d0, dAc + j * 256, dB + j * 128, (ch | j) != 0);
          }
          mma2_commit_mc_e(e, &empty_bar[st], 3);
        }
        __syncwarp();
        mma2_commit_mc_e(elect_one(), &tfull_bar[acc], 3);
        new_group = w.next(a);
        __syncwarp();
        if (new_group || it + 1 == n_it) mma2_commit_mc_e(elect_one(), &aempty_bar[ab], 3);
        __syncwarp();
      }
    } else if (n_it && lane == 0) {  // peer: forward A / B fill completions to the leader
      Tc2Walk w;
      w.start(a, pt0);
      uint32_t g = 0;
      bool new_group = true;
      for (uint32_t it = 0; it < n_it; ++it) {
        if (new_group) {
          mb_wait(&afull_bar[g % ABUFS], (g / ABUFS) & 1u);
          mb_arrive_remote(&pafull_bar[g % ABUFS], 0);
          ++g;
        }
        new_group = w.next(a);
      }
    }
    __syncwarp();
  } else if (warp == 2) {
    if (n_it && rank == 1 && lane == 0) {  // peer: forward accumulator releases to the leader
      for (uint32_t it = 0; it + NACC < n_it; ++it) {  // the leader waits releases of tiles 0 .. n_it - 1 - NACC
        const uint32_t acc = it % NACC;
        mb_wait(&tempty_bar[acc], (it / NACC) & 1u);
        mb_arrive_remote(&ptempty_bar[acc], 0);
      }
    }
    __syncwarp();
  } else {  // epilogue warps 3..18: group eg (accumulator it % 2), lane quarter q, column half h
    const uint32_t ew = threadIdx.x >> 5;
    const uint32_t q = ew & 3, eg = (ew - 3) >> 3, h = ((ew - 3) >> 2) & 1;
    const uint32_t wpr = a.g.words_per_row;
    const uint32_t two = a.two;
    Tc2Walk w;
    if (n_it) w.start(a, pt0);
    uint32_t cnt = 0;
    for (uint32_t it = 0; it < n_it; ++it) {
      const uint32_t acc = it % NACC;
      const uint32_t r = a.rb0 + w.p;
      const uint32_t bj = w.c;
      const uint32_t i = r * 128 + q * 32 + lane;
      if ((it & 1) == eg) {
        mb_wait_warp(&tfull_bar[acc], (it / NACC) & 1u);
        tc_fence_after();
        const bool valid = !w.ghost && r < a.rb1 && !(a.g.triangle && bj < r);
        uint32_t v0[32], v1[32];
        const uint32_t ta = tmem + ((q * 32u) << 16) + acc * 128 + h * 64;
        TC_LD32(ta, v0);
        TC_LD32(ta + 32, v1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mb_arrive(&tempty_bar[acc]);
        if (valid && !(a.dbg & 1)) {
          uint32_t b[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) b[k] = 0;
#pragma unroll
          for (int c = 7; c >= 0; --c) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              b[k] = __funnelshift_l(v0[8 * k + c], b[k], 1);
              b[4 + k] = __funnelshift_l(v1[8 * k + c], b[4 + k], 1);
            }
            b[3] = fma_pipe_shift_in(b[3], v0[24 + c], two);
            b[7] = fma_pipe_shift_in(b[7], v1[24 + c], two);
          }
          uint32_t m0 = ~__byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
          uint32_t m1 = ~__byte_perm(__byte_perm(b[4], b[5], 0x0040), __byte_perm(b[6], b[7], 0x0040), 0x5410);
          if ((a.g.triangle && bj == r) || bj + 1 == a.nbc) {
            const uint32_t c0 = bj * 128 + h * 64;
            m0 &= tc_col_mask(c0, i, a.g);
            m1 &= tc_col_mask(c0 + 32, i, a.g);
          }
          if (i < a.g.n_rows) {
            *reinterpret_cast<uint2*>(a.bitmap + static_cast<size_t>(i) * wpr + bj * 4 + h * 2) = make_uint2(m0, m1);
            cnt += __popc(m0) + __popc(m1);
          }
        }
      }
      if (w.next(a) || it + 1 == n_it) {
        if (cnt && i < a.g.n_rows) atomicAdd(a.rowcnt + i, cnt);
        cnt = 0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no commit or remote arrive still targets this CTA
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// Hamming on the tensor cores: with s = 2x - 1 in {-1, +1}^64 per
// fingerprint, s_a . s_b = 64 - 2 hd(a, b), so hd <= max_dist <=> s_a . s_b -
// (64 - 2 max_dist) >= 0 — an exact int8 MMA with s32 accumulators and the
// same folded-threshold trick as the MRC compare: row form [s_a | -thr | 0..],
// column form [s_b | 1 | 0..], K' = 96 bytes (three K=32 int8 steps), stored
// in the f16 kernel's panel layout (16-byte chunks [6][128 docs]), so the
// tile kernel and its sign-bit epilogue are reused unchanged.
constexpr uint32_t kHamKPBytes = 96;
__global__ void __launch_bounds__(256) ham_forms_kernel(const uint64_t* __restrict__ fp, uint32_t n, int thr,
                                                        uint8_t* __restrict__ rowf, uint8_t* __restrict__ colf) {
  // thread (chunk kc, doc dl) of panel blockIdx.x: 16 bytes at [kc][dl]
  const uint32_t pan = blockIdx.x;
  for (uint32_t idx = threadIdx.x; idx < 6 * 128; idx += blockDim.x) {
    const uint32_t kc = idx >> 7, dl = idx & 127, d = pan * 128 + dl;
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    uint32_t wr[4] = {0u, 0u, 0u, 0u};
    if (d < n) {
      if (kc < 4) {
        const uint32_t bits = static_cast<uint32_t>(fp[d] >> (16 * kc)) & 0xffffu;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t nib = (bits >> (4 * q)) & 0xfu;
          const uint32_t y = (nib * 0x00204081u) & 0x01010101u;  // bit t of the nibble -> byte t = 0 / 1
          w[q] = y | ((y ^ 0x01010101u) * 0xffu);                 // 1 -> +1 (0x01), 0 -> -1 (0xff)
          wr[q] = w[q];
        }
      } else if (kc == 4) {
        wr[0] = static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(-thr)));
        w[0] = 1u;
      }
    }
    const size_t off = (static_cast<size_t>(pan) * 6 * 128 + static_cast<size_t>(kc) * 128 + dl) * 16;
    if (rowf) *reinterpret_cast<uint4*>(rowf + off) = make_uint4(wr[0], wr[1], wr[2], wr[3]);
    if (colf) *reinterpret_cast<uint4*>(colf + off) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Row form [hi | hi | lo | -tau pieces] or column form [hi | lo | hi | 1 1 1]
// of every document, panel layout (see the top comment). CTA per 128-doc
// panel: threads convert ST[k][d] (coalesced along d) once into both forms
// in shared memory ([doc][K'] halves, row stride padded by 8 halves), then
// write each panel as 16-byte chunks in [chunk][doc] order (coalesced).
__global__ void __launch_bounds__(256) tc_forms_kernel(const float* __restrict__ ST, uint32_t ld, uint32_t n_docs,
                                                       uint32_t K, uint32_t KP, float tau, __half* __restrict__ rowf,
                                                       __half* __restrict__ colf, uint32_t* __restrict__ rowcnt,
                                                       uint32_t n_rowcnt, uint32_t col64) {
  extern __shared__ __align__(16) __half fsm[];
  pdl_wait();
  // the tile kernel's row counts start at zero: zeroed here, 128 per panel (no memset node before this PDL launch)
  if (rowcnt && threadIdx.x < 128 && blockIdx.x * 128 + threadIdx.x < n_rowcnt) rowcnt[blockIdx.x * 128 + threadIdx.x] = 0;
  const uint32_t stride = KP + 8;  // halves per doc row (16-byte aligned, staggers banks)
  __half* R = fsm;
  __half* C = fsm + 128 * stride;
  const uint32_t pan = blockIdx.x, d0 = pan * 128;
  const __half t0 = __float2half_rn(tau);
  const float r1 = tau - __half2float(t0);
  const __half t1 = __float2half_rn(r1);
  const __half t2 = __float2half_rn(r1 - __half2float(t1));
  const __half one = __float2half_rn(1.0f), zero = __float2half_rn(0.0f);
  {
    // thread (dl, k0): values k0, k0 + 2, ... of doc d0 + dl; all loads issued before any use
    constexpr uint32_t kPer = (kTcSmallKP / 3 + 1) / 2 + 1;  // ceil(41 / 2)
    const uint32_t dl = threadIdx.x & 127, k0 = threadIdx.x >> 7, d = d0 + dl;
    float v[kPer];
#pragma unroll
    for (uint32_t u = 0; u < kPer; ++u) {
      const uint32_t k = k0 + 2 * u;
      v[u] = (k < K && d < n_docs) ? ST[static_cast<size_t>(k) * ld + d] : 0.0f;
    }
    __half* rr = R + dl * stride;
    __half* cc = C + dl * stride;
#pragma unroll
    for (uint32_t u = 0; u < kPer; ++u) {
      const uint32_t k = k0 + 2 * u;
      if (k < K) {
        const __half hi = __float2half_rn(v[u]);
        const __half lo = __float2half_rn(v[u] - __half2float(hi));
        rr[k] = hi;
        rr[K + k] = hi;
        rr[2 * K + k] = lo;
        cc[k] = hi;
        cc[K + k] = lo;
        cc[2 * K + k] = hi;
      }
    }
  }
  for (uint32_t idx = threadIdx.x; idx < (KP - 3 * K) * 128; idx += blockDim.x) {
    const uint32_t j = idx >> 7, dl = idx & 127, p = 3 * K + j;
    __half rv = zero, cv = zero;
    if (j < 3) {
      const __half tj = j == 0 ? t0 : (j == 1 ? t1 : t2);
      rv = __half2float(tj) == 0.0f ? zero : __hneg(tj);  // +0, never -0: tau = 0 keeps dot = 0 a match
      cv = one;
    }
    R[dl * stride + p] = rv;
    C[dl * stride + p] = cv;
  }
  __syncthreads();
  const uint32_t chunks = KP / 8;
  const size_t base = static_cast<size_t>(pan) * chunks * 128 * 8;
  for (uint32_t idx = threadIdx.x; idx < chunks * 128; idx += blockDim.x) {
    const uint32_t kc = idx >> 7, dl = idx & 127;
    const size_t off = base + (static_cast<size_t>(kc) * 128 + dl) * 8;
    if (rowf) *reinterpret_cast<uint4*>(rowf + off) = *reinterpret_cast<const uint4*>(R + dl * stride + kc * 8);
    if (colf) {  // col64: 64-document panels (the B halves of the CTA-pair kernel)
      const size_t o = col64 ? (static_cast<size_t>(2 * pan + (dl >> 6)) * chunks + kc) * 64 * 8 +
                                   static_cast<size_t>(dl & 63) * 8
                             : off;
      *reinterpret_cast<uint4*>(colf + o) = *reinterpret_cast<const uint4*>(C + dl * stride + kc * 8);
    }
  }
}

// Any K': thread (8-value chunk kc, doc dl) computes its 8 halves of both
// forms straight from ST (reads coalesced along d; each ST value is read by
// the three chunks that hold its hi / lo copies) and stores 16 bytes at
// [kc][dl] (coalesced). Grid: (panels, ceil(K'/8 / 2)), 256 threads.
__global__ void __launch_bounds__(256) tc_forms_any_kernel(const float* __restrict__ ST, uint32_t ld, uint32_t n_docs,
                                                           uint32_t K, uint32_t KP, float tau,
                                                           __half* __restrict__ rowf, __half* __restrict__ colf,
                                                           uint32_t* __restrict__ rowcnt, uint32_t n_rowcnt,
                                                           uint32_t col64) {
  const uint32_t pan = blockIdx.x, dl = threadIdx.x & 127, kc = blockIdx.y * 2 + (threadIdx.x >> 7);
  pdl_wait();
  if (rowcnt && blockIdx.y == 0 && threadIdx.x < 128 && pan * 128 + threadIdx.x < n_rowcnt) rowcnt[pan * 128 + threadIdx.x] = 0;
  if (kc * 8 >= KP) return;
  const uint32_t d = pan * 128 + dl;
  const __half t0 = __float2half_rn(tau);
  const float r1 = tau - __half2float(t0);
  const __half t1 = __float2half_rn(r1);
  const __half t2 = __float2half_rn(r1 - __half2float(t1));
  __align__(16) __half rv[8], cv[8];
#pragma unroll
  for (uint32_t e = 0; e < 8; ++e) {
    const uint32_t pos = kc * 8 + e;
    __half r = __float2half_rn(0.0f), c = r;
    if (pos < 3 * K) {
      const uint32_t seg = pos / K, k = pos - seg * K;
      const float v = d < n_docs ? ST[static_cast<size_t>(k) * ld + d] : 0.0f;
      const __half hi = __float2half_rn(v);
      const __half lo = __float2half_rn(v - __half2float(hi));
      r = seg == 2 ? lo : hi;  // row form [hi | hi | lo]
      c = seg == 1 ? lo : hi;  // column form [hi | lo | hi]
    } else if (pos < 3 * K + 3) {
      const uint32_t j = pos - 3 * K;
      const __half tj = j == 0 ? t0 : (j == 1 ? t1 : t2);
      r = __half2float(tj) == 0.0f ? __float2half_rn(0.0f) : __hneg(tj);  // +0, never -0
      c = __float2half_rn(1.0f);
    }
    rv[e] = r;
    cv[e] = c;
  }
  const size_t off = (static_cast<size_t>(pan) * (KP / 8) + kc) * 128 * 8 + static_cast<size_t>(dl) * 8;
  if (rowf) *reinterpret_cast<uint4*>(rowf + off) = *reinterpret_cast<const uint4*>(rv);
  if (colf) {  // col64: 64-document panels (the B halves of the CTA-pair kernel)
    const size_t o = col64 ? (static_cast<size_t>(2 * pan + (dl >> 6)) * (KP / 8) + kc) * 64 * 8 +
                                 static_cast<size_t>(dl & 63) * 8
                           : off;
    *reinterpret_cast<uint4*>(colf + o) = *reinterpret_cast<const uint4*>(cv);
  }
}

// Shared-memory plan of mrc_tc_kernel for a K': row blocks per group, A
// buffers and B chunk stages (false when fewer than 3 stages fit).
constexpr uint32_t kTcSmemBudget = 225u * 1024u;
struct TcPlan {
  uint32_t rb, abufs, stages, CB;
  size_t smem;
};
bool tc_plan(uint32_t KP, TcPlan& pl) {
  const uint32_t PB = 256u * KP;
  if (KP <= kTcSmallKP) {  // one chunk = the whole panel: 2 x 2 resident A panels + S panels
    pl.rb = pl.abufs = 2;
    pl.CB = PB;
    pl.stages = std::max<uint32_t>(2u, std::min<uint32_t>(8u, (kTcSmemBudget - 4u * PB) / PB));
    pl.smem = std::max<size_t>(static_cast<size_t>(4 + pl.stages) * PB, 116u * 1024u);
    return true;
  }
  pl.CB = 256u * kTcChunkK;
  if (4u * PB + 4u * pl.CB <= kTcSmemBudget) {
    pl.rb = 2;
    pl.abufs = 2;
  } else if (2u * PB + 4u * pl.CB <= kTcSmemBudget) {
    pl.rb = 2;
    pl.abufs = 1;
  } else {
    pl.rb = 1;
    pl.abufs = (2u * PB + 4u * pl.CB <= kTcSmemBudget) ? 2u : 1u;
  }
  const uint32_t a_bytes = pl.abufs * pl.rb * PB;
  if (a_bytes + 4u * pl.CB > kTcSmemBudget) return false;  // >= 2 stages per issuer ring
  pl.stages = std::min<uint32_t>(kTcMaxStages, (kTcSmemBudget - a_bytes) / pl.CB);
  // at least ~116 KB so that exactly one CTA (the TMEM owner of all 512 columns) fits per SM
  pl.smem = std::max<size_t>(static_cast<size_t>(a_bytes) + static_cast<size_t>(pl.stages) * pl.CB, 116u * 1024u);
  return true;
}

}  // namespace

uint32_t mrc_tc_kp(uint32_t K) { return ((3 * K + 3) + 15) / 16 * 16; }

bool mrc_tc_supported(uint32_t K, float tau) {
  // fp16 pieces of tau: |tau| < 65504, and tau = 0 or |tau| >= 2^-14 (fp16
  // normal) so that the leading piece is nonzero and a zero signature never
  // matches a positive tau; the resident A panels plus 3+ B chunk stages fit
  // in shared memory (K <= 234; K = 128 -> K' = 400)
  const float at = fabsf(tau);
  TcPlan pl;
  return K >= 1 && tc_plan(mrc_tc_kp(K), pl) && at < 60000.0f && (at == 0.0f || at >= 6.103515625e-05f);
}

size_t mrc_tc_form_bytes(uint32_t K, uint32_t n_docs) {
  return static_cast<size_t>(ceil_div(n_docs, 128)) * 256u * mrc_tc_kp(K);
}

void launch_mrc_tc_forms(const float* ST, uint32_t ld, uint32_t n_docs, uint32_t K, float tau, void* rowf, void* colf,
                         uint32_t* rowcnt, uint32_t n_rowcnt, cudaStream_t s, bool col64) {
  const uint32_t KP = mrc_tc_kp(K);
  const uint32_t n_pan = static_cast<uint32_t>(ceil_div(n_docs, 128));
  if (!n_pan) return;
  if (KP > kTcSmallKP) {
    const dim3 grid(n_pan, static_cast<unsigned>(ceil_div(KP / 8, 2)));
    launch_pdl(tc_forms_any_kernel, grid, dim3(256), 0, s, ST, ld, n_docs, K, KP, tau, static_cast<__half*>(rowf),
               static_cast<__half*>(colf), rowcnt, n_rowcnt, col64 ? 1u : 0u);
    note_launch();
    return;
  }
  const size_t smem = 2ull * 128 * (KP + 8) * sizeof(__half);  // <= 69.6 KB at K' = 128
  ensure_smem(tc_forms_kernel, 72 * 1024);
  launch_pdl(tc_forms_kernel, dim3(n_pan), dim3(256), smem, s, ST, ld, n_docs, K, KP, tau, static_cast<__half*>(rowf),
             static_cast<__half*>(colf), rowcnt, n_rowcnt, col64 ? 1u : 0u);
  note_launch();
}

// The tile kernel over operand panels of K' = KP halves (i8: 2*KP int8 values).
static void launch_tc_tiles(const void* rowf, const void* colf, uint32_t KP, const PairGrid& g, uint32_t* bitmap,
                            uint32_t* rowcnt, cudaStream_t s, bool i8) {
  TcArgs a{};
  a.Ar = static_cast<const __half*>(rowf);
  a.Bc = static_cast<const __half*>(colf);
  a.KP = KP;
  a.g = g;
  a.nbr = static_cast<uint32_t>(ceil_div(g.n_rows, 128));
  a.nbc = static_cast<uint32_t>(ceil_div(g.n_cols, 128));
  a.rb0 = g.row_begin / 128;
  a.rb1 = static_cast<uint32_t>(ceil_div(g.row_end, 128));
  if (a.rb1 > a.nbr) a.rb1 = a.nbr;
  if (g.row_end <= g.row_begin || a.rb1 <= a.rb0 || a.nbc == 0) return;
  TcPlan pl;
  if (!tc_plan(a.KP, pl)) return;  // callers check mrc_tc_supported
  a.rb = pl.rb;
  a.abufs = pl.abufs;
  a.stages = pl.stages;
  a.CB = pl.CB;
  a.nch = a.KP <= kTcSmallKP ? 1u : static_cast<uint32_t>(ceil_div(a.KP, kTcChunkK));
  a.last_steps = a.KP <= kTcSmallKP ? a.KP / 16 : (a.KP - kTcChunkK * (a.nch - 1)) / 16;
  uint64_t T = 0;
  for (uint32_t r0 = a.rb0; r0 < a.rb1; r0 += a.rb) T += a.nbc - (g.triangle ? r0 : 0u);
  if (T == 0) return;
  a.n_tiles = T;
  a.bitmap = bitmap;
  a.rowcnt = rowcnt;
  a.two = 2;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(T, static_cast<uint64_t>(sms)));
  // rectangle with a database wider than a few column blocks per CTA: stripe-major walk.
  // REFSIG_TC_STRIPE: 0 never, 1 for every rectangle (tests), unset = when nbc >= 8 * grid
  static const int stripe_mode = [] {
    const char* m = std::getenv("REFSIG_TC_STRIPE");
    return m ? std::atoi(m) : -1;
  }();
  a.n_groups = static_cast<uint32_t>(ceil_div(a.rb1 - a.rb0, a.rb));
  if (!g.triangle && stripe_mode != 0 && (stripe_mode == 1 || (a.n_groups >= 2 && a.nbc >= 8ull * grid)))
    a.stripe = static_cast<uint32_t>(ceil_div(a.nbc, grid));
  // CTA pairs sharing every B chunk by cluster multicast (chunked path, stripe walk, even grid):
  // correct (tests) but measured no faster at configs[4] (7.40 vs 7.29 ms: one L2 read per pair, yet
  // each SM still ingests the whole 64 B/clk of B — the per-SM share, not L2, is the bound), so off
  // unless REFSIG_TC_MC=1
  static const int mc_mode = [] {
    const char* m = std::getenv("REFSIG_TC_MC");
    return m ? std::atoi(m) : 0;
  }();
  const bool mc = mc_mode == 1 && !i8 && a.KP > kTcSmallKP && a.stripe && grid >= 2 && a.n_groups >= 2;
  unsigned grid_mc = grid & ~1u;
  if (mc) a.stripe = static_cast<uint32_t>(ceil_div(a.nbc, grid_mc / 2));
  static const uint32_t dbg = [] {
    const char* m = std::getenv("REFSIG_TC_DEBUG");
    return m ? static_cast<uint32_t>(std::atoi(m)) : 0u;
  }();
  a.dbg = dbg;
  const size_t smem = pl.smem;
  // per launch: the attribute is per device context (a process may drive several GPUs)
  const uint32_t fs = a.KP <= kTcSmallKP ? a.KP / 16 : 0u;
  void (*kern)(TcArgs) = nullptr;
  switch (i8 ? 100u : fs) {
    case 100: kern = mrc_tc_kernel<kHamKPBytes / 32, true>; break;  // KP = 48 halves = 96 bytes
    case 1: kern = mrc_tc_kernel<1>; break;
    case 2: kern = mrc_tc_kernel<2>; break;
    case 3: kern = mrc_tc_kernel<3>; break;
    case 4: kern = mrc_tc_kernel<4>; break;
    case 5: kern = mrc_tc_kernel<5>; break;
    case 6: kern = mrc_tc_kernel<6>; break;
    case 7: kern = mrc_tc_kernel<7>; break;
    case 8: kern = mrc_tc_kernel<8>; break;
    default: kern = mc ? mrc_tc_kernel<0, false, true> : mrc_tc_kernel<0>; break;
  }
  ensure_smem(kern, smem);
#ifdef REFSIG_TC_TRACE
  if (dbg & 8) {
    static bool dumped = false;
    if (dumped) {
    } else {
      dumped = true;
      long long z[12][64] = {};
      cudaMemcpyToSymbolAsync(g_tc_trace, z, sizeof(z), 0, cudaMemcpyHostToDevice, s);
    }
  }
#endif
  if (std::getenv("REFSIG_TC_PRINT"))
    std::fprintf(stderr,
                 "mrc_tc: KP %u nch %u last %u CB %u rb %u abufs %u stages %u smem %zu grid %u tiles %llu rows %u cols "
                 "%u wpr %u tri %d rb0 %u rb1 %u nbc %u stripe %u groups %u mc %d Ar %p Bc %p bitmap %p\n",
                 a.KP, a.nch, a.last_steps, a.CB, a.rb, a.abufs, a.stages, smem, grid,
                 static_cast<unsigned long long>(a.n_tiles), g.n_rows, g.n_cols, g.words_per_row, g.triangle ? 1 : 0,
                 a.rb0, a.rb1, a.nbc, a.stripe, a.n_groups, mc ? 1 : 0, static_cast<const void*>(a.Ar),
                 static_cast<const void*>(a.Bc),
                 static_cast<void*>(a.bitmap));
  if (mc) {
    launch_pdl_cluster2(kern, dim3(grid_mc), dim3(kTcThreads), smem, s, a);
  } else {
    launch_pdl(kern, dim3(grid), dim3(kTcThreads), smem, s, a);
  }
#ifdef REFSIG_TC_TRACE
  if (dbg & 8) {
    static int calls = 0;
    if (++calls == 3) {
      long long z[12][64];
      cudaStreamSynchronize(s);
      cudaMemcpyFromSymbol(z, g_tc_trace, sizeof(z));
      const long long t0 = z[0][0];
      std::fprintf(stderr, "it  mma_start full tempty issued | epi_wait tfull ld0 c0 ld1 arrive c1 done\n");
      for (int it = 0; it < 40; it += 2)
        std::fprintf(stderr, "%2d %7lld %7lld %7lld %7lld | %7lld %7lld %7lld %7lld %7lld %7lld %7lld %7lld\n", it,
                     z[0][it] - t0, z[1][it] - t0, z[2][it] - t0, z[3][it] - t0, z[4][it] - t0, z[5][it] - t0,
                     z[8][it] - t0, z[9][it] - t0, z[10][it] - t0, z[6][it] - t0, z[11][it] - t0, z[7][it] - t0);
    }
  }
#endif
  note_launch();
}

void launch_mrc_tc(const void* rowf, const void* colf, uint32_t K, const PairGrid& g, uint32_t* bitmap,
                   uint32_t* rowcnt, cudaStream_t s) {
  launch_tc_tiles(rowf, colf, mrc_tc_kp(K), g, bitmap, rowcnt, s, false);
}

// CTA-pair kernel: chunked K' (> 128), query rectangle wide enough for the
// stripe walk; REFSIG_TC2=0 disables it (measurement), 1 forces it where it applies.
bool mrc_tc2_applies(uint32_t K, const PairGrid& g) {
  static const int mode = [] {
    const char* m = std::getenv("REFSIG_TC2");
    return m ? std::atoi(m) : -1;
  }();
  if (mode == 0) return false;
  const uint32_t KP = mrc_tc_kp(K);
  const uint32_t nbc = static_cast<uint32_t>(ceil_div(g.n_cols, 128));
  const uint32_t rb0 = g.row_begin / 128, rb1 = static_cast<uint32_t>(ceil_div(g.row_end, 128));
  if (KP > 512 || rb1 - rb0 < 2) return false;
  if (mode == 1) return true;
  if (g.triangle) return false;  // (measured below; see DESIGN)
  return KP > kTcSmallKP && nbc >= 8u * 74u;
}

bool launch_mrc_tc2(const void* rowf, const void* colf, uint32_t K, const PairGrid& g, uint32_t* bitmap,
                    uint32_t* rowcnt, cudaStream_t s) {
  TcArgs a{};
  a.Ar = static_cast<const __half*>(rowf);
  a.Bc = static_cast<const __half*>(colf);
  a.KP = mrc_tc_kp(K);
  a.g = g;
  a.nbr = static_cast<uint32_t>(ceil_div(g.n_rows, 128));
  a.nbc = static_cast<uint32_t>(ceil_div(g.n_cols, 128));
  a.rb0 = g.row_begin / 128;
  a.rb1 = std::min(static_cast<uint32_t>(ceil_div(g.row_end, 128)), a.nbr);
  if (g.row_end <= g.row_begin || a.rb1 <= a.rb0 || a.nbc == 0) return true;
  const uint32_t PB = 256u * a.KP;
  a.rb = 1;
  a.abufs = 2u * PB + 4u * kTc2ChunkBytes <= kTcSmemBudget ? 2u : 1u;
  a.stages = std::min<uint32_t>(kTcMaxStages, (kTcSmemBudget - a.abufs * PB) / kTc2ChunkBytes);
  a.CB = kTc2ChunkBytes;
  a.nch = static_cast<uint32_t>(ceil_div(a.KP, kTc2ChunkK));
  a.last_steps = (a.KP - kTc2ChunkK * (a.nch - 1)) / 16;
  a.n_groups = a.rb1 - a.rb0;
  a.bitmap = bitmap;
  a.rowcnt = rowcnt;
  a.two = 2;
  {
    const char* m = std::getenv("REFSIG_TC_DEBUG");  // timing experiments: 1 no epilogue math, 4 no MMA
    a.dbg = m ? static_cast<uint32_t>(std::atoi(m)) : 0u;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = static_cast<unsigned>(sms) & ~1u;
  if (g.triangle) {  // pair tiles: row-block pairs x their columns from the lower block
    uint64_t T = 0;
    for (uint32_t r0 = a.rb0; r0 < a.rb1; r0 += 2) T += a.nbc - r0;
    a.n_tiles = T;
    a.stripe = 0;
  } else {
    a.stripe = static_cast<uint32_t>(ceil_div(a.nbc, grid / 2));
  }
  const size_t smem = std::max<size_t>(static_cast<size_t>(a.abufs) * PB + static_cast<size_t>(a.stages) * kTc2ChunkBytes,
                                       116u * 1024u);
  ensure_smem(mrc_tc2_kernel, smem);
  // the column forms as 512-byte rows of u16 (a 2-D box of 256 x 16 = one contiguous 8 KB chunk; a
  // [8 halves][64 docs][chunks] 3-D view with 16-byte inner rows measured 9.25 vs 6.92 ms)
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return false;  // the caller reports it
  CUtensorMap bmap;
  const cuuint64_t n64 = 2ull * a.nbc;
  const cuuint64_t gdim[2] = {256, n64 * (a.KP / 8) * 2};
  const cuuint64_t gstride[1] = {512};
  const cuuint32_t box[2] = {256, kTc2ChunkBytes / 512};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult er = encode(&bmap, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(colf), gdim, gstride, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (er != CUDA_SUCCESS) return false;
  if (std::getenv("REFSIG_TC_PRINT"))
    std::fprintf(stderr, "mrc_tc2: KP %u nch %u last %u abufs %u stages %u smem %zu grid %u stripe %u groups %u nbc %u\n",
                 a.KP, a.nch, a.last_steps, a.abufs, a.stages, smem, grid, a.stripe, a.n_groups, a.nbc);
  launch_pdl_cluster2(mrc_tc2_kernel, dim3(grid), dim3(kTcThreads), smem, s, a, bmap);
  note_launch();
  return true;
}

size_t ham_tc_form_bytes(uint32_t n) { return static_cast<size_t>(ceil_div(n, 128)) * 128 * kHamKPBytes; }

void launch_ham_tc_forms(const uint64_t* fp, uint32_t n, int max_dist, void* rowf, void* colf, cudaStream_t s) {
  if (!n) return;
  ham_forms_kernel<<<static_cast<unsigned>(ceil_div(n, 128)), 256, 0, s>>>(fp, n, 64 - 2 * max_dist,
                                                                            static_cast<uint8_t*>(rowf),
                                                                            static_cast<uint8_t*>(colf));
  note_launch();
}

void launch_ham_tc(const void* rowf, const void* colf, const PairGrid& g, uint32_t* bitmap, uint32_t* rowcnt,
                   cudaStream_t s) {
  launch_tc_tiles(rowf, colf, kHamKPBytes / 2, g, bitmap, rowcnt, s, true);
}

}  // namespace refsig_gpu
