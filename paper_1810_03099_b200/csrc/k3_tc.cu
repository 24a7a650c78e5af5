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
// Kernel. Persistent, one CTA per SM, 320 threads: warp 0 = bulk-copy
// producer, warp 1 = TMEM owner + MMA issuer (one thread), warps 2..9 =
// epilogue. Tile = 128 rows x 256 columns (two N=128 MMAs per K step; the
// column tile starts at the row block on the triangle, so no tile lies below
// the diagonal), accumulators double-buffered in TMEM (2 x 256 of the 512
// columns) so the epilogue of tile t overlaps the MMAs of tile t+1. Epilogue
// warp w reads TMEM lanes 32*(w%4).. (its hardware lane quarter) and column
// half (w-2)/4: 4 x tcgen05.ld.32x32b.x32, sign bits -> four 32-bit words =
// the row's 128 bits of one bitmap block, written as one 16-byte store in
// the same bitmap/rowcnt format as the CUDA-core kernel (k3_pairs.cu), so
// the scan and emitter are shared.

#include <cuda_fp16.h>

#include "kernels.cuh"

namespace refsig_gpu {
namespace {

constexpr uint32_t kTcThreads = 320;
constexpr uint32_t kTcMaxKP = 128;  // 3K + 3 <= 128  <=>  K <= 41

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, no swizzle: LBO = 2048 B between 8-element K chunks, SBO = 128 B
// between 8-row groups, descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(2048u >> 4) << 16) |
         (static_cast<uint64_t>(128u >> 4) << 32) | (1ull << 46);
}
// kind::f16 instruction descriptor: D f32, A/B f16, K-major both, M=128, N=128.
constexpr uint32_t kIdesc = (1u << 4) | (0u << 7) | (0u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

#define TC_LD32(addr, v)                                                                                            \
  asm volatile(                                                                                                     \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%" \
      "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                                 \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), \
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),     \
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),    \
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                  \
      : "r"(addr))

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
  PairGrid g;
  uint32_t nbc;          // 128-column blocks
  uint32_t rb0, rb1;     // row blocks [rb0, rb1)
  uint64_t n_tiles;
  uint32_t stages;
  uint32_t* bitmap;
  uint32_t* rowcnt;
};

// Column tiles (256 wide) of row block r, and the first column block.
__device__ __forceinline__ uint32_t tc_ct(const TcArgs& a, uint32_t r) {
  return a.g.triangle ? (a.nbc - r + 1) / 2 : (a.nbc + 1) / 2;
}
__device__ __forceinline__ uint32_t tc_cs(const TcArgs& a, uint32_t r) { return a.g.triangle ? r : 0u; }

struct TileWalk {
  uint32_t r, c;
  __device__ void start(const TcArgs& a, uint64_t t) {
    r = a.rb0;
    while (t >= tc_ct(a, r)) {
      t -= tc_ct(a, r);
      ++r;
    }
    c = static_cast<uint32_t>(t);
  }
  __device__ void next(const TcArgs& a) {
    if (++c == tc_ct(a, r)) {
      c = 0;
      ++r;
    }
  }
};

__global__ void __launch_bounds__(kTcThreads, 1) mrc_tc_kernel(TcArgs a) {
  extern __shared__ __align__(1024) uint8_t tsm[];
  __shared__ __align__(8) uint64_t full_bar[8], empty_bar[8], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t t0 = a.n_tiles * blockIdx.x / gridDim.x, t1 = a.n_tiles * (blockIdx.x + 1) / gridDim.x;
  const uint32_t n_it = static_cast<uint32_t>(t1 - t0);
  const uint32_t PB = 256u * a.KP;  // bytes per operand panel
  const uint32_t S = a.stages;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mb_init(&full_bar[s], 1);
      mb_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
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

  if (warp == 0) {
    if (lane == 0) {  // producer: A panel + one or two B panels per tile
      TileWalk w;
      w.start(a, t0);
      for (uint32_t it = 0; it < n_it; ++it) {
        const uint32_t st = it % S;
        if (it >= S) mb_wait(&empty_bar[st], ((it / S) - 1) & 1u);
        const uint32_t bj = tc_cs(a, w.r) + 2 * w.c;
        const uint32_t nb = bj + 1 < a.nbc ? 2u : 1u;
        uint8_t* sA = tsm + static_cast<size_t>(st) * 3 * PB;
        mb_expect_tx(&full_bar[st], PB * (1 + nb));
        bulk_g2s(sA, reinterpret_cast<const uint8_t*>(a.Ar) + static_cast<size_t>(w.r) * PB, PB, &full_bar[st]);
        bulk_g2s(sA + PB, reinterpret_cast<const uint8_t*>(a.Bc) + static_cast<size_t>(bj) * PB, nb * PB,
                 &full_bar[st]);
        w.next(a);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      TileWalk w;
      w.start(a, t0);
      const uint32_t ksteps = a.KP / 16;
      for (uint32_t it = 0; it < n_it; ++it) {
        const uint32_t st = it % S, acc = it & 1;
        const uint32_t bj = tc_cs(a, w.r) + 2 * w.c;
        const uint32_t nb = bj + 1 < a.nbc ? 2u : 1u;
        mb_wait(&full_bar[st], (it / S) & 1u);
        if (it >= 2) mb_wait(&tempty_bar[acc], ((it >> 1) - 1) & 1u);
        tc_fence_after();
        const uint32_t sA = smem_u32(tsm + static_cast<size_t>(st) * 3 * PB);
        for (uint32_t h = 0; h < nb; ++h)
          for (uint32_t k = 0; k < ksteps; ++k)
            mma_f16(tmem + acc * 256 + h * 128, smem_desc(sA + k * 4096), smem_desc(sA + (1 + h) * PB + k * 4096),
                    k > 0);
        mma_commit(&empty_bar[st]);
        mma_commit(&tfull_bar[acc]);
        w.next(a);
      }
    }
    __syncwarp();
  } else {  // epilogue warps 2..9
    const uint32_t q = warp & 3, h = (warp - 2) >> 2;
    const uint32_t wpr = a.g.words_per_row;
    TileWalk w;
    w.start(a, t0);
    uint32_t cnt = 0;
    for (uint32_t it = 0; it < n_it; ++it) {
      const uint32_t acc = it & 1;
      const uint32_t r = w.r;
      const uint32_t bj = tc_cs(a, r) + 2 * w.c + h;
      mb_wait(&tfull_bar[acc], (it >> 1) & 1u);
      tc_fence_after();
      uint32_t v0[32], v1[32], v2[32], v3[32];
      const bool valid = bj < a.nbc;
      if (valid) {
        const uint32_t ta = tmem + ((q * 32u) << 16) + acc * 256 + h * 128;
        TC_LD32(ta, v0);
        TC_LD32(ta + 32, v1);
        TC_LD32(ta + 64, v2);
        TC_LD32(ta + 96, v3);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mb_arrive(&tempty_bar[acc]);
      if (valid) {
        uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;  // bit c = sign(dot - tau) of column 32j + c
#pragma unroll
        for (int c = 31; c >= 0; --c) {
          m0 = __funnelshift_l(v0[c], m0, 1);
          m1 = __funnelshift_l(v1[c], m1, 1);
          m2 = __funnelshift_l(v2[c], m2, 1);
          m3 = __funnelshift_l(v3[c], m3, 1);
        }
        m0 = ~m0, m1 = ~m1, m2 = ~m2, m3 = ~m3;
        const uint32_t i = r * 128 + q * 32 + lane;
        if ((a.g.triangle && bj == r) || bj + 1 == a.nbc) {
          const uint32_t c0 = bj * 128;
          m0 &= tc_col_mask(c0, i, a.g);
          m1 &= tc_col_mask(c0 + 32, i, a.g);
          m2 &= tc_col_mask(c0 + 64, i, a.g);
          m3 &= tc_col_mask(c0 + 96, i, a.g);
        }
        if (i < a.g.n_rows) {
          *reinterpret_cast<uint4*>(a.bitmap + static_cast<size_t>(i) * wpr + bj * 4) = make_uint4(m0, m1, m2, m3);
          cnt += __popc(m0) + __popc(m1) + __popc(m2) + __popc(m3);
        }
      }
      w.next(a);
      if (w.r != r || it + 1 == n_it) {
        const uint32_t i = r * 128 + q * 32 + lane;
        if (cnt && i < a.g.n_rows) atomicAdd(a.rowcnt + i, cnt);
        cnt = 0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// Row form [hi | hi | lo | -tau pieces] or column form [hi | lo | hi | 1 1 1]
// of every document, panel layout (see the top comment). Thread per (doc, K
// chunk of 8); consecutive threads = consecutive docs: reads of ST[k][d] and
// 16-byte writes are both coalesced.
__global__ void __launch_bounds__(256) tc_forms_kernel(const float* __restrict__ ST, uint32_t ld, uint32_t n_docs,
                                                       uint32_t K, uint32_t KP, uint32_t n_pan, float tau,
                                                       __half* __restrict__ rowf, __half* __restrict__ colf) {
  const uint32_t chunks = KP / 8;
  const uint64_t total = static_cast<uint64_t>(n_pan) * 128 * chunks;
  // tau = t0 + t1 + t2 in fp16 pieces (exact for any fp32 tau in fp16 range)
  const __half t0 = __float2half_rn(tau);
  const float r1 = tau - __half2float(t0);
  const __half t1 = __float2half_rn(r1);
  const __half t2 = __float2half_rn(r1 - __half2float(t1));
  const __half one = __float2half_rn(1.0f), zero = __float2half_rn(0.0f);
  for (uint64_t idx = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t dl = static_cast<uint32_t>(idx % 128);
    const uint64_t pc = idx / 128;
    const uint32_t kc = static_cast<uint32_t>(pc % chunks), pan = static_cast<uint32_t>(pc / chunks);
    const uint32_t d = pan * 128 + dl;
    __align__(16) __half rv[8], cv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t p = kc * 8 + e;
      __half rr = zero, cc = zero;
      if (p < 3 * K) {
        const uint32_t seg = p / K, k = p - seg * K;
        const float v = d < n_docs ? ST[static_cast<size_t>(k) * ld + d] : 0.0f;
        const __half hi = __float2half_rn(v);
        const __half lo = __float2half_rn(v - __half2float(hi));
        rr = seg == 2 ? lo : hi;
        cc = seg == 1 ? lo : hi;
      } else if (p < 3 * K + 3) {
        const uint32_t j = p - 3 * K;
        const __half tj = j == 0 ? t0 : (j == 1 ? t1 : t2);
        rr = __hneg(tj);
        if (__half2float(tj) == 0.0f) rr = zero;  // +0, never -0: tau = 0 keeps dot = 0 a match
        cc = one;
      }
      rv[e] = rr;
      cv[e] = cc;
    }
    const size_t off = ((static_cast<size_t>(pan) * chunks + kc) * 128 + dl) * 8;
    if (rowf) *reinterpret_cast<uint4*>(rowf + off) = *reinterpret_cast<const uint4*>(rv);
    if (colf) *reinterpret_cast<uint4*>(colf + off) = *reinterpret_cast<const uint4*>(cv);
  }
}

}  // namespace

uint32_t mrc_tc_kp(uint32_t K) { return ((3 * K + 3) + 15) / 16 * 16; }

bool mrc_tc_supported(uint32_t K, float tau) {
  // fp16 pieces of tau: |tau| < 65504, and tau = 0 or |tau| >= 2^-14 (fp16
  // normal) so that the leading piece is nonzero and a zero signature never
  // matches a positive tau; K' <= 128 keeps 2+ stages in smem
  const float at = fabsf(tau);
  return K >= 1 && mrc_tc_kp(K) <= kTcMaxKP && at < 60000.0f && (at == 0.0f || at >= 6.103515625e-05f);
}

size_t mrc_tc_form_bytes(uint32_t K, uint32_t n_docs) {
  return static_cast<size_t>(ceil_div(n_docs, 128)) * 256u * mrc_tc_kp(K);
}

void launch_mrc_tc_forms(const float* ST, uint32_t ld, uint32_t n_docs, uint32_t K, float tau, void* rowf, void* colf,
                         cudaStream_t s) {
  const uint32_t KP = mrc_tc_kp(K);
  const uint32_t n_pan = static_cast<uint32_t>(ceil_div(n_docs, 128));
  const uint64_t total = static_cast<uint64_t>(n_pan) * 128 * (KP / 8);
  if (!total) return;
  const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 148ull * 8));
  tc_forms_kernel<<<blocks, 256, 0, s>>>(ST, ld, n_docs, K, KP, n_pan, tau, static_cast<__half*>(rowf),
                                         static_cast<__half*>(colf));
  note_launch();
}

void launch_mrc_tc(const void* rowf, const void* colf, uint32_t K, const PairGrid& g_in, uint32_t* bitmap,
                   uint32_t* rowcnt, cudaStream_t s) {
  PairGrid g = g_in;
  TcArgs a{};
  a.Ar = static_cast<const __half*>(rowf);
  a.Bc = static_cast<const __half*>(colf);
  a.KP = mrc_tc_kp(K);
  a.g = g;
  a.nbc = static_cast<uint32_t>(ceil_div(g.n_cols, 128));
  a.rb0 = g.row_begin / 128;
  a.rb1 = static_cast<uint32_t>(ceil_div(g.row_end, 128));
  if (g.row_end <= g.row_begin || a.rb1 <= a.rb0 || a.nbc == 0) return;
  uint64_t T = 0;
  for (uint32_t r = a.rb0; r < a.rb1; ++r) T += g.triangle ? (a.nbc - r + 1) / 2 : (a.nbc + 1) / 2;
  if (T == 0) return;
  a.n_tiles = T;
  a.bitmap = bitmap;
  a.rowcnt = rowcnt;
  const uint32_t stage_bytes = 3u * 256u * a.KP;
  a.stages = std::max<uint32_t>(2u, std::min<uint32_t>(8u, (200u * 1024u) / stage_bytes));
  // at least ~116 KB so that exactly one CTA (the TMEM owner of all 512 columns) fits per SM
  const size_t smem = std::max<size_t>(static_cast<size_t>(a.stages) * stage_bytes, 116u * 1024u);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(mrc_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(T, static_cast<uint64_t>(sms)));
  mrc_tc_kernel<<<grid, kTcThreads, smem, s>>>(a);
  note_launch();
}

}  // namespace refsig_gpu
