// k5_tc.cu — the dense contractions of the exact-cosine evaluation on the
// 5th-generation tensor cores (north_star item 5: "tensor cores only on
// densified tiles where it truly is a dense contraction").
//
// SPEC eval (Eq. 2/3 of PAPER.md:207-215): for every pair
// i<j, the exact cosine (reference ngram.hpp:184-202) against the MRC compare
// score and the Simhash similarity (simhash.hpp:49-52). The
// exact cosine is split (k5_exact.cu) into a dense head — the H highest-df
// terms, rows A[d][H] — and a sparse tail summed exactly in fixed point by
// exact_tail_kernel (dump mode: T[i][j] * 2^-30). Per pair this kernel needs
// two dense dot products: head A_i . A_j (H terms) and the MRC dot
// S^_i . S^_j (K terms). Both are N x N contractions over the same pair
// tiles, so one tcgen05 kernel computes them as two MMA chains of one K
// walk: each document's operand is
//   row form    [head hi | head hi | head lo | mrc hi | mrc hi | mrc lo]
//   column form [head hi | head lo | head hi | mrc hi | mrc lo | mrc hi]
// (split fp16 as in k3_tc.cu: hi = rn(v), lo = rn(v - hi); the dropped
// lo*lo term is < 2^-22), each part padded to a multiple of 16; the first
// K_h/16 k-steps accumulate the head dot into TMEM columns [0, 128) of the
// tile's accumulator, the rest the MRC dot into [128, 256).
//
// Kernel: persistent, one CTA per SM, 608 threads: warp 0 bulk-copy producer
// (A = 128-row block resident, double-buffered when two fit; B = 128-column
// panel streamed in 64-wide K chunks), warp 1 the MMA issuer, warps 3..18 the
// epilogue in two groups (one per double-buffered 256-column accumulator),
// each warp 32 rows (its TMEM lane quarter) x 64 columns. Epilogue per pair:
// exact = min(head + T_ij 2^-30, 1), e_mrc = min(mrc, 1) - exact, e_sim =
// (1 - popc(F_i ^ F_j)/64) - exact, accumulated in double per thread (n, sum
// e, sum e^2, sum |e| per method) and reduced in a fixed order per CTA; the
// host adds the CTAs in index order (deterministic).

#include <cuda_fp16.h>

#include <algorithm>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace refsig_gpu {
namespace {

constexpr uint32_t kEvThreads = 608;
constexpr uint32_t kEvChunk = 64;  // K halves per B stage chunk (16 KB per 128-doc panel)
constexpr uint32_t kEvMaxStages = 8;
constexpr uint32_t kEvBudget = 225u * 1024u;

struct EvTcArgs {
  const __half* Ar;  // row forms, 128-doc panels (k3_tc.cu layout)
  const __half* Bc;  // column forms
  uint32_t KP;       // K' of a document operand (multiple of 64)
  uint32_t SH;       // k-steps of the head part (K_h / 16)
  uint32_t nch;      // 64-wide chunks per tile (KP / 64)
  uint32_t abufs, stages;
  uint32_t n_docs, rb0, rb1, nbc;  // row blocks [rb0, rb1) of the triangle, nbc column blocks
  uint32_t row_lo, row_hi;         // pairs i<j with row_lo <= i < row_hi
  uint64_t n_tiles;
  const uint32_t* T;  // tail sums, row-major [row_hi-row_lo][ldT] (valid for j > i)
  uint32_t ldT;
  const uint64_t* fp;  // fingerprints (NULL: no Simhash errors)
  double* out;         // [grid][8]
};

struct EvWalk {  // triangle tiles of 128-row blocks: block r has column blocks r .. nbc-1
  uint32_t r, c;
  __device__ void start(const EvTcArgs& a, uint64_t t) {
    r = a.rb0;
    while (t >= a.nbc - r) {
      t -= a.nbc - r;
      ++r;
    }
    c = r + static_cast<uint32_t>(t);
  }
  __device__ bool next(const EvTcArgs& a) {  // true when the next tile starts a new row block
    if (++c == a.nbc) {
      ++r;
      c = r;
      return true;
    }
    return false;
  }
};

__global__ void __launch_bounds__(kEvThreads, 1) eval_tc_kernel(EvTcArgs a) {
  extern __shared__ __align__(1024) uint8_t tsm[];
  __shared__ __align__(8) uint64_t full_bar[kEvMaxStages], empty_bar[kEvMaxStages], afull_bar[2], aempty_bar[2],
      tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ double red[16][8];
  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
  const uint64_t t0 = a.n_tiles * blockIdx.x / gridDim.x, t1 = a.n_tiles * (blockIdx.x + 1) / gridDim.x;
  const uint32_t n_it = static_cast<uint32_t>(t1 - t0);
  const uint32_t PB = 256u * a.KP, CB = 256u * kEvChunk, S = a.stages, NCH = a.nch, AB = a.abufs;
  uint8_t* sA = tsm;
  uint8_t* sB = tsm + AB * PB;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mb_init(&full_bar[s], 1);
      mb_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mb_init(&afull_bar[s], 1);
      mb_init(&aempty_bar[s], 1);
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

  double acc7[7] = {0, 0, 0, 0, 0, 0, 0};  // n, sum e, sum e^2, sum |e| (MRC), the same for Simhash
  if (warp == 0) {
    if (lane == 0 && n_it) {  // producer
      EvWalk w;
      w.start(a, t0);
      uint32_t g = 0, q = 0;
      bool new_block = true;
      for (uint32_t it = 0; it < n_it; ++it) {
        if (new_block) {
          const uint32_t ab = g % AB;
          if (g >= AB) mb_wait(&aempty_bar[ab], ((g / AB) - 1) & 1u);
          mb_expect_tx(&afull_bar[ab], PB);
          bulk_g2s(sA + ab * PB, reinterpret_cast<const uint8_t*>(a.Ar) + static_cast<size_t>(w.r) * PB, PB,
                   &afull_bar[ab]);
          ++g;
        }
        const uint8_t* src = reinterpret_cast<const uint8_t*>(a.Bc) + static_cast<size_t>(w.c) * PB;
        for (uint32_t ch = 0; ch < NCH; ++ch, ++q) {
          const uint32_t st = q % S;
          if (q >= S) mb_wait(&empty_bar[st], ((q / S) - 1) & 1u);
          mb_expect_tx(&full_bar[st], CB);
          bulk_g2s(sB + static_cast<size_t>(st) * CB, src + static_cast<size_t>(ch) * CB, CB, &full_bar[st]);
        }
        new_block = w.next(a);
      }
    }
    __syncwarp();
  } else if (warp == 1) {  // the MMA issuer: every tile, accumulator it % 2; one ring consumer
    if (n_it) {
      EvWalk w;
      w.start(a, t0);
      const uint64_t dA0 = smem_desc(smem_u32(sA)), dB0 = smem_desc(smem_u32(sB));
      const uint64_t dPB = PB >> 4, dCB = CB >> 4;
      uint32_t g = 0, q = 0;
      bool new_block = true;
      for (uint32_t it = 0; it < n_it; ++it) {
        if (new_block) {
          mb_wait_warp(&afull_bar[g % AB], (g / AB) & 1u);
          ++g;
        }
        const uint32_t ab = (g - 1) % AB, acc = it & 1;
        if (it >= 2) mb_wait_warp(&tempty_bar[acc], ((it >> 1) - 1) & 1u);
        const uint64_t dA = dA0 + ab * dPB;
        const uint32_t dh = tmem + acc * 256, dm = dh + 128;
        for (uint32_t ch = 0; ch < NCH; ++ch, ++q) {
          const uint32_t st = q % S;
          mb_wait_warp(&full_bar[st], (q / S) & 1u);
          const uint32_t e = elect_one();
          tc_fence_after();
          const uint64_t dB = dB0 + st * dCB;
#pragma unroll
          for (uint32_t j = 0; j < kEvChunk / 16; ++j) {
            const uint32_t s = ch * (kEvChunk / 16) + j;  // k-step of the document operand
            const bool head = s < a.SH;
            mma_f16_e(e, head ? dh : dm, dA + s * 256u, dB + j * 256u, head ? (s != 0) : (s != a.SH));
          }
          mma_commit_e(e, &empty_bar[st]);
        }
        __syncwarp();
        mma_commit_e(elect_one(), &tfull_bar[acc]);
        new_block = w.next(a);
        __syncwarp();
        if (new_block || it + 1 == n_it) mma_commit_e(elect_one(), &aempty_bar[ab]);
        __syncwarp();
      }
    }
    __syncwarp();
  } else if (warp >= 3) {  // epilogue: group eg (accumulator), lane quarter q, column half c2
    const uint32_t ew = threadIdx.x / 32 - 3;
    const uint32_t q = (threadIdx.x / 32) & 3, eg = ew >> 3, c2 = (ew >> 2) & 1;
    EvWalk w;
    if (n_it) w.start(a, t0);
    for (uint32_t it = 0; it < n_it; ++it) {
      const uint32_t acc = it & 1;
      const uint32_t r = w.r, bj = w.c;
      if (acc == eg) {
        const uint32_t i = r * 128 + q * 32 + lane;
        const bool row_ok = i >= a.row_lo && i < a.row_hi && i < a.n_docs;
        const uint64_t fi = (a.fp && row_ok) ? a.fp[i] : 0ull;
        const uint32_t* trow = a.T + static_cast<size_t>(row_ok ? i - a.row_lo : 0) * a.ldT;
        mb_wait_warp(&tfull_bar[acc], (it >> 1) & 1u);
        tc_fence_after();
#pragma unroll 1
        for (int h = 0; h < 4; ++h) {  // 16-column quarters of this warp's 64 columns
          const uint32_t j0 = bj * 128 + c2 * 64 + h * 16;
          // this row's 16 tail sums (4 x 16 B; ldT is padded to whole 128-column blocks) and the
          // columns' fingerprints, loaded before the TMEM wait
          uint4 tv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tv[k] = row_ok ? *reinterpret_cast<const uint4*>(trow + j0 + 4 * k) : make_uint4(0, 0, 0, 0);
          const uint64_t fl = (a.fp && j0 + (lane & 15) < a.n_docs) ? a.fp[j0 + (lane & 15)] : 0ull;
          uint32_t hv[16], mv[16];
          const uint32_t ta = tmem + ((q * 32u) << 16) + acc * 256 + c2 * 64 + h * 16;
          TC_LD16(ta, hv);
          TC_LD16(ta + 128, mv);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (h == 3) {  // accumulator fully read: hand it back
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mb_arrive(&tempty_bar[acc]);
          }
          const uint32_t tt[16] = {tv[0].x, tv[0].y, tv[0].z, tv[0].w, tv[1].x, tv[1].y, tv[1].z, tv[1].w,
                                   tv[2].x, tv[2].y, tv[2].z, tv[2].w, tv[3].x, tv[3].y, tv[3].z, tv[3].w};
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const uint32_t j = j0 + c;
            const uint64_t fj = __shfl_sync(0xffffffffu, fl, c);
            if (!row_ok || j <= i || j >= a.n_docs) continue;
            const float ex =
                fminf(__uint_as_float(hv[c]) + static_cast<float>(tt[c]) * (1.0f / 1073741824.0f), 1.0f);
            const double em = static_cast<double>(fminf(__uint_as_float(mv[c]), 1.0f)) - static_cast<double>(ex);
            acc7[0] += 1.0;
            acc7[1] += em;
            acc7[2] = fma(em, em, acc7[2]);
            acc7[3] += fabs(em);
            if (a.fp) {
              const double es = (1.0 - __popcll(fi ^ fj) / 64.0) - static_cast<double>(ex);
              acc7[4] += es;
              acc7[5] = fma(es, es, acc7[5]);
              acc7[6] += fabs(es);
            }
          }
        }
      }
      w.next(a);
    }
  }
  // fixed-order reduction over the 16 epilogue warps (warp tree, then warps in order)
  if (warp >= 3) {
#pragma unroll
    for (int k = 0; k < 7; ++k)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc7[k] += __shfl_xor_sync(0xffffffffu, acc7[k], o);
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < 7; ++k) red[threadIdx.x / 32 - 3][k] = acc7[k];
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 7) {
    double x = 0;
    for (int w2 = 0; w2 < 16; ++w2) x += red[w2][threadIdx.x];
    a.out[blockIdx.x * 8 + threadIdx.x] = x;
  }
  if (threadIdx.x == 7) a.out[blockIdx.x * 8 + 7] = 0.0;
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// Operand forms of the evaluation: document d's row and column forms (see
// the top comment) from AT[H][ld] (head rows, transposed) and ST[K][ld]
// (unit signatures), 128-doc panels in the k3_tc.cu layout. Thread (8-half
// chunk kc, doc dl); grid (panels, ceil(KP/8 / 2)).
__global__ void __launch_bounds__(256) eval_forms_kernel(const float* __restrict__ AT, uint32_t H,
                                                         const float* __restrict__ ST, uint32_t K, uint32_t ld,
                                                         uint32_t n_docs, uint32_t KH, uint32_t KP,
                                                         __half* __restrict__ rowf, __half* __restrict__ colf) {
  const uint32_t pan = blockIdx.x, dl = threadIdx.x & 127, kc = blockIdx.y * 2 + (threadIdx.x >> 7);
  if (kc * 8 >= KP) return;
  const uint32_t d = pan * 128 + dl;
  __align__(16) __half rv[8], cv[8];
#pragma unroll
  for (uint32_t e = 0; e < 8; ++e) {
    uint32_t pos = kc * 8 + e;
    const float* src = AT;
    uint32_t n = H;
    if (pos >= KH) {  // the MRC part
      pos -= KH;
      src = ST;
      n = K;
    }
    __half r = __float2half_rn(0.0f), c = r;
    if (pos < 3 * n) {
      const uint32_t seg = pos / n, k = pos - seg * n;
      const float v = d < n_docs ? src[static_cast<size_t>(k) * ld + d] : 0.0f;
      const __half hi = __float2half_rn(v);
      const __half lo = __float2half_rn(v - __half2float(hi));
      r = seg == 2 ? lo : hi;  // row form [hi | hi | lo]
      c = seg == 1 ? lo : hi;  // column form [hi | lo | hi]
    }
    rv[e] = r;
    cv[e] = c;
  }
  const size_t off = (static_cast<size_t>(pan) * (KP / 8) + kc) * 128 * 8 + static_cast<size_t>(dl) * 8;
  *reinterpret_cast<uint4*>(rowf + off) = *reinterpret_cast<const uint4*>(rv);
  *reinterpret_cast<uint4*>(colf + off) = *reinterpret_cast<const uint4*>(cv);
}

uint32_t eval_kh(uint32_t H) { return (3 * H + 15) / 16 * 16; }
// head and MRC parts; the total rounded to whole 64-wide chunks (zero padding)
uint32_t eval_kp(uint32_t H, uint32_t K) { return (eval_kh(H) + (3 * K + 15) / 16 * 16 + 63) / 64 * 64; }

}  // namespace

size_t eval_tc_form_bytes(uint32_t H, uint32_t K, uint32_t n_docs) {
  return static_cast<size_t>(ceil_div(n_docs, 128)) * 256u * eval_kp(H, K);
}

bool eval_tc_supported(uint32_t H, uint32_t K) {
  const uint32_t PB = 256u * eval_kp(H, K);
  return PB + 4u * 256u * kEvChunk <= kEvBudget;  // one A panel and >= 4 B stages
}

void launch_eval_tc_forms(const float* AT, uint32_t H, const float* ST, uint32_t K, uint32_t ld, uint32_t n_docs,
                          void* rowf, void* colf, cudaStream_t s) {
  const uint32_t KP = eval_kp(H, K);
  const uint32_t n_pan = static_cast<uint32_t>(ceil_div(n_docs, 128));
  if (!n_pan) return;
  eval_forms_kernel<<<dim3(n_pan, static_cast<unsigned>(ceil_div(KP / 8, 2))), 256, 0, s>>>(
      AT, H, ST, K, ld, n_docs, eval_kh(H), KP, static_cast<__half*>(rowf), static_cast<__half*>(colf));
  note_launch();
}

uint32_t launch_eval_tc(const void* rowf, const void* colf, uint32_t H, uint32_t K, uint32_t n_docs, uint32_t row_lo,
                        uint32_t row_hi, const uint32_t* T, uint32_t ldT, const uint64_t* fp, double* out,
                        cudaStream_t s) {
  EvTcArgs a{};
  a.Ar = static_cast<const __half*>(rowf);
  a.Bc = static_cast<const __half*>(colf);
  a.KP = eval_kp(H, K);
  a.SH = eval_kh(H) / 16;
  a.nch = a.KP / kEvChunk;
  const uint32_t PB = 256u * a.KP, CB = 256u * kEvChunk;
  a.abufs = 2u * PB + 4u * CB <= kEvBudget ? 2u : 1u;
  a.stages = std::min<uint32_t>(kEvMaxStages, (kEvBudget - a.abufs * PB) / CB);
  a.n_docs = n_docs;
  a.rb0 = row_lo / 128;
  a.rb1 = static_cast<uint32_t>(ceil_div(row_hi, 128));
  a.nbc = static_cast<uint32_t>(ceil_div(n_docs, 128));
  a.row_lo = row_lo;
  a.row_hi = row_hi;
  uint64_t T_tiles = 0;
  for (uint32_t r = a.rb0; r < a.rb1; ++r) T_tiles += a.nbc - r;
  a.n_tiles = T_tiles;
  a.T = T;
  a.ldT = ldT;
  a.fp = fp;
  a.out = out;
  if (!T_tiles) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(T_tiles, static_cast<uint64_t>(sms)));
  const size_t smem = std::max<size_t>(static_cast<size_t>(a.abufs) * PB + static_cast<size_t>(a.stages) * CB,
                                       116u * 1024u);
  ensure_smem(eval_tc_kernel, smem);
  eval_tc_kernel<<<grid, kEvThreads, smem, s>>>(a);
  note_launch();
  return grid;
}

}  // namespace refsig_gpu
