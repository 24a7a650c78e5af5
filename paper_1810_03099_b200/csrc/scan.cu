// scan.cu — device exclusive prefix sums (u32 counts -> u64 offsets).
//
// Three phases, all on the caller's stream, no host round trip:
//   1. each 4096-element block reduces to one u64 partial,
//   2. one CTA scans the partials (serially per thread chunk + block scan),
//   3. each block rescans its elements and adds its partial offset.
// Used for row offsets of the pair emitters and the compact CSR rowptr.

#include "kernels.cuh"

namespace refsig_gpu {
namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanIpt = 4;
constexpr uint64_t kScanBlock = kScanThreads * kScanIpt;

__device__ __forceinline__ uint64_t warp_inclusive_scan_u64(uint64_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

__device__ __forceinline__ uint64_t block_exscan_u64(uint64_t v, uint64_t* sh, uint64_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t inc = warp_inclusive_scan_u64(v, lane);
  if (lane == 31) sh[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint64_t x = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
    uint64_t xi = warp_inclusive_scan_u64(x, lane);
    sh[lane] = xi - x;
    if (lane == 31) sh[32] = xi;
  }
  __syncthreads();
  uint64_t r = sh[wid] + inc - v;
  *total = sh[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t* __restrict__ in, uint64_t n,
                                                                   uint64_t* __restrict__ partial) {
  __shared__ uint64_t sh[33];
  const uint64_t base = blockIdx.x * kScanBlock + threadIdx.x * kScanIpt;
  uint64_t s = 0;
#pragma unroll
  for (int q = 0; q < kScanIpt; ++q)
    if (base + q < n) s += in[base + q];
  uint64_t tot;
  block_exscan_u64(s, sh, &tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) scan_partials_kernel(uint64_t* partial, uint64_t nb) {
  __shared__ uint64_t sh[33];
  // each thread owns a contiguous chunk of partials
  const uint64_t per = (nb + kScanThreads - 1) / kScanThreads;
  const uint64_t lo = threadIdx.x * per;
  uint64_t s = 0;
  for (uint64_t i = lo; i < lo + per && i < nb; ++i) s += partial[i];
  uint64_t tot;
  uint64_t off = block_exscan_u64(s, sh, &tot);
  for (uint64_t i = lo; i < lo + per && i < nb; ++i) {
    uint64_t x = partial[i];
    partial[i] = off;
    off += x;
  }
  if (threadIdx.x == 0) partial[nb] = tot;
}

__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const uint32_t* __restrict__ in, uint64_t n,
                                                                  const uint64_t* __restrict__ partial,
                                                                  uint64_t nb, uint64_t* __restrict__ out,
                                                                  uint64_t* total_out) {
  __shared__ uint64_t sh[33];
  const uint64_t base = blockIdx.x * kScanBlock + threadIdx.x * kScanIpt;
  uint32_t v[kScanIpt];
  uint64_t s = 0;
#pragma unroll
  for (int q = 0; q < kScanIpt; ++q) {
    v[q] = base + q < n ? in[base + q] : 0u;
    s += v[q];
  }
  uint64_t tot;
  uint64_t off = partial[blockIdx.x] + block_exscan_u64(s, sh, &tot);
#pragma unroll
  for (int q = 0; q < kScanIpt; ++q) {
    if (base + q < n) out[base + q] = off;
    off += v[q];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[n] = partial[nb];
    if (total_out) *total_out = partial[nb];
  }
}

// n <= kSmallScan: one 256-thread CTA per tile of 1024 values (thread t owns
// values 4t..4t+3: one 16-byte load, two 16-byte stores). Each CTA first
// reduces all values before its tile itself (<= 128 KB of L2-resident reads),
// so the tiles are independent: one launch, no serial chain across CTAs.
constexpr uint64_t kSmallScan = 32768;
constexpr int kSmallThreads = 256;
constexpr uint32_t kSmallTile = 4 * kSmallThreads;

__device__ __forceinline__ uint4 load4(const uint32_t* __restrict__ in, uint32_t i, uint32_t n) {
  if (i + 4 <= n) return __ldg(reinterpret_cast<const uint4*>(in + i));
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  if (i < n) v.x = in[i];
  if (i + 1 < n) v.y = in[i + 1];
  if (i + 2 < n) v.z = in[i + 2];
  return v;
}

__global__ void __launch_bounds__(kSmallThreads) scan_small_kernel(const uint32_t* __restrict__ in, uint64_t n,
                                                                   uint64_t* __restrict__ out, uint64_t* total_out) {
  pdl_wait();
  __shared__ uint64_t sh[33];
  const uint32_t nn = static_cast<uint32_t>(n);
  const uint32_t t0 = blockIdx.x * kSmallTile;
  const uint32_t i = t0 + threadIdx.x * 4;
  const uint4 v = load4(in, i, nn);
  // prefix = sum of in[0 .. t0): 4 independent 16-byte loads per step
  uint64_t pre = 0;
  for (uint32_t j0 = threadIdx.x * 4; j0 < t0; j0 += 4 * kSmallTile) {
    uint4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t j = j0 + u * kSmallTile;
      x[u] = j < t0 ? __ldg(reinterpret_cast<const uint4*>(in + j)) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) pre += static_cast<uint64_t>(x[u].x) + x[u].y + x[u].z + x[u].w;
  }
  uint64_t pre_tot;
  block_exscan_u64(pre, sh, &pre_tot);
  const uint64_t s = static_cast<uint64_t>(v.x) + v.y + v.z + v.w;
  uint64_t tot;
  const uint64_t o0 = pre_tot + block_exscan_u64(s, sh, &tot);
  const uint64_t o1 = o0 + v.x, o2 = o1 + v.y, o3 = o2 + v.z;
  if (i + 4 <= nn) {
    reinterpret_cast<ulonglong2*>(out + i)[0] = make_ulonglong2(o0, o1);
    reinterpret_cast<ulonglong2*>(out + i)[1] = make_ulonglong2(o2, o3);
  } else {
    if (i < nn) out[i] = o0;
    if (i + 1 < nn) out[i + 1] = o1;
    if (i + 2 < nn) out[i + 2] = o2;
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    out[n] = pre_tot + tot;
    if (total_out) *total_out = pre_tot + tot;  // e.g. mapped pinned memory: the host reads it after a sync
  }
}

}  // namespace

size_t scan_tmp_bytes(uint64_t n) { return sizeof(uint64_t) * (ceil_div(n, kScanBlock) + 2); }

void launch_exclusive_scan_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t n, void* tmp, cudaStream_t s,
                                      uint64_t* total_out) {
  uint64_t nb = ceil_div(n, kScanBlock);
  if (nb == 0) {
    cudaMemsetAsync(out, 0, sizeof(uint64_t), s);
    if (total_out) launch_words_to_host(reinterpret_cast<const uint32_t*>(out), 2, reinterpret_cast<uint32_t*>(total_out), s);
    return;
  }
  if (n <= kSmallScan) {
    launch_pdl(scan_small_kernel, dim3(static_cast<unsigned>(ceil_div(n, kSmallTile))), dim3(kSmallThreads), 0, s, in,
               n, out, total_out);
    note_launch();
    return;
  }
  uint64_t* partial = static_cast<uint64_t*>(tmp);
  scan_reduce_kernel<<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, partial);
  note_launch();
  scan_partials_kernel<<<1, kScanThreads, 0, s>>>(partial, nb);
  note_launch();
  scan_apply_kernel<<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, partial, nb, out, total_out);
  note_launch();
}

}  // namespace refsig_gpu
