// common.cuh — shared device helpers for the refsig B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace refsig_gpu {

constexpr int kWarp = 32;
constexpr uint32_t kPadKey = 0xFFFFFFFFu;
constexpr int kTile = 128;  // pair-tile edge (rows and columns) of the all-pairs kernels

// Packed per-term info gathered once per nonzero: x = idf32 bits, y = row of
// the term in the compact reference table (or -1 when not in the union U).
struct __align__(8) TermInfo {
  float idf;
  int32_t ref_row;
};
static_assert(sizeof(TermInfo) == 8, "TermInfo is one 8-byte gather");

// Read-only loads that do not allocate in L1: streamed count entries and the
// per-nonzero TermInfo gathers, so L1 keeps the reused reference-table rows.
__device__ __forceinline__ uint2 ld_na(const uint2* p) {
  uint2 v;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ TermInfo ld_na(const TermInfo* p) {
  TermInfo v;
  asm("ld.global.nc.L1::no_allocate.v2.b32 {%0, %1}, [%2];" : "=f"(v.idf), "=r"(v.ref_row) : "l"(p));
  return v;
}

// L1 eviction-priority variants (K2 cache-policy A/B, REFSIG_K2_HINT 3/4).
__device__ __forceinline__ uint2 ld_ef(const uint2* p) {
  uint2 v;
  asm("ld.global.nc.L1::evict_first.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ TermInfo ld_el(const TermInfo* p) {
  TermInfo v;
  asm("ld.global.nc.L1::evict_last.v2.b32 {%0, %1}, [%2];" : "=f"(v.idf), "=r"(v.ref_row) : "l"(p));
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
  return __reduce_add_sync(0xffffffffu, v);
}

// Inclusive warp scan (Kogge-Stone over shuffles).
__device__ __forceinline__ uint32_t warp_inclusive_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// splitmix64 term hash, SURVEY.md Appendix A6 (replaces the MD5 word hash of
// reference simhash.hpp:23-29 for integer term ids).
__device__ __forceinline__ uint64_t term_hash64(uint64_t seed, uint32_t t) {
  uint64_t z = seed + (static_cast<uint64_t>(t) + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

}  // namespace refsig_gpu

namespace refsig_gpu {
// Counts kernel launches issued by this library (refsig_gpu_launch_count).
void note_launch();
// cudaFuncAttributeMaxDynamicSharedMemorySize >= bytes for `func` on the
// current device (the attribute is per device context; remembered per
// (function, device) so repeated launches skip the driver call).
void ensure_smem_attr(const void* func, int bytes);
template <typename... KArgs>
inline void ensure_smem(void (*kernel)(KArgs...), size_t bytes) {
  ensure_smem_attr(reinterpret_cast<const void*>(kernel), static_cast<int>(bytes));
}

// Programmatic dependent launch: a kernel launched with launch_pdl may be
// scheduled while its predecessor in the stream drains; it must call
// pdl_wait() before touching the predecessor's output (a no-op when launched
// without the attribute). Predecessors may call pdl_trigger() once their
// remaining work no longer produces data the dependent reads early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// REFSIG_NO_PDL=1 launches the PDL kernels as plain stream-ordered launches (debugging).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// launch_pdl with 2-CTA clusters (CTAs 2k, 2k+1 co-scheduled on one TPC).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster2(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
}  // namespace refsig_gpu
