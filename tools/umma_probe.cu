// umma_probe.cu — tcgen05.mma issue/throughput microbenchmark (kind::f16,
// M=128, K=16, smem operands in the K-major no-swizzle layout K3-TC uses).
// One CTA per SM, one thread issues `iters` MMAs then commits and waits;
// reports cycles per MMA for N in {64,128,256} and 1 vs 2 accumulators.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/umma_probe tools/umma_probe.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(lbo >> 4) << 16) |
         (static_cast<uint64_t>(sbo >> 4) << 32) | (1ull << 46);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}

template <bool WARP>
__global__ void __launch_bounds__(128, 1) probe(int iters, int N, int naccs, int kchunk_stride, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | ((static_cast<uint32_t>(N) >> 3) << 17) | ((128u >> 4) << 24);
  if (WARP ? threadIdx.x < 32 : threadIdx.x == 0) {
    const uint32_t a0 = su32(sm), b0 = su32(sm + 32 * 1024);
    long long t0 = clock64();
    const uint64_t ad0 = desc(a0, kchunk_stride, 128), bd0 = desc(b0, kchunk_stride, 128);
    const uint64_t kstep = static_cast<uint64_t>((2 * kchunk_stride) >> 4);
    for (int i = 0; i < iters; i += 4) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t acc = (naccs == 2 && (k & 1)) ? N : 0;
        if (!WARP || elect_one())
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase + acc),
              "l"(ad0 + k * kstep), "l"(bd0 + k * kstep), "r"(idesc), "r"(1));
        if (WARP) __syncwarp();
      }
    }
    if (!WARP || elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile(
        "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
            su32(&bar)));
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    const uint32_t w = threadIdx.x >> 5;
    uint32_t v[32], x[32];
    long long t0 = clock64();
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%"
        "20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(tbase + ((w * 32u) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    uint32_t acc = 0;
    for (int i = 0; i < 32; ++i) acc += v[i];
    long long t1 = clock64();
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%"
        "20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]), "=r"(x[8]),
          "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]), "=r"(x[15]), "=r"(x[16]),
          "=r"(x[17]), "=r"(x[18]), "=r"(x[19]), "=r"(x[20]), "=r"(x[21]), "=r"(x[22]), "=r"(x[23]), "=r"(x[24]),
          "=r"(x[25]), "=r"(x[26]), "=r"(x[27]), "=r"(x[28]), "=r"(x[29]), "=r"(x[30]), "=r"(x[31])
        : "r"(tbase + ((w * 32u) << 16) + 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 32; ++i) acc += x[i];
    long long t2 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) { out[1] = t1 - t0; out[2] = t2 - t1; out[3] = acc; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 32);
  cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int iters = 4096;
  for (int w = 0; w < 2; ++w)
  for (int N : {64, 128, 256})
    for (int naccs : {1, 2}) {
      if (N * naccs > 512) continue;
      const int stride = N == 256 ? 4096 : 2048;  // K-chunk stride: rows x 16 B
      for (int rep = 0; rep < 2; ++rep) {
        if (w) probe<true><<<148, 128, 96 * 1024>>>(iters, N, naccs, stride, d);
        else probe<false><<<148, 128, 96 * 1024>>>(iters, N, naccs, stride, d);
      }
      unsigned long long cc[4] = {};
      cudaError_t e = cudaMemcpy(cc, d, 32, cudaMemcpyDeviceToHost);
      const unsigned long long c = cc[0];
      std::printf("  ldtm x32 + wait + 32 adds: %llu, %llu cycles\n", cc[1], cc[2]);
      const double cyc = double(c) / iters;
      const double macs = 128.0 * N * 16;
      std::printf("%s N=%3d accs=%d: %7.1f cycles/MMA  %6.0f MAC/clk/SM  (%s)\n", w ? "warp  " : "thread", N, naccs, cyc, macs / cyc,
                  cudaGetErrorString(e));
    }
  return 0;
}
