// alu_peaks.cu — microbenchmarks for the ALU roofline denominators that
// MEASURED_PEAKS.json does not carry (FP32 FFMA, POPC, FP64 DADD, INT64 add).
// Prints one JSON object; per-clock rates come from clock64() so they do not
// depend on the DVFS clock. Build: make tools; run on the GPU box.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

constexpr int kIters = 4096;
constexpr int kChains = 8;

__global__ void ffma_kernel(float* out, float a, float b, long long* cyc) {
  float r[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) r[c] = threadIdx.x * 1e-3f + c;
  long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) r[c] = fmaf(r[c], a, b);
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += r[c];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__device__ __forceinline__ unsigned long long ffma2u(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// FFMA2 (fma.rn.f32x2): 2 FMAs per lane per instruction.
__global__ void ffma2_kernel(float* out, float a, float b, long long* cyc) {
  unsigned long long r[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) r[c] = 0x3f8000003f800000ull + threadIdx.x + c;
  const unsigned long long aa = (static_cast<unsigned long long>(__float_as_uint(a)) << 32) | __float_as_uint(a);
  const unsigned long long bb = (static_cast<unsigned long long>(__float_as_uint(b)) << 32) | __float_as_uint(b);
  long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) r[c] = ffma2u(r[c], aa, bb);
  }
  long long t1 = clock64();
  unsigned long long s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s ^= r[c];
  if (s == 12345ull) out[0] = 1.0f;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void popc_kernel(unsigned* out, unsigned m, long long* cyc) {
  unsigned r[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) r[c] = threadIdx.x * 7919u + c;
  long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) r[c] = __popc(r[c] ^ m) + r[c];
  }
  long long t1 = clock64();
  unsigned s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += r[c];
  if (s == 12345u) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void dadd_kernel(double* out, double a, long long* cyc) {
  double r[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) r[c] = threadIdx.x * 1e-3 + c;
  long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) r[c] = r[c] + a;
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += r[c];
  if (s == 12345.0) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <class F>
void run(const char* name, F launch, double ops_per_thread_iter, int sms, bool last) {
  long long* cyc;
  cudaMalloc(&cyc, 8);
  const int blocks = sms * 8, threads = 256;
  launch(blocks, threads, cyc);  // warm
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  launch(blocks, threads, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double ops = double(blocks) * threads * kIters * kChains * ops_per_thread_iter;
  // per-clock rate per SM: ops of one SM's resident CTAs / cycles of one CTA
  const double per_clk_sm = double(8) * threads * kIters * kChains * ops_per_thread_iter / double(c);
  std::printf("  \"%s\": {\"ops_per_s\": %.6g, \"per_clk_per_sm\": %.4g, \"ms\": %.4f, \"implied_mhz\": %.1f}%s\n",
              name, ops / (ms * 1e-3), per_clk_sm, ms, double(c) / (ms * 1e3), last ? "" : ",");
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* fo;
  cudaMalloc(&fo, 64);
  std::printf("{\n  \"sms\": %d,\n", sms);
  run("ffma", [&](int g, int t, long long* c) { ffma_kernel<<<g, t>>>(fo, 1.0001f, 1e-7f, c); }, 1.0, sms, false);
  run("ffma2_fma_ops", [&](int g, int t, long long* c) { ffma2_kernel<<<g, t>>>(fo, 1.0001f, 1e-7f, c); }, 2.0, sms,
      false);
  run("popc_xor_add", [&](int g, int t, long long* c) {
    popc_kernel<<<g, t>>>(reinterpret_cast<unsigned*>(fo), 0x9E3779B9u, c);
  }, 1.0, sms, false);
  run("dadd", [&](int g, int t, long long* c) { dadd_kernel<<<g, t>>>(reinterpret_cast<double*>(fo), 1e-9, c); },
      1.0, sms, true);
  std::printf("}\n");
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
