// fp32_peak.cu — measures the B200's FP32 SIMT peak (MEASURED_PEAKS.json has HBM and bf16
// tensor peaks only). Independent FFMA2 (packed f32x2) and FFMA chains, all SMs, CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp32_peak tools/fp32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 1 << 14;

__global__ void __launch_bounds__(256) ffma2_loop(float* out, float a, float b) {
  unsigned long long acc[kChains];
  unsigned long long va, vb;
  asm("mov.b64 %0, {%1, %1};" : "=l"(va) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(vb) : "f"(b));
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    float x = threadIdx.x * 1e-3f + c;
    asm("mov.b64 %0, {%1, %1};" : "=l"(acc[c]) : "f"(x));
  }
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c)
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[c]) : "l"(va), "l"(vb));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[c]));
    s += lo + hi;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) ffma_loop(float* out, float a, float b) {
  float acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(acc[c]) : "f"(a), "f"(b));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int blocks = prop.multiProcessorCount * 8, threads = 256;
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best2 = 0, best1 = 0;
  for (int rep = 0; rep < 20; ++rep) {
    cudaEventRecord(e0);
    ffma2_loop<<<blocks, threads>>>(out, 0.9999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 2.0 * kChains * double(kIters) * blocks * threads;
    if (rep) best2 = flops / (ms * 1e-3) / 1e12 > best2 ? flops / (ms * 1e-3) / 1e12 : best2;
    cudaEventRecord(e0);
    ffma_loop<<<blocks, threads>>>(out, 0.9999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops1 = 2.0 * kChains * double(kIters) * blocks * threads;
    if (rep) best1 = flops1 / (ms * 1e-3) / 1e12 > best1 ? flops1 / (ms * 1e-3) / 1e12 : best1;
  }
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  std::printf("{\"gpu\": \"%s\", \"sms\": %d, \"fp32_ffma2_tflops\": %.2f, \"fp32_ffma_tflops\": %.2f, "
              "\"nominal_tflops_at_max_clock\": %.2f, \"max_clock_mhz\": %.0f, "
              "\"how\": \"best of 19 launches, %d CTAs x 256 threads x %d independent chains x %d FMA (packed f32x2 and scalar), CUDA events\"}\n",
              prop.name, prop.multiProcessorCount, best2, best1,
              256.0 * prop.multiProcessorCount * clk * 1e3 / 1e12, clk / 1e3, blocks, kChains, kIters);
  return 0;
}
