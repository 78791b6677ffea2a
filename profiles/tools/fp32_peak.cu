// FP32 CUDA-core peak of this GPU (the compute roofline of the SIMT
// kernels; BASELINE.md §2 "FP32 SIMT: to be measured").  Two dependent-chain
// free FMA streams per thread, 8 independent accumulators, scalar FFMA and
// packed FFMA2 (fma.rn.f32x2) variants; grid = 148 SMs x 8 CTAs x 256
// threads.  Built by __graft_entry__.build() into profiles/tools/
// libfp32peak.so; bench.py loads it and times it with CUDA events.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) ffma_kernel(float* out, float a, float b) {
  float x[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) x[t] = threadIdx.x * 1e-3f + t;
#pragma unroll 4
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) x[t] = fmaf(x[t], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += x[t];
  if (s == 1234.5f) out[0] = s;  // never true; keeps the chains live
}

__global__ void __launch_bounds__(256) ffma2_kernel(float* out, float a, float b) {
  unsigned long long x[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const float lo = threadIdx.x * 1e-3f + t, hi = lo + 0.5f;
    x[t] = (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
  }
  const unsigned long long av = (unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(a) << 32);
  const unsigned long long bv = (unsigned long long)__float_as_uint(b) | ((unsigned long long)__float_as_uint(b) << 32);
#pragma unroll 4
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[t]) : "l"(av), "l"(bv));
  }
  float s = 0.f;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += __uint_as_float((unsigned)x[t]) + __uint_as_float((unsigned)(x[t] >> 32));
  if (s == 1234.5f) out[0] = s;
}

}  // namespace

extern "C" {

// Returns the best-of-`reps` FP32 TFLOP/s (2 flops per FMA) of the scalar
// (packed = 0) or packed f32x2 (packed = 1) kernel, or a negative value on error.
double es_fp32_peak_tflops(int packed, int reps) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1.0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out = nullptr;
  if (cudaMalloc(&out, 4) != cudaSuccess) return -2.0;
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int r = 0; r < reps + 1; ++r) {
    cudaEventRecord(e0);
    if (packed) ffma2_kernel<<<blocks, threads>>>(out, 0.999f, 1e-4f);
    else ffma_kernel<<<blocks, threads>>>(out, 0.999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = (double)blocks * threads * kIters * 8 * (packed ? 2 : 1);
    const double tf = 2.0 * fmas / (ms * 1e-3) / 1e12;
    if (r > 0 && tf > best) best = tf;  // r = 0 is warm-up
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? best : -3.0;
}

}  // extern "C"
