// tcgen05.mma issue-to-completion rate for the operand layouts the key pass and
// the forward use (M=128, K=16 per instruction, bf16 -> f32): cycles per MMA of a
// long back-to-back stream on one SM, one CTA per SM on every SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2601_16622_b200/csrc \
//        mma_rate.cu -o mma_rate && ./mma_rate
#include <cstdio>
#include <cuda_runtime.h>
#include "umma.cuh"

using namespace es;

// mode 0: A smem no-swizzle K-major, B smem no-swizzle K-major, N=144 (the value / dV MMA)
// mode 1: A smem SW32 K-major,       B smem no-swizzle MN-major, N=144 (the key pass's D MMA)
// mode 2: A TMEM,                    B smem SW64 K-major,       N=16  (the S MMA)
// mode 3: A smem SW128 K-major,      B smem SW128 K-major,      N=144 (reference: swizzled)
// mode 4: A smem no-swizzle K-major, B smem no-swizzle K-major, N=256
// mode 5: A smem SW128 K-major,      B smem SW128 K-major,      N=256
__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int mode, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (umma::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 160 * 1024);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    umma::mbar_init(bar, 1);
    umma::fence_barrier_init();
  }
  if (threadIdx.x < 32) umma::tmem_alloc(tslot, 512);
  umma::fence_proxy_async();
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = umma::smem_u32(sm), b = umma::smem_u32(sm + 64 * 1024);
    const int N = (mode == 2) ? 16 : (mode >= 4 ? 256 : 144);
    const uint32_t idesc = umma::idesc_bf16(128, N, 0, mode == 1 ? 1 : 0);
    long long t0 = clock64();
    if (mode >= 6) {  // 6: constant descriptors, one accumulator; 7: four accumulators round-robin; 8: N=16 x4 acc
      const uint64_t ad = umma::sdesc(a, 128, 2304, 0), bd = umma::sdesc(b, 128, 2304, 0);
      const uint32_t id = umma::idesc_bf16(128, mode == 8 ? 16 : 144, 0, 0);
      for (int it = 0; it < iters; it += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          umma::mma_f16(tmem + (mode >= 7 ? 128 * u : 0), ad, bd, id, 1);
      }
      umma::mma_commit(bar);
      umma::mbar_wait(bar, 0);
      long long t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
    } else
    for (int it = 0; it < iters; ++it) {
      const int s = it % 9;
      switch (mode) {
        case 0:
          umma::mma_f16(tmem, umma::sdesc(a + s * 256, 128, 2304, 0), umma::sdesc(b + s * 256, 128, 2304, 0), idesc, 1);
          break;
        case 1:
          umma::mma_f16(tmem, umma::sdesc(a + s * 4096, 16, 256, 6), umma::sdesc(b + s * 4608, 2304, 128, 0), idesc, 1);
          break;
        case 2:
          umma::mma_f16_ts(tmem + 448, tmem + 8 * (s * 2), umma::sdesc(b + s * 1024, 16, 512, 4), idesc, 1);
          break;
        case 3:
          umma::mma_f16(tmem, umma::sdesc(a + (s & 3) * 32, 16, 1024, 2), umma::sdesc(b + (s & 3) * 32, 16, 1024, 2), idesc, 1);
          break;
        case 4:
          umma::mma_f16(tmem, umma::sdesc(a + s * 256, 128, 2304, 0), umma::sdesc(b + s * 256, 128, 2304, 0), idesc, 1);
          break;
        default:
          umma::mma_f16(tmem, umma::sdesc(a + (s & 3) * 32, 16, 1024, 2), umma::sdesc(b + (s & 3) * 32, 16, 1024, 2), idesc, 1);
          break;
      }
    }
    if (mode < 6) {
      umma::mma_commit(bar);
      umma::mbar_wait(bar, 0);
      long long t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  const int smem = 161 * 1024 + 1024;
  cudaFuncSetAttribute(mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"A nosw K  , B nosw K , N144 (value/dV)", "A SW32 K  , B nosw MN, N144 (key-pass D)",
                         "A TMEM    , B SW64 K , N16  (S)", "A SW128 K , B SW128 K, N144",
                         "A nosw K  , B nosw K , N256", "A SW128 K , B SW128 K, N256",
                         "const desc, 1 acc, N144", "const desc, 4 acc, N144", "const desc, 4 acc, N16"};
  for (int mode = 0; mode < 9; ++mode) {
    const int iters = 4096;
    mma_rate_kernel<<<148, 128, smem>>>(mode, iters, d);
    mma_rate_kernel<<<148, 128, smem>>>(mode, iters, d);
    long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const int N = (mode == 2 || mode == 8) ? 16 : (mode == 4 || mode == 5) ? 256 : 144;
    const double flops = 2.0 * 128 * N * 16;
    printf("mode %d  %-42s %7.1f cycles/MMA  %6.0f flop/cycle/SM  (%s)\n", mode, names[mode], (double)c / iters,
           flops * iters / c, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
