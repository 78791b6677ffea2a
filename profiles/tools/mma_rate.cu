// tcgen05.mma throughput on one SM (one CTA per SM on every SM): a long
// back-to-back stream of M=128, K=16 (bf16 -> f32) MMAs with constant
// descriptors, one template instance per operand form, so the issuing thread
// does nothing but issue.  Also the same stream with the descriptors rebuilt
// per MMA (what the kernels did before round 2's descriptor change).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2601_16622_b200/csrc \
//        mma_rate.cu -o mma_rate && ./mma_rate
#include <cstdio>
#include <cuda_runtime.h>
#include "umma.cuh"

using namespace es;

// A: 0 smem no-swizzle K-major, 1 smem SW64 K-major, 2 TMEM
// B: 0 no-swizzle K-major, 1 SW64 K-major, 2 no-swizzle MN-major
template <int A, int B, int N, bool REBUILD>
__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int iters, long long* out) {
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
    const uint64_t ad = A == 0 ? umma::sdesc(a, 128, 2304, 0) : umma::sdesc(a, 16, 512, 4);
    const uint64_t bd = B == 0 ? umma::sdesc(b, 128, 2304, 0) : B == 1 ? umma::sdesc(b, 16, 512, 4)
                                                                       : umma::sdesc(b, 2304, 128, 0);
    constexpr uint32_t id = umma::idesc_bf16(128, N, 0, B == 2 ? 1 : 0);
    const uint32_t d = tmem + 256;
    long long t0 = clock64();
    for (int it = 0; it < iters; it += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        uint64_t bb = bd, aa = ad;
        if (REBUILD) {  // descriptors rebuilt from the address each time (the pre-change issue loops)
          const int s = (it + u) % 9;
          bb = umma::sdesc(b + s * 256, 128, 2304, 0);
          aa = umma::sdesc(a + s * 256, 128, 2304, 0);
        }
        if (A == 2) umma::mma_f16_ts(d, tmem + 8 * (u & 7), bb, id, 1);
        else umma::mma_f16(d, aa, bb, id, 1);
      }
    }
    umma::mma_commit(bar);
    umma::mbar_wait(bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  umma::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_dealloc(tmem, 512);
}

template <int A, int B, int N, bool REBUILD = false>
void run(const char* name, long long* d) {
  const int smem = 161 * 1024 + 1024, iters = 8192;
  cudaFuncSetAttribute(mma_rate_kernel<A, B, N, REBUILD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_rate_kernel<A, B, N, REBUILD><<<148, 128, smem>>>(iters, d);
  mma_rate_kernel<A, B, N, REBUILD><<<148, 128, smem>>>(iters, d);
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 128 * N * 16;
  printf("%-46s N=%3d %7.1f cycles/MMA %6.0f flop/cycle/SM (%s)\n", name, N, (double)c / iters, flops * iters / c,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<0, 0, 144>("A smem nosw, B nosw K (value / dV MMA)", d);
  run<0, 0, 144, true>("  same, descriptors rebuilt per MMA", d);
  run<0, 2, 144>("A smem nosw, B nosw MN (key-pass D, A as nosw)", d);
  run<2, 1, 16>("A TMEM, B SW64 K (the S MMA)", d);
  run<2, 1, 32>("A TMEM, B SW64 K", d);
  run<2, 1, 64>("A TMEM, B SW64 K", d);
  run<2, 1, 128>("A TMEM, B SW64 K", d);
  run<2, 0, 16>("A TMEM, B nosw K", d);
  run<0, 0, 16>("A smem nosw, B nosw K", d);
  run<1, 1, 16>("A smem SW64, B SW64 K", d);
  run<0, 0, 64>("A smem nosw, B nosw K", d);
  run<0, 0, 256>("A smem nosw, B nosw K", d);
  run<1, 1, 256>("A smem SW64, B SW64 K", d);
  return 0;
}
