// Per-degree Q/K/V projections (Eq. 6 PAPER.md:277-287, SPEC.md:257-265 +
// W_H) and their backward -- SIMT fp32-accumulate tiled GEMM path.
//
// For degree l the rows are (n, m) of the irreps layout, h[(n*M + l*l + m)*C],
// i.e. a row-strided [N(2l+1)] x C operand multiplied by W[l] = [C][2Dq+Cv];
// output column o scatters to q (o < Dq), k (o < 2Dq) or v.  The channel
// mixing never touches m (it commutes with D^l), so q.k stays invariant.
#include <cuda_bf16.h>

#include <cstdlib>

#include "es_internal.h"

namespace es {

namespace {
template <typename T>
__device__ __forceinline__ float ld(const T* p) {
  if constexpr (sizeof(T) == 4) return __ldg(reinterpret_cast<const float*>(p));
  else return __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(p)));
}
template <typename T>
__device__ __forceinline__ void st(T* p, float v) {
  if constexpr (sizeof(T) == 4) *reinterpret_cast<float*>(p) = v;
  else *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
}

constexpr int BM = 64, BN = 64, BK = 16;

// C[rows x cols] = A[rows x Kd] * B[Kd x cols], element access through
// functors; 256 threads, 4x4 outputs each, fp32 accumulation.
template <class FA, class FB, class FC>
__device__ __forceinline__ void gemm_tile(int rows, int cols, int k0, int k1, int rb, int cb, const FA& fa,
                                          const FB& fb, const FC& fc) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tr = tid / 16, tc = tid % 16;
  float acc[4][4] = {};
  for (int kk = k0; kk < k1; kk += BK) {
    for (int t = tid; t < BM * BK; t += 256) {
      const int r = t / BK, k = t % BK;
      const int gr = rb + r, gk = kk + k;
      As[k][r] = (gr < rows && gk < k1) ? fa(gr, gk) : 0.f;
    }
    for (int t = tid; t < BK * BN; t += 256) {
      const int k = t / BN, c = t % BN;
      const int gk = kk + k, gc = cb + c;
      Bs[k][c] = (gk < k1 && gc < cols) ? fb(gk, gc) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[4], b[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) a[x] = As[k][tr * 4 + x];
#pragma unroll
      for (int y = 0; y < 4; ++y) b[y] = Bs[k][tc * 4 + y];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(a[x], b[y], acc[x][y]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int gr = rb + tr * 4 + x, gc = cb + tc * 4 + y;
      if (gr < rows && gc < cols) fc(gr, gc, acc[x][y]);
    }
}

struct PK {
  int N, M, C, Dq, Cv, Wc, l, d;  // d = 2l+1
};

__device__ __forceinline__ size_t rowaddr(const PK& p, int r) {  // (n, m) -> row index n*M + l*l + m
  const int n = r / p.d, m = r - n * p.d;
  return (size_t)n * p.M + p.l * p.l + m;
}

template <typename T>
__global__ void __launch_bounds__(256) proj_fwd_kernel(PK p, const T* __restrict__ h, const T* __restrict__ W,
                                                       T* __restrict__ q, T* __restrict__ k, T* __restrict__ v) {
  const int rows = p.N * p.d;
  const T* Wl = W + (size_t)p.l * p.C * p.Wc;
  auto fa = [&](int r, int c) { return ld(h + rowaddr(p, r) * p.C + c); };
  auto fb = [&](int c, int o) { return ld(Wl + (size_t)c * p.Wc + o); };
  auto fc = [&](int r, int o, float val) {
    const size_t ra = rowaddr(p, r);
    if (o < p.Dq) st(q + ra * p.Dq + o, val);
    else if (o < 2 * p.Dq) st(k + ra * p.Dq + (o - p.Dq), val);
    else st(v + ra * p.Cv + (o - 2 * p.Dq), val);
  };
  gemm_tile(rows, p.Wc, 0, p.C, blockIdx.x * BM, blockIdx.y * BN, fa, fb, fc);
}

template <typename T>
__device__ __forceinline__ float gfetch(const PK& p, const T* dq, const T* dk, const T* dv, size_t ra, int o) {
  if (o < p.Dq) return ld(dq + ra * p.Dq + o);
  if (o < 2 * p.Dq) return ld(dk + ra * p.Dq + (o - p.Dq));
  return ld(dv + ra * p.Cv + (o - 2 * p.Dq));
}

template <typename T>
__global__ void __launch_bounds__(256) proj_bwd_dh_kernel(PK p, const T* __restrict__ W, const T* __restrict__ dq,
                                                          const T* __restrict__ dk, const T* __restrict__ dv,
                                                          T* __restrict__ dh) {
  const int rows = p.N * p.d;
  const T* Wl = W + (size_t)p.l * p.C * p.Wc;
  auto fa = [&](int r, int o) { return gfetch(p, dq, dk, dv, rowaddr(p, r), o); };
  auto fb = [&](int o, int c) { return ld(Wl + (size_t)c * p.Wc + o); };
  auto fc = [&](int r, int c, float val) { st(dh + rowaddr(p, r) * p.C + c, val); };
  gemm_tile(rows, p.C, 0, p.Wc, blockIdx.x * BM, blockIdx.y * BN, fa, fb, fc);
}

// dW[l] (C x Wc) += h^T G over a chunk of rows (split-K, fp32 atomics).
template <typename T>
__global__ void __launch_bounds__(256) proj_bwd_dw_kernel(PK p, int chunk, const T* __restrict__ h,
                                                          const T* __restrict__ dq, const T* __restrict__ dk,
                                                          const T* __restrict__ dv, float* __restrict__ dW) {
  const int rows = p.N * p.d;
  const int r0 = blockIdx.z * chunk, r1 = min(rows, r0 + chunk);
  float* dWl = dW + (size_t)p.l * p.C * p.Wc;
  auto fa = [&](int c, int r) { return ld(h + rowaddr(p, r) * p.C + c); };
  auto fb = [&](int r, int o) { return gfetch(p, dq, dk, dv, rowaddr(p, r), o); };
  auto fc = [&](int c, int o, float val) { atomicAdd(dWl + (size_t)c * p.Wc + o, val); };
  gemm_tile(p.C, p.Wc, r0, r1, blockIdx.x * BM, blockIdx.y * BN, fa, fb, fc);
}

template <typename T>
es_status fwd_t(const ProjArgs& a, const void* h, const void* W, void* q, void* k, void* v, cudaStream_t s) {
  for (int l = 0; l <= a.L; ++l) {
    PK p{a.N, (a.L + 1) * (a.L + 1), a.C, a.Dq, a.Cv, 2 * a.Dq + a.Cv, l, 2 * l + 1};
    const int rows = a.N * p.d;
    dim3 grid((rows + BM - 1) / BM, (p.Wc + BN - 1) / BN);
    proj_fwd_kernel<T><<<grid, 256, 0, s>>>(p, (const T*)h, (const T*)W, (T*)q, (T*)k, (T*)v);
  }
  return cuda_status(cudaGetLastError(), "proj_fwd_kernel");
}

template <typename T>
es_status bwd_t(const ProjArgs& a, const void* h, const void* W, const void* dq, const void* dk, const void* dv,
                void* dh, float* dW, cudaStream_t s) {
  const int Wc = 2 * a.Dq + a.Cv;
  if (dW) cudaMemsetAsync(dW, 0, sizeof(float) * (size_t)(a.L + 1) * a.C * Wc, s);
  for (int l = 0; l <= a.L; ++l) {
    PK p{a.N, (a.L + 1) * (a.L + 1), a.C, a.Dq, a.Cv, Wc, l, 2 * l + 1};
    const int rows = a.N * p.d;
    dim3 g1((rows + BM - 1) / BM, (a.C + BN - 1) / BN);
    proj_bwd_dh_kernel<T><<<g1, 256, 0, s>>>(p, (const T*)W, (const T*)dq, (const T*)dk, (const T*)dv, (T*)dh);
    if (dW) {
      const int tiles = ((a.C + BM - 1) / BM) * ((Wc + BN - 1) / BN);
      int splits = (148 * 4 + tiles - 1) / tiles;
      int chunk = (rows + splits - 1) / splits;
      chunk = ((chunk + BK - 1) / BK) * BK;
      if (chunk < BK) chunk = BK;
      splits = (rows + chunk - 1) / chunk;
      dim3 g2((a.C + BM - 1) / BM, (Wc + BN - 1) / BN, splits);
      proj_bwd_dw_kernel<T><<<g2, 256, 0, s>>>(p, chunk, (const T*)h, (const T*)dq, (const T*)dk, (const T*)dv, dW);
    }
  }
  return cuda_status(cudaGetLastError(), "proj_bwd kernels");
}
}  // namespace

static bool force_simt() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ES_PROJ_SIMT");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

es_status proj_fwd_launch(const ProjArgs& a, const void* h, const void* W, void* q, void* k, void* v,
                          cudaStream_t st) {
  if (a.N == 0) return ES_OK;
  if (!force_simt() && proj_tc_supported(a)) return proj_fwd_tc_launch(a, h, W, q, k, v, st);
  return a.dtype == ES_BF16 ? fwd_t<__nv_bfloat16>(a, h, W, q, k, v, st) : fwd_t<float>(a, h, W, q, k, v, st);
}

es_status proj_bwd_launch(const ProjArgs& a, const void* h, const void* W, const void* dq, const void* dk,
                          const void* dv, void* dh, float* dW, cudaStream_t st) {
  if (a.N == 0)  // dW is overwritten even with no rows (an empty shard all-reduces zeros)
    return dW ? cuda_status(cudaMemsetAsync(dW, 0, sizeof(float) * (size_t)(a.L + 1) * a.C * (2 * a.Dq + a.Cv), st),
                            "project_bwd: dW")
              : ES_OK;
  if (!force_simt() && proj_tc_supported(a)) return proj_bwd_tc_launch(a, h, W, dq, dk, dv, dh, dW, st);
  return a.dtype == ES_BF16 ? bwd_t<__nv_bfloat16>(a, h, W, dq, dk, dv, dh, dW, st)
                            : bwd_t<float>(a, h, W, dq, dk, dv, dh, dW, st);
}

}  // namespace es
