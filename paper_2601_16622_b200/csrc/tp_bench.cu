// Dense-CG vs EAAS tensor-product microbenchmark on the GPU (
// run_tp_bench SPEC.md:449-457, Figure 2): P independent
// (feature, direction) pairs, each producing the per-pair value of the
// attention's path set
//     x = sum_(li,lf,lo) (v^li (x) R^lf(r))^lo        (all degrees <= L, weight 1)
// either by the dense Clebsch-Gordan product (every (2li+1)(2lf+1)(2lo+1)
// coupling coefficient, the e3nn-style SO(3) product) or by EAAS (per-pair
// frame, Wigner blocks, sparse parity re-index: Prop. 1) -- the same device
// code the fused attention kernels run.  fp32, v [P][M][C], r [P][3], x [P][M][C].
#include <vector>

#include "attention_common.cuh"

namespace es {
namespace {

constexpr int kDenseMax = 13200;  // >= 13075 coefficients of the L = 4 path set
struct DenseTab {
  int npath;
  int li[70], lf[70], lo[70], off[71];  // paths (15 at L = 2, 65 at L = 4) and their offsets into g_dense_coef
};
__constant__ DenseTab c_dense;
__device__ float g_dense_coef[kDenseMax];  // per path [2lo+1][2li+1][2lf+1] (global: > the constant bank)

int dense_madds(int L) {
  int n = 0;
  for (int li = 0; li <= L; ++li)
    for (int lf = 0; lf <= L; ++lf)
      for (int lo = std::abs(li - lf); lo <= std::min(li + lf, L); ++lo) n += (2 * li + 1) * (2 * lf + 1) * (2 * lo + 1);
  return n;
}

es_status upload_dense(int L) {
  static int done[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && done[dev] == L + 1) return ES_OK;
  DenseTab t{};
  std::vector<float> coef;
  int n = 0;
  for (int li = 0; li <= L; ++li)
    for (int lf = 0; lf <= L; ++lf)
      for (int lo = std::abs(li - lf); lo <= std::min(li + lf, L); ++lo) {
        if (n >= 70) return fail(ES_UNSUPPORTED, "tp_bench: path table overflow");
        t.li[n] = li; t.lf[n] = lf; t.lo[n] = lo; t.off[n] = (int)coef.size();
        for (int mo = -lo; mo <= lo; ++mo)
          for (int mi = -li; mi <= li; ++mi)
            for (int mf = -lf; mf <= lf; ++mf) coef.push_back((float)real_cg(li, mi, lf, mf, lo, mo));
        ++n;
      }
  t.npath = n;
  t.off[n] = (int)coef.size();
  if (coef.size() > (size_t)kDenseMax) return fail(ES_UNSUPPORTED, "tp_bench: dense table overflow");
  cudaError_t e = cudaMemcpyToSymbol(c_dense, &t, sizeof(t));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_dense_coef, coef.data(), coef.size() * sizeof(float));
  if (e != cudaSuccess) return cuda_status(e, "tp_bench tables");
  if (dev < 64) done[dev] = L + 1;
  return ES_OK;
}

// one CTA per pair, one thread per channel: the dense product, all coefficients
template <int L>
__global__ void tp_dense_kernel(int C, const float* __restrict__ v, const float* __restrict__ r,
                                float* __restrict__ x) {
  constexpr int M = (L + 1) * (L + 1);
  const int p = blockIdx.x, c = threadIdx.x;
  __shared__ float Y[M];
  if (c == 0) {
    float y[9];
#pragma unroll
    for (int l = 0; l <= L; ++l) {
      if (l == 0) sh_degree<0>(r[3 * p], r[3 * p + 1], r[3 * p + 2], y);
      if (l == 1) sh_degree<1>(r[3 * p], r[3 * p + 1], r[3 * p + 2], y);
      if (l == 2) sh_degree<2>(r[3 * p], r[3 * p + 1], r[3 * p + 2], y);
      if (l == 3) sh_degree<3>(r[3 * p], r[3 * p + 1], r[3 * p + 2], y);
      if (l == 4) sh_degree<4>(r[3 * p], r[3 * p + 1], r[3 * p + 2], y);
      for (int m = 0; m < 2 * l + 1; ++m) Y[l * l + m] = y[m];
    }
  }
  __syncthreads();
  if (c >= C) return;
  float vi[M], acc[M];
#pragma unroll
  for (int a = 0; a < M; ++a) {
    vi[a] = v[((size_t)p * M + a) * C + c];
    acc[a] = 0.f;
  }
  for (int q = 0; q < c_dense.npath; ++q) {
    const int li = c_dense.li[q], lf = c_dense.lf[q], lo = c_dense.lo[q];
    const float* cf = g_dense_coef + c_dense.off[q];
    const int di = 2 * li + 1, df = 2 * lf + 1;
    for (int mo = 0; mo < 2 * lo + 1; ++mo) {
      float s = 0.f;
      for (int mi = 0; mi < di; ++mi)
        for (int mf = 0; mf < df; ++mf) s = fmaf(cf[(mo * di + mi) * df + mf], vi[li * li + mi] * Y[lf * lf + mf], s);
      acc[lo * lo + mo] += s;
    }
  }
#pragma unroll
  for (int a = 0; a < M; ++a) x[((size_t)p * M + a) * C + c] = acc[a];
}

// BP pairs per CTA: records prepared one pair per thread, then every thread
// applies EAAS to its channels for each pair (the attention kernels' scheme)
template <int L, int CPL>
__global__ void tp_eaas_kernel(KParams kp, int P, const float* __restrict__ v, const float* __restrict__ r,
                               float* __restrict__ x) {
  using LY = Lay<L>;
  constexpr int M = LY::M, REC = LY::REC, BP = LY::BP;
  extern __shared__ float4 smem4[];
  float* recs = reinterpret_cast<float*>(smem4);
  const int C = kp.C, c0 = threadIdx.x * CPL;
  const int p0 = blockIdx.x * BP, nb = min(BP, P - p0);
  for (int t = threadIdx.x; t < nb; t += blockDim.x)
    pair_prepare_vec<L, true>(kp, r[3 * (p0 + t)], r[3 * (p0 + t) + 1], r[3 * (p0 + t) + 2], p0 + t, recs + t * REC);
  __syncthreads();
  for (int e = 0; e < nb; ++e) {
    const int p = p0 + e;
    float vv[M][CPL], acc[M][CPL];
#pragma unroll
    for (int a = 0; a < M; ++a)
#pragma unroll
      for (int u = 0; u < CPL; ++u) {
        vv[a][u] = v[((size_t)p * M + a) * C + c0 + u];
        acc[a][u] = 0.f;
      }
    value_apply<L, CPL, false>(recs + e * REC, vv, 1.f, acc);
#pragma unroll
    for (int a = 0; a < M; ++a)
#pragma unroll
      for (int u = 0; u < CPL; ++u) x[((size_t)p * M + a) * C + c0 + u] = acc[a][u];
  }
}

template <int L, int CPL>
es_status run_eaas(int C, int P, const float* v, const float* r, float* x, cudaStream_t st) {
  KParams kp{};
  kp.C = C; kp.phi_mode = 1; kp.r_cut = 1e30f; kp.inv_rcut = 0.f;
  const size_t smem = (size_t)Lay<L>::BP * Lay<L>::REC * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(tp_eaas_kernel<L, CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tp_eaas_kernel<L, CPL><<<(P + Lay<L>::BP - 1) / Lay<L>::BP, C / CPL, smem, st>>>(kp, P, v, r, x);
  return cuda_status(cudaGetLastError(), "tp_eaas_kernel");
}

es_status check_tp(int L, int C, int P) {
  if (L != 2 && L != 4) return fail(ES_UNSUPPORTED, "tp_bench: L must be 2 or 4");
  if (C < 32 || C % 32 != 0 || C > 256 || P < 0) return fail(ES_INVALID_ARGUMENT, "tp_bench: C a multiple of 32 <= 256");
  return ES_OK;
}

}  // namespace
}  // namespace es

using namespace es;

extern "C" {

es_status es_tp_madds(int32_t L, int64_t* dense, int64_t* eaas) {
  if (L < 0 || L > kMaxL || !dense || !eaas) return fail(ES_INVALID_ARGUMENT, "tp_madds: L in [0, 4]");
  *dense = dense_madds(L);
  // EAAS per channel: align sum_l (2l+1)^2, re-index (non-zero rule entries), un-align sum_l (2l+1)^2
  int64_t d2 = 0;
  for (int l = 0; l <= L; ++l) d2 += (2 * l + 1) * (2 * l + 1);
  // re-index: one multiply-add per non-zero (entry, source) of the rule polynomials
  const HostTables& t = host_tables();
  int64_t re = 0;
  for (int lo = 0; lo <= L; ++lo)
    for (int li = 0; li <= L; ++li)
      for (int m = -std::min(lo, li); m <= std::min(lo, li); ++m) {
        const int e = entry_index(lo, li, m);
        bool a = false, b = false;
        for (int f = 0; f <= kMaxL; ++f) {
          a |= std::fabs(t.ca[L][e][f]) > 1e-12;
          b |= std::fabs(t.cb[L][e][f]) > 1e-12;
        }
        re += (a ? 1 : 0) + (b ? 1 : 0);
      }
  *eaas = 2 * d2 + re;
  return ES_OK;
}

es_status es_tp_bench_dense(int32_t L, int32_t C, int32_t P, const float* v, const float* r, float* x, void* stream) {
  es_status s = check_tp(L, C, P);
  if (s != ES_OK || P == 0) return s;
  if ((s = upload_tables_tu()) != ES_OK || (s = upload_dense(L)) != ES_OK) return s;
  if (L == 2) tp_dense_kernel<2><<<P, C, 0, (cudaStream_t)stream>>>(C, v, r, x);
  else tp_dense_kernel<4><<<P, C, 0, (cudaStream_t)stream>>>(C, v, r, x);
  return cuda_status(cudaGetLastError(), "tp_dense_kernel");
}

es_status es_tp_bench_eaas(int32_t L, int32_t C, int32_t P, const float* v, const float* r, float* x, void* stream) {
  es_status s = check_tp(L, C, P);
  if (s != ES_OK || P == 0) return s;
  if ((s = upload_tables_tu()) != ES_OK) return s;
  return L == 2 ? run_eaas<2, 2>(C, P, v, r, x, (cudaStream_t)stream)
                : run_eaas<4, 1>(C, P, v, r, x, (cudaStream_t)stream);
}

}  // extern "C"
