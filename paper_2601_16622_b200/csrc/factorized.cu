// Node-centric factorized message (Eq. 5
// PAPER.md:228-235, the three-stage flow of PAPER.md:299-322), fp64 on the
// GPU:
//
//   m_i = sum_j alpha_ij sum_paths (h_j^li (x) R^lf(r_j - r_i))^lo
//       = sum_(li,lf,lo) sum_u w(lf,u) sum_l' c(li,u,lb,lf,lo,l')
//             ( [sum_j alpha_ij (h_j^li (x) R^lb(r_j - o))^l'] (x) R^u(o - r_i) )^lo,   lb = lf - u
//
// R^lf(a + b) = sum_u w(lf,u) (R^u(a) (x) R^{lf-u}(b))^lf is the binomial
// translation identity (weights: conventions.hpp:32-34) and c the recoupling
// (h (x) (A (x) B)^lf)^lo = sum_l' c_l' ((h (x) B)^l' (x) A)^lo (the Wigner-6j
// step of Eq. 5), both solved once on the host by least squares -- the SPEC
// ledger's primary construction ("6j-vs-solve").  Three kernels:
//   source_term : S_j = (h_j (x) R(r_j - o))  -- per node j, all (li, lb, l')
//   aggregate   : A_i = sum_j alpha_ij S_j     -- per edge only a scalar alpha
//   target      : m_i = T(R(o - r_i)) A_i      -- per node i
// so the per-edge work is O(1) CG-free multiply-adds per component, the
// path's defining property.  Shipped for L <= 2 (SPEC ledger
// "degree budget"); origin o = the caller's recentring point (centroid).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "es_internal.h"

namespace es {
namespace {

constexpr int kFmMaxL = 2;

struct SrcEnt {
  int t;     // source component row
  int hrow;  // feature row li*li + mi
  int yidx;  // solid-harmonic index lb*lb + mb
  double c;
};
struct TgtEnt {
  int orow;  // output row lo*lo + mo
  int t;     // aggregated component row
  int yidx;  // u*u + ma
  double c;
};

int ncomp(int L) { return (L + 1) * (L + 1) * (L + 1) * (L + 1); }
int comp_offset(int L, int li, int lb, int l2) {
  int o = 0;
  for (int a = 0; a <= L; ++a)
    for (int b = 0; b <= L; ++b)
      for (int c = std::abs(a - b); c <= a + b; ++c) {
        if (a == li && b == lb && c == l2) return o;
        o += 2 * c + 1;
      }
  return -1;
}
bool tri(int a, int b, int c) { return c >= std::abs(a - b) && c <= a + b; }

// dense real CG product of single vectors: out[mo] = sum C(l1,l2,lo)[mo][m1][m2] u[m1] v[m2]
void tp(int l1, const double* u, int l2, const double* v, int lo, double* out) {
  for (int mo = -lo; mo <= lo; ++mo) {
    double s = 0.0;
    for (int m1 = -l1; m1 <= l1; ++m1)
      for (int m2 = -l2; m2 <= l2; ++m2) s += real_cg(l1, m1, l2, m2, lo, mo) * u[m1 + l1] * v[m2 + l2];
    out[mo + lo] = s;
  }
}

// small dense least squares (normal equations, Gauss-Jordan with pivoting)
bool solve(std::vector<double>& A, std::vector<double>& b, int n) {
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (std::fabs(A[r * n + col]) > std::fabs(A[piv * n + col])) piv = r;
    if (std::fabs(A[piv * n + col]) < 1e-300) return false;
    if (piv != col) {
      for (int k = 0; k < n; ++k) std::swap(A[col * n + k], A[piv * n + k]);
      std::swap(b[col], b[piv]);
    }
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      const double f = A[r * n + col] / A[col * n + col];
      for (int k = col; k < n; ++k) A[r * n + k] -= f * A[col * n + k];
      b[r] -= f * b[col];
    }
  }
  for (int r = 0; r < n; ++r) b[r] /= A[r * n + r];
  return true;
}

struct Lcg {
  unsigned long long s = 0x9E3779B97F4A7C15ull;
  double next() {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return ((s >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
  }
};

// translation weights w[u], u = 0..l (least squares over random (a, b))
bool translation_lsq(int l, double* w) {
  const int d = 2 * l + 1, nu = l + 1;
  std::vector<double> A(nu * nu, 0.0), b(nu, 0.0);
  Lcg g;
  double ya[9], yb[9], yab[9], cp[kMaxL + 1][9];
  for (int s = 0; s < 16 * nu; ++s) {
    const double a[3] = {g.next(), g.next(), g.next()}, bb[3] = {g.next(), g.next(), g.next()};
    const double ab[3] = {a[0] + bb[0], a[1] + bb[1], a[2] + bb[2]};
    solid_harmonics_host(l, ab, yab);
    for (int u = 0; u <= l; ++u) {
      solid_harmonics_host(u, a, ya);
      solid_harmonics_host(l - u, bb, yb);
      tp(u, ya, l - u, yb, l, cp[u]);
    }
    for (int m = 0; m < d; ++m)
      for (int p = 0; p < nu; ++p) {
        b[p] += cp[p][m] * yab[m];
        for (int q = 0; q < nu; ++q) A[p * nu + q] += cp[p][m] * cp[q][m];
      }
  }
  if (!solve(A, b, nu)) return false;
  for (int u = 0; u <= l; ++u) w[u] = b[u];
  return true;
}

// recoupling c[l'] of (h^li (x) (A^u (x) B^lb)^lf)^lo onto ((h (x) B)^l' (x) A)^lo
bool recouple_lsq(int li, int u, int lb, int lf, int lo, double* c) {
  for (int k = 0; k < 2 * kMaxL + 1; ++k) c[k] = 0.0;
  std::vector<int> ls;
  for (int l2 = std::abs(li - lb); l2 <= li + lb; ++l2)
    if (tri(l2, u, lo)) ls.push_back(l2);
  const int nl = (int)ls.size();
  if (!tri(u, lb, lf) || !tri(li, lf, lo) || nl == 0) return true;
  std::vector<double> A(nl * nl, 0.0), b(nl, 0.0);
  Lcg g;
  double h[9], av[9], bv[9], ab[9], lhs[9], hb[17], rhs[9][9];
  for (int s = 0; s < 12 * nl + 4; ++s) {
    for (int m = 0; m < 2 * li + 1; ++m) h[m] = g.next();
    for (int m = 0; m < 2 * u + 1; ++m) av[m] = g.next();
    for (int m = 0; m < 2 * lb + 1; ++m) bv[m] = g.next();
    tp(u, av, lb, bv, lf, ab);
    tp(li, h, lf, ab, lo, lhs);
    for (int p = 0; p < nl; ++p) {
      tp(li, h, lb, bv, ls[p], hb);
      tp(ls[p], hb, u, av, lo, rhs[p]);
    }
    for (int m = 0; m < 2 * lo + 1; ++m)
      for (int p = 0; p < nl; ++p) {
        b[p] += rhs[p][m] * lhs[m];
        for (int q = 0; q < nl; ++q) A[p * nl + q] += rhs[p][m] * rhs[q][m];
      }
  }
  if (!solve(A, b, nl)) return false;
  for (int p = 0; p < nl; ++p) c[ls[p]] = b[p];
  return true;
}

struct FmTables {
  int L = -1;
  SrcEnt* src = nullptr;
  TgtEnt* tgt = nullptr;
  int nsrc = 0, ntgt = 0;
};

// host build of the source / target entry lists for max degree L
bool build_tables(int L, std::vector<SrcEnt>& src, std::vector<TgtEnt>& tgt) {
  for (int li = 0; li <= L; ++li)
    for (int lb = 0; lb <= L; ++lb)
      for (int l2 = std::abs(li - lb); l2 <= li + lb; ++l2) {
        const int t0 = comp_offset(L, li, lb, l2);
        for (int m2 = -l2; m2 <= l2; ++m2)
          for (int mi = -li; mi <= li; ++mi)
            for (int mb = -lb; mb <= lb; ++mb) {
              const double c = real_cg(li, mi, lb, mb, l2, m2);
              if (std::fabs(c) > 1e-14) src.push_back({t0 + m2 + l2, li * li + mi + li, lb * lb + mb + lb, c});
            }
      }
  double w[kMaxL + 1][kMaxL + 1];
  for (int lf = 0; lf <= L; ++lf)
    if (!translation_lsq(lf, w[lf])) return false;
  // accumulate coefficients per (orow, t, yidx)
  const int M = (L + 1) * (L + 1), NS = ncomp(L);
  std::vector<double> acc((size_t)M * NS * M, 0.0);
  for (int li = 0; li <= L; ++li)
    for (int lf = 0; lf <= L; ++lf)
      for (int lo = 0; lo <= L; ++lo) {
        if (!tri(li, lf, lo)) continue;
        for (int u = 0; u <= lf; ++u) {
          const int lb = lf - u;
          double c[2 * kMaxL + 1];
          if (!recouple_lsq(li, u, lb, lf, lo, c)) return false;
          for (int l2 = std::abs(li - lb); l2 <= li + lb; ++l2) {
            const double k = w[lf][u] * c[l2];
            if (k == 0.0 || !tri(l2, u, lo)) continue;
            const int t0 = comp_offset(L, li, lb, l2);
            for (int mo = -lo; mo <= lo; ++mo)
              for (int m2 = -l2; m2 <= l2; ++m2)
                for (int ma = -u; ma <= u; ++ma) {
                  const double cg = real_cg(l2, m2, u, ma, lo, mo);
                  if (cg == 0.0) continue;
                  acc[((size_t)(lo * lo + mo + lo) * NS + t0 + m2 + l2) * M + u * u + ma + u] += k * cg;
                }
          }
        }
      }
  for (int o = 0; o < M; ++o)
    for (int t = 0; t < NS; ++t)
      for (int y = 0; y < M; ++y) {
        const double c = acc[((size_t)o * NS + t) * M + y];
        if (std::fabs(c) > 1e-14) tgt.push_back({o, t, y, c});
      }
  return true;
}

FmTables g_fm[64][kFmMaxL + 1];
std::mutex g_fm_mu;

es_status fm_tables(int L, FmTables* out) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 64) return fail(ES_UNSUPPORTED, "factorized: device index >= 64");
  std::lock_guard<std::mutex> lock(g_fm_mu);
  FmTables& t = g_fm[dev][L];
  if (t.L != L) {
    std::vector<SrcEnt> src;
    std::vector<TgtEnt> tgt;
    if (!build_tables(L, src, tgt)) return fail(ES_CUDA_ERROR, "factorized: table solve failed");
    if (cudaMalloc(&t.src, src.size() * sizeof(SrcEnt)) != cudaSuccess ||
        cudaMalloc(&t.tgt, tgt.size() * sizeof(TgtEnt)) != cudaSuccess)
      return fail(ES_CUDA_ERROR, "factorized: table allocation failed");
    cudaMemcpy(t.src, src.data(), src.size() * sizeof(SrcEnt), cudaMemcpyHostToDevice);
    cudaMemcpy(t.tgt, tgt.data(), tgt.size() * sizeof(TgtEnt), cudaMemcpyHostToDevice);
    t.nsrc = (int)src.size();
    t.ntgt = (int)tgt.size();
    t.L = L;
  }
  *out = t;
  return ES_OK;
}

// real solid harmonics |r|^l Y_lm of degrees 0..L (fp64, l <= 2), library convention
__device__ void solid_all(int L, double x, double y, double z, double* Y) {
  const double c0 = 0.28209479177387814, c1 = 0.4886025119029199, c2 = 1.0925484305920792,
               c20 = 0.31539156525252005;
  Y[0] = c0;
  if (L >= 1) {
    Y[1] = c1 * y; Y[2] = c1 * z; Y[3] = -c1 * x;
  }
  if (L >= 2) {
    Y[4] = c2 * x * y; Y[5] = c2 * y * z; Y[6] = c20 * (2.0 * z * z - x * x - y * y);
    Y[7] = -c2 * x * z; Y[8] = 0.5 * c2 * (x * x - y * y);
  }
}

// one CTA per atom, one thread per channel
__global__ void fm_source_kernel(int L, int C, int NS, double ox, double oy, double oz, const double* __restrict__ pos,
                                 const double* __restrict__ h, const SrcEnt* __restrict__ ent, int nent,
                                 double* __restrict__ S) {
  const int j = blockIdx.x, c = threadIdx.x;
  __shared__ double Y[25];
  const int M = (L + 1) * (L + 1);
  if (c == 0) solid_all(L, pos[3 * j] - ox, pos[3 * j + 1] - oy, pos[3 * j + 2] - oz, Y);
  __syncthreads();
  if (c >= C) return;
  double hv[9];
  for (int r = 0; r < M; ++r) hv[r] = h[((size_t)j * M + r) * C + c];
  double* o = S + (size_t)j * NS * C + c;
  for (int t = 0; t < NS; ++t) o[(size_t)t * C] = 0.0;
  for (int e = 0; e < nent; ++e) {
    const SrcEnt s = ent[e];
    o[(size_t)s.t * C] += s.c * hv[s.hrow] * Y[s.yidx];
  }
}

__global__ void fm_aggregate_kernel(int K, int H, int C, int NS, const int* __restrict__ nbr,
                                    const double* __restrict__ alpha, const double* __restrict__ S,
                                    double* __restrict__ A) {
  const int i = blockIdx.x, c = threadIdx.x;
  if (c >= C) return;
  const int hh = c / (C / H);
  double* a = A + (size_t)i * NS * C + c;
  for (int t = 0; t < NS; ++t) a[(size_t)t * C] = 0.0;
  for (int kk = 0; kk < K; ++kk) {
    const int j = nbr[(size_t)i * K + kk];
    if (j < 0) continue;
    const double al = alpha[((size_t)i * K + kk) * H + hh];
    const double* s = S + (size_t)j * NS * C + c;
    for (int t = 0; t < NS; ++t) a[(size_t)t * C] += al * s[(size_t)t * C];  // a scalar per edge: no CG work
  }
}

__global__ void fm_target_kernel(int L, int C, int NS, double ox, double oy, double oz, const double* __restrict__ pos,
                                 const double* __restrict__ A, const TgtEnt* __restrict__ ent, int nent,
                                 double* __restrict__ out) {
  const int i = blockIdx.x, c = threadIdx.x;
  __shared__ double Y[25];
  const int M = (L + 1) * (L + 1);
  if (c == 0) solid_all(L, ox - pos[3 * i], oy - pos[3 * i + 1], oz - pos[3 * i + 2], Y);
  __syncthreads();
  if (c >= C) return;
  double acc[9];
  for (int r = 0; r < M; ++r) acc[r] = 0.0;
  const double* a = A + (size_t)i * NS * C + c;
  for (int e = 0; e < nent; ++e) {
    const TgtEnt t = ent[e];
    acc[t.orow] += t.c * Y[t.yidx] * a[(size_t)t.t * C];
  }
  for (int r = 0; r < M; ++r) out[((size_t)i * M + r) * C + c] = acc[r];
}

es_status check_msg(const es_msg_desc* d) {
  if (!d) return fail(ES_INVALID_ARGUMENT, "factorized: null descriptor");
  if (d->N < 0 || d->K < 1 || d->H < 1 || d->C < 1 || d->C % d->H != 0)
    return fail(ES_INVALID_ARGUMENT, "factorized: N >= 0, K >= 1, C a multiple of H");
  if (d->L < 0 || d->L > kFmMaxL) return fail(ES_UNSUPPORTED, "factorized: L must be in [0, 2]");
  if (d->C > 1024) return fail(ES_UNSUPPORTED, "factorized: C <= 1024");
  return ES_OK;
}

}  // namespace
}  // namespace es

using namespace es;

extern "C" {

es_status es_translation_coefficients(int32_t l, double* w) {
  if (l < 0 || l > kMaxL || !w) return fail(ES_INVALID_ARGUMENT, "translation_coefficients: l in [0, 4]");
  return translation_lsq(l, w) ? ES_OK : fail(ES_CUDA_ERROR, "translation_coefficients: singular solve");
}

size_t es_factorized_workspace_size(const es_msg_desc* d) {
  if (check_msg(d) != ES_OK) return 0;
  return 2 * sizeof(double) * (size_t)d->N * ncomp(d->L) * d->C + 256;
}

es_status es_source_term(const es_msg_desc* d, const double* pos, const double* h, double* S, void* stream) {
  es_status s = check_msg(d);
  if (s != ES_OK) return s;
  if (d->N == 0) return ES_OK;
  if (!pos || !h || !S) return fail(ES_INVALID_ARGUMENT, "source_term: null buffer");
  FmTables t;
  if ((s = fm_tables(d->L, &t)) != ES_OK) return s;
  fm_source_kernel<<<d->N, (d->C + 31) / 32 * 32, 0, (cudaStream_t)stream>>>(
      d->L, d->C, ncomp(d->L), d->origin[0], d->origin[1], d->origin[2], pos, h, t.src, t.nsrc, S);
  return cuda_status(cudaGetLastError(), "fm_source_kernel");
}

es_status es_message_aggregate(const es_msg_desc* d, const int32_t* nbr, const double* alpha, const double* S,
                               double* A, void* stream) {
  es_status s = check_msg(d);
  if (s != ES_OK) return s;
  if (d->N == 0) return ES_OK;
  if (!nbr || !alpha || !S || !A) return fail(ES_INVALID_ARGUMENT, "message_aggregate: null buffer");
  fm_aggregate_kernel<<<d->N, (d->C + 31) / 32 * 32, 0, (cudaStream_t)stream>>>(d->K, d->H, d->C, ncomp(d->L), nbr,
                                                                               alpha, S, A);
  return cuda_status(cudaGetLastError(), "fm_aggregate_kernel");
}

es_status es_target_couple(const es_msg_desc* d, const double* pos, const double* A, double* out, void* stream) {
  es_status s = check_msg(d);
  if (s != ES_OK) return s;
  if (d->N == 0) return ES_OK;
  if (!pos || !A || !out) return fail(ES_INVALID_ARGUMENT, "target_couple: null buffer");
  FmTables t;
  if ((s = fm_tables(d->L, &t)) != ES_OK) return s;
  fm_target_kernel<<<d->N, (d->C + 31) / 32 * 32, 0, (cudaStream_t)stream>>>(
      d->L, d->C, ncomp(d->L), d->origin[0], d->origin[1], d->origin[2], pos, A, t.tgt, t.ntgt, out);
  return cuda_status(cudaGetLastError(), "fm_target_kernel");
}

es_status es_factorized_message(const es_msg_desc* d, const double* pos, const double* h, const int32_t* nbr,
                                const double* alpha, double* out, void* workspace, size_t workspace_bytes,
                                void* stream) {
  es_status s = check_msg(d);
  if (s != ES_OK) return s;
  if (d->N == 0) return ES_OK;
  if (!workspace || workspace_bytes < es_factorized_workspace_size(d))
    return fail(ES_INVALID_ARGUMENT, "factorized_message: workspace too small");
  double* S = (double*)workspace;
  double* A = S + (size_t)d->N * ncomp(d->L) * d->C;
  if ((s = es_source_term(d, pos, h, S, stream)) != ES_OK) return s;
  if ((s = es_message_aggregate(d, nbr, alpha, S, A, stream)) != ES_OK) return s;
  return es_target_couple(d, pos, A, out, stream);
}

}  // extern "C"
