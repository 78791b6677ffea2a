// Host-side SO(3) constant tables for the fused kernels (double precision,
// built once per process, first-writer-wins under std::call_once -- the
// reference's cache discipline, clebsch.hpp:179-191 / SPEC.md:140).
//
// Independent C++ restatement of the reference conventions:
//  * real orthonormal solid harmonics, (-1)^m on positive m (harmonics.hpp:36-81)
//  * complex CG by the Racah sum (clebsch.hpp:26-52), complex->real change of
//    basis on all three legs with phase -i on odd paths (clebsch.hpp:89-173)
//  * EAAS re-index coefficients = the m_f = 0 slice of cg_real
//    (conventions.hpp:29-31) times Y_lf0(e_z)
//  * Wigner-D by an exact fit to the harmonic identity
//    solid(l, R p) = D solid(l, p) on 2l+1 fixed points (the SPEC's own
//    oracle for D): D = B A^-1 with A^-1 precomputed here.
#include <cmath>
#include <complex>
#include <mutex>

#include "es_internal.h"

namespace es {
namespace {

double fact(int n) {
  double r = 1.0;
  for (int k = 2; k <= n; ++k) r *= k;
  return r;
}
int psign(int n) { return (n % 2 == 0) ? 1 : -1; }
bool tri(int a, int b, int c) { return c >= std::abs(a - b) && c <= a + b; }

double complex_cg(int j1, int m1, int j2, int m2, int J, int M) {
  if (std::abs(m1) > j1 || std::abs(m2) > j2 || std::abs(M) > J || M != m1 + m2 || !tri(j1, j2, J)) return 0.0;
  const double delta = fact(j1 + j2 - J) * fact(j1 - j2 + J) * fact(-j1 + j2 + J) / fact(j1 + j2 + J + 1);
  const double pre = std::sqrt((2 * J + 1) * delta * fact(J + M) * fact(J - M) * fact(j1 + m1) * fact(j1 - m1) *
                               fact(j2 + m2) * fact(j2 - m2));
  double s = 0.0;
  for (int k = 0; k <= j1 + j2 - J; ++k) {
    const int a = j1 - m1 - k, b = j2 + m2 - k, c = J - j2 + m1 + k, d = J - j1 - m2 + k;
    if (a < 0 || b < 0 || c < 0 || d < 0) continue;
    s += psign(k) / (fact(k) * fact(j1 + j2 - J - k) * fact(a) * fact(b) * fact(c) * fact(d));
  }
  return pre * s;
}

// u(m, mu): row = real order m, column = complex order mu.
std::complex<double> ubasis(int m, int mu) {
  const double s = 1.0 / std::sqrt(2.0);
  if (m == 0) return mu == 0 ? 1.0 : 0.0;
  if (m > 0) {
    if (mu == m) return s;
    if (mu == -m) return psign(m) * s;
    return 0.0;
  }
  const int a = -m;
  if (mu == -a) return {0.0, s};
  if (mu == a) return {0.0, -psign(a) * s};
  return 0.0;
}

void invert(double* A, int n, double* out) {  // Gauss-Jordan, partial pivoting
  double aug[9][18];
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < 2 * n; ++c) aug[r][c] = c < n ? A[r * n + c] : (c - n == r ? 1.0 : 0.0);
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (std::fabs(aug[r][col]) > std::fabs(aug[piv][col])) piv = r;
    for (int c = 0; c < 2 * n; ++c) std::swap(aug[col][c], aug[piv][c]);
    const double d = aug[col][col];
    for (int c = 0; c < 2 * n; ++c) aug[col][c] /= d;
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      const double f = aug[r][col];
      for (int c = 0; c < 2 * n; ++c) aug[r][c] -= f * aug[col][c];
    }
  }
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) out[r * n + c] = aug[r][n + c];
}

// Fixed fit points: 9 unit vectors chosen offline (max condition number of
// the per-degree harmonic matrices A^l, l = 1..4, is 4.96 -> fp32-safe).
const double kFitPts[9][3] = {
    {-0.02253313821940293, -0.8539075592261686, 0.5199366672763067},
    {-0.4828586021383436, 0.8068987672323669, 0.34023807808634743},
    {0.9649931962101184, -0.20321038788424253, -0.16581215131622845},
    {0.8383752290779996, 0.47748391727098904, -0.26293741463694964},
    {0.6441588202098021, -0.4689532009893899, -0.6042700634879414},
    {-0.38199621792014643, -0.6917058465307652, 0.6128800138443589},
    {0.34916331310175835, 0.3418216231434718, 0.872492383196189},
    {-0.20213941235167712, 0.5988208311867272, -0.7749537212704741},
    {0.82318138755364, 0.5643060569515284, 0.0626983035901483}};

HostTables g_tables;
std::once_flag g_once;

void build_tables() {
  HostTables& t = g_tables;
  for (int k = 0; k < 9; ++k) {
    const double n = std::sqrt(kFitPts[k][0] * kFitPts[k][0] + kFitPts[k][1] * kFitPts[k][1] +
                               kFitPts[k][2] * kFitPts[k][2]);
    for (int a = 0; a < 3; ++a) t.fit_pts[k][a] = kFitPts[k][a] / n;
  }
  for (int l = 0; l <= kMaxL; ++l)
    for (int mu = 0; mu <= kMaxL; ++mu) {
      t.shnorm[l][mu] = 0.0;
      if (mu > l) continue;
      const double nrm = std::sqrt((2 * l + 1) / (4.0 * M_PI) * fact(l - mu) / fact(l + mu));
      t.shnorm[l][mu] = mu == 0 ? nrm : std::sqrt(2.0) * nrm;
    }
  for (int l = 1; l <= kMaxL; ++l) {
    const int d = 2 * l + 1;
    double A[81], Ai[81], y[9];
    for (int k = 0; k < d; ++k) {  // A[m][k] = Y^l_m(p_k)
      solid_harmonics_host(l, t.fit_pts[k], y);
      for (int m = 0; m < d; ++m) A[m * d + k] = y[m];
    }
    invert(A, d, Ai);  // Ai[k][m'] with D = B Ai
    for (int i = 0; i < d * d; ++i) t.ainv[l][i] = Ai[i];
  }
  for (int L = 0; L <= kMaxL; ++L)
    for (int e = 0; e < 85; ++e)
      for (int f = 0; f <= kMaxL; ++f) t.ca[L][e][f] = t.cb[L][e][f] = 0.0;
  for (int L = 0; L <= kMaxL; ++L)
    for (int lo = 0; lo <= L; ++lo)
      for (int li = 0; li <= L; ++li)
        for (int lf = 0; lf <= L; ++lf) {
          if (!tri(li, lf, lo)) continue;
          const double yf = std::sqrt((2 * lf + 1) / (4.0 * M_PI));
          const bool odd = (li + lf + lo) % 2 != 0;
          const int mm = std::min(li, lo);
          for (int m = -mm; m <= mm; ++m) {
            const int e = entry_index(lo, li, m);
            // even path: out[m] <- in[m];  odd path: out[m] <- in[-m]
            const double c = real_cg(li, odd ? -m : m, lf, 0, lo, m) * yf;
            if (odd) t.cb[L][e][lf] += c;
            else t.ca[L][e][lf] += c;
          }
        }
}

}  // namespace

int entry_index(int lo, int li, int m) {
  int s = 0;
  for (int a = 0; a <= kMaxL; ++a)
    for (int b = 0; b <= kMaxL; ++b) {
      const int mm = std::min(a, b);
      if (a == lo && b == li) return s + m + mm;
      s += 2 * mm + 1;
    }
  return -1;
}

double real_cg(int l1, int m1, int l2, int m2, int lo, int mo) {
  if (!tri(l1, l2, lo)) return 0.0;
  std::complex<double> acc(0.0, 0.0);
  const int mu1s[2] = {m1, -m1}, mu2s[2] = {m2, -m2}, mus[2] = {mo, -mo};
  for (int a = 0; a < (m1 == 0 ? 1 : 2); ++a)
    for (int b = 0; b < (m2 == 0 ? 1 : 2); ++b)
      for (int c = 0; c < (mo == 0 ? 1 : 2); ++c) {
        const int mu1 = mu1s[a], mu2 = mu2s[b], muo = mus[c];
        if (muo != mu1 + mu2) continue;
        acc += ubasis(mo, muo) * std::conj(ubasis(m1, mu1)) * std::conj(ubasis(m2, mu2)) *
               complex_cg(l1, mu1, l2, mu2, lo, muo);
      }
  if ((l1 + l2 + lo) % 2 != 0) acc *= std::complex<double>(0.0, -1.0);
  return acc.real();
}

void solid_harmonics_host(int l, const double* r, double* out) {
  const double x = r[0], y = r[1], z = r[2], r2 = x * x + y * y + z * z;
  if (l == 0) { out[0] = 0.28209479177387814; return; }
  double a = 1.0, b = 0.0;
  for (int mu = 0; mu <= l; ++mu) {
    if (mu > 0) { const double an = a * x - b * y, bn = a * y + b * x; a = an; b = bn; }
    double p2 = 0.0, pc = 1.0;
    for (int k = 2 * mu - 1; k > 1; k -= 2) pc *= k;
    for (int ll = mu + 1; ll <= l; ++ll) {
      const double pn = ((2 * ll - 1) * z * pc - (ll + mu - 1) * r2 * p2) / (ll - mu);
      p2 = pc; pc = pn;
    }
    const double nrm = std::sqrt((2 * l + 1) / (4.0 * M_PI) * fact(l - mu) / fact(l + mu));
    if (mu == 0) out[l] = nrm * pc;
    else {
      out[l + mu] = psign(mu) * std::sqrt(2.0) * nrm * pc * a;
      out[l - mu] = std::sqrt(2.0) * nrm * pc * b;
    }
  }
}

const HostTables& host_tables() {
  std::call_once(g_once, build_tables);
  return g_tables;
}

}  // namespace es
