// C wrapper around the REFERENCE so3 headers (compiled where they lie under
// /root/reference through the Eigen shim).  ORACLE TEST INFRASTRUCTURE ONLY:
// lets tests pin oracle/esoracle.c against the reference's own code.
// Layout conversions: reference blocks are Eigen C x (2l+1) matrices
// (irreps.hpp:69-71); the oracle/GPU use [2l+1][C] row-major, the same bytes.
#include <cstring>
#include <string>

#include "equistream/core/counters.hpp"
#include "equistream/core/factorials.hpp"
#include "equistream/so3/clebsch.hpp"
#include "equistream/so3/conventions.hpp"
#include "equistream/so3/harmonics.hpp"
#include "equistream/so3/irreps.hpp"
#include "equistream/so3/rotation.hpp"
#include "equistream/so3/tensor_product.hpp"
#include "equistream/so3/wigner.hpp"
#include "legendre_oracle.hpp"

using namespace equistream;

extern "C" {

int esref_solid_harmonics(int l, const double* r, double* out) {
  try {
    const auto v = so3::solid_harmonics(l, Eigen::Vector3d(r[0], r[1], r[2]));
    for (int m = 0; m < 2 * l + 1; ++m) out[m] = v[m];
    return 0;
  } catch (...) { return -1; }
}

int esref_legendre_real_sph(int l, const double* u, double* out) {
  const auto v = oracle::real_sph_trig(l, Eigen::Vector3d(u[0], u[1], u[2]));
  for (int m = 0; m < 2 * l + 1; ++m) out[m] = v[m];
  return 0;
}

double esref_on_axis(int l, double r) { return so3::on_axis_solid_harmonic(l, r); }
double esref_complex_cg(int j1, int m1, int j2, int m2, int J, int M) { return so3::complex_cg(j1, m1, j2, m2, J, M); }
double esref_wigner_6j(int a, int b, int c, int d, int e, int f) { return so3::wigner_6j(a, b, c, d, e, f); }
double esref_factorial(int n) { return static_cast<double>(factorial(n)); }

int esref_cg_real(int l1, int l2, int lo, double* out) {
  try {
    if (!so3::triangle_valid(l1, l2, lo)) return -1;
    const auto& t = so3::cg_real(l1, l2, lo);
    const int d1 = 2 * l1 + 1, d2 = 2 * l2 + 1;
    for (int mo = -lo; mo <= lo; ++mo)
      for (int m1 = -l1; m1 <= l1; ++m1)
        for (int m2 = -l2; m2 <= l2; ++m2) out[(mo + lo) * d1 * d2 + (m1 + l1) * d2 + (m2 + l2)] = t.coeff(m1, m2, mo);
    return 0;
  } catch (...) { return -2; }
}

// u: [2l1+1][cu], v: [2l2+1][cv] -> out [2lo+1][max(cu,cv)]; returns madds.
long long esref_tensor_product_dense(const double* u, int l1, int cu, const double* v, int l2, int cv, int lo,
                                     double* out) {
  Eigen::MatrixXd U(cu, 2 * l1 + 1), V(cv, 2 * l2 + 1);
  for (int m = 0; m < 2 * l1 + 1; ++m) for (int c = 0; c < cu; ++c) U(c, m) = u[m * cu + c];
  for (int m = 0; m < 2 * l2 + 1; ++m) for (int c = 0; c < cv; ++c) V(c, m) = v[m * cv + c];
  counters().reset();
  const auto r = so3::tensor_product_dense(U, l1, V, l2, lo);
  if (!r) return -1;
  const int C = static_cast<int>(r->rows());
  for (int m = 0; m < 2 * lo + 1; ++m) for (int c = 0; c < C; ++c) out[m * C + c] = (*r)(c, m);
  return static_cast<long long>(counters().madds);
}

// The reference's wigner_d as shipped (defect F3 included): R row-major.
int esref_wigner_d(int l, const double* R, double* out) {
  try {
    Eigen::Matrix3d m;
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) m(i, j) = R[i * 3 + j];
    const auto d = so3::wigner_d(l, so3::Rotation(m));
    const int n = 2 * l + 1;
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) out[i * n + j] = d.matrix(i, j);
    return 0;
  } catch (...) { return -1; }
}

int esref_conventions_manifest(char* buf, int n) {
  const std::string s = so3::conventions_manifest();
  if (static_cast<int>(s.size()) + 1 > n) return -static_cast<int>(s.size()) - 1;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

}  // extern "C"
