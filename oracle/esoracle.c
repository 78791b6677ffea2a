/*
 * esoracle.c -- CPU ORACLE for the equistream-b200 hot path.  TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py, and never by the product
 * (paper_2601_16622_b200/), which fails loudly without its CUDA library.
 *
 * Plain C (C11, double precision, OpenMP over target atoms) restatement of
 * the reference's algorithm for the fused equivariant attention path.  Every
 * function cites the reference file:line (relative to /root/reference) it
 * follows.  The reference headers themselves need Eigen (absent here); the
 * so3 pieces of this file are pinned against those very headers compiled
 * through a small Eigen shim (oracle/build_ref.sh -> oracle/_ref/libesref.so,
 * see tests/test_oracle_vs_ref.py), the rest against the SPEC known-answer
 * examples and the dense tensor-product oracle.
 *
 * Build: oracle/Makefile  (-O2 -ffp-contract=off -fopenmp; no FMA contraction
 * so that neighbour distances are bit-identical to the GPU builder's
 * __dmul_rn/__dadd_rn sequence).
 *
 * Feature layout ("irreps layout"): a node feature is [M][C] with
 * M = (L+1)^2, row index ll = l*l + (m + l), channels innermost.  This is the
 * byte order of the reference IrrepsFeature blocks (Eigen column-major
 * C_l x (2l+1), irreps.hpp:69-71) stacked over l.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ESO_MAXL 8
#define ESO_PI 3.14159265358979323846

/* ------------------------------------------------------------------ */
/* factorials.hpp:11-46                                                */
/* ------------------------------------------------------------------ */
static long double g_fact[65];
static int g_fact_init = 0;
static void fact_init(void) {
  if (g_fact_init) return;
  g_fact[0] = 1.0L;
  for (int n = 1; n <= 64; ++n) g_fact[n] = g_fact[n - 1] * (long double)n;
  g_fact_init = 1;
}
static long double factl(int n) { return g_fact[n]; }
double eso_factorial(int n) {
  fact_init();
  if (n < 0 || n > 64) return -1.0;
  return (double)g_fact[n];
}
static double dfact_odd(int n) { /* (2n-1)!!, factorials.hpp:35-39 */
  double r = 1.0;
  for (int k = 2 * n - 1; k > 1; k -= 2) r *= k;
  return r;
}
static int psign(int n) { return (n % 2 == 0) ? 1 : -1; }

/* ------------------------------------------------------------------ */
/* harmonics.hpp:36-81 -- real orthonormal solid harmonics, m=-l..l,   */
/* (-1)^m on the positive-m tesseral components (harmonics.hpp:76).    */
/* ------------------------------------------------------------------ */
void eso_solid_harmonics(int l, const double* r, double* out) {
  fact_init();
  const double x = r[0], y = r[1], z = r[2];
  const double r2 = x * x + y * y + z * z;
  if (l == 0) { out[0] = 0.28209479177387814; return; }
  double a = 1.0, b = 0.0; /* Re/Im (x+iy)^mu */
  for (int mu = 0; mu <= l; ++mu) {
    if (mu > 0) {
      const double an = a * x - b * y, bn = a * y + b * x;
      a = an; b = bn;
    }
    double p2 = 0.0, pc = dfact_odd(mu);
    for (int ll = mu + 1; ll <= l; ++ll) {
      const double pn = ((2 * ll - 1) * z * pc - (ll + mu - 1) * r2 * p2) / (double)(ll - mu);
      p2 = pc; pc = pn;
    }
    const double norm = sqrt((2 * l + 1) / (4.0 * ESO_PI) * (double)(factl(l - mu) / factl(l + mu)));
    if (mu == 0) out[l] = norm * pc;
    else {
      const double s = sqrt(2.0) * norm * pc;
      out[l + mu] = psign(mu) * s * a;
      out[l - mu] = s * b;
    }
  }
}

/* harmonics.hpp:93-97 */
double eso_on_axis_solid_harmonic(int l, double rn) {
  return pow(rn, l) * sqrt((2 * l + 1) / (4.0 * ESO_PI));
}

/* ------------------------------------------------------------------ */
/* clebsch.hpp:26-52 -- complex (Condon-Shortley) CG, Racah sum         */
/* ------------------------------------------------------------------ */
static int tri_ok(int a, int b, int c) { return c >= abs(a - b) && c <= a + b; }

double eso_complex_cg(int j1, int m1, int j2, int m2, int J, int M) {
  fact_init();
  if (abs(m1) > j1 || abs(m2) > j2 || abs(M) > J) return 0.0;
  if (M != m1 + m2) return 0.0;
  if (!tri_ok(j1, j2, J)) return 0.0;
  const long double delta = factl(j1 + j2 - J) * factl(j1 - j2 + J) * factl(-j1 + j2 + J) / factl(j1 + j2 + J + 1);
  const long double pre = sqrtl((long double)(2 * J + 1) * delta * factl(J + M) * factl(J - M) * factl(j1 + m1) *
                                factl(j1 - m1) * factl(j2 + m2) * factl(j2 - m2));
  int kmin = 0, kmax = j1 + j2 - J;
  if (j2 - J - m1 > kmin) kmin = j2 - J - m1;
  if (j1 - J + m2 > kmin) kmin = j1 - J + m2;
  if (j1 - m1 < kmax) kmax = j1 - m1;
  if (j2 + m2 < kmax) kmax = j2 + m2;
  long double sum = 0.0L;
  for (int k = kmin; k <= kmax; ++k) {
    const long double t = factl(k) * factl(j1 + j2 - J - k) * factl(j1 - m1 - k) * factl(j2 + m2 - k) *
                          factl(J - j2 + m1 + k) * factl(J - j1 - m2 + k);
    sum += psign(k) / t;
  }
  return (double)(pre * sum);
}

/* clebsch.hpp:56-85 -- Wigner 6j (Racah).  Used only by the factorized
 * path; exposed for the known-answer test. */
double eso_wigner_6j(int j1, int j2, int j3, int j4, int j5, int j6) {
  fact_init();
#define TOK(a, b, c) ((a) >= 0 && (b) >= 0 && (c) >= 0 && tri_ok(a, b, c))
  if (!TOK(j1, j2, j3) || !TOK(j1, j5, j6) || !TOK(j4, j2, j6) || !TOK(j4, j5, j3)) return 0.0;
#undef TOK
#define TRI(a, b, c) (factl((a) + (b) - (c)) * factl((a) - (b) + (c)) * factl(-(a) + (b) + (c)) / factl((a) + (b) + (c) + 1))
  const long double pre = sqrtl(TRI(j1, j2, j3) * TRI(j1, j5, j6) * TRI(j4, j2, j6) * TRI(j4, j5, j3));
#undef TRI
  int tmin = j1 + j2 + j3;
  if (j1 + j5 + j6 > tmin) tmin = j1 + j5 + j6;
  if (j4 + j2 + j6 > tmin) tmin = j4 + j2 + j6;
  if (j4 + j5 + j3 > tmin) tmin = j4 + j5 + j3;
  int tmax = j1 + j2 + j4 + j5;
  if (j2 + j3 + j5 + j6 < tmax) tmax = j2 + j3 + j5 + j6;
  if (j3 + j1 + j6 + j4 < tmax) tmax = j3 + j1 + j6 + j4;
  long double sum = 0.0L;
  for (int t = tmin; t <= tmax; ++t) {
    const long double den = factl(t - j1 - j2 - j3) * factl(t - j1 - j5 - j6) * factl(t - j4 - j2 - j6) *
                            factl(t - j4 - j5 - j3) * factl(j1 + j2 + j4 + j5 - t) * factl(j2 + j3 + j5 + j6 - t) *
                            factl(j3 + j1 + j6 + j4 - t);
    sum += psign(t) * factl(t + 1) / den;
  }
  return (double)(pre * sum);
}

/* ------------------------------------------------------------------ */
/* clebsch.hpp:89-103 -- complex->real basis change u(m, mu)           */
/* returned as re/im parts; clebsch.hpp:120-173 real table             */
/* ------------------------------------------------------------------ */
static void ubasis(int l, int m, int mu, double* re, double* im) {
  const double s = 1.0 / sqrt(2.0);
  *re = 0.0; *im = 0.0;
  if (m == 0) { if (mu == 0) *re = 1.0; return; }
  if (m > 0) {
    if (mu == m) *re = s;
    else if (mu == -m) *re = psign(m) * s;
  } else {
    const int a = -m; /* row l-a */
    if (mu == -a) *im = s;                 /* u(l-a, l-a) = i/sqrt2 */
    else if (mu == a) *im = -psign(a) * s; /* u(l-a, l+a) = -i (-1)^a /sqrt2 */
  }
  (void)l;
}

/* out[(mo+lo)*d1*d2 + (m1+l1)*d2 + (m2+l2)], returns 0 ok, -1 triangle
 * violation, -2 imaginary residue (clebsch.hpp:164-167). */
int eso_cg_real(int l1, int l2, int lo, double* out) {
  if (!tri_ok(l1, l2, lo)) return -1;
  const int d1 = 2 * l1 + 1, d2 = 2 * l2 + 1;
  const int odd = ((l1 + l2 + lo) % 2) != 0;
  for (int mo = -lo; mo <= lo; ++mo)
    for (int m1 = -l1; m1 <= l1; ++m1)
      for (int m2 = -l2; m2 <= l2; ++m2) {
        double are = 0.0, aim = 0.0;
        const int mu1s[2] = {m1, -m1}, mu2s[2] = {m2, -m2}, mus[2] = {mo, -mo};
        for (int a = 0; a < (m1 == 0 ? 1 : 2); ++a)
          for (int b = 0; b < (m2 == 0 ? 1 : 2); ++b)
            for (int c = 0; c < (mo == 0 ? 1 : 2); ++c) {
              const int mu1 = mu1s[a], mu2 = mu2s[b], muo = mus[c];
              if (muo != mu1 + mu2) continue;
              double uo_r, uo_i, u1_r, u1_i, u2_r, u2_i;
              ubasis(lo, mo, muo, &uo_r, &uo_i);
              ubasis(l1, m1, mu1, &u1_r, &u1_i);
              ubasis(l2, m2, mu2, &u2_r, &u2_i);
              u1_i = -u1_i; u2_i = -u2_i; /* conj */
              /* w = uo * u1c * u2c */
              const double t_r = uo_r * u1_r - uo_i * u1_i, t_i = uo_r * u1_i + uo_i * u1_r;
              const double w_r = t_r * u2_r - t_i * u2_i, w_i = t_r * u2_i + t_i * u2_r;
              if (w_r == 0.0 && w_i == 0.0) continue;
              const double cg = eso_complex_cg(l1, mu1, l2, mu2, lo, muo);
              are += w_r * cg; aim += w_i * cg;
            }
        if (odd) { /* multiply by -i */
          const double nr = aim, ni = -are;
          are = nr; aim = ni;
        }
        if (fabs(aim) > 1e-12) return -2;
        out[(mo + lo) * d1 * d2 + (m1 + l1) * d2 + (m2 + l2)] = are;
      }
  return 0;
}

/* Cached tables for l <= ESO_MAXL/2 paths used by attention (l <= 4). */
#define ESO_LT 5
static double* g_cg[ESO_LT][ESO_LT][ESO_LT];
static int g_cg_init = 0;
static void cg_cache_init(void) {
  if (g_cg_init) return;
#pragma omp critical(eso_cg_cache)
  {
    if (!g_cg_init) {
      for (int a = 0; a < ESO_LT; ++a)
        for (int b = 0; b < ESO_LT; ++b)
          for (int c = 0; c < ESO_LT; ++c) {
            g_cg[a][b][c] = NULL;
            if (!tri_ok(a, b, c)) continue;
            double* t = (double*)calloc((size_t)(2 * a + 1) * (2 * b + 1) * (2 * c + 1), sizeof(double));
            eso_cg_real(a, b, c, t);
            g_cg[a][b][c] = t;
          }
      g_cg_init = 1;
    }
  }
}
static const double* cgt(int a, int b, int c) { return g_cg[a][b][c]; }

/* ------------------------------------------------------------------ */
/* tensor_product.hpp:18-49 -- literal dense CG product, per channel.  */
/* Blocks are [2l+1][C] (m-major, channel innermost).                  */
/* ------------------------------------------------------------------ */
static void tp_dense_tab(const double* tab, const double* u, int l1, int cu, const double* v, int l2, int cv, int lo,
                         double* out) {
  const int C = cu > cv ? cu : cv;
  const int d1 = 2 * l1 + 1, d2 = 2 * l2 + 1;
  for (int mo = 0; mo < 2 * lo + 1; ++mo)
    for (int c = 0; c < C; ++c) {
      const int c1 = cu == 1 ? 0 : c, c2 = cv == 1 ? 0 : c;
      double acc = 0.0;
      for (int m1 = 0; m1 < d1; ++m1)
        for (int m2 = 0; m2 < d2; ++m2) acc += tab[mo * d1 * d2 + m1 * d2 + m2] * u[m1 * cu + c1] * v[m2 * cv + c2];
      out[mo * C + c] = acc;
    }
}

int eso_tensor_product_dense(const double* u, int l1, int cu, const double* v, int l2, int cv, int lo, double* out) {
  if (!tri_ok(l1, l2, lo)) return -1;
  if (cu != cv && cu != 1 && cv != 1) return -3;
  if (l1 < ESO_LT && l2 < ESO_LT && lo < ESO_LT) {
    cg_cache_init();
    tp_dense_tab(cgt(l1, l2, lo), u, l1, cu, v, l2, cv, lo, out);
    return 0;
  }
  const int d1 = 2 * l1 + 1, d2 = 2 * l2 + 1;
  double* tab = (double*)malloc(sizeof(double) * (size_t)(2 * lo + 1) * d1 * d2);
  eso_cg_real(l1, l2, lo, tab);
  tp_dense_tab(tab, u, l1, cu, v, l2, cv, lo, out);
  free(tab);
  return 0;
}

/* ------------------------------------------------------------------ */
/* Wigner-D.  The reference wigner.hpp:31-56 builds G_y with the wrong  */
/* sign and is an anti-homomorphism; the oracle instead     */
/* follows the convention anchor itself (wigner.hpp:19-20,              */
/* SPEC.md:89,126): D(R) is the least-squares solution of               */
/*   solid(l, R p_k) = D solid(l, p_k)  over 4(2l+1) spiral points      */
/* ("least-squares fit of D from harmonic evaluations").     */
/* D is row-major [(2l+1)][(2l+1)], acting on value vectors.            */
/* ------------------------------------------------------------------ */
static int solve_inplace(double* A, double* B, int n, int nrhs) { /* A X = B, X -> B */
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (fabs(A[r * n + col]) > fabs(A[piv * n + col])) piv = r;
    if (fabs(A[piv * n + col]) < 1e-300) return -1;
    if (piv != col) {
      for (int k = 0; k < n; ++k) { double t = A[col * n + k]; A[col * n + k] = A[piv * n + k]; A[piv * n + k] = t; }
      for (int k = 0; k < nrhs; ++k) { double t = B[col * nrhs + k]; B[col * nrhs + k] = B[piv * nrhs + k]; B[piv * nrhs + k] = t; }
    }
    const double d = A[col * n + col];
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      const double f = A[r * n + col] / d;
      if (f == 0.0) continue;
      for (int k = col; k < n; ++k) A[r * n + k] -= f * A[col * n + k];
      for (int k = 0; k < nrhs; ++k) B[r * nrhs + k] -= f * B[col * nrhs + k];
    }
  }
  for (int r = 0; r < n; ++r)
    for (int k = 0; k < nrhs; ++k) B[r * nrhs + k] /= A[r * n + r];
  return 0;
}

int eso_wigner_d(int l, const double* R, double* D) {
  const int d = 2 * l + 1;
  if (l == 0) { D[0] = 1.0; return 0; }
  const int np = 4 * d;
  double* Y = (double*)malloc(sizeof(double) * d * np);  /* Y[m][k] = solid(l, p_k) */
  double* Z = (double*)malloc(sizeof(double) * d * np);  /* Z[m][k] = solid(l, R p_k) */
  double tmp[2 * ESO_MAXL + 1];
  const double ga = ESO_PI * (3.0 - sqrt(5.0));
  for (int k = 0; k < np; ++k) { /* golden spiral points on the unit sphere */
    const double zz = 1.0 - (2.0 * k + 1.0) / np;
    const double rr = sqrt(1.0 - zz * zz);
    const double p[3] = {rr * cos(ga * k), rr * sin(ga * k), zz};
    const double q[3] = {R[0] * p[0] + R[1] * p[1] + R[2] * p[2], R[3] * p[0] + R[4] * p[1] + R[5] * p[2],
                         R[6] * p[0] + R[7] * p[1] + R[8] * p[2]};
    eso_solid_harmonics(l, p, tmp);
    for (int m = 0; m < d; ++m) Y[m * np + k] = tmp[m];
    eso_solid_harmonics(l, q, tmp);
    for (int m = 0; m < d; ++m) Z[m * np + k] = tmp[m];
  }
  /* D Y = Z  ->  (Y Y^T) D^T = Y Z^T */
  double* A = (double*)malloc(sizeof(double) * d * d);
  double* B = (double*)malloc(sizeof(double) * d * d);
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      double s = 0.0, t = 0.0;
      for (int k = 0; k < np; ++k) { s += Y[a * np + k] * Y[b * np + k]; t += Y[a * np + k] * Z[b * np + k]; }
      A[a * d + b] = s; B[a * d + b] = t;
    }
  int st = solve_inplace(A, B, d, d); /* B = D^T */
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) D[a * d + b] = B[b * d + a];
  free(Y); free(Z); free(A); free(B);
  return st;
}

/* The same least-squares D in closed form for the per-pair hot loops of
 * the CPU baseline: D = Z Y^T (Y Y^T)^-1 with the fixed-point factor
 * Pinv = Y^T (Y Y^T)^-1 ([np][d]) computed once per l. */
static double* g_pinv[ESO_LT];
static void pinv_init(void) {
#pragma omp critical(eso_pinv_cache)
  if (!g_pinv[ESO_LT - 1]) {
    for (int l = 0; l < ESO_LT; ++l) {
      const int d = 2 * l + 1, np = 4 * d;
      double* P = (double*)malloc(sizeof(double) * np * d);
      double* Y = (double*)malloc(sizeof(double) * d * np);
      double* A = (double*)malloc(sizeof(double) * d * d);
      double* Bt = (double*)malloc(sizeof(double) * d * np); /* (Y Y^T)^-1 Y  -> [d][np] */
      double tmp[2 * ESO_MAXL + 1];
      const double ga = ESO_PI * (3.0 - sqrt(5.0));
      for (int k = 0; k < np; ++k) {
        const double zz = 1.0 - (2.0 * k + 1.0) / np, rr = sqrt(1.0 - zz * zz);
        const double p[3] = {rr * cos(ga * k), rr * sin(ga * k), zz};
        eso_solid_harmonics(l, p, tmp);
        for (int m = 0; m < d; ++m) Y[m * np + k] = tmp[m];
      }
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
          double t = 0.0;
          for (int k = 0; k < np; ++k) t += Y[a * np + k] * Y[b * np + k];
          A[a * d + b] = t;
        }
      memcpy(Bt, Y, sizeof(double) * d * np);
      solve_inplace(A, Bt, d, np);
      for (int k = 0; k < np; ++k)
        for (int m = 0; m < d; ++m) P[k * d + m] = Bt[m * np + k];
      free(Y); free(A); free(Bt);
      g_pinv[l] = P;
    }
  }
}
static void wigner_d_fast(int l, const double* R, double* D) {
  const int d = 2 * l + 1, np = 4 * d;
  if (l == 0) { D[0] = 1.0; return; }
  const double* P = g_pinv[l];
  const double ga = ESO_PI * (3.0 - sqrt(5.0));
  double z[2 * ESO_MAXL + 1];
  for (int a = 0; a < d * d; ++a) D[a] = 0.0;
  for (int k = 0; k < np; ++k) {
    const double zz = 1.0 - (2.0 * k + 1.0) / np, rr = sqrt(1.0 - zz * zz);
    const double p[3] = {rr * cos(ga * k), rr * sin(ga * k), zz};
    const double q[3] = {R[0] * p[0] + R[1] * p[1] + R[2] * p[2], R[3] * p[0] + R[4] * p[1] + R[5] * p[2],
                         R[6] * p[0] + R[7] * p[1] + R[8] * p[2]};
    eso_solid_harmonics(l, q, z);
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) D[a * d + b] += z[a] * P[k * d + b];
  }
}

/* ------------------------------------------------------------------ */
/* SPEC eaas (gauge SPEC.md:216): R with R r = |r| e_z */
/* rotating about (r^ x e_z)/|.| by arccos(r^.e_z); identity / pi about */
/* e_x within 1e-6 of +/- e_z.  Row-major 3x3.                          */
/* ------------------------------------------------------------------ */
int eso_alignment_rotation(const double* r, double* R) {
  const double n = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  if (n <= 1e-8) return -1; /* degenerate */
  const double u[3] = {r[0] / n, r[1] / n, r[2] / n};
  const double s = sqrt(u[0] * u[0] + u[1] * u[1]);
  for (int i = 0; i < 9; ++i) R[i] = 0.0;
  if (s < 1e-6 && u[2] > 0) { R[0] = R[4] = R[8] = 1.0; return 0; }
  if (s < 1e-6 && u[2] < 0) { R[0] = 1.0; R[4] = -1.0; R[8] = -1.0; return 0; }
  /* axis k = u x e_z = (u_y, -u_x, 0)/s; angle t: cos t = u_z, sin t = s */
  const double kx = u[1] / s, ky = -u[0] / s, kz = 0.0;
  const double c = u[2], sn = s, C1 = 1.0 - c;
  R[0] = c + kx * kx * C1;      R[1] = kx * ky * C1 - kz * sn; R[2] = kx * kz * C1 + ky * sn;
  R[3] = ky * kx * C1 + kz * sn; R[4] = c + ky * ky * C1;     R[5] = ky * kz * C1 - kx * sn;
  R[6] = kz * kx * C1 - ky * sn; R[7] = kz * ky * C1 + kx * sn; R[8] = c + kz * kz * C1;
  return 0;
}

/* for each m_o the surviving source m_i and coefficient
 * cg_real(li,lf,lo)[m_o](m_i, 0) (the m_f = 0 slice; conventions.hpp:29-31).
 * src[m_o+lo] = m_i or -1000 when absent.  Returns the entry count. */
int eso_reindex_rule(int li, int lf, int lo, int* src, double* coef) {
  cg_cache_init();
  if (!tri_ok(li, lf, lo) || li >= ESO_LT || lf >= ESO_LT || lo >= ESO_LT) return -1;
  const double* t = cgt(li, lf, lo);
  const int d1 = 2 * li + 1, d2 = 2 * lf + 1;
  int cnt = 0;
  for (int mo = -lo; mo <= lo; ++mo) {
    src[mo + lo] = -1000; coef[mo + lo] = 0.0;
    for (int mi = -li; mi <= li; ++mi) {
      const double c = t[(mo + lo) * d1 * d2 + (mi + li) * d2 + lf];
      if (fabs(c) > 1e-14) {
        src[mo + lo] = mi; coef[mo + lo] = c; ++cnt;
      }
    }
  }
  return cnt;
}

typedef struct { int src[2 * ESO_LT + 1]; double coef[2 * ESO_LT + 1]; } eso_rule;
static eso_rule g_rule[ESO_LT][ESO_LT][ESO_LT];
static int g_rule_init = 0;
static const eso_rule* rule_of(int li, int lf, int lo) {
  if (!g_rule_init) {
#pragma omp critical(eso_rule_cache)
    {
      if (!g_rule_init) {
        for (int a = 0; a < ESO_LT; ++a)
          for (int b = 0; b < ESO_LT; ++b)
            for (int c = 0; c < ESO_LT; ++c)
              if (tri_ok(a, b, c)) eso_reindex_rule(a, b, c, g_rule[a][b][c].src, g_rule[a][b][c].coef);
        g_rule_init = 1;
      }
    }
  }
  return &g_rule[li][lf][lo];
}

/* apply_reindex: out[m_o] = coef * h~[m_i] * rmag */
void eso_apply_reindex(int li, int lf, int lo, const double* ht, int C, double rmag, double* out) {
  int src[2 * ESO_LT + 1];
  double coef[2 * ESO_LT + 1];
  eso_reindex_rule(li, lf, lo, src, coef);
  for (int mo = 0; mo < 2 * lo + 1; ++mo)
    for (int c = 0; c < C; ++c)
      out[mo * C + c] = (src[mo] == -1000) ? 0.0 : coef[mo] * ht[(src[mo] + li) * C + c] * rmag;
}

/* eaas_tensor_product: align -> reindex -> unalign.
 * h: [2li+1][C]; Rgauge optional (NULL -> SPEC gauge).  r = 0 returns the
 * exact dense result. */
int eso_eaas_tp(const double* h, int li, int C, const double* r, int lf, int lo, const double* Rgauge, double* out) {
  if (!tri_ok(li, lf, lo)) return -1;
  const double n = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  const int di = 2 * li + 1, dout = 2 * lo + 1;
  if (n <= 1e-8) {
    double y[2 * ESO_LT + 1];
    eso_solid_harmonics(lf, r, y);
    return eso_tensor_product_dense(h, li, C, y, lf, 1, lo, out);
  }
  double R[9];
  if (Rgauge) memcpy(R, Rgauge, sizeof(R));
  else eso_alignment_rotation(r, R);
  double Di[(2 * ESO_LT + 1) * (2 * ESO_LT + 1)], Do[(2 * ESO_LT + 1) * (2 * ESO_LT + 1)];
  eso_wigner_d(li, R, Di);
  eso_wigner_d(lo, R, Do);
  double* ht = (double*)malloc(sizeof(double) * di * C);
  double* w = (double*)malloc(sizeof(double) * dout * C);
  for (int a = 0; a < di; ++a) /* align: h~ = D_i h (per channel value vector) */
    for (int c = 0; c < C; ++c) {
      double s = 0.0;
      for (int b = 0; b < di; ++b) s += Di[a * di + b] * h[b * C + c];
      ht[a * C + c] = s;
    }
  eso_apply_reindex(li, lf, lo, ht, C, eso_on_axis_solid_harmonic(lf, n), w);
  for (int a = 0; a < dout; ++a) /* unalign: out = D_o^T w */
    for (int c = 0; c < C; ++c) {
      double s = 0.0;
      for (int b = 0; b < dout; ++b) s += Do[b * dout + a] * w[b * C + c];
      out[a * C + c] = s;
    }
  free(ht); free(w);
  return 0;
}

/* ------------------------------------------------------------------ */
/* Neighbour index (build_neighbors SPEC.md:431-439):  */
/* per atom the K nearest j != i with d^2 < r_cut^2 (strict), sorted by */
/* (d^2, j), sentinel -1.  Atoms only pair inside their segment          */
/* (seg_ptr[B+1], molecule batches) and, with box != NULL, under the      */
/* minimum-image convention (the PBC extension of SURVEY F7).  d^2 is     */
/* ((dx*dx + dy*dy) + dz*dz) in double, no contraction -- the exact      */
/* sequence the GPU builder uses, so lists are bit-identical.            */
/* ------------------------------------------------------------------ */
static inline double pair_d2(const double* pi, const double* pj, const double* box) {
  double dx = pj[0] - pi[0], dy = pj[1] - pi[1], dz = pj[2] - pi[2];
  if (box) {
    dx = dx - box[0] * rint(dx / box[0]);
    dy = dy - box[1] * rint(dy / box[1]);
    dz = dz - box[2] * rint(dz / box[2]);
  }
  const double xx = dx * dx, yy = dy * dy, zz = dz * dz;
  const double s = xx + yy;
  return s + zz;
}

typedef struct { double d2; int j; } eso_cand;
static int cand_cmp(const void* a, const void* b) {
  const eso_cand* x = (const eso_cand*)a;
  const eso_cand* y = (const eso_cand*)b;
  if (x->d2 < y->d2) return -1;
  if (x->d2 > y->d2) return 1;
  return (x->j > y->j) - (x->j < y->j);
}

/* Returns 0, or -1 if an atom has more than max_cand in-cutoff
 * candidates (never for sane systems; max_cand = 4096). */
int eso_build_neighbors(int N, const double* pos, int nseg, const int* seg_ptr, const double* box, int K, double r_cut,
                        int* nbr, double* dist, int* count) {
  const double rc2 = r_cut * r_cut;
  int err = 0;
  int one_seg[2] = {0, N};
  if (!seg_ptr) { seg_ptr = one_seg; nseg = 1; }
  for (int s = 0; s < nseg; ++s) {
    const int a0 = seg_ptr[s], a1 = seg_ptr[s + 1];
#pragma omp parallel for schedule(dynamic, 16)
    for (int i = a0; i < a1; ++i) {
      eso_cand* cand = (eso_cand*)malloc(sizeof(eso_cand) * 4096);
      int nc = 0;
      for (int j = a0; j < a1; ++j) {
        if (j == i) continue;
        const double d2 = pair_d2(pos + 3 * i, pos + 3 * j, box);
        if (d2 < rc2) {
          if (nc < 4096) { cand[nc].d2 = d2; cand[nc].j = j; }
          ++nc;
        }
      }
      if (nc > 4096) {
#pragma omp atomic write
        err = -1;
        nc = 4096;
      }
      qsort(cand, (size_t)nc, sizeof(eso_cand), cand_cmp);
      const int keep = nc < K ? nc : K;
      for (int k = 0; k < K; ++k) {
        nbr[(size_t)i * K + k] = k < keep ? cand[k].j : -1;
        if (dist) dist[(size_t)i * K + k] = k < keep ? sqrt(cand[k].d2) : 0.0;
      }
      count[i] = keep;
      free(cand);
    }
  }
  return err;
}

/* ------------------------------------------------------------------ */
/* Projections, Eq. (6) PAPER.md:277-287 / SPEC.md:257-265, plus W_H.  */
/* W: [(L+1)][C][Dq + Dq + Cv]  (per-l channel mixing, never mixing m).  */
/* q,k: [N][M][Dq], v: [N][M][Cv].                                      */
/* ------------------------------------------------------------------ */
void eso_project(int N, int L, int C, int Dq, int Cv, const double* h, const double* W, double* q, double* k, double* v) {
  const int M = (L + 1) * (L + 1), Wc = 2 * Dq + Cv;
#pragma omp parallel for schedule(static)
  for (int n = 0; n < N; ++n)
    for (int l = 0; l <= L; ++l)
      for (int m = 0; m < 2 * l + 1; ++m) {
        const int mm = l * l + m;
        const double* x = h + ((size_t)n * M + mm) * C;
        const double* w = W + (size_t)l * C * Wc;
        for (int o = 0; o < Wc; ++o) {
          double s = 0.0;
          for (int c = 0; c < C; ++c) s += x[c] * w[(size_t)c * Wc + o];
          if (o < Dq) q[((size_t)n * M + mm) * Dq + o] = s;
          else if (o < 2 * Dq) k[((size_t)n * M + mm) * Dq + (o - Dq)] = s;
          else v[((size_t)n * M + mm) * Cv + (o - 2 * Dq)] = s;
        }
      }
}

/* Backward of eso_project: dh and dW from dq, dk, dv. */
void eso_project_bwd(int N, int L, int C, int Dq, int Cv, const double* h, const double* W, const double* dq,
                     const double* dk, const double* dv, double* dh, double* dW) {
  const int M = (L + 1) * (L + 1), Wc = 2 * Dq + Cv;
#pragma omp parallel for schedule(static)
  for (int n = 0; n < N; ++n)
    for (int l = 0; l <= L; ++l)
      for (int m = 0; m < 2 * l + 1; ++m) {
        const int mm = l * l + m;
        const double* w = W + (size_t)l * C * Wc;
        for (int c = 0; c < C; ++c) {
          double s = 0.0;
          for (int o = 0; o < Wc; ++o) {
            double g;
            if (o < Dq) g = dq[((size_t)n * M + mm) * Dq + o];
            else if (o < 2 * Dq) g = dk[((size_t)n * M + mm) * Dq + (o - Dq)];
            else g = dv[((size_t)n * M + mm) * Cv + (o - 2 * Dq)];
            s += g * w[(size_t)c * Wc + o];
          }
          dh[((size_t)n * M + mm) * C + c] = s;
        }
      }
  if (!dW) return;
  /* dW[l][c][o] = sum_(n, m) h[n][lm][c] g[n][lm][o]: per (l, c) row, outputs innermost (contiguous) */
#pragma omp parallel for schedule(static)
  for (int lc = 0; lc < (L + 1) * C; ++lc) {
    const int l = lc / C, c = lc % C;
    double* row = dW + ((size_t)l * C + c) * Wc;
    for (int o = 0; o < Wc; ++o) row[o] = 0.0;
    for (int n = 0; n < N; ++n)
      for (int m = 0; m < 2 * l + 1; ++m) {
        const int mm = l * l + m;
        const double hv = h[((size_t)n * M + mm) * C + c];
        const double* gq = dq + ((size_t)n * M + mm) * Dq;
        const double* gk = dk + ((size_t)n * M + mm) * Dq;
        const double* gv = dv + ((size_t)n * M + mm) * Cv;
        for (int o = 0; o < Dq; ++o) row[o] += hv * gq[o];
        for (int o = 0; o < Dq; ++o) row[Dq + o] += hv * gk[o];
        for (int o = 0; o < Cv; ++o) row[2 * Dq + o] += hv * gv[o];
      }
  }
}

/* ------------------------------------------------------------------ */
/* Stream attention (Alg. 1).         */
/* ------------------------------------------------------------------ */
typedef struct {
  int N, K, H, L;
  int Dq, Cv;        /* q/k channels per (l,m) row; value channels */
  double r_cut;
  int value_mode;    /* 0 = plain (phi * v_j, SPEC stream_aggregate),
                        1 = dense CG (v_j (x) R^lf(r_ij) summed over paths; the
                            edge_centric_message oracle SPEC.md:342-350),
                        2 = EAAS per pair (the reference CPU path) */
  int phi_mode;      /* 0 = cosine cutoff, 1 = phi == 1 */
  const double* box; /* NULL or [3] minimum image */
  int bias_mode;     /* RadialScalars b: 0 = b == 0, 1 = b0 + b1 r + b2 r^2 */
  double bias[3];
} eso_attn_desc;

static inline void pair_vec(const double* pos, int i, int j, const double* box, double* r) {
  r[0] = pos[3 * j] - pos[3 * i]; r[1] = pos[3 * j + 1] - pos[3 * i + 1]; r[2] = pos[3 * j + 2] - pos[3 * i + 2];
  if (box) for (int a = 0; a < 3; ++a) r[a] = r[a] - box[a] * rint(r[a] / box[a]);
}
static inline double bias_of(const eso_attn_desc* d, double rn) { /* score(q,k,r) = tau q.k + b(r), Eq. 18 */
  return d->bias_mode ? d->bias[0] + d->bias[1] * rn + d->bias[2] * rn * rn : 0.0;
}
static inline double phi_of(const eso_attn_desc* d, double rn) {
  if (d->phi_mode == 1) return 1.0;
  return rn < d->r_cut ? 0.5 * (cos(ESO_PI * rn / d->r_cut) + 1.0) : 0.0;
}

/* Value message x[M][Cv] of pair (i,j) for the chosen value mode, phi included.
 * Mode 1 is the literal per-path dense CG product (tensor_product.hpp:18-49).
 * Mode 2 is EAAS organised the way a CPU implementation
 * would: one alignment rotation and D^l per pair, align each l_i block
 * once, sparse re-index every path, un-align each l_o block once. */
static void pair_value(const eso_attn_desc* d, const double* v, int j, const double* r, double phi, double* x,
                       double* scratch /* [2][M][Cv] */) {
  const int L = d->L, M = (L + 1) * (L + 1), Cv = d->Cv;
  const double* vj = v + (size_t)j * M * Cv;
  if (d->value_mode == 0) {
    for (int t = 0; t < M * Cv; ++t) x[t] = phi * vj[t];
    return;
  }
  memset(x, 0, sizeof(double) * M * Cv);
  const double rn = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  if (d->value_mode == 1 || rn <= 1e-8) {
    double* tmp = scratch;
    double y[2 * ESO_LT + 1];
    for (int li = 0; li <= L; ++li)
      for (int lf = 0; lf <= L; ++lf) {
        eso_solid_harmonics(lf, r, y);
        for (int lo = 0; lo <= L; ++lo) {
          if (!tri_ok(li, lf, lo)) continue;
          tp_dense_tab(cgt(li, lf, lo), vj + (size_t)li * li * Cv, li, Cv, y, lf, 1, lo, tmp);
          double* xo = x + (size_t)lo * lo * Cv;
          for (int t = 0; t < (2 * lo + 1) * Cv; ++t) xo[t] += phi * tmp[t];
        }
      }
    return;
  }
  double R[9];
  eso_alignment_rotation(r, R);
  double* ht = scratch;
  double* w = scratch + (size_t)M * Cv;
  memset(w, 0, sizeof(double) * M * Cv);
  double D[ESO_LT][(2 * ESO_LT - 1) * (2 * ESO_LT - 1)];
  for (int l = 0; l <= L; ++l) {
    const int dl = 2 * l + 1;
    wigner_d_fast(l, R, D[l]);
    for (int a = 0; a < dl; ++a)
      for (int c = 0; c < Cv; ++c) {
        double s = 0.0;
        for (int b = 0; b < dl; ++b) s += D[l][a * dl + b] * vj[(size_t)(l * l + b) * Cv + c];
        ht[(size_t)(l * l + a) * Cv + c] = s;
      }
  }
  for (int li = 0; li <= L; ++li)
    for (int lf = 0; lf <= L; ++lf) {
      const double rmag = eso_on_axis_solid_harmonic(lf, rn);
      for (int lo = 0; lo <= L; ++lo) {
        if (!tri_ok(li, lf, lo)) continue;
        const eso_rule* ru = rule_of(li, lf, lo);
        for (int mo = 0; mo < 2 * lo + 1; ++mo) {
          if (ru->src[mo] == -1000) continue;
          const double cf = ru->coef[mo] * rmag;
          const double* hs = ht + (size_t)(li * li + ru->src[mo] + li) * Cv;
          double* wo = w + (size_t)(lo * lo + mo) * Cv;
          for (int c = 0; c < Cv; ++c) wo[c] += cf * hs[c];
        }
      }
    }
  for (int l = 0; l <= L; ++l) {
    const int dl = 2 * l + 1;
    for (int a = 0; a < dl; ++a)
      for (int c = 0; c < Cv; ++c) {
        double s = 0.0;
        for (int b = 0; b < dl; ++b) s += D[l][b * dl + a] * w[(size_t)(l * l + b) * Cv + c];
        x[(size_t)(l * l + a) * Cv + c] = phi * s;
      }
  }
}

/* stream_aggregate: one pass per atom with (mu, z, A)
 * per head in double, zero output for zero-neighbour rows
 * (SPEC.md:311).  out [N][M][Cv]; lse [N][H] = mu + log z (or -inf). */
void eso_attn_fwd(const eso_attn_desc* d, const double* q, const double* k, const double* v, const double* pos,
                  const int* nbr, double* out, double* lse) {
  const int N = d->N, K = d->K, H = d->H, L = d->L, M = (L + 1) * (L + 1);
  const int Dq = d->Dq, Cv = d->Cv, dqh = Dq / H, cvh = Cv / H;
  const double tau = 1.0 / sqrt((double)M * dqh);
  cg_cache_init();
  pinv_init();
#pragma omp parallel
  {
    double* x = (double*)malloc(sizeof(double) * M * Cv);
    double* scr = (double*)malloc(sizeof(double) * 2 * M * Cv);
    double* A = (double*)malloc(sizeof(double) * M * Cv);
    double* mu = (double*)malloc(sizeof(double) * H);
    double* z = (double*)malloc(sizeof(double) * H);
    double* s = (double*)malloc(sizeof(double) * H);
#pragma omp for schedule(dynamic, 4)
    for (int i = 0; i < N; ++i) {
      for (int h = 0; h < H; ++h) { mu[h] = -INFINITY; z[h] = 0.0; }
      memset(A, 0, sizeof(double) * M * Cv);
      for (int kk = 0; kk < K; ++kk) {
        const int j = nbr[(size_t)i * K + kk];
        if (j < 0) continue; /* Alg. 1 line "if j is padding: continue" */
        double r[3];
        pair_vec(pos, i, j, d->box, r);
        const double rn = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
        for (int h = 0; h < H; ++h) {
          double acc = 0.0;
          for (int mm = 0; mm < M; ++mm)
            for (int c = h * dqh; c < (h + 1) * dqh; ++c)
              acc += q[((size_t)i * M + mm) * Dq + c] * k[((size_t)j * M + mm) * Dq + c];
          s[h] = tau * acc + bias_of(d, rn); /* Eq. 18 */
        }
        pair_value(d, v, j, r, phi_of(d, rn), x, scr);
        for (int h = 0; h < H; ++h) { /* Eqs. 15-17 */
          const double mu2 = s[h] > mu[h] ? s[h] : mu[h];
          const double sc = exp(mu[h] - mu2), e = exp(s[h] - mu2);
          z[h] = z[h] * sc + e;
          for (int mm = 0; mm < M; ++mm)
            for (int c = h * cvh; c < (h + 1) * cvh; ++c)
              A[mm * Cv + c] = A[mm * Cv + c] * sc + e * x[mm * Cv + c];
          mu[h] = mu2;
        }
      }
      for (int h = 0; h < H; ++h) {
        const int empty = !(z[h] > 0.0);
        for (int mm = 0; mm < M; ++mm)
          for (int c = h * cvh; c < (h + 1) * cvh; ++c)
            out[((size_t)i * M + mm) * Cv + c] = empty ? 0.0 : A[mm * Cv + c] / z[h];
        if (lse) lse[(size_t)i * H + h] = empty ? -INFINITY : mu[h] + log(z[h]);
      }
    }
    free(x); free(scr); free(A); free(mu); free(z); free(s);
  }
}

/* dense_reference_aggregate: materialise the N x K x H
 * score matrix, two-pass stable softmax, then the weighted sum. */
void eso_attn_dense_ref(const eso_attn_desc* d, const double* q, const double* k, const double* v, const double* pos,
                        const int* nbr, double* out) {
  const int N = d->N, K = d->K, H = d->H, L = d->L, M = (L + 1) * (L + 1);
  const int Dq = d->Dq, Cv = d->Cv, dqh = Dq / H, cvh = Cv / H;
  const double tau = 1.0 / sqrt((double)M * dqh);
  cg_cache_init();
  pinv_init();
  double* S = (double*)malloc(sizeof(double) * (size_t)N * K * H);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < N; ++i)
    for (int kk = 0; kk < K; ++kk) {
      const int j = nbr[(size_t)i * K + kk];
      for (int h = 0; h < H; ++h) {
        double acc = -INFINITY;
        if (j >= 0) {
          double r[3];
          pair_vec(pos, i, j, d->box, r);
          acc = 0.0;
          for (int mm = 0; mm < M; ++mm)
            for (int c = h * dqh; c < (h + 1) * dqh; ++c)
              acc += q[((size_t)i * M + mm) * Dq + c] * k[((size_t)j * M + mm) * Dq + c];
          acc = acc * tau + bias_of(d, sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]));
        }
        S[((size_t)i * K + kk) * H + h] = acc;
      }
    }
#pragma omp parallel
  {
    double* x = (double*)malloc(sizeof(double) * M * Cv);
    double* scr = (double*)malloc(sizeof(double) * 2 * M * Cv);
#pragma omp for schedule(dynamic, 4)
    for (int i = 0; i < N; ++i) {
      double* o = out + (size_t)i * M * Cv;
      memset(o, 0, sizeof(double) * M * Cv);
      for (int h = 0; h < H; ++h) { /* pass 1: max and normaliser */
        double mx = -INFINITY, z = 0.0;
        for (int kk = 0; kk < K; ++kk) { double sv = S[((size_t)i * K + kk) * H + h]; if (sv > mx) mx = sv; }
        if (mx == -INFINITY) continue;
        for (int kk = 0; kk < K; ++kk) { double sv = S[((size_t)i * K + kk) * H + h]; if (sv != -INFINITY) z += exp(sv - mx); }
        for (int kk = 0; kk < K; ++kk) S[((size_t)i * K + kk) * H + h] =
            (S[((size_t)i * K + kk) * H + h] == -INFINITY) ? 0.0 : exp(S[((size_t)i * K + kk) * H + h] - mx) / z;
      }
      for (int kk = 0; kk < K; ++kk) {
        const int j = nbr[(size_t)i * K + kk];
        if (j < 0) continue;
        double r[3];
        pair_vec(pos, i, j, d->box, r);
        const double rn = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
        pair_value(d, v, j, r, phi_of(d, rn), x, scr);
        for (int h = 0; h < H; ++h) {
          const double a = S[((size_t)i * K + kk) * H + h];
          for (int mm = 0; mm < M; ++mm)
            for (int c = h * cvh; c < (h + 1) * cvh; ++c) o[mm * Cv + c] += a * x[mm * Cv + c];
        }
      }
    }
    free(x); free(scr);
  }
  free(S);
}

/* Per-pair linear value operator T (x = T v per channel, phi included):
 * T[(lo,mo)][(li,mi)] = phi sum_lf sum_mf C^{lo mo}_{li mi, lf mf} R^lf_mf(r)
 * for value_mode 1/2 (identical maps, Prop. 1), identity*phi for mode 0. */
static void pair_T(const eso_attn_desc* d, const double* r, double phi, double* T) {
  const int L = d->L, M = (L + 1) * (L + 1);
  memset(T, 0, sizeof(double) * M * M);
  if (d->value_mode == 0) { for (int a = 0; a < M; ++a) T[a * M + a] = phi; return; }
  double y[2 * ESO_LT + 1];
  for (int li = 0; li <= L; ++li)
    for (int lf = 0; lf <= L; ++lf) {
      eso_solid_harmonics(lf, r, y);
      for (int lo = 0; lo <= L; ++lo) {
        if (!tri_ok(li, lf, lo)) continue;
        const double* t = cgt(li, lf, lo);
        const int d1 = 2 * li + 1, d2 = 2 * lf + 1;
        for (int mo = 0; mo < 2 * lo + 1; ++mo)
          for (int mi = 0; mi < d1; ++mi) {
            double s = 0.0;
            for (int mf = 0; mf < d2; ++mf) s += t[mo * d1 * d2 + mi * d2 + mf] * y[mf];
            T[(lo * lo + mo) * M + li * li + mi] += phi * s;
          }
      }
    }
}

/* stream_aggregate_backward: gradients of
 * sum <dout, out> w.r.t. q, k, v by recomputation from (q,k,v,lse).
 * Two race-free parallel phases, the GPU's split: (1) query-centric over i:
 * Delta_i, per-pair p and ds = p (dout_i . x_ij - Delta_i), dq_i; (2)
 * key-centric over j through the transposed relation (pairs of key j in
 * ascending (i, slot) order, so sums are deterministic): dv_j += p T^T dout_i,
 * dk_j += tau ds q_i.  Only O(N K H) scalars are kept between the phases. */
void eso_attn_bwd(const eso_attn_desc* d, const double* q, const double* k, const double* v, const double* pos,
                  const int* nbr, const double* out, const double* lse, const double* dout, double* dq, double* dk,
                  double* dv) {
  const int N = d->N, K = d->K, H = d->H, L = d->L, M = (L + 1) * (L + 1);
  const int Dq = d->Dq, Cv = d->Cv, dqh = Dq / H, cvh = Cv / H;
  const double tau = 1.0 / sqrt((double)M * dqh);
  cg_cache_init();
  double* P = (double*)malloc(sizeof(double) * ((size_t)N * K * H + 1));
  double* DS = (double*)malloc(sizeof(double) * ((size_t)N * K * H + 1));
  int* rptr = (int*)calloc((size_t)N + 2, sizeof(int));
  int* rpair = (int*)malloc(sizeof(int) * ((size_t)N * K + 1));
#pragma omp parallel
  {
    double* T = (double*)malloc(sizeof(double) * M * M);
    double* y = (double*)malloc(sizeof(double) * M * Cv);
    double* Delta = (double*)malloc(sizeof(double) * H);
#pragma omp for schedule(dynamic, 4)
    for (int i = 0; i < N; ++i) {
      double* dqi = dq + (size_t)i * M * Dq;
      memset(dqi, 0, sizeof(double) * M * Dq);
      for (int h = 0; h < H; ++h) {
        double s = 0.0;
        for (int mm = 0; mm < M; ++mm)
          for (int c = h * cvh; c < (h + 1) * cvh; ++c)
            s += dout[((size_t)i * M + mm) * Cv + c] * out[((size_t)i * M + mm) * Cv + c];
        Delta[h] = s;
      }
      for (int kk = 0; kk < K; ++kk) {
        const int j = nbr[(size_t)i * K + kk];
        if (j < 0) continue;
        double r[3];
        pair_vec(pos, i, j, d->box, r);
        const double rn = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
        pair_T(d, r, phi_of(d, rn), T);
        for (int a = 0; a < M; ++a) /* y = T^T dout_i  [M][Cv] */
          for (int c = 0; c < Cv; ++c) {
            double s = 0.0;
            for (int o = 0; o < M; ++o) s += T[o * M + a] * dout[((size_t)i * M + o) * Cv + c];
            y[a * Cv + c] = s;
          }
        for (int h = 0; h < H; ++h) {
          double sc = 0.0;
          for (int mm = 0; mm < M; ++mm)
            for (int c = h * dqh; c < (h + 1) * dqh; ++c)
              sc += q[((size_t)i * M + mm) * Dq + c] * k[((size_t)j * M + mm) * Dq + c];
          const double p = exp(tau * sc + bias_of(d, rn) - lse[(size_t)i * H + h]);
          double dp = 0.0;
          for (int mm = 0; mm < M; ++mm)
            for (int c = h * cvh; c < (h + 1) * cvh; ++c) dp += y[mm * Cv + c] * v[((size_t)j * M + mm) * Cv + c];
          const double ds = p * (dp - Delta[h]);
          P[((size_t)i * K + kk) * H + h] = p;
          DS[((size_t)i * K + kk) * H + h] = ds;
          for (int mm = 0; mm < M; ++mm)
            for (int c = h * dqh; c < (h + 1) * dqh; ++c)
              dqi[mm * Dq + c] += tau * ds * k[((size_t)j * M + mm) * Dq + c];
        }
      }
    }
#pragma omp single
    { /* transposed relation (counting sort; ascending pair index per key) */
      for (size_t e = 0; e < (size_t)N * K; ++e)
        if (nbr[e] >= 0) rptr[nbr[e] + 1]++;
      for (int j = 0; j < N; ++j) rptr[j + 1] += rptr[j];
      int* cur = (int*)malloc(sizeof(int) * ((size_t)N + 1));
      memcpy(cur, rptr, sizeof(int) * ((size_t)N + 1));
      for (size_t e = 0; e < (size_t)N * K; ++e)
        if (nbr[e] >= 0) rpair[cur[nbr[e]]++] = (int)e;
      free(cur);
    }
#pragma omp for schedule(dynamic, 4)
    for (int j = 0; j < N; ++j) {
      double* dkj = dk + (size_t)j * M * Dq;
      double* dvj = dv + (size_t)j * M * Cv;
      memset(dkj, 0, sizeof(double) * M * Dq);
      memset(dvj, 0, sizeof(double) * M * Cv);
      for (int e = rptr[j]; e < rptr[j + 1]; ++e) {
        const int pe = rpair[e], i = pe / K;
        double r[3];
        pair_vec(pos, i, j, d->box, r);
        const double rn = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
        pair_T(d, r, phi_of(d, rn), T);
        for (int a = 0; a < M; ++a)
          for (int c = 0; c < Cv; ++c) {
            double s = 0.0;
            for (int o = 0; o < M; ++o) s += T[o * M + a] * dout[((size_t)i * M + o) * Cv + c];
            y[a * Cv + c] = s;
          }
        for (int h = 0; h < H; ++h) {
          const double p = P[(size_t)pe * H + h], ds = DS[(size_t)pe * H + h];
          for (int mm = 0; mm < M; ++mm)
            for (int c = h * cvh; c < (h + 1) * cvh; ++c) dvj[mm * Cv + c] += p * y[mm * Cv + c];
          for (int mm = 0; mm < M; ++mm)
            for (int c = h * dqh; c < (h + 1) * dqh; ++c)
              dkj[mm * Dq + c] += tau * ds * q[((size_t)i * M + mm) * Dq + c];
        }
      }
    }
    free(T); free(y); free(Delta);
  }
  free(P); free(DS); free(rptr); free(rpair);
}

/* Per-pair operator for tests (exposes pair_T). */
void eso_pair_operator(int L, int value_mode, double r_cut, int phi_mode, const double* r, double* T) {
  eso_attn_desc d;
  memset(&d, 0, sizeof(d));
  d.L = L; d.value_mode = value_mode; d.r_cut = r_cut; d.phi_mode = phi_mode;
  cg_cache_init();
  const double rn = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  pair_T(&d, r, phi_of(&d, rn), T);
}

int eso_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
void eso_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ------------------------------------------------------------------ */
/* Node-centric factorized message (Eq. 5 PAPER.md:   */
/* 228-235; three-stage flow PAPER.md:299-322).                         */
/*   m_i = sum_j alpha_ij sum_paths (h_j^li (x) R^lf(r_j - r_i))^lo     */
/* with R^lf(a + b) = sum_u w(lf,u) (R^u(a) (x) R^{lf-u}(b))^lf         */
/* (translation weights, conventions.hpp:32-34), a = -(r_i - o),        */
/* b = r_j - o, and (h (x) (A (x) B)^lf)^lo recoupled to                */
/* sum_l' c_l' ((h (x) B)^l' (x) A)^lo (Wigner-6j recoupling; the       */
/* coefficients solved by least squares, SPEC ledger "6j-vs-solve").    */
/* Source terms depend on j only, targets on i only: per edge only the  */
/* scalar alpha_ij multiplies.                            */
/* ------------------------------------------------------------------ */
static double binom_d(int n, int k) {
  double r = 1.0;
  for (int a = 1; a <= k; ++a) r = r * (n - k + a) / a;
  return r;
}
/* closed form printed by the reference manifest (conventions.hpp:32-34) */
double eso_translation_weight(int l, int u) {
  return sqrt(binom_d(2 * l, 2 * u) * 4.0 * ESO_PI * (2 * l + 1) / ((2.0 * u + 1.0) * (2.0 * (l - u) + 1.0)));
}

static unsigned long long g_lcg = 88172645463325252ull;
static double lcg_unit(void) { /* deterministic sample points for the least-squares solves */
  g_lcg = g_lcg * 6364136223846793005ull + 1442695040888963407ull;
  return ((g_lcg >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

/* translation_coefficients: least-squares w[u], u = 0..l, of
 * R^l(a+b) = sum_u w[u] (R^u(a) (x) R^{l-u}(b))^l over 8(l+1)(2l+1) samples. */
int eso_translation_coefficients(int l, double* w) {
  cg_cache_init();
  const int d = 2 * l + 1, nu = l + 1, ns = 8 * nu * d;
  double* A = (double*)calloc((size_t)nu * nu, sizeof(double));
  double* B = (double*)calloc((size_t)nu, sizeof(double));
  double ya[2 * ESO_LT + 1], yb[2 * ESO_LT + 1], yab[2 * ESO_LT + 1], cp[ESO_LT + 1][2 * ESO_LT + 1];
  for (int s = 0; s < ns / d; ++s) {
    const double a[3] = {lcg_unit(), lcg_unit(), lcg_unit()}, b[3] = {lcg_unit(), lcg_unit(), lcg_unit()};
    const double ab[3] = {a[0] + b[0], a[1] + b[1], a[2] + b[2]};
    eso_solid_harmonics(l, ab, yab);
    for (int u = 0; u <= l; ++u) {
      eso_solid_harmonics(u, a, ya);
      eso_solid_harmonics(l - u, b, yb);
      tp_dense_tab(cgt(u, l - u, l), ya, u, 1, yb, l - u, 1, l, cp[u]);
    }
    for (int m = 0; m < d; ++m)
      for (int p = 0; p < nu; ++p) {
        B[p] += cp[p][m] * yab[m];
        for (int q = 0; q < nu; ++q) A[p * nu + q] += cp[p][m] * cp[q][m];
      }
  }
  const int st = solve_inplace(A, B, nu, 1);
  for (int u = 0; u <= l; ++u) w[u] = B[u];
  free(A); free(B);
  return st;
}

/* recoupling (h^li (x) (A^u (x) B^lb)^lf)^lo = sum_l' c[l'] ((h (x) B)^l' (x) A)^lo;
 * c indexed by l' (entries outside |li-lb|..li+lb or not triangle with (l', u, lo) are 0). */
int eso_recouple(int li, int u, int lb, int lf, int lo, double* c) {
  cg_cache_init();
  const int lmin = abs(li - lb), lmax = li + lb;
  int nl = 0, ls[2 * ESO_LT + 1];
  for (int l2 = lmin; l2 <= lmax; ++l2)
    if (l2 < ESO_LT && tri_ok(l2, u, lo)) ls[nl++] = l2;
  for (int l2 = 0; l2 <= 2 * (ESO_LT - 1); ++l2) c[l2] = 0.0;
  if (!tri_ok(u, lb, lf) || !tri_ok(li, lf, lo) || nl == 0) return -1;
  const int dl = 2 * lo + 1;
  double* A = (double*)calloc((size_t)nl * nl, sizeof(double));
  double* B = (double*)calloc((size_t)nl, sizeof(double));
  double h[2 * ESO_LT + 1], av[2 * ESO_LT + 1], bv[2 * ESO_LT + 1], ab[2 * ESO_LT + 1], lhs[2 * ESO_LT + 1];
  double hb[4 * ESO_LT + 1], rhs[2 * ESO_LT + 1][2 * ESO_LT + 1];
  for (int s = 0; s < 12 * nl + 4; ++s) {
    for (int m = 0; m < 2 * li + 1; ++m) h[m] = lcg_unit();
    for (int m = 0; m < 2 * u + 1; ++m) av[m] = lcg_unit();
    for (int m = 0; m < 2 * lb + 1; ++m) bv[m] = lcg_unit();
    tp_dense_tab(cgt(u, lb, lf), av, u, 1, bv, lb, 1, lf, ab);
    tp_dense_tab(cgt(li, lf, lo), h, li, 1, ab, lf, 1, lo, lhs);
    for (int p = 0; p < nl; ++p) {
      tp_dense_tab(cgt(li, lb, ls[p]), h, li, 1, bv, lb, 1, ls[p], hb);
      tp_dense_tab(cgt(ls[p], u, lo), hb, ls[p], 1, av, u, 1, lo, rhs[p]);
    }
    for (int m = 0; m < dl; ++m)
      for (int p = 0; p < nl; ++p) {
        B[p] += rhs[p][m] * lhs[m];
        for (int q = 0; q < nl; ++q) A[p * nl + q] += rhs[p][m] * rhs[q][m];
      }
  }
  const int st = solve_inplace(A, B, nl, 1);
  for (int p = 0; p < nl; ++p) c[ls[p]] = B[p];
  free(A); free(B);
  return st;
}

/* source-term component layout: for li = 0..L, lb = 0..L, l' = |li-lb|..li+lb:
 * (2l'+1) rows; M^2 rows in total. */
static int src_ncomp(int L) { return (L + 1) * (L + 1) * (L + 1) * (L + 1); }
static int src_offset(int L, int li, int lb, int l2) {
  int o = 0;
  for (int a = 0; a <= L; ++a)
    for (int b = 0; b <= L; ++b)
      for (int c = abs(a - b); c <= a + b; ++c) {
        if (a == li && b == lb && c == l2) return o;
        o += 2 * c + 1;
      }
  return -1;
}

/* source_term: S_j^(li,lb,l') = (h_j^li (x) R^lb(r_j - o))^l'  [N][M^2][C] */
void eso_source_term(int N, int L, int C, const double* pos, const double* origin, const double* h, double* S) {
  cg_cache_init();
  const int M = (L + 1) * (L + 1), NS = src_ncomp(L);
#pragma omp parallel for schedule(static)
  for (int j = 0; j < N; ++j) {
    const double r[3] = {pos[3 * j] - origin[0], pos[3 * j + 1] - origin[1], pos[3 * j + 2] - origin[2]};
    double y[2 * ESO_LT + 1];
    for (int li = 0; li <= L; ++li)
      for (int lb = 0; lb <= L; ++lb) {
        eso_solid_harmonics(lb, r, y);
        for (int l2 = abs(li - lb); l2 <= li + lb; ++l2)
          tp_dense_tab(cgt(li, lb, l2), h + ((size_t)j * M + li * li) * C, li, C, y, lb, 1, l2,
                       S + ((size_t)j * NS + src_offset(L, li, lb, l2)) * C);
      }
  }
}

/* alpha-weighted aggregation: A_i = sum_j alpha_ij^{head(c)} S_j (only scalar work per edge) */
void eso_aggregate(int N, int K, int H, int NS, int C, const int* nbr, const double* alpha, const double* S,
                   double* A) {
  const int ch = C / H;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < N; ++i) {
    double* a = A + (size_t)i * NS * C;
    memset(a, 0, sizeof(double) * NS * C);
    for (int kk = 0; kk < K; ++kk) {
      const int j = nbr[(size_t)i * K + kk];
      if (j < 0) continue;
      const double* s = S + (size_t)j * NS * C;
      for (int t = 0; t < NS; ++t)
        for (int c = 0; c < C; ++c) a[t * C + c] += alpha[((size_t)i * K + kk) * H + c / ch] * s[t * C + c];
    }
  }
}

/* target_couple + translation (Eq. 5):
 * m_i^lo = sum_(li,lf) sum_u w(lf,u) sum_l' c (A_i^(li, lf-u, l') (x) R^u(o - r_i))^lo */
void eso_target_couple(int N, int L, int C, const double* pos, const double* origin, const double* A, double* out) {
  cg_cache_init();
  const int M = (L + 1) * (L + 1), NS = src_ncomp(L);
  double w[ESO_LT][ESO_LT];
  for (int lf = 0; lf <= L; ++lf) eso_translation_coefficients(lf, w[lf]);
  static double cc[ESO_LT][ESO_LT][ESO_LT][ESO_LT][2 * ESO_LT]; /* [li][u][lb][lo][l'] (lf = u + lb) */
#pragma omp critical(eso_recouple_cache)
  for (int li = 0; li <= L; ++li)
    for (int u = 0; u <= L; ++u)
      for (int lb = 0; lb + u <= L; ++lb)
        for (int lo = 0; lo <= L; ++lo) eso_recouple(li, u, lb, u + lb, lo, cc[li][u][lb][lo]);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < N; ++i) {
    const double a[3] = {origin[0] - pos[3 * i], origin[1] - pos[3 * i + 1], origin[2] - pos[3 * i + 2]};
    double ya[ESO_LT][2 * ESO_LT + 1];
    for (int u = 0; u <= L; ++u) eso_solid_harmonics(u, a, ya[u]);
    double* o = out + (size_t)i * M * C;
    memset(o, 0, sizeof(double) * M * C);
    double* tmp = (double*)malloc(sizeof(double) * (2 * L + 1) * C);
    for (int li = 0; li <= L; ++li)
      for (int lf = 0; lf <= L; ++lf)
        for (int lo = 0; lo <= L; ++lo) {
          if (!tri_ok(li, lf, lo)) continue;
          for (int u = 0; u <= lf; ++u) {
            const int lb = lf - u;
            for (int l2 = abs(li - lb); l2 <= li + lb; ++l2) {
              const double coef = w[lf][u] * cc[li][u][lb][lo][l2];
              if (coef == 0.0 || !tri_ok(l2, u, lo)) continue;
              tp_dense_tab(cgt(l2, u, lo), A + ((size_t)i * NS + src_offset(L, li, lb, l2)) * C, l2, C, ya[u], u, 1,
                           lo, tmp);
              for (int t = 0; t < (2 * lo + 1) * C; ++t) o[lo * lo * C + t] += coef * tmp[t];
            }
          }
        }
    free(tmp);
  }
}

/* factorized_message: source -> aggregate -> target */
void eso_factorized_message(int N, int K, int H, int L, int C, const double* pos, const double* origin, const double* h,
                            const int* nbr, const double* alpha, double* out) {
  const int NS = src_ncomp(L);
  double* S = (double*)malloc(sizeof(double) * (size_t)N * NS * C);
  double* A = (double*)malloc(sizeof(double) * (size_t)N * NS * C);
  eso_source_term(N, L, C, pos, origin, h, S);
  eso_aggregate(N, K, H, NS, C, nbr, alpha, S, A);
  eso_target_couple(N, L, C, pos, origin, A, out);
  free(S); free(A);
}

/* edge_centric_message: the oracle -- per edge the dense CG
 * product h_j (x) R^lf(r_j - r_i) over all paths, weighted by alpha_ij. */
void eso_edge_message(int N, int K, int H, int L, int C, const double* pos, const double* h, const int* nbr,
                      const double* alpha, double* out) {
  eso_attn_desc d;
  memset(&d, 0, sizeof(d));
  d.N = N; d.K = K; d.H = H; d.L = L; d.Cv = C; d.value_mode = 1; d.phi_mode = 1; d.r_cut = 1e300;
  cg_cache_init();
  const int M = (L + 1) * (L + 1), ch = C / H;
#pragma omp parallel
  {
    double* x = (double*)malloc(sizeof(double) * M * C);
    double* scr = (double*)malloc(sizeof(double) * 2 * M * C);
#pragma omp for schedule(dynamic, 4)
    for (int i = 0; i < N; ++i) {
      double* o = out + (size_t)i * M * C;
      memset(o, 0, sizeof(double) * M * C);
      for (int kk = 0; kk < K; ++kk) {
        const int j = nbr[(size_t)i * K + kk];
        if (j < 0) continue;
        double r[3];
        pair_vec(pos, i, j, NULL, r);
        pair_value(&d, h, j, r, 1.0, x, scr);
        for (int t = 0; t < M; ++t)
          for (int c = 0; c < C; ++c) o[t * C + c] += alpha[((size_t)i * K + kk) * H + c / ch] * x[t * C + c];
      }
    }
    free(x); free(scr);
  }
}
