#pragma once
// Fused on-the-fly equivariant attention with per-pair EAAS (sm_100a) --
// shared device code (tables, per-pair preparation, EAAS operator).
//
// Forward  = stream_aggregate (Alg. 1),
// backward = stream_aggregate_backward by recomputation,
// with the north-star value path: for every (i, j) pair the kernel builds in
// registers/shared memory the relative direction, the SO(3)->SO(2) edge frame
// R (R r_ij = |r_ij| e_z), the Wigner blocks D^l(R), the radial factors
// |r|^lf Y_lf0(e_z) and applies the EAAS sparse parity re-index
// (Def. 1 / Prop. 1) per channel:
//     x_ij = phi(r_ij) * D^T P(|r_ij|) D v_j      (== sum over CG paths of v_j (x) R^lf(r_ij))
// No per-edge tensor reaches HBM: the per-pair operator lives in shared
// memory for one neighbour batch, the softmax state (mu, z, A) in registers.
//
// Work decomposition: one CTA per target atom (forward / dq) or per key atom
// (dk, dv).  The CTA's WQ = C / (32*CPL) warps split the value channels
// (CPL channels per lane, whole heads per warp), so scores reduce inside a
// warp with shuffles.  Each neighbour batch of BP pairs is prepared by BP
// threads in parallel (one pair per thread: frame, D^l fit, reindex
// polynomials), then every warp streams the batch for its channels.
#include <cuda_bf16.h>


#include "es_internal.h"

namespace es {
namespace {

// ------------------------------------------------------------------ tables
struct DevTables {
  float fit_pts[9][3];
  float ainv[kMaxL + 1][81];
  float shnorm[kMaxL + 1][kMaxL + 1];
  float cab[kMaxL + 1][85][2][kMaxL + 1];  // [L][canonical entry][a|b][lf]
};
static __constant__ DevTables c_tab;

__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int canon_entry(int lo, int li, int m) {
  int s = 0;
  for (int a = 0; a <= kMaxL; ++a)
    for (int b = 0; b <= kMaxL; ++b) {
      const int mm = cmin(a, b);
      if (a == lo && b == li) return s + m + mm;
      s += 2 * mm + 1;
    }
  return -1;
}

template <int L>
struct Lay {
  static constexpr int M = (L + 1) * (L + 1);
  __host__ __device__ static constexpr int doff(int l) {
    int s = 0;
    for (int a = 1; a < l; ++a) s += (2 * a + 1) * (2 * a + 1);
    return s;
  }
  __host__ __device__ static constexpr int eoff(int lo, int li) {
    int s = 0;
    for (int a = 0; a <= L; ++a)
      for (int b = 0; b <= L; ++b) {
        if (a == lo && b == li) return s;
        s += 2 * cmin(a, b) + 1;
      }
    return s;
  }
  static constexpr int ND = doff(L + 1);
  static constexpr int NE = eoff(L + 1, 0);
  static constexpr int OFF_AB = ND;
  static constexpr int OFF_PHI = ND + 2 * NE;
  static constexpr int OFF_J = OFF_PHI + 1;
  static constexpr int OFF_X = OFF_PHI + 2;  // spare (query slot in backward)
  static constexpr int OFF_DPHI = OFF_PHI + 3;  // dphi/dr (position gradients)
  static constexpr int OFF_R = OFF_PHI + 4;     // r_ij as fp32 (3)
  static constexpr int OFF_B = OFF_PHI + 7;     // radial score bias b(r_ij)
  static constexpr int OFF_DB = OFF_PHI + 8;    // db/dr (position gradients)
  static constexpr int OFF_SI = OFF_PHI + 9;    // backward: the pair's index into the saved scores
  static constexpr int REC = ((OFF_PHI + 10) + 3) / 4 * 4;
  static constexpr int BP = (L <= 2) ? 64 : 32;  // pairs per batch
};

inline es_status upload_tables_tu() {
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && done[dev]) return ES_OK;
  const HostTables& h = host_tables();
  DevTables t;
  for (int k = 0; k < 9; ++k)
    for (int a = 0; a < 3; ++a) t.fit_pts[k][a] = (float)h.fit_pts[k][a];
  for (int l = 0; l <= kMaxL; ++l) {
    for (int i = 0; i < 81; ++i) t.ainv[l][i] = (float)h.ainv[l][i];
    for (int mu = 0; mu <= kMaxL; ++mu) t.shnorm[l][mu] = (float)h.shnorm[l][mu];
  }
  for (int L = 0; L <= kMaxL; ++L)
    for (int e = 0; e < 85; ++e)
      for (int f = 0; f <= kMaxL; ++f) {
        t.cab[L][e][0][f] = (float)h.ca[L][e][f];
        t.cab[L][e][1][f] = (float)h.cb[L][e][f];
      }
  cudaError_t e = cudaMemcpyToSymbol(c_tab, &t, sizeof(t));
  if (e != cudaSuccess) return cuda_status(e, "upload_tables");
  if (dev < 64) done[dev] = true;
  return ES_OK;
}

// ------------------------------------------------------------------ helpers
// L1 prefetch of the line holding p (no register cost): used to put the next
// pair's gathered rows in flight while the current pair is being processed.
__device__ __forceinline__ void pf_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
template <typename T>
__device__ __forceinline__ float ldf(const T* p);
template <>
__device__ __forceinline__ float ldf<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(__ldg(p)); }

__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

// Load n (1, 2, 4, 8) consecutive elements as floats (bf16: exact widening by bit shifts).
template <int n, typename T>
__device__ __forceinline__ void ldvec(const T* p, float* o) {
  if constexpr (n == 8 && sizeof(T) == 2) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    o[0] = bf_lo(u.x); o[1] = bf_hi(u.x); o[2] = bf_lo(u.y); o[3] = bf_hi(u.y);
    o[4] = bf_lo(u.z); o[5] = bf_hi(u.z); o[6] = bf_lo(u.w); o[7] = bf_hi(u.w);
  } else if constexpr (n == 8) {
    ldvec<4>(p, o);
    ldvec<4>(p + 4, o + 4);
  } else if constexpr (sizeof(T) == 4) {
    if constexpr (n == 4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(p));
      o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else if constexpr (n == 2) {
      const float2 v = __ldg(reinterpret_cast<const float2*>(p));
      o[0] = v.x; o[1] = v.y;
    } else {
#pragma unroll
      for (int a = 0; a < n; ++a) o[a] = ldf(p + a);
    }
  } else {
    if constexpr (n == 4) {
      const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
      o[0] = bf_lo(u.x); o[1] = bf_hi(u.x); o[2] = bf_lo(u.y); o[3] = bf_hi(u.y);
    } else if constexpr (n == 2) {
      const unsigned u = __ldg(reinterpret_cast<const unsigned*>(p));
      o[0] = bf_lo(u); o[1] = bf_hi(u);
    } else {
#pragma unroll
      for (int a = 0; a < n; ++a) o[a] = ldf(p + a);
    }
  }
}

template <int n, typename T>
__device__ __forceinline__ void stvec(T* p, const float* v) {
  if constexpr (sizeof(T) == 4) {
    if constexpr (n == 4) *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    else if constexpr (n == 2) *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    else {
#pragma unroll
      for (int a = 0; a < n; ++a) p[a] = v[a];
    }
  } else {
#pragma unroll
    for (int a = 0; a < n; ++a) p[a] = __float2bfloat16_rn(v[a]);
  }
}

// Real solid harmonics of one degree l at a point (harmonics.hpp:36-81
// recursion; orthonormal, (-1)^m on positive m).
template <int l>
__device__ __forceinline__ void sh_degree(float x, float y, float z, float* out) {
  if constexpr (l == 0) {
    out[0] = 0.28209479177387814f;
  } else {
    const float r2 = x * x + y * y + z * z;
    float a = 1.f, b = 0.f;
#pragma unroll
    for (int mu = 0; mu <= l; ++mu) {
      if (mu > 0) {
        const float an = a * x - b * y, bn = a * y + b * x;
        a = an; b = bn;
      }
      float p2 = 0.f, pc = 1.f;
#pragma unroll
      for (int k = 2 * mu - 1; k > 1; k -= 2) pc *= (float)k;
#pragma unroll
      for (int ll = mu + 1; ll <= l; ++ll) {
        const float pn = ((2 * ll - 1) * z * pc - (ll + mu - 1) * r2 * p2) * (1.f / (float)(ll - mu));
        p2 = pc; pc = pn;
      }
      const float nrm = c_tab.shnorm[l][mu] * pc;
      if (mu == 0) out[l] = nrm;
      else {
        out[l + mu] = ((mu & 1) ? -nrm : nrm) * a;
        out[l - mu] = nrm * b;
      }
    }
  }
}

// D^l(R) = B A^-1 with B[:,k] = Y^l(R p_k): written row-major into rec.
template <int l>
__device__ __forceinline__ void fit_wigner(const float (&R)[9], float* rec) {
  constexpr int d = 2 * l + 1;
  float acc[d * d];
#pragma unroll
  for (int t = 0; t < d * d; ++t) acc[t] = 0.f;
#pragma unroll
  for (int k = 0; k < d; ++k) {
    const float px = c_tab.fit_pts[k][0], py = c_tab.fit_pts[k][1], pz = c_tab.fit_pts[k][2];
    const float qx = R[0] * px + R[1] * py + R[2] * pz;
    const float qy = R[3] * px + R[4] * py + R[5] * pz;
    const float qz = R[6] * px + R[7] * py + R[8] * pz;
    float y[d];
    sh_degree<l>(qx, qy, qz, y);
#pragma unroll
    for (int m = 0; m < d; ++m)
#pragma unroll
      for (int mp = 0; mp < d; ++mp) acc[m * d + mp] = fmaf(y[m], c_tab.ainv[l][k * d + mp], acc[m * d + mp]);
  }
#pragma unroll
  for (int t = 0; t < d * d; ++t) rec[t] = acc[t];
}

template <int L, int l>
__device__ __forceinline__ void fit_all(const float (&R)[9], float* rec) {
  if constexpr (l <= L) {
    if constexpr (l == 1) {
      // D^1 = Pi R Pi^T with Y^1 = c (y, z, -x): idx (1,2,0), sign (+,+,-)
      const int idx[3] = {1, 2, 0};
      const float sg[3] = {1.f, 1.f, -1.f};
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) rec[Lay<L>::doff(1) + a * 3 + b] = sg[a] * sg[b] * R[idx[a] * 3 + idx[b]];
    } else {
      fit_wigner<l>(R, rec + Lay<L>::doff(l));
    }
    fit_all<L, l + 1>(R, rec);
  }
}

// Real solid harmonics of degree <= 2 in the library convention (row
// l*l+m+l; Y^1 = c1 (y, z, -x)) and their gradients -- the R^{l_f}(r) of the
// per-pair value map x = phi sum_f Y^f(r) G_f v (same map as EAAS, Prop. 1),
// differentiated for the position gradients.
__device__ __forceinline__ void solid2_grad(float x, float y, float z, float (&Y)[9], float (&G)[9][3]) {
  const float c0 = 0.28209479177387814f, c1 = 0.4886025119029199f, c2 = 1.0925484305920792f,
              c20 = 0.6307831305050401f;
  Y[0] = c0; G[0][0] = 0.f; G[0][1] = 0.f; G[0][2] = 0.f;
  Y[1] = c1 * y; G[1][0] = 0.f; G[1][1] = c1; G[1][2] = 0.f;
  Y[2] = c1 * z; G[2][0] = 0.f; G[2][1] = 0.f; G[2][2] = c1;
  Y[3] = -c1 * x; G[3][0] = -c1; G[3][1] = 0.f; G[3][2] = 0.f;
  Y[4] = c2 * x * y; G[4][0] = c2 * y; G[4][1] = c2 * x; G[4][2] = 0.f;
  Y[5] = c2 * y * z; G[5][0] = 0.f; G[5][1] = c2 * z; G[5][2] = c2 * y;
  Y[6] = c20 * (z * z - 0.5f * (x * x + y * y)); G[6][0] = -c20 * x; G[6][1] = -c20 * y; G[6][2] = 2.f * c20 * z;
  Y[7] = -c2 * x * z; G[7][0] = -c2 * z; G[7][1] = 0.f; G[7][2] = -c2 * x;
  Y[8] = 0.5f * c2 * (x * x - y * y); G[8][0] = c2 * x; G[8][1] = -c2 * y; G[8][2] = 0.f;
}

// Forward-mode derivative (value + gradient in x, y, z): the solid harmonics of
// any degree and their gradients from the same recursion (position gradients
// for every L).
struct D3 {
  float v, x, y, z;
};
__device__ __forceinline__ D3 operator+(D3 a, D3 b) { return {a.v + b.v, a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ D3 operator-(D3 a, D3 b) { return {a.v - b.v, a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ D3 operator*(D3 a, D3 b) {
  return {a.v * b.v, a.v * b.x + a.x * b.v, a.v * b.y + a.y * b.v, a.v * b.z + a.z * b.v};
}
__device__ __forceinline__ D3 operator*(float s, D3 a) { return {s * a.v, s * a.x, s * a.y, s * a.z}; }

// sh_degree<l> with its gradient: out[m] = |r|^l Y_lm(r) and d/d(x, y, z)
template <int l>
__device__ __forceinline__ void sh_degree_d3(float px, float py, float pz, D3* out) {
  if constexpr (l == 0) {
    out[0] = {0.28209479177387814f, 0.f, 0.f, 0.f};
  } else {
    const D3 x = {px, 1.f, 0.f, 0.f}, y = {py, 0.f, 1.f, 0.f}, z = {pz, 0.f, 0.f, 1.f};
    const D3 r2 = x * x + y * y + z * z;
    D3 a = {1.f, 0.f, 0.f, 0.f}, b = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int mu = 0; mu <= l; ++mu) {
      if (mu > 0) {
        const D3 an = a * x - b * y, bn = a * y + b * x;
        a = an; b = bn;
      }
      float pcs = 1.f;
#pragma unroll
      for (int k = 2 * mu - 1; k > 1; k -= 2) pcs *= (float)k;
      D3 p2 = {0.f, 0.f, 0.f, 0.f}, pc = {pcs, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ll = mu + 1; ll <= l; ++ll) {
        const D3 pn = (1.f / (float)(ll - mu)) * ((float)(2 * ll - 1) * (z * pc) - (float)(ll + mu - 1) * (r2 * p2));
        p2 = pc; pc = pn;
      }
      const D3 nrm = c_tab.shnorm[l][mu] * pc;
      if (mu == 0) out[l] = nrm;
      else {
        out[l + mu] = ((mu & 1) ? -1.f : 1.f) * (nrm * a);
        out[l - mu] = nrm * b;
      }
    }
  }
}

struct KParams {
  int N, K, H, C, Dq;
  int row0, Nk;  // query i <-> atom row0 + i (pos); keys j index k/v/pos in [0, Nk)
  int phi_mode, periodic;
  float tau, r_cut, inv_rcut;
  double bx, by, bz;
  int bias_mode;       // 0: b == 0; 1: b(r) = b0 + b1 r + b2 r^2 (RadialScalars b)
  float b0, b1, b2;
  float* scores_out;        // optional [N][K][H] scores of the valid slots (forward)
  const float* scores_in;   // optional saved scores (backward)
  const int* rank_of;       // saved scores in rank space (tensor-core forward): slot -> rank, else NULL
};

// radial score bias and its r-derivative
__device__ __forceinline__ float bias_of(const KParams& p, float rn) {
  return p.bias_mode ? fmaf(fmaf(p.b2, rn, p.b1), rn, p.b0) : 0.f;
}
__device__ __forceinline__ float dbias_of(const KParams& p, float rn) {
  return p.bias_mode ? fmaf(2.f * p.b2, rn, p.b1) : 0.f;
}

// Per-pair preparation (one thread): r_ij = pos_j - pos_i (double difference,
// minimum image if periodic), phi, and for EAAS the frame / D^l / reindex
// coefficients.  Gauge: R = R' P with P = diag(1,-1,-1) when u_z < 0 so that
// the closed-form frame R' (rows e1, e2, u') is used only for u'_z >= 0 --
// branch-stable; any gauge gives the same composite.
template <int L, bool EAAS>
__device__ void pair_prepare_vec(const KParams& p, float rx, float ry, float rz, int j, float* rec);

template <int L, bool EAAS>
__device__ void pair_prepare(const KParams& p, const double* __restrict__ pos, int i, int j, float* rec) {
  const int ia = p.row0 + i;
  double dx = pos[3 * j] - pos[3 * ia], dy = pos[3 * j + 1] - pos[3 * ia + 1], dz = pos[3 * j + 2] - pos[3 * ia + 2];
  if (p.periodic) {
    dx -= p.bx * rint(dx / p.bx);
    dy -= p.by * rint(dy / p.by);
    dz -= p.bz * rint(dz / p.bz);
  }
  pair_prepare_vec<L, EAAS>(p, (float)dx, (float)dy, (float)dz, j, rec);
}

// the per-pair record from the relative vector r_ij itself
template <int L, bool EAAS>
__device__ void pair_prepare_vec(const KParams& p, float rx, float ry, float rz, int j, float* rec) {
  const float rn = sqrtf(rx * rx + ry * ry + rz * rz);
  float phi = 1.f;
  if (p.phi_mode == 0) phi = rn < p.r_cut ? 0.5f * (cospif(rn * p.inv_rcut) + 1.f) : 0.f;
  rec[Lay<L>::OFF_PHI] = phi;
  rec[Lay<L>::OFF_J] = __int_as_float(j);
  // phi'(r) = -(pi / 2 r_cut) sin(pi r / r_cut) inside the cutoff
  rec[Lay<L>::OFF_DPHI] =
      (p.phi_mode == 0 && rn < p.r_cut) ? -0.5f * 3.14159265358979f * p.inv_rcut * sinpif(rn * p.inv_rcut) : 0.f;
  rec[Lay<L>::OFF_R] = rx;
  rec[Lay<L>::OFF_R + 1] = ry;
  rec[Lay<L>::OFF_R + 2] = rz;
  rec[Lay<L>::OFF_B] = bias_of(p, rn);
  rec[Lay<L>::OFF_DB] = dbias_of(p, rn);
  if constexpr (EAAS) {
    float R[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f};
    if (rn > 1e-8f) {
      const float inv = 1.f / rn;
      const float ux = rx * inv;
      const bool flip = rz < 0.f;
      const float uy = flip ? -ry * inv : ry * inv;
      const float uz = flip ? -rz * inv : rz * inv;
      const float f = 1.f / (1.f + uz);
      R[0] = 1.f - ux * ux * f; R[1] = -ux * uy * f; R[2] = -ux;
      R[3] = -ux * uy * f;      R[4] = 1.f - uy * uy * f; R[5] = -uy;
      R[6] = ux;                R[7] = uy;                R[8] = uz;
      if (flip) {  // R' P: negate columns 1 and 2
        R[1] = -R[1]; R[2] = -R[2]; R[4] = -R[4]; R[5] = -R[5]; R[7] = -R[7]; R[8] = -R[8];
      }
    }
    fit_all<L, 1>(R, rec);
    float rp[L + 1];
    rp[0] = 1.f;
#pragma unroll
    for (int f = 1; f <= L; ++f) rp[f] = rp[f - 1] * rn;
#pragma unroll
    for (int lo = 0; lo <= L; ++lo)
#pragma unroll
      for (int li = 0; li <= L; ++li) {
        const int mm = cmin(lo, li);
#pragma unroll
        for (int m = -mm; m <= mm; ++m) {
          const int ce = canon_entry(lo, li, m);
          const int e = Lay<L>::eoff(lo, li) + m + mm;
          float a = 0.f, b = 0.f;
#pragma unroll
          for (int f = 0; f <= L; ++f) {
            a = fmaf(c_tab.cab[L][ce][0][f], rp[f], a);
            b = fmaf(c_tab.cab[L][ce][1][f], rp[f], b);
          }
          rec[Lay<L>::OFF_AB + 2 * e] = a;
          rec[Lay<L>::OFF_AB + 2 * e + 1] = b;
        }
      }
  }
}

// acc[c] += a * x[c] over a thread's channels: channel pairs go through the
// packed FFMA2 (sm_100: two fp32 FMAs per issue slot, the scalar broadcast is
// an operand modifier), so the FMA-bound per-pair value work issues half the
// instructions.  Same rounding as fmaf per lane.
__device__ __forceinline__ void ffma2(float a, float x0, float x1, float& c0, float& c1) {
  asm("{\n\t.reg .b64 a2, x2, c2;\n\t"
      "mov.b64 a2, {%2, %2};\n\t"
      "mov.b64 x2, {%3, %4};\n\t"
      "mov.b64 c2, {%0, %1};\n\t"
      "fma.rn.f32x2 c2, a2, x2, c2;\n\t"
      "mov.b64 {%0, %1}, c2;\n\t}"
      : "+f"(c0), "+f"(c1)
      : "f"(a), "f"(x0), "f"(x1));
}
// acc[c] += x[c] * y[c] (element-wise pairs)
__device__ __forceinline__ void ffma2v(float x0, float x1, float y0, float y1, float& c0, float& c1) {
  asm("{\n\t.reg .b64 x2, y2, c2;\n\t"
      "mov.b64 x2, {%2, %3};\n\t"
      "mov.b64 y2, {%4, %5};\n\t"
      "mov.b64 c2, {%0, %1};\n\t"
      "fma.rn.f32x2 c2, x2, y2, c2;\n\t"
      "mov.b64 {%0, %1}, c2;\n\t}"
      : "+f"(c0), "+f"(c1)
      : "f"(x0), "f"(x1), "f"(y0), "f"(y1));
}
template <int CPL>
__device__ __forceinline__ void fmac(float a, const float (&x)[CPL], float (&acc)[CPL]) {
#pragma unroll
  for (int c = 0; c + 1 < CPL; c += 2) ffma2(a, x[c], x[c + 1], acc[c], acc[c + 1]);
  if constexpr (CPL & 1) acc[CPL - 1] = fmaf(a, x[CPL - 1], acc[CPL - 1]);
}
// acc[c] += x[c] * y[c]
template <int CPL>
__device__ __forceinline__ void fmav(const float (&x)[CPL], const float (&y)[CPL], float (&acc)[CPL]) {
#pragma unroll
  for (int c = 0; c + 1 < CPL; c += 2) ffma2v(x[c], x[c + 1], y[c], y[c + 1], acc[c], acc[c + 1]);
  if constexpr (CPL & 1) acc[CPL - 1] = fmaf(x[CPL - 1], y[CPL - 1], acc[CPL - 1]);
}

// Odd channel counts per thread (CPL = 1: the L = 4 kernels): the scalar
// form, whose register allocation the packed form would disturb.
template <int L, int CPL, bool ADJ>
__device__ __forceinline__ void eaas_apply_scalar(const float* __restrict__ rec, const float (&v)[Lay<L>::M][CPL], float s,
                                           float (&acc)[Lay<L>::M][CPL]) {
  constexpr int M = Lay<L>::M;
  float vt[M][CPL];
  // align: vt^l = D^l v^l
#pragma unroll
  for (int c = 0; c < CPL; ++c) vt[0][c] = v[0][c];
#pragma unroll
  for (int l = 1; l <= L; ++l) {
    const float* D = rec + Lay<L>::doff(l);
    const int d = 2 * l + 1;
#pragma unroll
    for (int m = 0; m < d; ++m)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        float t = 0.f;
#pragma unroll
        for (int mp = 0; mp < d; ++mp) t = fmaf(D[m * d + mp], v[l * l + mp][c], t);
        vt[l * l + m][c] = t;
      }
  }
  // sparse re-index in the aligned frame (forward P or adjoint P^T)
  float w[M][CPL];
#pragma unroll
  for (int t = 0; t < M; ++t)
#pragma unroll
    for (int c = 0; c < CPL; ++c) w[t][c] = 0.f;
#pragma unroll
  for (int lo = 0; lo <= L; ++lo)
#pragma unroll
    for (int li = 0; li <= L; ++li) {
      const int mm = cmin(lo, li);
#pragma unroll
      for (int m = -mm; m <= mm; ++m) {
        const int e = Lay<L>::eoff(lo, li) + m + mm;
        const float a = rec[Lay<L>::OFF_AB + 2 * e];
        const float b = rec[Lay<L>::OFF_AB + 2 * e + 1];
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          if constexpr (!ADJ) {
            w[lo * lo + lo + m][c] = fmaf(a, vt[li * li + li + m][c], w[lo * lo + lo + m][c]);
            if (m != 0) w[lo * lo + lo + m][c] = fmaf(b, vt[li * li + li - m][c], w[lo * lo + lo + m][c]);
          } else {
            w[li * li + li + m][c] = fmaf(a, vt[lo * lo + lo + m][c], w[li * li + li + m][c]);
            if (m != 0) w[li * li + li - m][c] = fmaf(b, vt[lo * lo + lo + m][c], w[li * li + li - m][c]);
          }
        }
      }
    }
  // un-align and accumulate: acc^l += s * D^l^T w^l
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[0][c] = fmaf(s, w[0][c], acc[0][c]);
#pragma unroll
  for (int l = 1; l <= L; ++l) {
    const float* D = rec + Lay<L>::doff(l);
    const int d = 2 * l + 1;
#pragma unroll
    for (int m = 0; m < d; ++m)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        float t = 0.f;
#pragma unroll
        for (int mp = 0; mp < d; ++mp) t = fmaf(D[mp * d + m], w[l * l + mp][c], t);
        acc[l * l + m][c] = fmaf(s, t, acc[l * l + m][c]);
      }
  }
}

// The same three EAAS steps ordered by target degree (L >= 3): the aligned
// vector vt is built first, then for each target degree t its re-indexed block
// w^t (at most 2L+1 rows instead of M) is formed and un-aligned into acc at
// once, so vt, one w block and acc are live together (the M-row w of the
// forms above is what spills at L = 4).  Each output element accumulates its
// terms in the same order as eaas_apply_scalar: bit-identical results.
template <int L, int CPL, bool ADJ>
__device__ __forceinline__ void eaas_apply_blk(const float* __restrict__ rec, const float (&v)[Lay<L>::M][CPL], float s,
                                               float (&acc)[Lay<L>::M][CPL]) {
  constexpr int M = Lay<L>::M;
  float vt[M][CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) vt[0][c] = v[0][c];
#pragma unroll
  for (int l = 1; l <= L; ++l) {
    const float* D = rec + Lay<L>::doff(l);
    const int d = 2 * l + 1;
#pragma unroll
    for (int m = 0; m < d; ++m) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) vt[l * l + m][c] = 0.f;
#pragma unroll
      for (int mp = 0; mp < d; ++mp) fmac<CPL>(D[m * d + mp], v[l * l + mp], vt[l * l + m]);
    }
  }
#pragma unroll
  for (int tl = 0; tl <= L; ++tl) {
    float w[2 * L + 1][CPL];
#pragma unroll
    for (int t = 0; t < 2 * tl + 1; ++t)
#pragma unroll
      for (int c = 0; c < CPL; ++c) w[t][c] = 0.f;
#pragma unroll
    for (int sl = 0; sl <= L; ++sl) {
      const int lo = ADJ ? sl : tl, li = ADJ ? tl : sl;
      const int mm = cmin(lo, li);
#pragma unroll
      for (int m = -mm; m <= mm; ++m) {
        const int e = Lay<L>::eoff(lo, li) + m + mm;
        const float a = rec[Lay<L>::OFF_AB + 2 * e];
        const float b = rec[Lay<L>::OFF_AB + 2 * e + 1];
        fmac<CPL>(a, vt[sl * sl + sl + m], w[tl + m]);
        if (m != 0) {
          if constexpr (!ADJ) fmac<CPL>(b, vt[sl * sl + sl - m], w[tl + m]);
          else fmac<CPL>(b, vt[sl * sl + sl + m], w[tl - m]);
        }
      }
    }
    if (tl == 0) {
      fmac<CPL>(s, w[0], acc[0]);
    } else {
      const float* D = rec + Lay<L>::doff(tl);
      const int d = 2 * tl + 1;
#pragma unroll
      for (int m = 0; m < d; ++m) {
        float t[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) t[c] = 0.f;
#pragma unroll
        for (int mp = 0; mp < d; ++mp) fmac<CPL>(D[mp * d + m], w[mp], t);
        fmac<CPL>(s, t, acc[tl * tl + m]);
      }
    }
  }
}

#ifndef ES_L34_BLK
#define ES_L34_BLK 1
#endif

// x += s * (D^T P D) v  per channel (EAAS forward value operator), or the
// adjoint y += s * (D^T P^T D) g when ADJ.  v: [M][CPL] registers.
template <int L, int CPL, bool ADJ>
__device__ __forceinline__ void eaas_apply(const float* __restrict__ rec, const float (&v)[Lay<L>::M][CPL], float s,
                                           float (&acc)[Lay<L>::M][CPL]) {
  if constexpr (ES_L34_BLK && L >= 3) {
    eaas_apply_blk<L, CPL, ADJ>(rec, v, s, acc);
    return;
  }
  if constexpr (CPL % 2 == 1) {
    eaas_apply_scalar<L, CPL, ADJ>(rec, v, s, acc);
    return;
  }
  constexpr int M = Lay<L>::M;
  float vt[M][CPL];
  // align: vt^l = D^l v^l
#pragma unroll
  for (int c = 0; c < CPL; ++c) vt[0][c] = v[0][c];
#pragma unroll
  for (int l = 1; l <= L; ++l) {
    const float* D = rec + Lay<L>::doff(l);
    const int d = 2 * l + 1;
#pragma unroll
    for (int m = 0; m < d; ++m) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) vt[l * l + m][c] = 0.f;
#pragma unroll
      for (int mp = 0; mp < d; ++mp) fmac<CPL>(D[m * d + mp], v[l * l + mp], vt[l * l + m]);
    }
  }
  // sparse re-index in the aligned frame (forward P or adjoint P^T)
  float w[M][CPL];
#pragma unroll
  for (int t = 0; t < M; ++t)
#pragma unroll
    for (int c = 0; c < CPL; ++c) w[t][c] = 0.f;
#pragma unroll
  for (int lo = 0; lo <= L; ++lo)
#pragma unroll
    for (int li = 0; li <= L; ++li) {
      const int mm = cmin(lo, li);
#pragma unroll
      for (int m = -mm; m <= mm; ++m) {
        const int e = Lay<L>::eoff(lo, li) + m + mm;
        const float a = rec[Lay<L>::OFF_AB + 2 * e];
        const float b = rec[Lay<L>::OFF_AB + 2 * e + 1];
        if constexpr (!ADJ) {
          fmac<CPL>(a, vt[li * li + li + m], w[lo * lo + lo + m]);
          if (m != 0) fmac<CPL>(b, vt[li * li + li - m], w[lo * lo + lo + m]);
        } else {
          fmac<CPL>(a, vt[lo * lo + lo + m], w[li * li + li + m]);
          if (m != 0) fmac<CPL>(b, vt[lo * lo + lo + m], w[li * li + li - m]);
        }
      }
    }
  // un-align and accumulate: acc^l += s * D^l^T w^l
  fmac<CPL>(s, w[0], acc[0]);
#pragma unroll
  for (int l = 1; l <= L; ++l) {
    const float* D = rec + Lay<L>::doff(l);
    const int d = 2 * l + 1;
#pragma unroll
    for (int m = 0; m < d; ++m) {
      float t[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) t[c] = 0.f;
#pragma unroll
      for (int mp = 0; mp < d; ++mp) fmac<CPL>(D[mp * d + m], w[l * l + mp], t);
      fmac<CPL>(s, t, acc[l * l + m]);
    }
  }
}

// The per-pair value operator of the SIMT kernels: the three sparse EAAS
// steps.  (Composing them into the M x M operator T = D^T P D once per pair
// costs 81 instead of 107 MACs per channel at L = 2 but was measured slower on
// B200: the per-pair composition lengthens the batch-preparation chain.)
template <int L, int CPL, bool ADJ>
__device__ __forceinline__ void value_apply(const float* __restrict__ rec, const float (&v)[Lay<L>::M][CPL], float s,
                                            float (&acc)[Lay<L>::M][CPL]) {
  eaas_apply<L, CPL, ADJ>(rec, v, s, acc);
}

}  // namespace
}  // namespace es
