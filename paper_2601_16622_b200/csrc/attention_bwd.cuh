// Backward of the fused equivariant attention: kernel templates shared by the
// per-degree translation units attention_bwd_l{0..4}.cu (each instantiates one
// L -- the kernels of one degree compile in parallel) and the launcher in
// attention_bwd.cu; see attention_common.cuh for the per-pair machinery.
#pragma once
#include <type_traits>

#include "_gen_cg.h"
#include "attention_common.cuh"

namespace es {
namespace {

// ------------------------------------------------------------------ backward
// Delta_i^h = sum_{rows, head channels} dout * out.  C/V threads per atom,
// V channels each (same head; V = 8: 16-byte loads of bf16), shuffle-reduced
// over the C_h/V lanes of a head.
template <typename T, int V>
__global__ void __launch_bounds__(256) attn_delta_kernel(int N, int M, int C, int H, const T* __restrict__ out,
                                                         const T* __restrict__ dout, float* __restrict__ delta) {
  const int tpa = C / V;
  const int i = blockIdx.x * (blockDim.x / tpa) + threadIdx.x / tpa;
  const int t = threadIdx.x % tpa;
  if (i >= N) return;
  float acc[V];
#pragma unroll
  for (int c = 0; c < V; ++c) acc[c] = 0.f;
  for (int mm = 0; mm < M; ++mm) {
    float a[V], b[V];
    ldvec<V>(out + ((size_t)i * M + mm) * C + V * t, a);
    ldvec<V>(dout + ((size_t)i * M + mm) * C + V * t, b);
    fmav<V>(a, b, acc);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < V; ++c) s += acc[c];
  const int g = (C / H) / V;  // threads per head (power of two <= 32)
  for (int o = g >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (t % g == 0) delta[(size_t)i * H + (V * t) / (C / H)] = s;
}

// Key-centric pass: CTA per key atom j over the transposed relation; yields
// dk_j, dv_j exclusively (no atomics) and the per-pair-head dscore.
// CC, HH > 0: channels / heads fixed at compile time (the BASELINE shape C=128,
// H=8): row strides become immediates, no per-row 64-bit address arithmetic.
// FORCE: also the position gradients (every L): per pair
//   dL/dr_ij = sum_h P_ij^h [phi'(r) r^ sum_f Y^f(r) D_f^h + phi sum_f grad Y^f(r) D_f^h],
//   D_f^h = dO_i^h . (G_f v_j)^h   (the value map x = phi sum_f Y^f G_f v, == EAAS),
// scattered to dpos_j (+) and dpos_i (-) with fp64 atomics.
// CTAs per SM the C=128 specialisation (64 threads) is compiled for (register cap)
#ifndef ES_BWD_MINB
#define ES_BWD_MINB 0
#endif
// DK = false: dk is left to the tensor-core dk pass (attn_dk_tc_kernel), so the
// gathered q_i rows are needed only for the score -- and not at all when the
// forward's scores are supplied (p.scores_in).
// L >= 3 at C = 128 (configs[3]): 128-thread CTAs; the query rows of a pair
// are re-read (L1) for the dk update instead of held across the EAAS adjoint
// (2 M registers), and ES_L34_BWD_MINB CTAs reside per SM.
#ifndef ES_L34_BWD_MINB
#define ES_L34_BWD_MINB 2
#endif
#ifndef ES_L34_QRELOAD
#define ES_L34_QRELOAD 1
#endif
template <int L, int CC>
struct KvShape {
  static constexpr bool BIG = L >= 3 && CC == 128;
  static constexpr int THREADS = BIG ? 128 : (ES_BWD_MINB > 0 && CC == 128 && L <= 2 ? 64 : (L <= 2 ? 192 : 256));
  static constexpr int MINB = BIG ? ES_L34_BWD_MINB : (ES_BWD_MINB > 0 && CC == 128 && L <= 2 ? ES_BWD_MINB : (L <= 2 ? 2 : 1));
  static constexpr bool QRELOAD = BIG && ES_L34_QRELOAD;
};

template <int L, int CPL, bool EAAS, typename T, int CC = 0, int HH = 0, bool FORCE = false, bool DK = true>
__global__ void __launch_bounds__(KvShape<L, CC>::THREADS, KvShape<L, CC>::MINB)
    attn_bwd_kv_kernel(KParams p, const T* __restrict__ q, const T* __restrict__ k,
                                                          const T* __restrict__ v, const double* __restrict__ pos,
                                                          const int* __restrict__ rev_ptr,
                                                          const int* __restrict__ rev_pair,
                                                          const float* __restrict__ lse, const T* __restrict__ dout,
                                                          const float* __restrict__ delta, T* __restrict__ dk,
                                                          T* __restrict__ dv, float* __restrict__ dsbuf,
                                                          double* __restrict__ dpos) {
  const int PC = CC ? CC : p.C, PH = HH ? HH : p.H, PDq = CC ? 2 * CC : p.Dq;
  using LY = Lay<L>;
  constexpr int M = LY::M;
  constexpr int REC = LY::REC;
  constexpr int BP = LY::BP;
  extern __shared__ float4 smem4[];
  float* recs = reinterpret_cast<float*>(smem4);

  const int j = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = (warp * 32 + lane) * CPL;
  const int Ch = PC / PH;
  const int lph = Ch / CPL;
  const int head = c0 / Ch;
  const int Dq = PDq;

  // k_j / v_j: this thread's channels staged once as fp32 in shared memory
  // ([mm][thread][2 CPL] and [mm][thread][CPL], conflict-free vector LDS)
  // instead of registers (halves the live state) or per-pair bf16 re-reads.
  float dkr[DK ? M : 1][2 * CPL], dvr[M][CPL];
  double fj[3] = {0.0, 0.0, 0.0};  // FORCE: this warp's share of dL/dpos_j
  const int nthr = blockDim.x;
  float* ks = recs + BP * REC;
  float* vs = ks + M * nthr * 2 * CPL;
  {
    const T* kj = k + (size_t)j * M * Dq + 2 * c0;
    const T* vj = v + (size_t)j * M * PC + c0;
#pragma unroll
    for (int mm = 0; mm < M; ++mm) {
      float kr[2 * CPL], vr[CPL];
      ldvec<2 * CPL>(kj + (size_t)mm * Dq, kr);
      ldvec<CPL>(vj + (size_t)mm * PC, vr);
#pragma unroll
      for (int c = 0; c < 2 * CPL; ++c) ks[(mm * nthr + threadIdx.x) * 2 * CPL + c] = kr[c];
#pragma unroll
      for (int c = 0; c < CPL; ++c) vs[(mm * nthr + threadIdx.x) * CPL + c] = vr[c];
    }
  }
#pragma unroll
  for (int mm = 0; mm < M; ++mm) {
    if constexpr (DK) {
#pragma unroll
      for (int c = 0; c < 2 * CPL; ++c) dkr[mm][c] = 0.f;
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) dvr[mm][c] = 0.f;
  }
  const int rs = rev_ptr[j], re = rev_ptr[j + 1];
  for (int base = rs; base < re; base += BP) {
    const int nb = min(BP, re - base);
    __syncthreads();
    for (int t = threadIdx.x; t < nb; t += blockDim.x) {
      const int pr = rev_pair[base + t];
      const int i = pr / p.K;
      float* rec = recs + t * REC;
      pair_prepare<L, EAAS>(p, pos, i, j, rec);
      rec[LY::OFF_J] = __int_as_float(i);
      rec[LY::OFF_X] = __int_as_float(pr);
      if (p.scores_in) rec[LY::OFF_SI] = __int_as_float(p.rank_of ? i * p.K + __ldg(p.rank_of + pr) : pr);
    }
    __syncthreads();
    for (int e = 0; e < nb; ++e) {
      const float* rec = recs + e * REC;
      const int i = __float_as_int(rec[LY::OFF_J]);
      const int pr = __float_as_int(rec[LY::OFF_X]);
      // packed FFMA2 forms only for even CPL: with CPL = 1 (L = 4) the
      // register pairing they impose costs spills
      constexpr bool PK = CPL % 2 == 0;
      constexpr bool QH = DK && !KvShape<L, CC>::QRELOAD;  // hold q_i in registers for the dk update
      float qv[QH ? M : 1][2 * CPL];
      float score;
      if (!DK && p.scores_in) {
        score = p.scores_in[(size_t)head * p.N * p.K + __float_as_int(rec[LY::OFF_SI])];  // [H][N][K]
      } else {
        float sc[2 * CPL];
#pragma unroll
        for (int c = 0; c < 2 * CPL; ++c) sc[c] = 0.f;
#pragma unroll
        for (int mm = 0; mm < M; ++mm) {
          float qt[2 * CPL];
          ldvec<2 * CPL>(q + ((size_t)i * M + mm) * Dq + 2 * c0, qt);
          if constexpr (QH) {
#pragma unroll
            for (int c = 0; c < 2 * CPL; ++c) qv[mm][c] = qt[c];
          }
          float kr[2 * CPL];
#pragma unroll
          for (int c = 0; c < 2 * CPL; ++c) kr[c] = ks[(mm * nthr + threadIdx.x) * 2 * CPL + c];
          if constexpr (PK) {
            fmav<2 * CPL>(qt, kr, sc);
          } else {
#pragma unroll
            for (int c = 0; c < 2 * CPL; ++c) sc[0] = fmaf(qt[c], kr[c], sc[0]);
          }
        }
        float s = 0.f;
#pragma unroll
        for (int c = 0; c < 2 * CPL; ++c) s += sc[c];
        for (int o = lph >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        score = fmaf(s, p.tau, rec[LY::OFF_B]);
      }
      const float P = expf(score - lse[(size_t)i * PH + head]);
      const float phi = rec[LY::OFF_PHI];
      float g[M][CPL], y[M][CPL];
#pragma unroll
      for (int mm = 0; mm < M; ++mm) {
        ldvec<CPL>(dout + ((size_t)i * M + mm) * PC + c0, g[mm]);
#pragma unroll
        for (int c = 0; c < CPL; ++c) y[mm][c] = 0.f;
      }
      if constexpr (EAAS) {
        value_apply<L, CPL, true>(rec, g, phi, y);
      } else {
#pragma unroll
        for (int mm = 0; mm < M; ++mm)
#pragma unroll
          for (int c = 0; c < CPL; ++c) y[mm][c] = phi * g[mm][c];
      }
      float dpc[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) dpc[c] = 0.f;
#pragma unroll
      for (int mm = 0; mm < M; ++mm) {
        float vr[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) vr[c] = vs[(mm * nthr + threadIdx.x) * CPL + c];
        fmac<CPL>(P, y[mm], dvr[mm]);
        fmav<CPL>(y[mm], vr, dpc);
      }
      float dp = 0.f;
#pragma unroll
      for (int c = 0; c < CPL; ++c) dp += dpc[c];
      for (int o = lph >> 1; o > 0; o >>= 1) dp += __shfl_xor_sync(0xffffffffu, dp, o);
      const float ds = P * (dp - delta[(size_t)i * PH + head]);
      if constexpr (FORCE) {
        const float rx = rec[LY::OFF_R], ry = rec[LY::OFF_R + 1], rz = rec[LY::OFF_R + 2];
        const float rn = sqrtf(rx * rx + ry * ry + rz * rz);
        const float inv = rn > 1e-12f ? 1.f / rn : 0.f;
        const float dphi = rec[LY::OFF_DPHI];
        float gx, gy, gz;
        if constexpr (EAAS && L != 2) {
          // any L: D_f = dO_i . (G_f v_j) by the generated straight-line contraction, then
          // s0 = sum_f Y^f D_f and s1 = sum_f grad Y^f D_f from the forward-mode harmonics
          float Df[M];
#pragma unroll
          for (int f = 0; f < M; ++f) Df[f] = 0.f;
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            float gc[M], vc[M];
#pragma unroll
            for (int mm = 0; mm < M; ++mm) {
              gc[mm] = g[mm][c];
              vc[mm] = vs[(mm * nthr + threadIdx.x) * CPL + c];
            }
            es_force_df<L>(gc, vc, Df);
          }
#pragma unroll
          for (int f = 0; f < M; ++f)
            for (int o = lph >> 1; o > 0; o >>= 1) Df[f] += __shfl_xor_sync(0xffffffffu, Df[f], o);
          float s0 = 0.f, s1x = 0.f, s1y = 0.f, s1z = 0.f;
          auto deg = [&](auto lc) {
            constexpr int l = decltype(lc)::value;
            D3 Y[2 * l + 1];
            sh_degree_d3<l>(rx, ry, rz, Y);
#pragma unroll
            for (int m = 0; m < 2 * l + 1; ++m) {
              const float d = Df[l * l + m];
              s0 = fmaf(Y[m].v, d, s0);
              s1x = fmaf(Y[m].x, d, s1x);
              s1y = fmaf(Y[m].y, d, s1y);
              s1z = fmaf(Y[m].z, d, s1z);
            }
          };
          deg(std::integral_constant<int, 0>{});
          if constexpr (L >= 1) deg(std::integral_constant<int, 1>{});
          if constexpr (L >= 2) deg(std::integral_constant<int, 2>{});
          if constexpr (L >= 3) deg(std::integral_constant<int, 3>{});
          if constexpr (L >= 4) deg(std::integral_constant<int, 4>{});
          const float a = dphi * inv * s0;
          gx = P * (a * rx + phi * s1x);
          gy = P * (a * ry + phi * s1y);
          gz = P * (a * rz + phi * s1z);
        } else if constexpr (EAAS) {
          float vv[M][2];
#pragma unroll
          for (int mm = 0; mm < M; ++mm) {
            vv[mm][0] = vs[(mm * nthr + threadIdx.x) * CPL];
            vv[mm][1] = CPL > 1 ? vs[(mm * nthr + threadIdx.x) * CPL + (CPL > 1 ? 1 : 0)] : 0.f;
          }
          float Df[M];
#pragma unroll
          for (int f = 0; f < M; ++f) Df[f] = 0.f;
          es_vg_all(vv, [&](int o, int f, float x0, float x1) {
            Df[f] = fmaf(g[o][0], x0, Df[f]);
            if constexpr (CPL > 1) Df[f] = fmaf(g[o][CPL > 1 ? 1 : 0], x1, Df[f]);
          });
#pragma unroll
          for (int f = 0; f < M; ++f)
            for (int o = lph >> 1; o > 0; o >>= 1) Df[f] += __shfl_xor_sync(0xffffffffu, Df[f], o);
          float Y[9], dY[9][3];
          solid2_grad(rx, ry, rz, Y, dY);
          float s0 = 0.f, s1x = 0.f, s1y = 0.f, s1z = 0.f;
#pragma unroll
          for (int f = 0; f < M; ++f) {
            s0 = fmaf(Y[f], Df[f], s0);
            s1x = fmaf(dY[f][0], Df[f], s1x);
            s1y = fmaf(dY[f][1], Df[f], s1y);
            s1z = fmaf(dY[f][2], Df[f], s1z);
          }
          const float a = dphi * inv * s0;
          gx = P * (a * rx + phi * s1x);
          gy = P * (a * ry + phi * s1y);
          gz = P * (a * rz + phi * s1z);
        } else {  // x = phi v_j: only phi depends on r
          const float dpr = phi != 0.f ? dp / phi : 0.f;
          const float a = P * dphi * inv * dpr;
          gx = a * rx; gy = a * ry; gz = a * rz;
        }
        {  // the score's radial bias: dL/dr += dscore b'(r) r^
          const float bb = ds * rec[LY::OFF_DB] * inv;
          gx = fmaf(bb, rx, gx); gy = fmaf(bb, ry, gy); gz = fmaf(bb, rz, gz);
        }
        // every lane holds its head's value: sum the heads of this warp
        for (int o = lph; o < 32; o <<= 1) {
          gx += __shfl_xor_sync(0xffffffffu, gx, o);
          gy += __shfl_xor_sync(0xffffffffu, gy, o);
          gz += __shfl_xor_sync(0xffffffffu, gz, o);
        }
        if (lane == 0) {
          const size_t ia = (size_t)(p.row0 + i);
          atomicAdd(dpos + 3 * ia, -(double)gx);
          atomicAdd(dpos + 3 * ia + 1, -(double)gy);
          atomicAdd(dpos + 3 * ia + 2, -(double)gz);
          fj[0] += gx; fj[1] += gy; fj[2] += gz;
        }
      }
      if constexpr (DK) {
        const float tds = p.tau * ds;
#pragma unroll
        for (int mm = 0; mm < M; ++mm) {
          float qt[2 * CPL];
          if constexpr (QH) {
#pragma unroll
            for (int c = 0; c < 2 * CPL; ++c) qt[c] = qv[mm][c];
          } else {
            ldvec<2 * CPL>(q + ((size_t)i * M + mm) * Dq + 2 * c0, qt);
          }
          if constexpr (PK) {
            fmac<2 * CPL>(tds, qt, dkr[mm]);
          } else {
#pragma unroll
            for (int c = 0; c < 2 * CPL; ++c) dkr[mm][c] = fmaf(tds, qt[c], dkr[mm][c]);
          }
        }
      }
      if ((lane % lph) == 0) dsbuf[(size_t)pr * PH + head] = ds;
    }
  }
  if constexpr (FORCE) {
    if (lane == 0) {
      atomicAdd(dpos + 3 * (size_t)j, fj[0]);
      atomicAdd(dpos + 3 * (size_t)j + 1, fj[1]);
      atomicAdd(dpos + 3 * (size_t)j + 2, fj[2]);
    }
  }
#pragma unroll
  for (int mm = 0; mm < M; ++mm) {
    if constexpr (DK) stvec<2 * CPL>(dk + ((size_t)j * M + mm) * Dq + 2 * c0, dkr[mm]);
    stvec<CPL>(dv + ((size_t)j * M + mm) * PC + c0, dvr[mm]);
  }
}

// Query-centric pass: dq_i = tau * sum_slot ds[i,slot,h] k_j.  Each thread
// owns 8 consecutive q-channels of one (l,m) row (one head).  Warp 0 first
// compacts the valid slots of row i (ballot over the row, so any sentinel
// pattern works) and their per-head dscore rows into shared memory; the
// gather loop then runs over valid pairs only, UNR k_j rows in flight.
// UNR k rows in flight per thread: the pass is an L2 gather of k rows (12.8 KB
// per pair at L = 4); 8 in flight instead of 4 took dq from 4.73 to 3.91 ms on
// configs[3], 1.81 to 1.62 ms on the 100k box, 0.32 to 0.30 ms at 20k atoms
template <typename T, int UNR = 8>
__global__ void __launch_bounds__(1024) attn_bwd_q_kernel(int M, int K, int H, int Dq, float tau,
                                                          const T* __restrict__ k, const int* __restrict__ nbr,
                                                          const float* __restrict__ dsbuf, T* __restrict__ dq) {
  extern __shared__ int bq_smem[];
  int* js = bq_smem;                                   // [K]
  float* dss = reinterpret_cast<float*>(bq_smem + K);  // [K][H]
  __shared__ int nvalid;
  const int i = blockIdx.x;
  const int dqh = Dq / H;
  const int n = M * Dq;
  // parallel compaction: warp w ballots slots [32 w, 32 w + 32), warp
  // counts -> exclusive prefix, then every valid lane copies its (j, dscore row)
  __shared__ int wcnt[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (K + 31) / 32;  // <= blockDim.x / 32 (checked at launch)
  int j = -1, s = warp * 32 + lane;
  unsigned m = 0;
  if (warp < nw) {
    j = s < K ? __ldg(nbr + (size_t)i * K + s) : -1;
    m = __ballot_sync(0xffffffffu, j >= 0);
    if (lane == 0) wcnt[warp] = __popc(m);
  }
  __syncthreads();
  if (warp < nw && j >= 0) {
    int p = __popc(m & ((1u << lane) - 1u));
    for (int w = 0; w < warp; ++w) p += wcnt[w];
    js[p] = j;
    const float* src = dsbuf + ((size_t)i * K + s) * H;
    if ((H & 3) == 0) {
      for (int h = 0; h < H; h += 4)
        *reinterpret_cast<float4*>(dss + p * H + h) = __ldg(reinterpret_cast<const float4*>(src + h));
    } else {
      for (int h = 0; h < H; ++h) dss[p * H + h] = __ldg(src + h);
    }
  }
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < nw; ++w) t += wcnt[w];
    nvalid = t;
  }
  __syncthreads();
  const int nv = nvalid;
  for (int e0 = threadIdx.x * 8; e0 < n; e0 += blockDim.x * 8) {
    const int h = (e0 % Dq) / dqh;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int e = 0;
    for (; e + UNR <= nv; e += UNR) {
      float kv[UNR][8];
#pragma unroll
      for (int u = 0; u < UNR; ++u) ldvec<8>(k + (size_t)js[e + u] * n + e0, kv[u]);
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const float ds = dss[(e + u) * H + h];
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t] = fmaf(ds, kv[u][t], acc[t]);
      }
    }
    for (; e < nv; ++e) {
      const float ds = dss[e * H + h];
      float kv[8];
      ldvec<8>(k + (size_t)js[e] * n + e0, kv);
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] = fmaf(ds, kv[t], acc[t]);
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[t] *= tau;
    stvec<4>(dq + (size_t)i * n + e0, acc);
    stvec<4>(dq + (size_t)i * n + e0 + 4, acc + 4);
  }
}

template <int L, int CPL, bool EAAS, typename T>
es_status run_bwd(const KParams& kp, const void* q, const void* k, const void* v, const double* pos,
                  const int32_t* nbr, const int32_t* rev_ptr, const int32_t* rev_pair, const void* out,
                  const float* lse, const void* dout, void* dq, void* dk, void* dv, float* delta, float* dsbuf,
                  double* dpos, bool skip_dq, bool skip_dk, cudaStream_t st) {
  constexpr int M = Lay<L>::M;
  const int g8 = (kp.C / kp.H) / 8;
  if ((kp.C / kp.H) % 8 == 0 && (g8 & (g8 - 1)) == 0) {
    const int apb = 256 / (kp.C / 8);
    attn_delta_kernel<T, 8><<<(kp.N + apb - 1) / apb, apb * (kp.C / 8), 0, st>>>(kp.N, M, kp.C, kp.H, (const T*)out,
                                                                                 (const T*)dout, delta);
  } else {
    const int apb = 256 / (kp.C / 2);
    attn_delta_kernel<T, 2><<<(kp.N + apb - 1) / apb, apb * (kp.C / 2), 0, st>>>(kp.N, M, kp.C, kp.H, (const T*)out,
                                                                                 (const T*)dout, delta);
  }
  es_status s = cuda_status(cudaGetLastError(), "attn_delta_kernel");
  if (s != ES_OK) return s;
  const int threads = kp.C / CPL;
  const size_t smem = (size_t)Lay<L>::BP * Lay<L>::REC * 4 + (size_t)M * threads * 3 * CPL * 4;
  auto fn = (kp.C == 128 && kp.H == 8) ? attn_bwd_kv_kernel<L, CPL, EAAS, T, 128, 8>
                                                               : attn_bwd_kv_kernel<L, CPL, EAAS, T>;
  if (dpos) {  // position gradients (forces), every L
    fn = attn_bwd_kv_kernel<L, CPL, EAAS, T, 0, 0, true>;
    s = cuda_status(cudaMemsetAsync(dpos, 0, sizeof(double) * 3 * (size_t)kp.Nk, st), "attn_bwd: dpos");
    if (s != ES_OK) return s;
  }
  // dk on the tensor cores (the tcgen05 shape): the key pass keeps dv and the dscores only
  if constexpr (L == 2 && CPL == 2 && EAAS && sizeof(T) == 2) {
    if (skip_dk) {
      if (kp.C != 128 || kp.H != 8) return fail(ES_CUDA_ERROR, "attn_bwd: tensor-core dk outside its shape");
      fn = dpos ? attn_bwd_kv_kernel<L, CPL, EAAS, T, 0, 0, true, false>
                : attn_bwd_kv_kernel<L, CPL, EAAS, T, 128, 8, false, false>;
    }
  } else {
    if (skip_dk) return fail(ES_CUDA_ERROR, "attn_bwd: tensor-core dk outside its shape");
  }
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fn<<<kp.Nk, threads, smem, st>>>(kp, (const T*)q, (const T*)k, (const T*)v, pos, rev_ptr, rev_pair, lse,
                                  (const T*)dout, delta, (T*)dk, (T*)dv, dsbuf, dpos);
  s = cuda_status(cudaGetLastError(), "attn_bwd_kv_kernel");
  if (s != ES_OK || skip_dq) return s;  // skip_dq: the tcgen05 dq kernel runs next
  {
    int tq = (M * kp.Dq / 8 + 31) / 32 * 32;
    if (tq > 1024) tq = 1024;
    if (tq < (kp.K + 31) / 32 * 32) tq = (kp.K + 31) / 32 * 32;  // one slot per thread in the compaction
    if (tq > 1024) return fail(ES_UNSUPPORTED, "attn_bwd: K > 1024");
    const size_t qsm = (size_t)kp.K * (1 + kp.H) * 4;
    if (qsm > 200 * 1024) return fail(ES_UNSUPPORTED, "attn_bwd: K * (H + 1) too large for the dq pass");
    auto qfn = attn_bwd_q_kernel<T>;
    if (qsm > 48 * 1024) cudaFuncSetAttribute(qfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsm);
    qfn<<<kp.N, tq, qsm, st>>>(M, kp.K, kp.H, kp.Dq, kp.tau, (const T*)k, nbr, dsbuf, (T*)dq);
  }
  return cuda_status(cudaGetLastError(), "attn_bwd_q_kernel");
}

KParams make_params(const AttnArgs& a) {
  KParams kp;
  kp.N = a.N; kp.K = a.K; kp.H = a.H; kp.C = a.C; kp.Dq = a.Dq;
  kp.row0 = a.row0; kp.Nk = a.Nk;
  kp.phi_mode = a.phi_mode; kp.periodic = a.periodic;
  kp.tau = a.tau; kp.r_cut = a.r_cut; kp.inv_rcut = 1.f / a.r_cut;
  kp.bx = a.box[0]; kp.by = a.box[1]; kp.bz = a.box[2];
  kp.bias_mode = a.bias_mode; kp.b0 = a.bias[0]; kp.b1 = a.bias[1]; kp.b2 = a.bias[2];
  kp.scores_out = a.scores_out; kp.scores_in = a.scores_in;
  kp.rank_of = nullptr;
  return kp;
}

}  // namespace

// the backward for one degree L (instantiated in attention_bwd_l<L>.cu)
template <int LL>
es_status bwd_run_L(const AttnArgs& a, const int* rank_of, const void* q, const void* k, const void* v,
                    const double* pos, const int32_t* nbr, const int32_t* rev_ptr, const int32_t* rev_pair,
                    const void* out, const float* lse, const void* dout, void* dq, void* dk, void* dv, float* delta,
                    float* dsbuf, double* dpos, bool skip_dq, bool skip_dk, cudaStream_t st)
#ifdef ES_BWD_DEFINE
{
  es_status s = upload_tables_tu();  // this translation unit's constant tables
  if (s != ES_OK) return s;
  KParams kp = make_params(a);
  kp.rank_of = rank_of;
  const bool eaas = a.value_mode == ES_VALUE_EAAS;
  const bool bf = a.dtype == ES_BF16;
  const int cpl = (LL <= 2 && a.C % 64 == 0 && (a.C / a.H) % 2 == 0) ? 2 : 1;
#define ES_RUN(CC)                                                                                          \
  {                                                                                                        \
    if (eaas)                                                                                              \
      return bf ? run_bwd<LL, CC, true, __nv_bfloat16>(kp, q, k, v, pos, nbr, rev_ptr, rev_pair, out, lse, dout, dq,  \
                                                       dk, dv, delta, dsbuf, dpos, skip_dq, skip_dk, st)   \
                : run_bwd<LL, CC, true, float>(kp, q, k, v, pos, nbr, rev_ptr, rev_pair, out, lse, dout, dq, dk, dv, \
                                               delta, dsbuf, dpos, skip_dq, skip_dk, st);                  \
    return bf ? run_bwd<LL, CC, false, __nv_bfloat16>(kp, q, k, v, pos, nbr, rev_ptr, rev_pair, out, lse, dout, dq, \
                                                      dk, dv, delta, dsbuf, dpos, skip_dq, skip_dk, st)    \
              : run_bwd<LL, CC, false, float>(kp, q, k, v, pos, nbr, rev_ptr, rev_pair, out, lse, dout, dq, dk, dv, \
                                              delta, dsbuf, dpos, skip_dq, skip_dk, st);                   \
  }
  if constexpr (LL <= 2) {
    if (cpl == 2) ES_RUN(2)
  }
  ES_RUN(1)
#undef ES_RUN
}
#else
;
#endif

}  // namespace es
