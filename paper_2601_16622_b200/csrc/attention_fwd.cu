// Forward of the fused equivariant attention; see attention_common.cuh.
#include <cstdlib>

#include "attention_common.cuh"

namespace es {
namespace {

// ------------------------------------------------------------------ forward
// CC, HH > 0: channels / heads fixed at compile time (the BASELINE shape C=128,
// H=8): row strides become immediates, no per-row 64-bit address arithmetic.
// L >= 3 at C = 128 (the OMol25-like shape of configs[3]): one 128-thread CTA
// per query atom, CPL = 1.  The query rows are staged in shared memory for the
// score phase instead of 2 M registers per thread (50 at L = 4), which frees
// the registers the value phase needs and lets ES_L34_FWD_MINB CTAs reside.
#ifndef ES_L34_FWD_MINB
#define ES_L34_FWD_MINB 2
#endif
#ifndef ES_L34_QSMEM
#define ES_L34_QSMEM 1
#endif
// ES_L34_FWD_CPL = 2: two channels per thread (64-thread CTAs, packed FFMA2 in
// the target-degree-ordered EAAS form, half the broadcast shared-memory loads
// of the per-pair operator per FMA)
// pairs per neighbour batch at L >= 3, C = 128: 16 (half of Lay<L>::BP) keeps the
// records + staged q under a quarter of shared memory, so the register limit
// (4 CTAs of 64 threads at 255 registers) and not shared memory bounds occupancy
#ifndef ES_L34_FWD_BP
#define ES_L34_FWD_BP 16
#endif
#ifndef ES_L34_FWD_CPL
#define ES_L34_FWD_CPL 2
#endif
template <int L, int CC, int CPL>
struct FwdShape {
  static constexpr bool BIG = L >= 3 && CC == 128;
  static constexpr bool QS = ES_L34_QSMEM && BIG;
  static constexpr int THREADS = BIG ? 128 / CPL : 256;
  static constexpr int MINB = BIG ? ES_L34_FWD_MINB * CPL : (L <= 2 ? 2 : 1);
  static constexpr int BP = BIG ? ES_L34_FWD_BP : Lay<L>::BP;
};

template <int L, int CPL, bool EAAS, typename T, int CC = 0, int HH = 0>
__global__ void __launch_bounds__(FwdShape<L, CC, CPL>::THREADS, FwdShape<L, CC, CPL>::MINB) attn_fwd_kernel(KParams p, const T* __restrict__ q, const T* __restrict__ k,
                                                       const T* __restrict__ v, const double* __restrict__ pos,
                                                       const int* __restrict__ nbr, T* __restrict__ out,
                                                       float* __restrict__ lse) {
  const int PC = CC ? CC : p.C, PH = HH ? HH : p.H, PDq = CC ? 2 * CC : p.Dq;
  using LY = Lay<L>;
  constexpr int M = LY::M;
  constexpr int REC = LY::REC;
  constexpr int BP = FwdShape<L, CC, CPL>::BP;
  extern __shared__ float4 smem4[];
  __shared__ int cnt_w[32];
  float* recs = reinterpret_cast<float*>(smem4);
  float* sc = recs + BP * REC;  // [BP][H]
  const int tpq = blockDim.x;
  const int i = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = (warp * 32 + lane) * CPL;  // first value channel of this lane
  const int Ch = PC / PH;                 // value channels per head
  const int lph = Ch / CPL;                 // lanes per head
  const int head = c0 / Ch;
  const int Dq = PDq;

  constexpr bool QS = FwdShape<L, CC, CPL>::QS;
  float qr[QS ? 1 : M][2 * CPL];
  float* qs = sc + BP * PH;  // QS: [M][tpq][2 CPL] fp32 (conflict-free vector LDS)
  if constexpr (QS) {
#pragma unroll
    for (int mm = 0; mm < M; ++mm) {
      float t[2 * CPL];
      ldvec<2 * CPL>(q + ((size_t)i * M + mm) * Dq + 2 * c0, t);
#pragma unroll
      for (int c = 0; c < 2 * CPL; ++c) qs[(mm * tpq + threadIdx.x) * 2 * CPL + c] = t[c];
    }
  } else {
#pragma unroll
    for (int mm = 0; mm < M; ++mm) ldvec<2 * CPL>(q + ((size_t)i * M + mm) * Dq + 2 * c0, qr[mm]);
  }
  // this thread's query channels of row mm (registers, or the staged copy)
  auto qrow = [&](int mm, int c) -> float {
    if constexpr (QS) return qs[(mm * tpq + threadIdx.x) * 2 * CPL + c];
    else return qr[mm][c];
  };
  float A[M][CPL];
#pragma unroll
  for (int mm = 0; mm < M; ++mm)
#pragma unroll
    for (int c = 0; c < CPL; ++c) A[mm][c] = 0.f;
  float mu = -INFINITY, z = 0.f;

  for (int base = 0; base < p.K; base += BP) {
    const int nslot = min(BP, p.K - base);
    __syncthreads();
    // compact this batch's valid slots: rec e < nb holds the e-th valid pair
    int nb = 0;
    for (int t0 = 0; t0 < nslot; t0 += tpq) {
      const int t = t0 + warp * 32 + lane;
      const int j = t < nslot ? nbr[(size_t)i * p.K + base + t] : -1;
      const unsigned m = __ballot_sync(0xffffffffu, j >= 0);
      if (lane == 0) cnt_w[warp] = __popc(m);
      __syncthreads();
      int before = nb;
      for (int w = 0; w < warp; ++w) before += cnt_w[w];
      int tot = 0;
      for (int w = 0; w < (tpq >> 5); ++w) tot += cnt_w[w];
      if (j >= 0) {
        float* rec = recs + (before + __popc(m & ((1u << lane) - 1u))) * REC;
        pair_prepare<L, EAAS>(p, pos, i, j, rec);
        rec[LY::OFF_X] = __int_as_float(base + t);  // slot (score store)
      }
      nb += tot;
      __syncthreads();
    }
    if (nb == 0) continue;
    // phase A: scores of this warp's heads for the whole batch (two pairs in flight)
    int e = 0;
    for (; e + 2 <= nb; e += 2) {
      const int j0 = __float_as_int(recs[e * REC + LY::OFF_J]);
      const int j1 = __float_as_int(recs[(e + 1) * REC + LY::OFF_J]);
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int mm = 0; mm < M; ++mm) {
        float k0[2 * CPL], k1[2 * CPL];
        ldvec<2 * CPL>(k + ((size_t)j0 * M + mm) * Dq + 2 * c0, k0);
        ldvec<2 * CPL>(k + ((size_t)j1 * M + mm) * Dq + 2 * c0, k1);
#pragma unroll
        for (int c = 0; c < 2 * CPL; ++c) {
          const float qc = qrow(mm, c);
          s0 = fmaf(qc, k0[c], s0);
          s1 = fmaf(qc, k1[c], s1);
        }
      }
      for (int o = lph >> 1; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      }
      if ((lane % lph) == 0) {
        sc[e * PH + head] = fmaf(s0, p.tau, recs[e * REC + LY::OFF_B]);
        sc[(e + 1) * PH + head] = fmaf(s1, p.tau, recs[(e + 1) * REC + LY::OFF_B]);
      }
    }
    for (; e < nb; ++e) {
      const int j = __float_as_int(recs[e * REC + LY::OFF_J]);
      float s = 0.f;
#pragma unroll
      for (int mm = 0; mm < M; ++mm) {
        float kv[2 * CPL];
        ldvec<2 * CPL>(k + ((size_t)j * M + mm) * Dq + 2 * c0, kv);
#pragma unroll
        for (int c = 0; c < 2 * CPL; ++c) s = fmaf(qrow(mm, c), kv[c], s);
      }
      for (int o = lph >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if ((lane % lph) == 0) sc[e * PH + head] = fmaf(s, p.tau, recs[e * REC + LY::OFF_B]);
    }
    __syncwarp();
    if (p.scores_out && (lane % lph) == 0)
      for (int e2 = 0; e2 < nb; ++e2)
        p.scores_out[((size_t)head * p.N + i) * p.K + __float_as_int(recs[e2 * REC + LY::OFF_X])] = sc[e2 * PH + head];
    float bm = -INFINITY;
    for (int e2 = 0; e2 < nb; ++e2) bm = fmaxf(bm, sc[e2 * PH + head]);
    const float mu2 = fmaxf(mu, bm);
    const float scale = __expf(mu - mu2);  // mu = -inf -> 0
    z *= scale;
#pragma unroll
    for (int mm = 0; mm < M; ++mm)
#pragma unroll
      for (int c = 0; c < CPL; ++c) A[mm][c] *= scale;
    mu = mu2;
    // phase B: values
    for (int e2 = 0; e2 < nb; ++e2) {
      const float* rec = recs + e2 * REC;
      const int j = __float_as_int(rec[LY::OFF_J]);
      if (e2 + 1 < nb) {
        const int jn = __float_as_int(recs[(e2 + 1) * REC + LY::OFF_J]);
#pragma unroll
        for (int mm = 0; mm < M; ++mm) pf_l1(v + ((size_t)jn * M + mm) * PC + c0);
      }
      const float pr = expf(sc[e2 * PH + head] - mu);
      z += pr;
      const float s = pr * rec[LY::OFF_PHI];
      float vv[M][CPL];
#pragma unroll
      for (int mm = 0; mm < M; ++mm) ldvec<CPL>(v + ((size_t)j * M + mm) * PC + c0, vv[mm]);
      if constexpr (EAAS) {
        value_apply<L, CPL, false>(rec, vv, s, A);
      } else {
#pragma unroll
        for (int mm = 0; mm < M; ++mm)
#pragma unroll
          for (int c = 0; c < CPL; ++c) A[mm][c] = fmaf(s, vv[mm][c], A[mm][c]);
      }
    }
  }
  const float inv = z > 0.f ? 1.f / z : 0.f;
#pragma unroll
  for (int mm = 0; mm < M; ++mm) {
    float o[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) o[c] = A[mm][c] * inv;
    stvec<CPL>(out + ((size_t)i * M + mm) * PC + c0, o);
  }
  if ((lane % lph) == 0) lse[(size_t)i * PH + head] = z > 0.f ? mu + logf(z) : -INFINITY;
}


template <int L, int CPL, bool EAAS, typename T>
es_status run_fwd(const KParams& kp, const void* q, const void* k, const void* v, const double* pos,
                  const int32_t* nbr, void* out, float* lse, cudaStream_t st) {
  const int tpq = kp.C / CPL;
  const bool fixed = kp.C == 128 && kp.H == 8;
  const int bp = fixed ? FwdShape<L, 128, CPL>::BP : Lay<L>::BP;
  size_t smem = (size_t)bp * Lay<L>::REC * 4 + (size_t)bp * kp.H * 4;
  if (fixed && FwdShape<L, 128, CPL>::QS) smem += (size_t)Lay<L>::M * tpq * 2 * CPL * 4;
  auto fn = fixed ? attn_fwd_kernel<L, CPL, EAAS, T, 128, 8> : attn_fwd_kernel<L, CPL, EAAS, T>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fn<<<kp.N, tpq, smem, st>>>(kp, (const T*)q, (const T*)k, (const T*)v, pos, nbr, (T*)out, lse);
  return cuda_status(cudaGetLastError(), "attn_fwd_kernel");
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
  return kp;
}

template <template <int, int, bool, typename> class Op, typename... Args>
es_status dispatch(const AttnArgs& a, Args&&... args) {
  const bool eaas = a.value_mode == ES_VALUE_EAAS;
  const bool bf = a.dtype == ES_BF16;
  const int cpl = (a.L <= 2 && a.C % 64 == 0 && (a.C / a.H) % 2 == 0) ? 2
                  : (a.L >= 3 && a.C == 128 && a.H == 8) ? ES_L34_FWD_CPL : 1;
#define ES_CASE(LL, CC)                                                                                  \
  if (a.L == LL && cpl == CC) {                                                                          \
    if (eaas) return bf ? Op<LL, CC, true, __nv_bfloat16>::run(args...) : Op<LL, CC, true, float>::run(args...); \
    return bf ? Op<LL, CC, false, __nv_bfloat16>::run(args...) : Op<LL, CC, false, float>::run(args...);        \
  }
  ES_CASE(0, 2) ES_CASE(1, 2) ES_CASE(2, 2) ES_CASE(0, 1) ES_CASE(1, 1) ES_CASE(2, 1) ES_CASE(3, 1) ES_CASE(4, 1)
#if ES_L34_FWD_CPL == 2
  ES_CASE(3, 2) ES_CASE(4, 2)
#endif
#undef ES_CASE
  return fail(ES_UNSUPPORTED, "attention: no kernel for this (L, C, H)");
}

template <int L, int CPL, bool EAAS, typename T>
struct FwdOp {
  template <typename... A>
  static es_status run(A... a) { return run_fwd<L, CPL, EAAS, T>(a...); }
};
}  // namespace

namespace {
bool use_tc_kernel(const AttnArgs& a) {
  // bf16 / L=2 / C=128 / H=8 (the BASELINE shapes): the tcgen05 kernel
  // (2.9 ms vs 4.5 ms for the SIMT kernel on configs[1]); ES_ATTN_TC=0 forces
  // the SIMT kernel (kept for the other shapes and for A/B measurements).
  // ES_ATTN_TC=1 forces it for any size (parity tests on small systems).
  static int use_tc = -1;
  if (use_tc < 0) {
    const char* e = getenv("ES_ATTN_TC");
    use_tc = (e && e[0] == '0') ? 0 : (e && e[0] == '1') ? 2 : 1;
  }
  // one 128-query tile per CTA: below ~half a wave of tiles (N < 74 * 128)
  // the per-atom SIMT kernel fills the GPU better (r01b sweep: SIMT faster
  // at N = 1k..5k, tie at 10k, tcgen05 faster from 20k)
  // and only for molecule batches: on one bulk system a tile's ~50-neighbour rows spread over ~150 key
  // chunks and the per-atom SIMT kernel wins (configs[2]/[4] at 20k / 100k atoms: 0.89 / 5.2 ms vs
  // 1.13 / 8.6 ms forward, profiles/r02_dispatch.txt)
  const bool enough_tiles = (a.N + 127) / 128 >= 74 && a.nseg > 0;
  return use_tc && (enough_tiles || use_tc == 2) && attn_tc_supported(a);
}
}  // namespace

size_t attn_fwd_workspace(const AttnArgs& a) { return use_tc_kernel(a) ? attn_fwd_tc_workspace(a) : 0; }

es_status attn_fwd_launch(const AttnArgs& a, const void* q, const void* k, const void* v, const double* pos,
                          const int32_t* nbr, void* out, float* lse, void* ws, size_t ws_bytes, cudaStream_t st) {
  es_status s = upload_tables_tu();
  if (s != ES_OK) return s;
  const KParams kp = make_params(a);
  if (a.N == 0) return ES_OK;
  if (use_tc_kernel(a)) return attn_fwd_tc_launch(a, q, k, v, pos, nbr, out, lse, ws, ws_bytes, st);
  return dispatch<FwdOp>(a, kp, q, k, v, pos, nbr, out, lse, st);
}

}  // namespace es
