// Tensor-core (tcgen05 / TMEM / TMA) fused equivariant attention, forward,
// bf16 storage, L = 2, C = 128, H = 8 (C_h = 16, d_k = 288) -- the shape of
// BASELINE configs 2, 3 and 5.
//
// Formulation (exact; same map as the per-pair EAAS kernel, Prop. 1):
//   x_ij = phi_ij sum_f Y^f(r_ij) G_f v_j,   G_f[o, i'] = C^{o}_{i', f}
// (the CG coupling of v_j with the solid harmonic basis function f, summed
// over the path set).  Per head h, with P_ij = exp(tau s_ij - lse_i):
//   out_i[(o,c)] = sum_{(f,j)} Wt[i,(f,j)] Vg[(f,j),(o,c)]
//   Wt[i,(f,j)]  = P_ij phi_ij Y^f(r_ij)          (9 scalars per pair: the only per-pair work)
//   Vg[(f,j),(o,c)] = sum_i' G_f[o,i'] v_j[i',c]   (per-key source coupling, 137 non-zeros)
// so both contractions run on the tensor cores:
//   S  = Q_h K_h^T            M=128 queries, N=16 keys,  K=288   (TMA, 64B swizzle)
//   O += Wt . Vg^T            M=128 queries, N=144 (o,c), K=144 (f,j)   (no-swizzle core matrices)
// A CTA owns a tile of 128 query atoms (whole molecules packed, or 128
// consecutive rows); key chunks of 16 atoms are the non-empty entries of the
// tile-skip mask.  One-pass online softmax: the running maximum only moves the
// exponent base when a chunk raises it by more than 5 (lazy rescale of the TMEM
// accumulator, rarely taken), and the epilogue divides by the row sum.  Invalid
// (non-neighbour) pairs get Wt = 0; pair validity comes from the neighbour
// index itself (never re-tested in fp32).
#include <cuda.h>
#include <cuda_bf16.h>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cub/cub.cuh>

#include "_gen_cg.h"
#include "es_internal.h"
#include "umma.cuh"

namespace es {

namespace {

using bf16 = __nv_bfloat16;

constexpr int TQ = 128;      // queries per tile (MMA M)
constexpr int KC = 16;       // keys per chunk (S MMA N)
constexpr int HD = 16;       // value channels per head
constexpr int DH = 32;       // q/k channels per head per (l,m) row
constexpr int MM = 9;        // (L+1)^2, L = 2
constexpr int KV = MM * KC;  // 144: value MMA K  ((f, j))
constexpr int NV = MM * HD;  // 144: value MMA N  ((o, c))

// shared memory map (bytes): 3 K/V/pos stages, double-buffered Wt and Vg
constexpr int NSTAGE = 3;
constexpr int KBYTES = MM * KC * DH * 2;               // 9 x [16 x 32] bf16 SW64   9216
constexpr int VBYTES = KC * MM * HD * 2;               // [16 keys][9][16] bf16     4608
constexpr int PBYTES = KC * 24;                        // [16 keys][3] f64          384
constexpr int WBYTES = TQ * KV * 2;                    // [128 x 144] core-matrix   36864
constexpr int GBYTES = NV * KV * 2;                    // [144 x 144] core-matrix   41472
constexpr int SM_K = 0;                                // NSTAGE x KBYTES
constexpr int SM_VST = SM_K + NSTAGE * KBYTES;         // NSTAGE x VBYTES
constexpr int SM_POS = SM_VST + NSTAGE * VBYTES;       // NSTAGE x PBYTES (chunk key positions)
constexpr int SM_WT = (SM_POS + NSTAGE * PBYTES + 1023) / 1024 * 1024;  // 2 x WBYTES (1024-aligned)
constexpr int SM_VG = SM_WT + 2 * WBYTES;              // 2 x GBYTES
constexpr int SM_BAR = SM_VG + 2 * GBYTES;
constexpr int SM_ZX = SM_BAR + 256;                    // [2][128] f32 softmax denominators of the key halves
constexpr int SM_PROW = SM_ZX + 2 * TQ * 4;            // [2][128 rows][16 keys] f32 softmax numerators
constexpr int SM_PAIRS = SM_PROW + 2 * TQ * KC * 4;    // [2][4 quadrants][512] u16 (row << 4 | key) pair lists
constexpr int SM_QTOT = SM_PAIRS + 2 * TQ * KC * 2;    // [2][4] i32 pairs per quadrant
constexpr int SM_QPOS = SM_QTOT + 64;                  // [128 rows][3] f64 query positions
constexpr int SM_TOTAL = SM_QPOS + TQ * 24;
static_assert(SM_TOTAL + 1024 <= 232448, "forward kernel exceeds 227 KB of shared memory");
static_assert(SM_POS + NSTAGE * PBYTES <= SM_WT, "smem map overlap");

struct TcTab {
  float ycoef[4];        // Y0, c1, c2, c20
  unsigned char ent_i[160];
  float ent_c[160];
  int ofs[MM * MM + 1];  // (o, f) -> entry range
};
__constant__ TcTab c_tc;
// Per-chunk event clocks of CTA 0 (compile with -DES_TC_TRACE, run with
// ES_TC_DBG=16): producer / MMA / row / Vg timelines, the tool used to find
// this kernel's critical path.
#ifdef ES_TC_TRACE
__device__ long long g_trace[8][128];
__device__ long long g_trace_w[8][128];  // per row warp: Wt arrive clock
__device__ long long g_trace_r[4][128];  // row thread 64: before / after the Wt-free wait, after the phase barrier
#define TC_TRACE(cond, slot) \
  do {                       \
    if (TRACE && (cond) && g < 128) slot = clock64(); \
  } while (0)
#else
#define TC_TRACE(cond, slot) \
  do {                       \
  } while (0)
#endif

struct TcArgs {
  int N, K, row0, Nk;
  int bias_mode;
  float b0, b1, b2;
  float* scores;       // optional [N][K][8] score store
  int score_rank;      // 1: scores indexed by (row, rank) -- the rank_of map of the tiles resolves slots
  const int* slots;    // the rows' ascending-j slot order (needed with scores)
  int dbg;  // profiling switches (ES_TC_DBG): 1 skip Vg math, 2 skip Wt math, 4 skip value MMA, 8 skip S MMA
  float tau, r_cut, inv_rcut;
  int phi_mode, periodic;
  double bx, by, bz;
};

// b(r_ij) of one pair from the staged key / query positions (kept out of line: the
// softmax phase it serves is register-bound)
__device__ __forceinline__ float tc_pair_bias(const TcArgs& a, const double* kp, const double* qp) {
  double dx = kp[0] - qp[0], dy = kp[1] - qp[1], dz = kp[2] - qp[2];
  if (a.periodic) {
    dx -= a.bx * rint(dx / a.bx);
    dy -= a.by * rint(dy / a.by);
    dz -= a.bz * rint(dz / a.bz);
  }
  const float rx = (float)dx, ry = (float)dy, rz = (float)dz;
  const float rn = sqrtf(rx * rx + ry * ry + rz * rz);
  return fmaf(fmaf(a.b2, rn, a.b1), rn, a.b0);
}

__device__ __forceinline__ void solid_l2(float x, float y, float z, float* Y) {
  const float r2 = x * x + y * y + z * z;
  const float c1 = c_tc.ycoef[1], c2 = c_tc.ycoef[2], c20 = c_tc.ycoef[3];
  Y[0] = c_tc.ycoef[0];
  Y[1] = c1 * y; Y[2] = c1 * z; Y[3] = -c1 * x;
  Y[4] = c2 * x * y; Y[5] = c2 * y * z; Y[6] = c20 * (1.5f * z * z - 0.5f * r2);
  Y[7] = -c2 * x * z; Y[8] = 0.5f * c2 * (x * x - y * y);
}

// no-swizzle K-major core-matrix layout: element (r, k) of an R x KV operand
__device__ __forceinline__ uint32_t cm_off(int r, int k) {
  return (uint32_t)((((r >> 3) * (KV / 8) + (k >> 3)) << 7) + ((r & 7) << 4) + ((k & 7) << 1));
}

__device__ __forceinline__ uint4 pack8(const float* v) {
  uint4 u;
  __nv_bfloat162 t;
  t = __floats2bfloat162_rn(v[0], v[1]); u.x = *reinterpret_cast<uint32_t*>(&t);
  t = __floats2bfloat162_rn(v[2], v[3]); u.y = *reinterpret_cast<uint32_t*>(&t);
  t = __floats2bfloat162_rn(v[4], v[5]); u.z = *reinterpret_cast<uint32_t*>(&t);
  t = __floats2bfloat162_rn(v[6], v[7]); u.w = *reinterpret_cast<uint32_t*>(&t);
  return u;
}

// Warp-specialised pipeline (448 threads):
//   warp 0, one lane : TMA producer (K, V, key positions; 3 stages)
//   warp 1, one lane : tcgen05 MMA issuer
//   warps 2-9        : the 128 query rows, two warps per TMEM lane quadrant:
//                      each reads the row's 16 scores, both run the identical
//                      online-softmax max/rescale decision, and each builds the
//                      Wt entries of one half of the chunk's keys (8 keys =
//                      one 16-byte store per f) -- no zero-fill pass, no
//                      shuffles, two warps per scheduler for latency hiding
//   warps 10-13      : per-key source coupling Vg (+ Q_h into TMEM)
// Q_h lives in tensor memory (the S MMA's A operand); Wt and Vg are double
// buffered, so chunk c+1's SIMT work overlaps chunk c's value MMA.
// TMEM: Q[2] [0,144) / [144,288) (next head's Q is loaded by the Vg warps
// while the current head runs), O [288,432), S[2] [448,464) / [480,496).
constexpr int TC_THREADS = 448;

template <bool BIAS, bool SCORES>
__global__ void __launch_bounds__(TC_THREADS, 1) attn_fwd_tc_kernel(
    const __grid_constant__ CUtensorMap mk, const __grid_constant__ CUtensorMap mv, TcArgs a,
    const bf16* __restrict__ q, const double* __restrict__ pos, const int* __restrict__ nbr,
    const int* __restrict__ cptr, const int* __restrict__ clist, const uint32_t* __restrict__ rowlist,
    const int* __restrict__ tstart, bf16* __restrict__ out, float* __restrict__ lse) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (umma::smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in .shared
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + SM_BAR);
  uint64_t* full_kv = bars + 0;    // [3] TMA landed (tx)
  uint64_t* empty_kv = bars + 3;   // [3] S MMA done with K + rows with key pos + Vg threads with V (385)
  uint64_t* s_full = bars + 6;     // [2] S MMA committed
  uint64_t* s_free = bars + 8;     // [2] rows read S (256)
  uint64_t* wt_full = bars + 10;   // [2] rows wrote Wt (256)
  uint64_t* vg_full = bars + 12;   // [2] Vg warps wrote Vg (128)
  uint64_t* wv_free = bars + 14;   // [2] value MMA committed (Wt / Vg free, O updated)
  uint64_t* acc_done = bars + 17;  // last value MMA of the head committed
  uint64_t* epi_done = bars + 18;  // rows finished reading O (256)
  uint64_t* q_ready = bars + 19;   // [2] Q_h stored into TMEM buffer h&1 (128, Vg warps)
  uint64_t* q_free = bars + 21;    // [2] last S MMA reading Q buffer committed
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 23);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q0 = tstart[blockIdx.x], q1 = tstart[blockIdx.x + 1];
  if (q0 >= q1) return;  // surplus (empty) tile: nothing to do, no barrier touched yet
#ifdef ES_TC_TRACE
  const bool TRACE = (a.dbg & 16) && blockIdx.x == 0;
#endif
  const int c_begin = cptr[blockIdx.x], nch = cptr[blockIdx.x + 1] - cptr[blockIdx.x];
  const bool is_row = warp >= 2 && warp <= 9;
  const int row = ((warp & 3) << 5) | lane;  // TMEM lane of a row thread (warp w -> lanes 32 (w%4) ..)
  const int qi = q0 + row;
  const bool qvalid = is_row && qi < q1;
  const bool qin = qi < q1;  // row exists (Vg warps load Q rows too)

  if (tid == 0) {
    umma::prefetch_tmap(&mk);
    umma::prefetch_tmap(&mv);
    for (int b = 0; b < NSTAGE; ++b) {
      umma::mbar_init(&full_kv[b], 1);
      umma::mbar_init(&empty_kv[b], 1 + 256 + 128);
    }
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&s_full[b], 1);
      umma::mbar_init(&s_free[b], 256);
      umma::mbar_init(&wt_full[b], 256);
      umma::mbar_init(&vg_full[b], 128);
      umma::mbar_init(&wv_free[b], 1);
    }
    umma::mbar_init(&q_ready[0], 128);
    umma::mbar_init(&q_ready[1], 128);
    umma::mbar_init(&q_free[0], 1);
    umma::mbar_init(&q_free[1], 1);
    umma::mbar_init(acc_done, 1);
    umma::mbar_init(epi_done, 256);
    umma::fence_barrier_init();
  }
  if (warp == 0) umma::tmem_alloc(tslot, 512);
  double* qpos = reinterpret_cast<double*>(sm + SM_QPOS);
  if (is_row && warp < 6) {
    const int qa = a.row0 + (qin ? qi : 0);
    qpos[3 * row] = qin ? pos[3 * qa] : 0.0;
    qpos[3 * row + 1] = qin ? pos[3 * qa + 1] : 0.0;
    qpos[3 * row + 2] = qin ? pos[3 * qa + 2] : 0.0;
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t t_q0 = tmem, t_out = tmem + 288, t_s0 = tmem + 448;  // Q[2] at 0 / 144
  constexpr uint32_t idesc_s = umma::idesc_bf16(128, KC, 0, 0);
  constexpr uint32_t idesc_v = umma::idesc_bf16(128, NV, 0, 0);

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer =================
      // L2 prefetch runs PF chunks ahead of the shared-memory stages (hides HBM latency)
      constexpr int PF = 4;
      auto prefetch = [&](int h, int c) {
        const int k0 = clist[c_begin + c] * KC;
        umma::tma_prefetch_3d(&mk, DH * h, k0, 0);
        umma::tma_prefetch_3d(&mv, HD * h, 0, k0);
      };
      for (int c = 0; c < nch && c < PF; ++c) prefetch(0, c);
      int g0 = 0;
      for (int h = 0; h < 8; ++h) {
        for (int c = 0; c < nch; ++c) {
          const int g = g0 + c, st = g % NSTAGE;
          {  // prefetch chunk c + PF (possibly of the next head)
            const int cp = c + PF;
            if (cp < nch) prefetch(h, cp);
            else if (h + 1 < 8 && cp - nch < nch) prefetch(h + 1, cp - nch);
          }
          TC_TRACE(true, g_trace[7][g]);
          if (g >= NSTAGE) umma::mbar_wait(&empty_kv[st], ((g / NSTAGE) - 1) & 1);
          const int k0 = clist[c_begin + c] * KC;
          const int nkeys = min(KC, a.Nk - k0);
          // bulk copies move multiples of 16 bytes: an odd key count leaves the last key's 24 bytes to a plain
          // load (stored before the arrive, whose release orders it for the consumers) -- never past pos[3*Nk]
          const uint32_t pbytes = (uint32_t)((nkeys & ~1) * 24);
          if (nkeys & 1) {
            double* tail = reinterpret_cast<double*>(sm + SM_POS + st * PBYTES) + 3 * (nkeys - 1);
            const double* src = pos + 3 * ((size_t)k0 + nkeys - 1);
            tail[0] = src[0]; tail[1] = src[1]; tail[2] = src[2];
          }
          uint8_t* kb = sm + SM_K + st * KBYTES;
          umma::mbar_arrive_expect_tx(&full_kv[st], KBYTES + VBYTES + pbytes);
          umma::tma_load_3d(kb, &mk, &full_kv[st], DH * h, k0, 0);  // 9 (l,m) blocks [16 keys][32 ch]
          umma::tma_load_3d(sm + SM_VST + st * VBYTES, &mv, &full_kv[st], HD * h, 0, k0);
        TC_TRACE(true, g_trace[0][g]);
          if (pbytes) umma::bulk_load(sm + SM_POS + st * PBYTES, pos + 3 * (size_t)k0, pbytes, &full_kv[st]);
        }
        g0 += nch;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ================= MMA issuer =================
      auto value_mma = [&](int g, int c, int h) {
        const int b = g & 1;
        umma::mbar_wait(&wt_full[b], (g >> 1) & 1);
        umma::mbar_wait(&vg_full[b], (g >> 1) & 1);
        if (c == 0 && h > 0) umma::mbar_wait(epi_done, (h - 1) & 1);  // O of the previous head read out
        umma::tc_fence_after();
        // descriptors advance by (byte offset >> 4) from one base: the single issuing thread
        // would otherwise spend ~100 cycles of dependent integer ops per MMA building them
        const uint64_t wd = umma::sdesc(umma::smem_u32(sm + SM_WT + b * WBYTES), 128, (KV / 8) * 128, 0);
        const uint64_t vd = umma::sdesc(umma::smem_u32(sm + SM_VG + b * GBYTES), 128, (KV / 8) * 128, 0);
        if (!(a.dbg & 4)) {
          umma::mma_f16(t_out, wd, vd, idesc_v, c > 0 ? 1u : 0u);
#pragma unroll
          for (int s = 1; s < MM; ++s) umma::mma_f16(t_out, wd + (uint64_t)(16 * s), vd + (uint64_t)(16 * s), idesc_v, 1u);
        }
        umma::mma_commit(&wv_free[b]);
        TC_TRACE(true, g_trace[6][g]);
      };
      auto issue_s = [&](int g, int h, bool last) {
        const int b = g & 1, st = g % NSTAGE;
        umma::mbar_wait(&full_kv[st], (g / NSTAGE) & 1);
        if (g >= 2) umma::mbar_wait(&s_free[b], ((g >> 1) - 1) & 1);
        umma::tc_fence_after();
        const uint64_t kd = umma::sdesc(umma::smem_u32(sm + SM_K + st * KBYTES), 16, 512, 4);
        const uint32_t tq = t_q0 + 144 * (h & 1), ts = t_s0 + 32 * b;
        if (!(a.dbg & 8)) {
#pragma unroll
          for (int s = 0; s < 2 * MM; ++s)
            umma::mma_f16_ts(ts, tq + 8 * s, kd + (uint64_t)(((s >> 1) * KC * DH * 2 + (s & 1) * 32) >> 4), idesc_s,
                             s > 0 ? 1u : 0u);
        }
        umma::mma_commit(&s_full[b]);
        TC_TRACE(true, g_trace[1][g]);
        umma::mma_commit(&empty_kv[st]);
        if (last) umma::mma_commit(&q_free[h & 1]);
      };
      int g0 = 0;
      for (int h = 0; h < 8; ++h) {
        umma::mbar_wait(&q_ready[h & 1], (h >> 1) & 1);
        if (nch > 0) issue_s(g0, h, nch == 1);
        else umma::mbar_arrive(&q_free[h & 1]);
        for (int c = 0; c < nch; ++c) {
          // S of the next chunk first, so the rows never wait behind a value MMA
          if (c + 1 < nch) issue_s(g0 + c + 1, h, c + 2 == nch);
          value_mma(g0 + c, c, h);
        }
        if (nch > 0) {
          umma::mma_commit(acc_done);
        } else {  // empty tile: keep acc_done one phase ahead of the epilogue at most (parity waits)
          if (h > 0) umma::mbar_wait(epi_done, (h - 1) & 1);
          umma::mbar_arrive(acc_done);
        }
        g0 += nch;
      }
    }
  } else if (is_row) {
    // ================= query rows =================
    const int half = (warp - 2) >> 2;  // this warp's keys: [8 half, 8 half + 8) of every chunk
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    float* zx = reinterpret_cast<float*>(sm + SM_ZX);  // [2][128] softmax denominators of the two halves
    int g0 = 0;
    for (int h = 0; h < 8; ++h) {
      float mu = -INFINITY, z = 0.f;
      int rbase = 0;  // valid keys of the row in earlier chunks (rank -> slot for the score store)
      // this row's (chunk, key-mask) list, ascending chunk, 0xffff terminator
      const uint32_t* rl = rowlist + (size_t)(qin ? qi : 0) * a.K;
      int rp = 0;
      uint32_t ent = qin ? __ldg(rl) : 0xffff0000u;
      for (int c = 0; c < nch; ++c) {
        const int g = g0 + c, b = g & 1, st = g % NSTAGE;
        unsigned vmask = 0u;
        if ((int)(ent >> 16) == c) {
          vmask = ent & 0xffffu;
          ++rp;
          ent = rp < a.K ? __ldg(rl + rp) : 0xffff0000u;
        }
        umma::mbar_wait(&s_full[b], (g >> 1) & 1);
        TC_TRACE(tid == 64, g_trace[2][g]);
        umma::mbar_wait(&full_kv[st], (g / NSTAGE) & 1);  // key positions landed (already complete)
        umma::tc_fence_after();
        uint32_t sr[16];
        umma::tmem_ld16(t_s0 + 32 * b + lane_base, sr);
        umma::tc_fence_before();
        umma::mbar_arrive(&s_free[b]);
        // scores s = tau q.k + b(r): identical in both halves (same scores, same instructions)
        // (in place: sr[t] becomes the score bits -- no second 16-register array)
#define svv(t) __uint_as_float(sr[t])
#pragma unroll
        for (int t = 0; t < KC; ++t) sr[t] = __float_as_uint(a.tau * __uint_as_float(sr[t]));
        if constexpr (BIAS) {  // radial bias: r_ij from the staged positions (separate instantiation: registers)
          if (vmask) {
            const double* kpos = reinterpret_cast<const double*>(sm + SM_POS + st * PBYTES);
#pragma unroll
            for (int t = 0; t < KC; ++t)
              if (vmask >> t & 1) sr[t] = __float_as_uint(svv(t) + tc_pair_bias(a, kpos + 3 * t, qpos + 3 * row));
          }
        }
        if (SCORES && qvalid) {  // keep the scores of my half's valid keys
          const unsigned hmask = (vmask >> (8 * half)) & 0xffu;
          if (hmask) {
            const int* srow = a.slots + (size_t)qi * a.K;
#pragma unroll
            for (int t = 0; t < 8; ++t)
              if (hmask >> t & 1) {
                const int kk = 8 * half + t;
                const int rank = rbase + __popc(vmask & ((1u << kk) - 1u));  // ascending-j position of the key
                // rank space (the tensor-core backward maps slots through rank_of) or slot space
                const int col = a.score_rank ? rank : __ldg(srow + rank);
                // head-major [H][N][K]: a row's scores of one head fill whole sectors within one head pass
                a.scores[((size_t)h * a.N + qi) * a.K + col] = half ? svv(8 + t) : svv(t);  // static indices
              }
          }
        }
        if constexpr (SCORES) rbase += __popc(vmask);
        float mc = -INFINITY;
#pragma unroll
        for (int t = 0; t < KC; ++t)
          if (vmask >> t & 1) mc = fmaxf(mc, svv(t));
        const bool need = (mu > -INFINITY) && (mc > mu + 5.f);
        float factor = 1.f;
        if (mu == -INFINITY && mc > -INFINITY) mu = mc;
        else if (need) { factor = __expf(mu - mc); mu = mc; z *= factor; }
        if (half == 0 && __any_sync(0xffffffffu, need)) {
          // O must be quiescent: every value MMA up to chunk c-1 complete (c >= 1 here)
          umma::mbar_wait(&wv_free[(g - 1) & 1], ((g - 1) >> 1) & 1);
          umma::tc_fence_after();
#pragma unroll
          for (int cc = 0; cc < NV / 16; ++cc) {
            uint32_t r[16];
            umma::tmem_ld16(t_out + lane_base + cc * 16, r);
#pragma unroll
            for (int t = 0; t < 16; ++t) r[t] = __float_as_uint(__uint_as_float(r[t]) * factor);
            umma::tmem_st16(t_out + lane_base + cc * 16, r);
          }
          umma::tc_fence_before();
        }
        const unsigned hm = (vmask >> (8 * half)) & 0xffu;  // my 8 keys
        float pw[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float sv = half ? svv(8 + t) : svv(t);
          pw[t] = (hm >> t & 1) ? __expf(sv - mu) : 0.f;
          z += pw[t];
        }
#undef svv
        // ---- phase 1 (row-bound): P row -> smem, zero my half of the Wt row,
        // per-row valid masks + quadrant-local prefix counts (half 0)
        const int pb = g & 1;  // phase-2 tables double buffered by chunk parity
        float* prow = reinterpret_cast<float*>(sm + SM_PROW) + pb * TQ * KC;
        int* qtot = reinterpret_cast<int*>(sm + SM_QTOT) + pb * 4;
        float4* pdst = reinterpret_cast<float4*>(prow + row * KC + 8 * half);
        pdst[0] = make_float4(pw[0], pw[1], pw[2], pw[3]);
        pdst[1] = make_float4(pw[4], pw[5], pw[6], pw[7]);
        if (half == 0) {
          const unsigned gm = (a.dbg & 2) ? 0u : vmask;
          const int cnt = __popc(gm);
          int incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          // this row's valid pairs, compacted into its quadrant's list
          uint16_t* pairs = reinterpret_cast<uint16_t*>(sm + SM_PAIRS) + pb * TQ * KC + (warp & 3) * 32 * KC;
          unsigned m = gm;
          int o = incl - cnt;
          while (m) {
            const int kk = __ffs(m) - 1;
            m &= m - 1;
            pairs[o++] = (uint16_t)((row << 4) | kk);
          }
          if (lane == 31) qtot[warp & 3] = incl;
        }
        TC_TRACE(tid == 64, g_trace_r[0][g] );
        if (g >= 2) umma::mbar_wait(&wv_free[b], ((g >> 1) - 1) & 1);  // Wt buffer b free
        TC_TRACE(tid == 64, g_trace_r[1][g] );
        uint8_t* wt = sm + SM_WT + b * WBYTES;
#pragma unroll
        for (int f = 0; f < MM; ++f)
          *reinterpret_cast<uint4*>(wt + cm_off(row, f * KC + 8 * half)) = make_uint4(0, 0, 0, 0);
        umma::named_bar(2, 256);
        TC_TRACE(tid == 64, g_trace_r[2][g] );
        // ---- phase 2 (balanced): the chunk's valid (row, key) pairs of the whole
        // tile are dealt round-robin to the 256 row threads (the pairs of a
        // molecule-sized chunk cluster in one quadrant; this spreads them)
        {
          const int q0n = qtot[0], q1n = q0n + qtot[1], q2n = q1n + qtot[2], total = q2n + qtot[3];
          const int rt = tid - 64;  // 0..255
          const double* kpos = reinterpret_cast<const double*>(sm + SM_POS + st * PBYTES);
#pragma unroll 1
          for (int p = rt; p < total; p += 256) {
            const int qd = (p >= q0n) + (p >= q1n) + (p >= q2n);
            const int local = p - (qd == 0 ? 0 : qd == 1 ? q0n : qd == 2 ? q1n : q2n);
            const int e = reinterpret_cast<const uint16_t*>(sm + SM_PAIRS)[pb * TQ * KC + qd * 32 * KC + local];
            const int orow = e >> 4, kk = e & 15;
            double dx = kpos[3 * kk] - qpos[3 * orow], dy = kpos[3 * kk + 1] - qpos[3 * orow + 1],
                   dz = kpos[3 * kk + 2] - qpos[3 * orow + 2];
            if (a.periodic) {
              dx -= a.bx * rint(dx / a.bx);
              dy -= a.by * rint(dy / a.by);
              dz -= a.bz * rint(dz / a.bz);
            }
            const float rx = (float)dx, ry = (float)dy, rz = (float)dz;
            const float rn = sqrtf(rx * rx + ry * ry + rz * rz);
            float phi = 1.f;
            // cutoff by the SFU cosine (|err| < 4e-7 on [0, pi]): cospif's range reduction is ~30
            // dependent instructions on this per-pair, per-head path
            if (a.phi_mode == 0) phi = rn < a.r_cut ? 0.5f * (__cosf(3.14159265358979f * rn * a.inv_rcut) + 1.f) : 0.f;
            float y[MM];
            solid_l2(rx, ry, rz, y);
            const float pp = prow[orow * KC + kk] * phi;
#pragma unroll
            for (int f = 0; f < MM; ++f)
              *reinterpret_cast<bf16*>(wt + cm_off(orow, f * KC + kk)) = __float2bfloat16_rn(pp * y[f]);
          }
        }
        umma::fence_proxy_async();
        umma::mbar_arrive(&wt_full[b]);
        TC_TRACE(tid == 64, g_trace[3][g]);
        TC_TRACE(lane == 0, g_trace_w[warp - 2][g] );
        umma::mbar_arrive(&empty_kv[st]);  // done with this stage's key positions
      }
      // ---- epilogue: O_h / z, the two halves each store half of the columns
      zx[half * TQ + row] = z;
      umma::named_bar(2, 256);
      const float zt = zx[row] + zx[TQ + row];
      umma::named_bar(2, 256);  // zx reusable by the next head
      umma::mbar_wait(acc_done, h & 1);
      umma::tc_fence_after();
      const float inv = zt > 0.f ? 1.f / zt : 0.f;
      if (qvalid && half == 0) lse[(size_t)qi * 8 + h] = zt > 0.f ? mu + __logf(zt) : -INFINITY;
      const int cc0 = half ? 5 : 0, cc1 = (a.dbg & 32) ? cc0 : half ? NV / 16 : 5;  // 32: no epilogue (profiling)
      for (int cc = cc0; cc < cc1; ++cc) {
        uint32_t r[16];
        if (nch > 0) umma::tmem_ld16(t_out + lane_base + cc * 16, r);
        float v[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) v[t] = nch > 0 ? __uint_as_float(r[t]) * inv : 0.f;
        if (qvalid) {
          uint4* dst = reinterpret_cast<uint4*>(out + ((size_t)qi * MM + cc) * 128 + HD * h);
          dst[0] = pack8(v);
          dst[1] = pack8(v + 8);
        }
      }
      umma::tc_fence_before();
      umma::mbar_arrive(epi_done);
      g0 += nch;
    }
  } else {
    // ================= per-key source coupling (warps 10-13) =================
    const int vt_id = tid - 320;
    const int vc = vt_id & 15, vjp = vt_id >> 4;  // channel, key pair (2 vjp, 2 vjp + 1)
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const bf16* qrow = q + (size_t)(qin ? qi : 0) * MM * 256;
    auto load_q = [&](int hh) {  // Q_hh row -> TMEM buffer hh&1 (A operand, packed bf16 pairs)
      const uint32_t tq = t_q0 + 144 * (hh & 1);
#pragma unroll
      for (int m0 = 0; m0 < MM; m0 += 3) {
        uint32_t r[3][16];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const uint4* src = reinterpret_cast<const uint4*>(qrow + (m0 + d) * 256 + DH * hh);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const uint4 u = qin ? __ldg(src + t) : make_uint4(0, 0, 0, 0);
            r[d][4 * t] = u.x; r[d][4 * t + 1] = u.y; r[d][4 * t + 2] = u.z; r[d][4 * t + 3] = u.w;
          }
        }
#pragma unroll
        for (int d = 0; d < 3; ++d) umma::tmem_st16(tq + lane_base + 16 * (m0 + d), r[d]);
      }
      umma::tc_fence_before();
      umma::mbar_arrive(&q_ready[hh & 1]);
    };
    load_q(0);
    int g0 = 0;
    for (int h = 0; h < 8; ++h) {
      if (h + 1 < 8) {
        if (h >= 1) umma::mbar_wait(&q_free[(h + 1) & 1], ((h - 1) >> 1) & 1);  // head h-1's S MMAs done
        load_q(h + 1);
      }
      for (int c = 0; c < nch; ++c) {
        const int g = g0 + c, b = g & 1, st = g % NSTAGE;
        umma::mbar_wait(&full_kv[st], (g / NSTAGE) & 1);
        TC_TRACE(vt_id == 0, g_trace[4][g]);
        // v_j[i'][c] of this thread's channel and two keys, read straight from the
        // TMA stage ([key][i'][16 c] bf16; lanes = consecutive channels)
        const unsigned short* vst = reinterpret_cast<const unsigned short*>(sm + SM_VST + st * VBYTES);
        float v2[MM][2];
#pragma unroll
        for (int ip = 0; ip < MM; ++ip) {
#pragma unroll
          for (int t = 0; t < 2; ++t)
            v2[ip][t] = __uint_as_float((uint32_t)vst[((2 * vjp + t) * MM + ip) * HD + vc] << 16);
        }
        umma::mbar_arrive(&empty_kv[st]);  // V stage consumed (every Vg thread arrives)
        if (g >= 2) umma::mbar_wait(&wv_free[b], ((g >> 1) - 1) & 1);  // Vg buffer b free
        uint8_t* vg = sm + SM_VG + b * GBYTES;
        // Vg[(f, j), (o, c)] for this thread's (c, 2 keys), all o: one straight-line code path
        // shared by the four warps (keeps the kernel's hot code small for the instruction cache)
        es_vg_all(v2, [&](int o, int f, float x0, float x1) {
          const __nv_bfloat162 pk = __floats2bfloat162_rn(x0, x1);
          *reinterpret_cast<uint32_t*>(vg + cm_off(o * HD + vc, f * KC + 2 * vjp)) =
              *reinterpret_cast<const uint32_t*>(&pk);
        });
        umma::fence_proxy_async();
        umma::mbar_arrive(&vg_full[b]);
        TC_TRACE(vt_id == 0, g_trace[5][g]);
      }
      g0 += nch;
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, 512);
#ifdef ES_TC_TRACE
  if (TRACE && tid == 0) {
    for (int g = 0; g < 128 && g < 8 * nch; ++g)
      printf("TRACE g=%d tma=%lld sI=%lld sR=%lld wt=%lld vgS=%lld vgD=%lld vI=%lld pw=%lld\n", g, g_trace[0][g],
             g_trace[1][g], g_trace[2][g], g_trace[3][g], g_trace[4][g], g_trace[5][g], g_trace[6][g], g_trace[7][g]);
    for (int g = 0; g < 128 && g < 8 * nch; ++g)
      printf("TRACEW g=%d %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld\n", g, g_trace_r[0][g], g_trace_r[1][g], g_trace_r[2][g], g_trace_w[0][g], g_trace_w[1][g],
             g_trace_w[2][g], g_trace_w[3][g], g_trace_w[4][g], g_trace_w[5][g], g_trace_w[6][g], g_trace_w[7][g]);
  }
#endif
}

// ---------------------------------------------------------------- tile chunk lists
__global__ void tc_count_kernel(int ntiles, int words, const uint32_t* __restrict__ mask, int* __restrict__ cnt) {
  const int t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (t >= ntiles) return;
  int c = 0;
  for (int w = lane; w < words; w += 32) c += __popc(mask[(size_t)t * words + w]);
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[t] = c;
}

__global__ void tc_fill_kernel(int ntiles, int words, const uint32_t* __restrict__ mask, const int* __restrict__ ptr,
                               int* __restrict__ list) {
  const int t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (t >= ntiles) return;
  int base = ptr[t];
  for (int w0 = 0; w0 < words; w0 += 32) {
    const int w = w0 + lane;
    const uint32_t m = w < words ? mask[(size_t)t * words + w] : 0u;
    const int c = __popc(m);
    int incl = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int pos = base + incl - c;
    uint32_t mm = m;
    while (mm) {
      const int b = __ffs(mm) - 1;
      list[pos++] = w * 32 + b;
      mm &= mm - 1;
    }
    base += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// Per query row: its valid neighbours folded into (tile chunk index << 16 | 16-bit key
// mask) entries, ascending chunk index, terminated by 0xffff0000 (the row-level
// tile-skip mask the attention kernels walk chunk by chunk); optionally the
// row's neighbour slots in the same (ascending j) order, for the dq kernel's
// dscore gathers.
__global__ void tc_rowlist_kernel(int N, int K, const int* __restrict__ nbr, const int* __restrict__ cptr,
                                  const int* __restrict__ clist, const int* __restrict__ rtile,
                                  uint32_t* __restrict__ rl, int* __restrict__ slots, int* __restrict__ rank_of) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int t = rtile[i], lo = cptr[t], n = cptr[t + 1] - lo;
  uint32_t* o = rl + (size_t)i * K;
  int cnt = 0, nv = 0;
  for (int s = 0; s < K; ++s) {
    const int j = nbr[(size_t)i * K + s];
    if (j < 0) continue;
    if (slots) {  // the row's slots in ascending-j order (= the (chunk, key-bit) order of the list)
      int* so = slots + (size_t)i * K;
      int p = nv++;
      while (p > 0 && nbr[(size_t)i * K + so[p - 1]] > j) { so[p] = so[p - 1]; --p; }
      so[p] = s;
    }
    const int kb = j / KC;
    int a = 0, b = n;
    while (a < b) {
      const int m = (a + b) >> 1;
      if (clist[lo + m] < kb) a = m + 1;
      else b = m;
    }
    const uint32_t key = (uint32_t)a << 16, bit = 1u << (j % KC);
    bool merged = false;
    for (int u = 0; u < cnt; ++u)
      if ((o[u] & 0xffff0000u) == key) { o[u] |= bit; merged = true; break; }
    if (!merged) {
      int p = cnt++;
      while (p > 0 && o[p - 1] > key) { o[p] = o[p - 1]; --p; }
      o[p] = key | bit;
    }
  }
  if (cnt < K) o[cnt] = 0xffff0000u;
  if (slots && rank_of)
    for (int r = 0; r < nv; ++r) rank_of[(size_t)i * K + slots[(size_t)i * K + r]] = r;
}

// Warp-per-row list builder for K <= 64 (two slots per lane): each valid
// slot finds its chunk's index in the tile list (binary search); the row's
// distinct chunks are then emitted in ascending order, one warp min-reduce
// (next chunk) and one OR-reduce (its 16-bit key mask) per entry -- a row
// touches a handful of chunks, so this replaces a 64-key sort.  A slot's
// position in the ascending-j slot order is the valid keys in earlier
// chunks plus the key bits below its own.
__global__ void tc_rowlist_warp_kernel(int N, int K, const int* __restrict__ nbr, const int* __restrict__ cptr,
                                       const int* __restrict__ clist, const int* __restrict__ rtile,
                                       uint32_t* __restrict__ rl, int* __restrict__ slots,
                                       int* __restrict__ rank_of) {
  const int i = (int)(((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= N) return;
  const int t = rtile[i], lo = cptr[t], n = cptr[t + 1] - lo;
  constexpr int NONE = 0x7fffffff;
  int ci[2];
  unsigned bit[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int s = lane + 32 * u;
    const int j = s < K ? __ldg(nbr + (size_t)i * K + s) : -1;
    ci[u] = NONE;
    bit[u] = 0u;
    if (j >= 0) {
      const int kb = j / KC;
      int a = 0, b = n;
      while (a < b) {
        const int m = (a + b) >> 1;
        if (clist[lo + m] < kb) a = m + 1;
        else b = m;
      }
      ci[u] = a;
      bit[u] = 1u << (j % KC);
    }
  }
  uint32_t* o = rl + (size_t)i * K;
  int nent = 0, before = 0;
  for (;;) {
    const int c = __reduce_min_sync(0xffffffffu, min(ci[0], ci[1]));
    if (c == NONE) break;
    const unsigned m = __reduce_or_sync(0xffffffffu, (ci[0] == c ? bit[0] : 0u) | (ci[1] == c ? bit[1] : 0u));
    if (lane == 0) o[nent] = ((uint32_t)c << 16) | m;
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (ci[u] == c) {
        if (slots) {
          const int r = before + __popc(m & (bit[u] - 1u));
          slots[(size_t)i * K + r] = lane + 32 * u;
          if (rank_of) rank_of[(size_t)i * K + lane + 32 * u] = r;  // slot -> rank (ascending-j position)
        }
        ci[u] = NONE;
      }
    ++nent;
    before += __popc(m);
  }
  if (lane == 0 && nent < K) o[nent] = 0xffff0000u;
}

// Query tiles.  Uniform: TQ consecutive rows.  Segment-packed (molecule
// batches): whole segments greedily packed up to TQ rows (a segment longer
// than TQ is split at TQ-row boundaries).  The greedy scan is sequential, so
// the segment list is cut into at most tc_pack_parts(N) parts of consecutive
// segments, each packed by one thread starting a fresh tile (a part costs at
// most one under-full tile); a block scan of the per-part tile counts places
// them.  Tiles past the last start at N (empty CTAs exit).
__host__ __device__ inline int tc_pack_parts(int N) { return min(1024, ((N + TQ - 1) / TQ) / 32 + 1); }

__global__ void tc_tiles_uniform_kernel(int N, int ntiles, int* __restrict__ tstart) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t <= ntiles) tstart[t] = min(N, t * TQ);
}

// greedy packing of segments [s0, s1) starting a tile at seg[s0]; emit(row)
// is called for every tile start
template <class F>
__device__ __forceinline__ int tc_pack_part(const int* __restrict__ seg, int s0, int s1, int N, F emit) {
  int nt = 0;
  if (s0 >= s1) return 0;
  int cur = s0 == 0 ? 0 : min(N, max(0, seg[s0]));  // the first tile starts at row 0
  emit(nt++, cur);
  int lo = cur;
  for (int x = s0; x < s1; ++x) {
    const int hi = min(N, max(lo, seg[x + 1]));
    if (hi - cur > TQ && lo > cur) {  // the segment does not fit: close the tile before it
      cur = lo;
      emit(nt++, cur);
    }
    while (hi - cur > TQ) {  // segment longer than a tile: split it
      cur += TQ;
      emit(nt++, cur);
    }
    lo = hi;
  }
  return nt;
}

__global__ void __launch_bounds__(1024) tc_tiles_packed_kernel(int N, int nseg, const int* __restrict__ seg,
                                                                int ntiles, int* __restrict__ tstart) {
  __shared__ int off[1025];
  const int parts = tc_pack_parts(N), G = (nseg + parts - 1) / parts;
  const int p = threadIdx.x;
  const int s0 = min(nseg, p * G), s1 = min(nseg, s0 + G);
  const int cnt = p < parts ? tc_pack_part(seg, s0, s1, N, [](int, int) {}) : 0;
  // block exclusive scan of the per-part tile counts
  off[p + 1] = cnt;
  if (p == 0) off[0] = 0;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {
    const int v = p + 1 >= d + 1 ? off[p + 1 - d] : 0;
    __syncthreads();
    off[p + 1] += v;
    __syncthreads();
  }
  const int base = off[p], total = min(ntiles, off[1024]);
  if (p < parts)
    tc_pack_part(seg, s0, s1, N, [&](int t, int row) {
      if (base + t < ntiles) tstart[base + t] = row;
    });
  for (int t = total + p; t <= ntiles; t += blockDim.x) tstart[t] = N;
}
__global__ void tc_rowtile_kernel(int ntiles, const int* __restrict__ tstart, int* __restrict__ rtile) {
  const int t = blockIdx.x;
  if (t >= ntiles) return;
  const int a = tstart[t], b = tstart[t + 1];
  for (int r = a + threadIdx.x; r < b; r += blockDim.x) rtile[r] = t;
}
// tile-skip mask: bit kb of tile t set iff a row of t has a key in chunk kb.
// vec (K % 4 == 0, 16-byte aligned table): four slots of one row per thread
// (one 16-byte load), bits of the same mask word OR-ed before the atomic.
__global__ void tc_mask_kernel(int N, int K, const int32_t* __restrict__ nbr, const int* __restrict__ rtile,
                               int words, uint32_t* __restrict__ mask, bool vec) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    if (t * 4 >= (size_t)N * K) return;
    const int4 jv = __ldg(reinterpret_cast<const int4*>(nbr) + t);
    const int js[4] = {jv.x, jv.y, jv.z, jv.w};
    if (js[0] < 0 && js[1] < 0 && js[2] < 0 && js[3] < 0) return;
    uint32_t* row = mask + (size_t)rtile[t * 4 / K] * words;
    int w = -1;
    uint32_t acc = 0u;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (js[e] < 0) continue;
      const int kb = js[e] / KC;
      if (kb / 32 != w) {
        if (acc) atomicOr(row + w, acc);
        w = kb / 32;
        acc = 0u;
      }
      acc |= 1u << (kb % 32);
    }
    if (acc) atomicOr(row + w, acc);
    return;
  }
  if (t >= (size_t)N * K) return;
  const int j = nbr[t];
  if (j < 0) return;
  const int kb = j / KC;
  atomicOr(&mask[(size_t)rtile[t / K] * words + kb / 32], 1u << (kb % 32));
}

// ---------------------------------------------------------------- key-side lists (dk pass)
// The transposed relation tiled the other way round: key tiles (rows = key
// atoms), 16-query chunks.  Mask bit (key tile, query chunk) from the forward
// table; per-key (chunk index << 16 | 16-bit query mask) entries from the
// key's ascending rev_pair segment, stored CSR at rev_ptr[j] (a key has at
// most as many entries as queries), terminated by 0xffff0000 when shorter.
__global__ void tc_maskT_kernel(int N, int K, const int32_t* __restrict__ nbr, const int* __restrict__ rtileT,
                                int words, uint32_t* __restrict__ mask) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (size_t)N * K) return;
  const int j = nbr[t];
  if (j < 0) return;
  const int qc = (int)(t / K) / KC;
  atomicOr(&mask[(size_t)rtileT[j] * words + qc / 32], 1u << (qc % 32));
}

__global__ void tc_rowlistT_kernel(int Nk, int K, const int* __restrict__ rev_ptr, const int* __restrict__ rev_pair,
                                   const int* __restrict__ cptr, const int* __restrict__ clist,
                                   const int* __restrict__ rtileT, uint32_t* __restrict__ rl) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= Nk) return;
  const int t = rtileT[j], lo = cptr[t], n = cptr[t + 1] - lo;
  const int e0 = rev_ptr[j], e1 = rev_ptr[j + 1];
  auto idx = [&](int qc) {
    int a = 0, b = n;
    while (a < b) {
      const int m = (a + b) >> 1;
      if (clist[lo + m] < qc) a = m + 1;
      else b = m;
    }
    return a;
  };
  int u = 0, cur = -1;
  uint32_t msk = 0u;
  for (int e = e0; e < e1; ++e) {
    const int i = rev_pair[e] / K, qc = i / KC;
    if (qc != cur) {
      if (cur >= 0) rl[e0 + u++] = ((uint32_t)idx(cur) << 16) | msk;
      cur = qc;
      msk = 0u;
    }
    msk |= 1u << (i % KC);
  }
  if (cur >= 0) rl[e0 + u++] = ((uint32_t)idx(cur) << 16) | msk;
  if (e0 + u < e1) rl[e0 + u] = 0xffff0000u;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}
bool map3(CUtensorMap* m, const void* base, int inner, int mid, int outer, int b0, int b1, int b2,
          CUtensorMapSwizzle sw) {
  EncodeTiledFn f = encode_fn();
  if (!f) return false;
  cuuint64_t gd[3] = {(cuuint64_t)inner, (cuuint64_t)mid, (cuuint64_t)outer};
  cuuint64_t gs[2] = {(cuuint64_t)inner * 2, (cuuint64_t)inner * mid * 2};
  cuuint32_t bd[3] = {(cuuint32_t)b0, (cuuint32_t)b1, (cuuint32_t)b2};
  cuuint32_t es_[3] = {1, 1, 1};
  return f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), gd, gs, bd, es_,
           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The same [outer][mid][inner] bf16 tensor with the mid and outer dimensions swapped, so one
// box {b_inner, b_outer rows, b_mid} lands as b_mid consecutive [b_outer][b_inner] blocks --
// e.g. a 16-atom chunk of all nine (l,m) rows of one head in a single TMA instead of nine.
bool map3t(CUtensorMap* m, const void* base, int inner, int mid, int outer, int b_inner, int b_outer, int b_mid,
           CUtensorMapSwizzle sw) {
  EncodeTiledFn f = encode_fn();
  if (!f) return false;
  cuuint64_t gd[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)mid};
  cuuint64_t gs[2] = {(cuuint64_t)inner * mid * 2, (cuuint64_t)inner * 2};
  cuuint32_t bd[3] = {(cuuint32_t)b_inner, (cuuint32_t)b_outer, (cuuint32_t)b_mid};
  cuuint32_t es_[3] = {1, 1, 1};
  return f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), gd, gs, bd, es_,
           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

es_status upload_tc_tables() {
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && done[dev]) return ES_OK;
  TcTab t;
  t.ycoef[0] = 0.28209479177387814f;
  t.ycoef[1] = (float)std::sqrt(3.0 / (4.0 * M_PI));
  t.ycoef[2] = (float)std::sqrt(15.0 / (4.0 * M_PI));
  t.ycoef[3] = (float)std::sqrt(5.0 / (4.0 * M_PI));
  // G_f[o, i'] for the path set of L = 2 (every degree <= 2), grouped by (o, f)
  int n = 0;
  for (int o = 0; o < MM; ++o)
    for (int f = 0; f < MM; ++f) {
      t.ofs[o * MM + f] = n;
      const int lo = o < 1 ? 0 : (o < 4 ? 1 : 2), mo = o - lo * lo - lo;
      const int lf = f < 1 ? 0 : (f < 4 ? 1 : 2), mf = f - lf * lf - lf;
      for (int ip = 0; ip < MM; ++ip) {
        const int li = ip < 1 ? 0 : (ip < 4 ? 1 : 2), mi = ip - li * li - li;
        const double c = real_cg(li, mi, lf, mf, lo, mo);
        if (std::fabs(c) > 1e-12) {
          if (n >= 160) return fail(ES_CUDA_ERROR, "attn_tc: CG table overflow");
          t.ent_i[n] = (unsigned char)ip;
          t.ent_c[n] = (float)c;
          ++n;
        }
      }
    }
  t.ofs[MM * MM] = n;
  const cudaError_t e = cudaMemcpyToSymbol(c_tc, &t, sizeof(t));
  if (e != cudaSuccess) return cuda_status(e, "attn_tc tables");
  if (dev < 64) done[dev] = true;
  return ES_OK;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

bool attn_tc_supported(const AttnArgs& a) {
  return a.dtype == ES_BF16 && a.value_mode == ES_VALUE_EAAS && a.L == 2 && a.C == 128 && a.H == 8 &&
         a.K <= 511 && encode_fn() != nullptr;
}

namespace {
struct TcScratch {
  int ntiles, nkb, words;  // ntiles: upper bound (segment-packed tiles are fewer)
  size_t chunks, cub_bytes, total, pairs;
};
// Query tiles are uniform TQ-row blocks, or -- with segments (molecule
// batches) -- whole segments greedily packed up to TQ rows, so a tile's key
// chunks cover only its own molecules.  Greedy packing closes a tile only
// when the next segment does not fit, so two consecutive tiles of one part
// hold > TQ rows: a part of R rows packs into <= 2 ceil(R / TQ) tiles, and
// 2 ceil(N / TQ) + 2 parts + 1 bounds the tile count of both schemes (the
// layout does not depend on which one built the buffer; surplus tiles are
// empty).
TcScratch tc_scratch(const AttnArgs& a) {
  TcScratch t;
  t.ntiles = 2 * ((a.N + TQ - 1) / TQ) + 2 * tc_pack_parts(a.N) + 1;
  t.nkb = (a.Nk + KC - 1) / KC;
  t.words = (t.nkb + 31) / 32;
  // a tile's chunk list is at most min(nkb, its valid pairs) long: the packed
  // lists of all tiles fit min(ntiles * nkb, N * K) entries
  const size_t dense = (size_t)t.ntiles * t.nkb, pairs = (size_t)a.N * a.K;
  t.pairs = pairs;
  t.chunks = dense < pairs ? dense : pairs;
  t.cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t.cub_bytes, (int*)nullptr, (int*)nullptr, t.ntiles + 1);
  t.total = align256((size_t)t.ntiles * t.words * 4) + 2 * align256((size_t)(t.ntiles + 1) * 4) +
            align256(t.chunks * 4) + align256(t.cub_bytes) + align256(pairs * 4) +
            align256((size_t)(t.ntiles + 1) * 4) + align256((size_t)a.N * 4);
  return t;
}
}  // namespace

size_t attn_fwd_tc_workspace(const AttnArgs& a) {
  return a.N > 0 ? tc_scratch(a).total + 2 * align256((size_t)a.N * a.K * 4) : 0;  // + slots, rank_of (score store)
}

namespace {
struct TcLists {
  const int* cptr;
  const int* clist;
  const uint32_t* rowlist;
  int ntiles;
  const int* tstart;  // [ntiles + 1] first query row of each tile (N past the last)
};
// the list arrays inside a tile / workspace buffer laid out by tc_scratch
struct TcPtrs {
  uint32_t* mask;
  int *cnt, *cptr, *clist;
  void* cub;
  uint32_t* rowlist;
  int* tstart;  // [ntiles + 1]
  int* rtile;   // [N] tile of each query row
  int* slots;    // only when the buffer holds them (tile buffers do)
  int* rank_of;  // [N*K] slot -> position in the row's ascending-j order (after slots)
};
TcPtrs tc_ptrs(void* base_, const TcScratch& t) {
  char* base = static_cast<char*>(base_);
  TcPtrs p;
  const int ntiles = t.ntiles, words = t.words;
  p.mask = (uint32_t*)base;
  size_t off = align256((size_t)ntiles * words * 4);
  p.cnt = (int*)(base + off);
  off += align256((size_t)(ntiles + 1) * 4);
  p.cptr = (int*)(base + off);
  off += align256((size_t)(ntiles + 1) * 4);
  p.clist = (int*)(base + off);
  off += align256(t.chunks * 4);
  p.cub = base + off;
  off += align256(t.cub_bytes);
  p.rowlist = (uint32_t*)(base + off);
  off += align256(t.pairs * 4);
  p.tstart = (int*)(base + off);
  off += align256((size_t)(ntiles + 1) * 4);
  p.rtile = (int*)(base + off);
  p.slots = (int*)(base + t.total);
  p.rank_of = (int*)(base + t.total + align256(t.pairs * 4));
  return p;
}

// tile-skip mask -> per-tile key-chunk lists -> per-row (chunk, key mask) lists
es_status tc_build_lists(const AttnArgs& a, const int32_t* nbr, void* ws, const TcScratch& t, int* slots,
                         TcLists* out, cudaStream_t st, const int32_t* seg = nullptr, int nseg = 0) {
  const int ntiles = t.ntiles, words = t.words;
  size_t cub_bytes = t.cub_bytes;
  const TcPtrs pp = tc_ptrs(ws, t);
  uint32_t* mask = pp.mask;
  int* cnt = pp.cnt;
  int* cptr = pp.cptr;
  int* clist = pp.clist;
  void* cub_ws = pp.cub;
  uint32_t* rowlist = pp.rowlist;
  if (seg && nseg > 0) tc_tiles_packed_kernel<<<1, 1024, 0, st>>>(a.N, nseg, seg, ntiles, pp.tstart);
  else tc_tiles_uniform_kernel<<<(ntiles + 256) / 256, 256, 0, st>>>(a.N, ntiles, pp.tstart);
  tc_rowtile_kernel<<<ntiles, 128, 0, st>>>(ntiles, pp.tstart, pp.rtile);
  cudaMemsetAsync(mask, 0, (size_t)ntiles * words * 4, st);
  cudaMemsetAsync(cnt, 0, (size_t)(ntiles + 1) * 4, st);
  {
    const size_t n = (size_t)a.N * a.K;
    const bool vec = (a.K & 3) == 0 && ((uintptr_t)nbr & 15) == 0;
    const size_t nt = vec ? n / 4 : n;
    tc_mask_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(a.N, a.K, nbr, pp.rtile, words, mask, vec);
  }
  tc_count_kernel<<<(ntiles + 7) / 8, 256, 0, st>>>(ntiles, words, mask, cnt);
  cudaError_t e = cub::DeviceScan::ExclusiveSum(cub_ws, cub_bytes, cnt, cptr, ntiles + 1, st);
  if (e != cudaSuccess) return cuda_status(e, "attn_tc scan");
  tc_fill_kernel<<<(ntiles + 7) / 8, 256, 0, st>>>(ntiles, words, mask, cptr, clist);
  // rank_of lives right after the slots (tile buffers and the workspaces that hold slots)
  int* rank_of = slots ? (int*)((char*)slots + align256(t.pairs * 4)) : nullptr;
  if (a.K <= 64)
    tc_rowlist_warp_kernel<<<(unsigned)(((size_t)a.N * 32 + 255) / 256), 256, 0, st>>>(a.N, a.K, nbr, cptr, clist,
                                                                                     pp.rtile, rowlist, slots, rank_of);
  else
    tc_rowlist_kernel<<<(a.N + 127) / 128, 128, 0, st>>>(a.N, a.K, nbr, cptr, clist, pp.rtile, rowlist, slots,
                                                         rank_of);
  *out = TcLists{cptr, clist, rowlist, ntiles, pp.tstart};
  return cuda_status(cudaGetLastError(), "attn_tc lists");
}
}  // namespace

// Scratch (tile mask, chunk lists, per-row chunk lists) lives in the caller's
// workspace (es_attn_fwd_workspace_size): no allocation on the launch path.
es_status attn_fwd_tc_launch(const AttnArgs& a, const void* q, const void* k, const void* v, const double* pos,
                             const int32_t* nbr, void* out, float* lse, void* ws, size_t ws_bytes,
                             cudaStream_t st) {
  es_status s = upload_tc_tables();
  if (s != ES_OK) return s;
  if (a.N == 0) return ES_OK;
  const TcScratch t = tc_scratch(a);
  TcLists lists;
  const int* slots = nullptr;
  if (a.tiles) {  // lists prebuilt for this neighbour index (es_attn_tiles_build)
    const TcPtrs pp = tc_ptrs(const_cast<void*>(a.tiles), t);
    lists = TcLists{pp.cptr, pp.clist, pp.rowlist, t.ntiles, pp.tstart};
    slots = pp.slots;
  } else {
    if (!ws || ws_bytes < attn_fwd_tc_workspace(a)) return fail(ES_INVALID_ARGUMENT, "attn_fwd: workspace too small");
    int* sl = a.scores_out ? (int*)((char*)ws + t.total) : nullptr;
    s = tc_build_lists(a, nbr, ws, t, sl, &lists, st);
    if (s != ES_OK) return s;
    slots = sl;
  }
  const int ntiles = lists.ntiles;
  const int* cptr = lists.cptr;
  const int* clist = lists.clist;
  const uint32_t* rowlist = lists.rowlist;

  CUtensorMap mk, mv;
  if (!map3t(&mk, k, 256, MM, a.Nk, DH, KC, MM, CU_TENSOR_MAP_SWIZZLE_64B) ||
      !map3(&mv, v, 128, MM, a.Nk, HD, MM, KC, CU_TENSOR_MAP_SWIZZLE_NONE))
    return fail(ES_CUDA_ERROR, "attn_fwd_tc: tensor map encode failed");
  TcArgs ta;
  ta.N = a.N; ta.K = a.K; ta.row0 = a.row0; ta.Nk = a.Nk;
  {
    const char* e = getenv("ES_TC_DBG");
    ta.dbg = e ? atoi(e) : 0;
  } ta.tau = a.tau; ta.r_cut = a.r_cut; ta.inv_rcut = 1.f / a.r_cut;
  ta.phi_mode = a.phi_mode; ta.periodic = a.periodic;
  ta.bx = a.box[0]; ta.by = a.box[1]; ta.bz = a.box[2];
  ta.bias_mode = a.bias_mode; ta.b0 = a.bias[0]; ta.b1 = a.bias[1]; ta.b2 = a.bias[2];
  ta.scores = a.scores_out;
  ta.slots = slots;
  ta.score_rank = attn_dq_tc_applicable(a) ? 1 : 0;
  const int smem = SM_TOTAL + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_fwd_tc_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(attn_fwd_tc_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(attn_fwd_tc_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(attn_fwd_tc_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  // bias and score store are separate instantiations: the default kernel carries neither
  auto kfn = a.bias_mode ? (ta.scores ? attn_fwd_tc_kernel<true, true> : attn_fwd_tc_kernel<true, false>)
                         : (ta.scores ? attn_fwd_tc_kernel<false, true> : attn_fwd_tc_kernel<false, false>);
  kfn<<<ntiles, TC_THREADS, smem, st>>>(mk, mv, ta, (const bf16*)q, pos, nbr, cptr, clist, rowlist,
                                                        lists.tstart, (bf16*)out, lse);
  return cuda_status(cudaGetLastError(), "attn_fwd_tc_kernel");
}


// ---------------------------------------------------------------- dq on the tensor cores
// dq_i^h = tau sum_j dS_ij^h k_j^h over the same 128-query tiles and 16-key
// chunks as the forward: per chunk one tcgen05 MMA group
//   D[128 queries, 288] += A[128, 16 keys] . B[16 keys, 288]
// with A = the chunk's dscore tile (bf16, built by the row warps from the
// backward's per-pair dscore buffer; zeros for non-neighbours) and B = the
// TMA-staged K chunk read MN-major (the 64-byte-swizzled [16 keys][32 ch]
// boxes of the forward's S MMA are exactly the MN-major SW64 atoms).
namespace {
constexpr int DQ_THREADS = 448;  // warp 0 TMA, warp 1 MMA, warps 2-5 rows (dscore tiles), warps 6-13 epilogue
constexpr int DQ_ABYTES = TQ * KC * 2;  // 4096: [128 rows][16 keys] bf16, no-swizzle core matrices
constexpr int DQ_SM_K = 0;
constexpr int DQ_NSTAGE = 8;  // deep K pipeline: per-chunk work is tiny, TMA latency dominates
constexpr int DQ_SM_A = DQ_NSTAGE * KBYTES;
constexpr int DQ_NA = 4;  // dscore tiles in flight: the rows run up to 4 chunks ahead of the MMA + commit latency
constexpr int DQ_SM_DS = DQ_SM_A + DQ_NA * DQ_ABYTES;  // [2 heads][128 rows][64] f32: the rows' dscores
constexpr int DQ_KMAX = 64;
constexpr int DQ_SM_OFF = DQ_SM_DS + 2 * TQ * DQ_KMAX * 4;  // [128 rows][64] i32: the rows' dscore gather offsets
constexpr int DQ_SM_STG = DQ_SM_OFF + TQ * DQ_KMAX * 4;     // [4 warps][32 rows][80 B] epilogue staging
constexpr int DQ_SM_BAR = DQ_SM_STG + 8 * 32 * 80;  // 8 epilogue warps
constexpr int DQ_SM_TOTAL = DQ_SM_BAR + 256;

// KEYS = false: dq (rows = query rows, chunks = key chunks, B = K chunk, dscores
//   gathered through the row's ascending-j slot order);
// KEYS = true: dk = tau dS^T Q (rows = key atoms, chunks = 16-query chunks of the
//   transposed relation, B = Q chunk, dscores gathered through the key's
//   ascending rev_pair entries -- the same ascending (chunk, bit) order).
template <bool KEYS>
__global__ void __launch_bounds__(DQ_THREADS, 1) attn_dqk_tc_kernel(
    const __grid_constant__ CUtensorMap mk, int N, int K, float tau, const int* __restrict__ cptr,
    const int* __restrict__ clist, const uint32_t* __restrict__ rowlist, const int* __restrict__ slots,
    const int* __restrict__ tstart, const int* __restrict__ rev_ptr, const float* __restrict__ dsbuf,
    bf16* __restrict__ dq, int dbg) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (umma::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + DQ_SM_BAR);
  uint64_t* full_kv = bars + 0;    // [8] TMA landed
  uint64_t* empty_kv = bars + 8;   // [8] MMA done with the K stage
  uint64_t* a_full = bars + 16;    // [DQ_NA] rows wrote the dscore tile (128)
  uint64_t* a_free = bars + 20;    // [DQ_NA] MMA done with the dscore tile
  uint64_t* acc_done = bars + 24;
  uint64_t* epi_done = bars + 25;  // epilogue warps read the accumulator (256)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 26);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q0 = tstart[blockIdx.x], q1 = tstart[blockIdx.x + 1];
  if (q0 >= q1) return;  // surplus (empty) tile
  const int c_begin = cptr[blockIdx.x], nch = cptr[blockIdx.x + 1] - cptr[blockIdx.x];
  if (tid == 0) {
    umma::prefetch_tmap(&mk);
    for (int b = 0; b < DQ_NSTAGE; ++b) {
      umma::mbar_init(&full_kv[b], 1);
      umma::mbar_init(&empty_kv[b], 1);
    }
    for (int b = 0; b < DQ_NA; ++b) {
      umma::mbar_init(&a_full[b], 128);
      umma::mbar_init(&a_free[b], 1);
    }
    umma::mbar_init(acc_done, 1);
    umma::mbar_init(epi_done, 256);
    umma::fence_barrier_init();
  }
  if (warp == 0) umma::tmem_alloc(tslot, 512);
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0) {
    if (lane == 0) {
      constexpr int PF = 4;  // L2 prefetch distance beyond the smem stages
      int g = 0;
      for (int h = 0; h < 8; ++h)
        for (int c = 0; c < nch; ++c, ++g) {
          const int st = g % DQ_NSTAGE;
          {
            const int cp = c + DQ_NSTAGE + PF;
            const int hp = h + cp / (nch > 0 ? nch : 1), ccp = cp % (nch > 0 ? nch : 1);
            if (hp < 8)
              umma::tma_prefetch_3d(&mk, DH * hp, clist[c_begin + ccp] * KC, 0);
          }
          if (g >= DQ_NSTAGE) umma::mbar_wait(&empty_kv[st], ((g / DQ_NSTAGE) - 1) & 1);
          const int k0 = clist[c_begin + c] * KC;
          uint8_t* kb = sm + DQ_SM_K + st * KBYTES;
          umma::mbar_arrive_expect_tx(&full_kv[st], KBYTES);
          umma::tma_load_3d(kb, &mk, &full_kv[st], DH * h, k0, 0);
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_a = umma::idesc_bf16(128, 256, 0, 1);
      constexpr uint32_t idesc_b = umma::idesc_bf16(128, 32, 0, 1);
      int g = 0;
      for (int h = 0; h < 8; ++h) {
        for (int c = 0; c < nch; ++c, ++g) {
          const int st = g % DQ_NSTAGE, b = g % DQ_NA;
          umma::mbar_wait(&full_kv[st], (g / DQ_NSTAGE) & 1);
          umma::mbar_wait(&a_full[b], (g / DQ_NA) & 1);
          if (c == 0 && h > 0) umma::mbar_wait(epi_done, (h - 1) & 1);
          umma::tc_fence_after();
          const uint32_t ka = umma::smem_u32(sm + DQ_SM_K + st * KBYTES);
          const uint64_t ad = umma::sdesc(umma::smem_u32(sm + DQ_SM_A + b * DQ_ABYTES), 128, 256, 0);
          // B: MN-major, 64B swizzle: 32-channel atoms 1024 B apart (one per (l,m) row), 8 keys = 512 B
          if (!(dbg & 1)) {
            umma::mma_f16(tmem, ad, umma::sdesc(ka, 1024, 512, 4), idesc_a, c > 0 ? 1u : 0u);
            umma::mma_f16(tmem + 256, ad, umma::sdesc(ka + 8 * 1024, 1024, 512, 4), idesc_b, c > 0 ? 1u : 0u);
          }
          umma::mma_commit(&empty_kv[st]);
          umma::mma_commit(&a_free[b]);
        }
        if (nch > 0) {
          umma::mma_commit(acc_done);
        } else {  // empty tile: keep acc_done one phase ahead of the epilogue at most (parity waits)
          if (h > 0) umma::mbar_wait(epi_done, (h - 1) & 1);
          umma::mbar_arrive(acc_done);
        }
      }
    }
  } else if (warp >= 6) {
    // ================= epilogue: out[row][mm][32 h .. 32 h + 32] = tau * D[row][32 mm ..].  The
    // accumulator is drained into registers (bf16, 144 per thread) and released at once; the global
    // stores then overlap the next head's MMAs, which the row warps keep fed (the drain used to stall
    // the whole pipeline once per head: ~a quarter of the kernel)
    // two warps per TMEM lane quadrant: (l,m) rows [0, 5) and [5, 9) (80 / 64 registers held)
    const int ehalf = (warp - 6) >> 2, m0 = ehalf ? 5 : 0, nm = ehalf ? MM - 5 : 5;
    const int erow0 = q0 + (warp & 3) * 32;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    uint8_t* stg = sm + DQ_SM_STG + (warp - 6) * (32 * 80);
    for (int h = 0; h < 8; ++h) {
      umma::mbar_wait(acc_done, h & 1);
      umma::tc_fence_after();
      uint32_t pk[5][16];  // [mm - m0][32 channels as bf16 pairs]
#pragma unroll
      for (int i = 0; i < 5; ++i) {  // one (l,m) row = 32 columns per TMEM load + wait
        if (i >= nm) break;
        uint32_t r[32];
        if (nch > 0 && !(dbg & 4)) umma::tmem_ld32(tmem + lane_base + 32 * (m0 + i), r);
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const float x0 = nch > 0 ? tau * __uint_as_float(r[2 * t]) : 0.f;
          const float x1 = nch > 0 ? tau * __uint_as_float(r[2 * t + 1]) : 0.f;
          const __nv_bfloat162 b2 = __floats2bfloat162_rn(x0, x1);
          pk[i][t] = *reinterpret_cast<const uint32_t*>(&b2);
        }
      }
      umma::tc_fence_before();
      umma::mbar_arrive(epi_done);
      if (dbg & 4) continue;
      // staged, coalesced stores: 4 lanes write one row's 64 bytes
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        if (i >= nm) break;
        const int mm = m0 + i;
        uint4* sw = reinterpret_cast<uint4*>(stg + lane * 80);
#pragma unroll
        for (int t = 0; t < 4; ++t) sw[t] = make_uint4(pk[i][4 * t], pk[i][4 * t + 1], pk[i][4 * t + 2], pk[i][4 * t + 3]);
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int rr = it * 8 + (lane >> 2), part = lane & 3;
          const int qq = erow0 + rr;
          if (qq < q1)
            *reinterpret_cast<uint4*>(dq + ((size_t)qq * MM + mm) * 256 + DH * h + part * 8) =
                *reinterpret_cast<const uint4*>(stg + rr * 80 + part * 16);
        }
        __syncwarp();
      }
    }
  } else {
    // ================= rows: dscore tiles
    const int row = ((warp & 3) << 5) | lane;
    const int qi = q0 + row;
    const bool qin = qi < q1;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    // the row's (chunk, mask) list, its gather order and the dscore row base
    const uint32_t* rl;
    const int* sl;
    size_t gbase;
    int lmax, nv = 0;
    if constexpr (KEYS) {
      const int e0 = qin ? rev_ptr[qi] : 0;
      nv = qin ? rev_ptr[qi + 1] - e0 : 0;
      rl = rowlist + e0;
      sl = slots + e0;
      gbase = 0;
      lmax = nv;
    } else {
      rl = rowlist + (size_t)(qin ? qi : 0) * K;
      sl = slots + (size_t)(qin ? qi : 0) * K;
      gbase = (size_t)(qin ? qi : 0) * K;
      lmax = K;
      if (qin)
        for (int u = 0; u < K; ++u) {  // valid pairs of the row (popcount over its chunk list)
          const uint32_t e = __ldg(rl + u);
          if ((e >> 16) == 0xffffu) break;
          nv += __popc(e & 0xffffu);
        }
    }
    // this row's dscores, double buffered by head: head h+1's values are
    // copied (cp.async, no registers) while head h's chunks run; a key with
    // more than DQ_KMAX queries reads the excess directly
    float* dsr0 = reinterpret_cast<float*>(sm + DQ_SM_DS) + row * DQ_KMAX;
    const int npf = nv < DQ_KMAX ? nv : DQ_KMAX;
    // the row's gather offsets (pair index * 8), loaded once for all heads: a slot load per
    // pair and head would put a dependent global load in front of every cp.async
    int* off = reinterpret_cast<int*>(sm + DQ_SM_OFF) + row * DQ_KMAX;
#pragma unroll 4
    for (int r0 = 0; r0 < npf; ++r0) off[r0] = (int)((gbase + __ldg(sl + r0)) * 8);
    auto fetch = [&](int hh) {
      float* dst = dsr0 + (hh & 1) * TQ * DQ_KMAX;
      for (int r0 = 0; r0 < npf; ++r0)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(umma::smem_u32(dst + r0)),
                     "l"(dsbuf + (off[r0] + hh))
                     : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    fetch(0);
    int g = 0;
    for (int h = 0; h < 8; ++h) {
      if (h + 1 < 8) {
        fetch(h + 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // head h's group landed
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      const float* dsr = dsr0 + (h & 1) * TQ * DQ_KMAX;
      int rp = 0, r = 0;
      uint32_t ent = (qin && lmax > 0) ? __ldg(rl) : 0xffff0000u;
      for (int c = 0; c < nch; ++c, ++g) {
        const int b = g % DQ_NA;
        unsigned vmask = 0u;
        if ((int)(ent >> 16) == c) {
          vmask = ent & 0xffffu;
          ++rp;
          ent = rp < lmax ? __ldg(rl + rp) : 0xffff0000u;
        }
        float d[KC];
        if (!KEYS || nv <= DQ_KMAX) {  // every dscore of the row is in the prefetch buffer
#pragma unroll
          for (int t = 0; t < KC; ++t) {
            d[t] = 0.f;
            if (vmask >> t & 1) d[t] = dsr[r++];
          }
        } else {  // a key with more than DQ_KMAX queries: the excess is read directly
#pragma unroll
          for (int t = 0; t < KC; ++t) d[t] = 0.f;
#pragma unroll 1
          for (int t = 0; t < KC; ++t)
            if (vmask >> t & 1) {
              const float x = r < DQ_KMAX ? dsr[r] : __ldg(dsbuf + (gbase + __ldg(sl + r)) * 8 + h);
              ++r;
#pragma unroll
              for (int u = 0; u < KC; ++u)
                if (u == t) d[u] = x;  // static register indices
            }
        }
        if (g >= DQ_NA) umma::mbar_wait(&a_free[b], ((g / DQ_NA) - 1) & 1);
        uint8_t* at = sm + DQ_SM_A + b * DQ_ABYTES + (row >> 3) * 256 + (row & 7) * 16;
        *reinterpret_cast<uint4*>(at) = pack8(d);
        *reinterpret_cast<uint4*>(at + 128) = pack8(d + 8);
        umma::fence_proxy_async();
        umma::mbar_arrive(&a_full[b]);
      }
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, 512);
}
}  // namespace

// profiling switches of the dq / dk kernels (ES_DQ_DBG, outputs wrong): 1 no MMAs, 4 no epilogue
int dq_dbg() {
  const char* e = getenv("ES_DQ_DBG");
  return e ? atoi(e) : 0;
}

bool attn_dq_tc_applicable(const AttnArgs& a) {
  static int use = -1;
  if (use < 0) {
    const char* e = getenv("ES_ATTN_TC");
    use = (e && e[0] == '0') ? 0 : (e && e[0] == '1') ? 2 : 1;
  }
  const bool enough_tiles = (a.N + TQ - 1) / TQ >= 74 && a.nseg > 0;  // molecule batches (see attn_fwd_launch)
  const bool idx32 = (size_t)a.N * a.K * 8 < ((size_t)1 << 31);  // 32-bit gather offsets
  return use && (enough_tiles || use == 2) && a.K <= DQ_KMAX && idx32 && attn_tc_supported(a);
}

size_t attn_dq_tc_workspace(const AttnArgs& a) {
  if (a.N <= 0) return 0;
  return tc_scratch(a).total + 2 * align256((size_t)a.N * a.K * 4);
}

es_status attn_dq_tc_launch(const AttnArgs& a, const void* k, const int32_t* nbr, const float* dsbuf, void* dq,
                            void* ws, size_t ws_bytes, cudaStream_t st) {
  if (a.N == 0) return ES_OK;
  const TcScratch t = tc_scratch(a);
  TcLists lists;
  int* slots;
  if (a.tiles) {  // lists + slot order prebuilt for this neighbour index
    const TcPtrs pp = tc_ptrs(const_cast<void*>(a.tiles), t);
    lists = TcLists{pp.cptr, pp.clist, pp.rowlist, t.ntiles, pp.tstart};
    slots = pp.slots;
  } else {
    if (!ws || ws_bytes < attn_dq_tc_workspace(a)) return fail(ES_INVALID_ARGUMENT, "attn_bwd: workspace too small");
    slots = (int*)((char*)ws + t.total);
    es_status s = tc_build_lists(a, nbr, ws, t, slots, &lists, st);
    if (s != ES_OK) return s;
  }
  CUtensorMap mk;
  if (!map3t(&mk, k, 256, MM, a.Nk, DH, KC, MM, CU_TENSOR_MAP_SWIZZLE_64B))
    return fail(ES_CUDA_ERROR, "attn_dq_tc: tensor map encode failed");
  const int smem = DQ_SM_TOTAL + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_dqk_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  attn_dqk_tc_kernel<false><<<lists.ntiles, DQ_THREADS, smem, st>>>(mk, a.N, a.K, a.tau, lists.cptr, lists.clist,
                                                                   lists.rowlist, slots, lists.tstart, nullptr,
                                                                   dsbuf, (bf16*)dq, dq_dbg());
  return cuda_status(cudaGetLastError(), "attn_dq_tc_kernel");
}

namespace {
// the key-side problem: rows = the Nk key atoms, chunks over the N query rows
AttnArgs key_side(const AttnArgs& a) {
  AttnArgs b = a;
  b.N = a.Nk;
  b.Nk = a.N;
  return b;
}

es_status tc_build_key_lists(const AttnArgs& a, const int32_t* nbr, const int32_t* rev_ptr, const int32_t* rev_pair,
                             void* ws, TcLists* out, cudaStream_t st, const int32_t* seg = nullptr, int nseg = 0,
                             const int* q_tstart = nullptr) {
  const AttnArgs b = key_side(a);
  const TcScratch t = tc_scratch(b);
  const TcPtrs pp = tc_ptrs(ws, t);
  size_t cub_bytes = t.cub_bytes;
  // key tiles: the query tiles' packing when keys and queries are the same atoms (molecule batches) --
  // copied from the query-side lists when the caller just built them (the packing is one CTA's serial scan)
  if (seg && nseg > 0 && a.N == a.Nk && q_tstart)
    cudaMemcpyAsync(pp.tstart, q_tstart, sizeof(int) * (size_t)(t.ntiles + 1), cudaMemcpyDeviceToDevice, st);
  else if (seg && nseg > 0 && a.N == a.Nk) tc_tiles_packed_kernel<<<1, 1024, 0, st>>>(b.N, nseg, seg, t.ntiles, pp.tstart);
  else tc_tiles_uniform_kernel<<<(t.ntiles + 256) / 256, 256, 0, st>>>(b.N, t.ntiles, pp.tstart);
  tc_rowtile_kernel<<<t.ntiles, 128, 0, st>>>(t.ntiles, pp.tstart, pp.rtile);
  cudaMemsetAsync(pp.mask, 0, (size_t)t.ntiles * t.words * 4, st);
  cudaMemsetAsync(pp.cnt, 0, (size_t)(t.ntiles + 1) * 4, st);
  const size_t np = (size_t)a.N * a.K;
  if (np > 0) tc_maskT_kernel<<<(unsigned)((np + 255) / 256), 256, 0, st>>>(a.N, a.K, nbr, pp.rtile, t.words, pp.mask);
  tc_count_kernel<<<(t.ntiles + 7) / 8, 256, 0, st>>>(t.ntiles, t.words, pp.mask, pp.cnt);
  cudaError_t e = cub::DeviceScan::ExclusiveSum(pp.cub, cub_bytes, pp.cnt, pp.cptr, t.ntiles + 1, st);
  if (e != cudaSuccess) return cuda_status(e, "attn_tc key scan");
  tc_fill_kernel<<<(t.ntiles + 7) / 8, 256, 0, st>>>(t.ntiles, t.words, pp.mask, pp.cptr, pp.clist);
  tc_rowlistT_kernel<<<(b.N + 127) / 128, 128, 0, st>>>(b.N, a.K, rev_ptr, rev_pair, pp.cptr, pp.clist, pp.rtile,
                                                        pp.rowlist);
  *out = TcLists{pp.cptr, pp.clist, pp.rowlist, t.ntiles, pp.tstart};
  return cuda_status(cudaGetLastError(), "attn_tc key lists");
}

size_t tiles_query_bytes(const AttnArgs& a) { return tc_scratch(a).total + 2 * align256((size_t)a.N * a.K * 4); }

}  // namespace

bool attn_dk_tc_applicable(const AttnArgs& a) {
  // Off by default (ES_DK_TC=1 enables it): on configs[1] the key pass without dk is gather-bound
  // (2.9 ms with the forward's kept scores, 4.2 ms recomputing them) and this pass adds 0.84 ms, while
  // keeping the scores costs the forward 0.47 ms -- 7.73 ms fwd+bwd against 7.50 ms for the SIMT
  // key pass with dk.
  const char* e = getenv("ES_DK_TC");  // read per call: the tests switch it
  return e && e[0] == '1' && attn_dq_tc_applicable(a);
}

// the tile buffer also carries the key-side lists (tensor-core key pass or dk)
bool tc_key_lists(const AttnArgs& a) { return attn_dk_tc_applicable(a) || attn_kv_tc_applicable(a); }

size_t attn_dk_tc_workspace(const AttnArgs& a) { return a.N > 0 ? tc_scratch(key_side(a)).total : 0; }

es_status attn_dk_tc_launch(const AttnArgs& a, const void* q, const int32_t* nbr, const int32_t* rev_ptr,
                            const int32_t* rev_pair, const float* dsbuf, void* dk, void* ws, size_t ws_bytes,
                            cudaStream_t st) {
  if (a.N == 0) return ES_OK;
  const TcScratch t = tc_scratch(key_side(a));
  TcLists lists;
  if (a.tiles) {  // key-side lists prebuilt after the query-side ones
    const TcPtrs pp = tc_ptrs(const_cast<char*>(static_cast<const char*>(a.tiles)) + tiles_query_bytes(a), t);
    lists = TcLists{pp.cptr, pp.clist, pp.rowlist, t.ntiles, pp.tstart};
  } else {
    if (!ws || ws_bytes < t.total) return fail(ES_INVALID_ARGUMENT, "attn_bwd: workspace too small (dk)");
    es_status s = tc_build_key_lists(a, nbr, rev_ptr, rev_pair, ws, &lists, st);
    if (s != ES_OK) return s;
  }
  CUtensorMap mq;
  if (!map3t(&mq, q, 256, MM, a.N, DH, KC, MM, CU_TENSOR_MAP_SWIZZLE_64B))
    return fail(ES_CUDA_ERROR, "attn_dk_tc: tensor map encode failed");
  const int smem = DQ_SM_TOTAL + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_dqk_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  attn_dqk_tc_kernel<true><<<lists.ntiles, DQ_THREADS, smem, st>>>(mq, a.Nk, a.K, a.tau, lists.cptr, lists.clist,
                                                                  lists.rowlist, rev_pair, lists.tstart, rev_ptr,
                                                                  dsbuf, (bf16*)dk, dq_dbg());
  return cuda_status(cudaGetLastError(), "attn_dk_tc_kernel");
}

void attn_tc_tiles_layout(const AttnArgs& a, es_attn_tiles_layout* out) {
  std::memset(out, 0, sizeof(*out));
  if (a.N <= 0 || !attn_tc_tiles_used(a)) return;
  auto side = [](const AttnArgs& b, int64_t base, es_attn_tiles_side* o, bool query) {
    const TcScratch t = tc_scratch(b);
    const TcPtrs p = tc_ptrs(nullptr, t);
    const char* z = nullptr;
    o->ntiles = t.ntiles;
    o->words = t.words;
    o->nchunk_max = (int64_t)t.chunks;
    o->mask = base + ((const char*)p.mask - z);
    o->cptr = base + ((const char*)p.cptr - z);
    o->clist = base + ((const char*)p.clist - z);
    o->rowlist = base + ((const char*)p.rowlist - z);
    o->tstart = base + ((const char*)p.tstart - z);
    o->rtile = base + ((const char*)p.rtile - z);
    o->slots = query ? base + ((const char*)p.slots - z) : -1;
    o->rank_of = query ? base + ((const char*)p.rank_of - z) : -1;
  };
  side(a, 0, &out->query, true);
  if (tc_key_lists(a)) side(key_side(a), (int64_t)tiles_query_bytes(a), &out->key, false);
}

const int* attn_tc_rank_of(const AttnArgs& a, const void* tiles) {
  if (!tiles) return nullptr;
  return reinterpret_cast<const int*>(static_cast<const char*>(tiles) + tc_scratch(a).total +
                                      align256((size_t)a.N * a.K * 4));
}

bool attn_tc_tiles_used(const AttnArgs& a) { return attn_dq_tc_applicable(a) || attn_fwd_workspace(a) > 0; }

size_t attn_tc_tiles_bytes(const AttnArgs& a) {
  if (a.N <= 0) return 0;
  return tiles_query_bytes(a) + (tc_key_lists(a) ? attn_dk_tc_workspace(a) : 0);
}

// The tile structures of one neighbour index, built once and reused by every
// forward / backward (and every layer) that uses the same index.
es_status attn_tc_tiles_build(const AttnArgs& a, const int32_t* nbr, const int32_t* seg, int nseg,
                              const int32_t* rev_ptr, const int32_t* rev_pair, void* tiles, size_t bytes,
                              cudaStream_t st) {
  if (a.N == 0) return ES_OK;
  const TcScratch t = tc_scratch(a);
  if (!tiles || bytes < attn_tc_tiles_bytes(a)) return fail(ES_INVALID_ARGUMENT, "attn_tiles: buffer too small");
  const bool keys = tc_key_lists(a);
  if (keys && (!rev_ptr || !rev_pair))
    return fail(ES_INVALID_ARGUMENT, "attn_tiles: the tensor-core backward needs rev_ptr / rev_pair (key-side lists)");
  TcLists lists;
  es_status s = tc_build_lists(a, nbr, tiles, t, (int*)((char*)tiles + t.total), &lists, st, seg, nseg);
  if (s != ES_OK || !keys) return s;
  return tc_build_key_lists(a, nbr, rev_ptr, rev_pair, (char*)tiles + tiles_query_bytes(a), &lists, st, seg, nseg,
                            lists.tstart);
}


// ---------------------------------------------------------------- key pass on the tensor cores
// dv_j and the per-pair dscores of the backward (stream_aggregate_backward,
// SPEC.md:293-301) over the key-side tiles (128 key atoms; 16-query chunks of
// the transposed relation), per head h and chunk three tcgen05 MMA groups:
//   S^T[j, i]     = K_h . Q_chunk^T                 M=128 keys, N=16,  K=288  (A = K_h in TMEM)
//   D[j, (f,i)]   = V_h . dOg^T                     M=128,      N=144, K=144  (A = V_h, TMA SW32;
//                                                                             B = dOg read MN-major)
//   dV[j,(i',c)] += Wt'[j,(f,i)] . dOg[(f,i),(i',c)] M=128,     N=144, K=144
// with the query-side source coupling dOg[(f,i),(i',c)] = sum_o G_f[o,i'] dO_i[o][c]
// (the transpose of the forward's per-key Vg) and per valid pair, on the key rows,
//   P = exp(tau s + b(r) - lse_i),  dP = phi sum_f Y^f D[j,(f,i)],  dS = P (dP - delta_i),
//   Wt'[j,(f,i)] = P phi Y^f       (zero for non-neighbours).
// This is the SIMT key pass's math (attn_bwd_kv_kernel: dv_j += P y, dP = y . v_j with
// y = phi (EAAS map)^T dO_i) with the map written as sum_f Y^f G_f (Prop. 1).  dk and dq
// follow from the dscores on the tensor cores (attn_dqk_tc_kernel).  The pair geometry
// (phi Y^f, b(r)) is head-independent: attn_pair_geom_kernel writes it once per pair in
// key-side order, and the eight head passes read it back (L2-resident).
// The (f, i) index of D, Wt' and dOg is quarter-major, k = 36 (i / 4) + 4 f + i % 4, so a
// row thread's 4 queries x 9 f of one quarter are 36 consecutive TMEM columns.
namespace {
constexpr int KV_NA = 2;                               // Q / dO stages (freed early: S MMA + coupling)
constexpr int KV_NB = 4;                               // position / lse / delta stages (freed by the rows)
constexpr int KV_QB = MM * KC * DH * 2;                // 9216: Q chunk, 9 SW64 boxes [16 q][32 ch]
constexpr int KV_OB = KC * MM * HD * 2;                // 4608: dO chunk [16 q][9][16 c]
constexpr int KV_ASTAGE = 14 * 1024;                   // Q | dO
constexpr int KV_B_L = KC * 24;                        // [16][3] f64 positions | [16][8] lse | [16][8] delta
constexpr int KV_B_D = KV_B_L + KC * 32;
constexpr int KV_BSTAGE = 1536;
static_assert(KV_QB + KV_OB <= KV_ASTAGE && KV_B_D + KC * 32 <= KV_BSTAGE, "kv stage overflow");
constexpr int KV_VHB = TQ * MM * HD * 2;               // 36864: V_h as 9 SW32 boxes [128 keys][16 c]
constexpr int KV_SM_B = KV_NA * KV_ASTAGE;
constexpr int KV_SM_WT = KV_SM_B + KV_NB * KV_BSTAGE;  // Wt' (single buffer: rows write it after dV(g-1))
constexpr int KV_SM_DOG = KV_SM_WT + WBYTES;           // 2 x GBYTES
constexpr int KV_SM_VH = KV_SM_DOG + 2 * GBYTES;       // 2 x KV_VHB: V_(h+1) lands while head h runs
constexpr int KV_SM_BAR = KV_SM_VH + 2 * KV_VHB;
constexpr int KV_SM_TOTAL = KV_SM_BAR + 512;
static_assert(KV_SM_TOTAL + 1024 <= 232448, "key-pass kernel exceeds 227 KB of shared memory");
static_assert(KV_SM_WT % 1024 == 0 && KV_SM_DOG % 1024 == 0 && KV_SM_VH % 1024 == 0, "kv smem alignment");

__device__ __forceinline__ int kv_k(int f, int i) { return (i >> 2) * 36 + 4 * f + (i & 3); }

#ifdef ES_TC_TRACE
__device__ long long g_ktrace[12][256];  // per-chunk event clocks of CTA 1 (ES_KV_DBG=64)
#define KV_TRACE(cond, ev, idx) \
  do {                          \
    if (KTRACE && (cond) && (idx) < 256) g_ktrace[ev][idx] = clock64(); \
  } while (0)
#else
#define KV_TRACE(cond, ev, idx) \
  do {                          \
  } while (0)
#endif

// Per-pair record of the key pass, key-side order (entry e of rev_pair): phi Y^f (9 x fp16),
// b(r) (f32), the pair index i K + slot.  32 bytes.
struct __align__(16) PairGeom {
  __half2 y01, y23, y45, y67;
  __half y8, pad;
  float bias;
  int pr;
  int pad2;
};
static_assert(sizeof(PairGeom) == 32, "pair record");

__global__ void __launch_bounds__(256) attn_pair_geom_kernel(TcArgs a, const double* __restrict__ pos,
                                                             const int* __restrict__ rev_ptr,
                                                             const int* __restrict__ rev_pair,
                                                             PairGeom* __restrict__ geom) {
  // 4 threads per key, entries strided by 4: independent loads in flight instead of one dependent chain
  const int j = (int)(((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 2), sub = threadIdx.x & 3;
  if (j >= a.Nk) return;
  const double kx = pos[3 * (size_t)j], ky = pos[3 * (size_t)j + 1], kz = pos[3 * (size_t)j + 2];
  const int e1 = rev_ptr[j + 1];
  for (int e = rev_ptr[j] + sub; e < e1; e += 4) {
    const int pr = rev_pair[e];
    const size_t i = (size_t)(pr / a.K);
    // r_ij = pos_j - pos_i, as the forward (key minus query)
    double dx = kx - pos[3 * i], dy = ky - pos[3 * i + 1], dz = kz - pos[3 * i + 2];
    if (a.periodic) {
      dx -= a.bx * rint(dx / a.bx);
      dy -= a.by * rint(dy / a.by);
      dz -= a.bz * rint(dz / a.bz);
    }
    const float rx = (float)dx, ry = (float)dy, rz = (float)dz;
    const float rn = sqrtf(rx * rx + ry * ry + rz * rz);
    float phi = 1.f;
    if (a.phi_mode == 0) phi = rn < a.r_cut ? 0.5f * (cospif(rn * a.inv_rcut) + 1.f) : 0.f;
    float y[MM];
    solid_l2(rx, ry, rz, y);
    PairGeom g;
    g.y01 = __floats2half2_rn(phi * y[0], phi * y[1]);
    g.y23 = __floats2half2_rn(phi * y[2], phi * y[3]);
    g.y45 = __floats2half2_rn(phi * y[4], phi * y[5]);
    g.y67 = __floats2half2_rn(phi * y[6], phi * y[7]);
    g.y8 = __float2half_rn(phi * y[8]);
    g.pad = __float2half_rn(0.f);
    g.bias = a.bias_mode ? fmaf(fmaf(a.b2, rn, a.b1), rn, a.b0) : 0.f;
    g.pr = pr;
    g.pad2 = 0;
    geom[e] = g;
  }
}

__global__ void __launch_bounds__(TC_THREADS, 1) attn_kv_tc_kernel(
    const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mo,
    const __grid_constant__ CUtensorMap mvh, TcArgs a, const bf16* __restrict__ k, const double* __restrict__ pos,
    const float* __restrict__ lse, const float* __restrict__ delta, const int* __restrict__ cptr,
    const int* __restrict__ clist, const uint32_t* __restrict__ rowlist, const int* __restrict__ tstart,
    const int* __restrict__ rev_ptr, const PairGeom* __restrict__ geom, float* __restrict__ dsbuf,
    bf16* __restrict__ dv) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (umma::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + KV_SM_BAR);
  uint64_t* full_a = bars + 0;     // [4] Q + dO landed (tx)
  uint64_t* empty_a = bars + 4;    // [4] S MMA + coupling threads done (129)
  uint64_t* full_b = bars + 8;     // [4] positions / lse / delta landed (tx)
  uint64_t* empty_b = bars + 12;   // [4] rows done (256)
  uint64_t* s_full = bars + 16;    // [2] S^T committed
  uint64_t* s_free = bars + 18;    // [2] rows read S^T (256)
  uint64_t* d_full = bars + 20;    // D committed
  uint64_t* d_free = bars + 21;    // rows read D (256)
  uint64_t* dog_full = bars + 22;  // [2] coupling threads wrote dOg (128)
  uint64_t* wv_free = bars + 24;   // [2] dV MMA committed (Wt', dOg buffer free)
  uint64_t* wt_full = bars + 26;   // rows wrote Wt' (256)
  uint64_t* acc_done = bars + 27;  // last dV MMA of the head committed
  uint64_t* epi_done = bars + 28;  // rows read dV (256)
  uint64_t* k_ready = bars + 29;   // K_h stored into TMEM (coupling warps, 128)
  uint64_t* k_free = bars + 30;    // last S MMA of the head committed
  uint64_t* vh_full = bars + 31;   // [2] V_h landed (tx)
  uint64_t* vh_free = bars + 33;   // [2] last D MMA of the head committed (V_h buffer free)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 35);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j0 = tstart[blockIdx.x], j1 = tstart[blockIdx.x + 1];
  if (j0 >= j1) return;  // surplus (empty) tile
  const int c_begin = cptr[blockIdx.x], nch = cptr[blockIdx.x + 1] - cptr[blockIdx.x];
#ifdef ES_TC_TRACE
  const bool KTRACE = (a.dbg & 64) && blockIdx.x == 1;
#endif
  const bool is_row = warp >= 2 && warp <= 9;
  const int row = ((warp & 3) << 5) | lane;  // TMEM lane = key row of the tile
  const int kj = j0 + row;
  const bool kin = kj < j1;

  if (tid == 0) {
    umma::prefetch_tmap(&mq);
    umma::prefetch_tmap(&mo);
    umma::prefetch_tmap(&mvh);
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&s_full[b], 1);
      umma::mbar_init(&s_free[b], 256);
      umma::mbar_init(&dog_full[b], 128);
      umma::mbar_init(&wv_free[b], 1);
    }
    for (int b = 0; b < KV_NA; ++b) {
      umma::mbar_init(&full_a[b], 1);
      umma::mbar_init(&empty_a[b], 1 + 128);
    }
    umma::mbar_init(&vh_full[0], 1);
    umma::mbar_init(&vh_full[1], 1);
    umma::mbar_init(&vh_free[0], 1);
    umma::mbar_init(&vh_free[1], 1);
    for (int b = 0; b < KV_NB; ++b) {
      umma::mbar_init(&full_b[b], 1);
      umma::mbar_init(&empty_b[b], 256);
    }
    umma::mbar_init(d_full, 1);
    umma::mbar_init(d_free, 256);
    umma::mbar_init(wt_full, 256);
    umma::mbar_init(acc_done, 1);
    umma::mbar_init(epi_done, 256);
    umma::mbar_init(k_ready, 128);
    umma::mbar_init(k_free, 1);
    umma::fence_barrier_init();
  }
  if (warp == 0) umma::tmem_alloc(tslot, 512);
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t t_k = tmem, t_d = tmem + 144, t_dv = tmem + 288, t_s0 = tmem + 448;
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  // K_hh rows (l,m) in [m0, m0 + 3) of this thread's key -> TMEM (the S MMA's A operand)
  const bf16* krow = k + (size_t)(kin ? kj : 0) * MM * 256;
  auto load_k3 = [&](int hh, int m0) {
    uint32_t rr[3][16];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const uint4* src = reinterpret_cast<const uint4*>(krow + (m0 + d) * 256 + DH * hh);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint4 u = kin ? __ldg(src + t) : make_uint4(0, 0, 0, 0);
        rr[d][4 * t] = u.x; rr[d][4 * t + 1] = u.y; rr[d][4 * t + 2] = u.z; rr[d][4 * t + 3] = u.w;
      }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) umma::tmem_st16(t_k + lane_base + 16 * (m0 + d), rr[d]);
  };
  auto load_k = [&](int hh) {  // the coupling warps: all nine (l,m) rows
    load_k3(hh, 0);
    load_k3(hh, 3);
    load_k3(hh, 6);
    umma::tc_fence_before();
    umma::mbar_arrive(k_ready);
  };

  if (nch == 0) {
    // no key of the tile is anyone's neighbour: dv = 0, no dscores
    if (is_row && kin) {
      const int half = (warp - 2) >> 2;
      for (int h = 0; h < 8; ++h)
        for (int cc = half ? 5 : 0; cc < (half ? MM : 5); ++cc) {
          uint4* dst = reinterpret_cast<uint4*>(dv + ((size_t)kj * MM + cc) * 128 + HD * h);
          dst[0] = make_uint4(0, 0, 0, 0);
          dst[1] = make_uint4(0, 0, 0, 0);
        }
    }
  } else if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer: query chunks (Q + dO; positions, lse, delta) and V_h
      constexpr int PF = 4;
      auto prefetch = [&](int h, int c) {
        const int i0 = clist[c_begin + c] * KC;
        umma::tma_prefetch_3d(&mq, DH * h, i0, 0);
        umma::tma_prefetch_3d(&mo, HD * h, 0, i0);
      };
      auto load_vh = [&](int h) {  // 9 i' blocks [128 keys][16 c] into buffer h & 1
        umma::mbar_arrive_expect_tx(&vh_full[h & 1], KV_VHB);
        umma::tma_load_3d(sm + KV_SM_VH + (h & 1) * KV_VHB, &mvh, &vh_full[h & 1], HD * h, j0, 0);
      };
      load_vh(0);
      load_vh(1);
      for (int c = 0; c < nch && c < PF; ++c) prefetch(0, c);
      int g = 0;
      for (int h = 0; h < 8; ++h) {
        for (int c = 0; c < nch; ++c, ++g) {
          {
            const int cp = c + PF;
            if (cp < nch) prefetch(h, cp);
            else if (h + 1 < 8 && cp - nch < nch) prefetch(h + 1, cp - nch);
          }
          const int i0 = clist[c_begin + c] * KC;
          const int nq = min(KC, a.N - i0);
          {
            const int st = g % KV_NA;
            if (g >= KV_NA) umma::mbar_wait(&empty_a[st], ((g / KV_NA) - 1) & 1);
            uint8_t* sa = sm + st * KV_ASTAGE;
            umma::mbar_arrive_expect_tx(&full_a[st], KV_QB + KV_OB);
            umma::tma_load_3d(sa, &mq, &full_a[st], DH * h, i0, 0);
            umma::tma_load_3d(sa + KV_QB, &mo, &full_a[st], HD * h, 0, i0);
            KV_TRACE(true, 0, g);
          }
          {
            const int st = g % KV_NB;
            if (g >= KV_NB) umma::mbar_wait(&empty_b[st], ((g / KV_NB) - 1) & 1);
            uint8_t* sb = sm + KV_SM_B + st * KV_BSTAGE;
            const uint32_t pbytes = (uint32_t)((nq & ~1) * 24), lbytes = (uint32_t)(nq * 32);
            if (nq & 1) {  // odd tail: the last query's 24 bytes by plain loads (ordered by the arrive)
              double* tail = reinterpret_cast<double*>(sb) + 3 * (nq - 1);
              const double* src = pos + 3 * ((size_t)i0 + nq - 1);
              tail[0] = src[0]; tail[1] = src[1]; tail[2] = src[2];
            }
            umma::mbar_arrive_expect_tx(&full_b[st], pbytes + 2 * lbytes);
            if (pbytes) umma::bulk_load(sb, pos + 3 * (size_t)i0, pbytes, &full_b[st]);
            umma::bulk_load(sb + KV_B_L, lse + (size_t)i0 * 8, lbytes, &full_b[st]);
            umma::bulk_load(sb + KV_B_D, delta + (size_t)i0 * 8, lbytes, &full_b[st]);
          }
          if (c == 0 && h >= 1 && h + 1 < 8) {  // V_(h+1) into the buffer head h-1 used
            umma::mbar_wait(&vh_free[(h + 1) & 1], ((h - 1) >> 1) & 1);
            load_vh(h + 1);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ================= MMA issuer
      constexpr uint32_t idesc_s = umma::idesc_bf16(128, KC, 0, 0);
      constexpr uint32_t idesc_d = umma::idesc_bf16(128, KV, 0, 1);
      constexpr uint32_t idesc_v = umma::idesc_bf16(128, NV, 0, 0);
      auto issue_s = [&](int g, bool last) {
        const int b = g & 1, st = g % KV_NA;
        umma::mbar_wait(&full_a[st], (g / KV_NA) & 1);
        if (g >= 2) umma::mbar_wait(&s_free[b], ((g >> 1) - 1) & 1);
        umma::tc_fence_after();
        // descriptors advance by (byte offset >> 4) from one base: the single issuing thread
        // would otherwise spend ~100 cycles of dependent integer ops per MMA building them
        const uint64_t qd = umma::sdesc(umma::smem_u32(sm + st * KV_ASTAGE), 16, 512, 4);
        const uint32_t ts = t_s0 + 32 * b;
        if (!(a.dbg & 16)) {
#pragma unroll
          for (int s = 0; s < 2 * MM; ++s)
            umma::mma_f16_ts(ts, t_k + 8 * s, qd + (uint64_t)(((s >> 1) * KC * DH * 2 + (s & 1) * 32) >> 4), idesc_s,
                             s > 0 ? 1u : 0u);
        }
        umma::mma_commit(&s_full[b]);
        umma::mma_commit(&empty_a[st]);
        if (last) umma::mma_commit(k_free);
        KV_TRACE(true, 1, g);
      };
      auto issue_d = [&](int g, int h, bool last) {
        const int b = g & 1;
        umma::mbar_wait(&dog_full[b], (g >> 1) & 1);
        if (g >= 1) umma::mbar_wait(d_free, (g - 1) & 1);
        umma::tc_fence_after();
        // A: V_h K-major SW32 (one 32-byte atom row per key, 8-key groups 256 B apart), one box per i';
        // B: dOg read MN-major (no swizzle: 8 (f,i) x 8 (i',c) core matrices, (f,i) groups 128 B
        //    apart (SBO), (i',c) groups 2304 B apart (LBO))
        const uint64_t vd = umma::sdesc(umma::smem_u32(sm + KV_SM_VH + (h & 1) * KV_VHB), 16, 256, 6);
        const uint64_t dd = umma::sdesc(umma::smem_u32(sm + KV_SM_DOG + b * GBYTES), (KV / 8) * 128, 128, 0);
        if (!(a.dbg & 4)) {
#pragma unroll
          for (int s = 0; s < MM; ++s)
            umma::mma_f16(t_d, vd + (uint64_t)((s * (KV_VHB / MM)) >> 4), dd + (uint64_t)((s * 2 * (KV / 8) * 128) >> 4),
                          idesc_d, s > 0 ? 1u : 0u);
        }
        umma::mma_commit(d_full);
        if (last) umma::mma_commit(&vh_free[h & 1]);
        KV_TRACE(true, 2, g);
      };
      auto issue_v = [&](int g, int c, int h) {
        const int b = g & 1;
        umma::mbar_wait(wt_full, g & 1);
        if (c == 0 && h > 0) umma::mbar_wait(epi_done, (h - 1) & 1);  // dV of the previous head read out
        umma::tc_fence_after();
        const uint64_t wd = umma::sdesc(umma::smem_u32(sm + KV_SM_WT), 128, (KV / 8) * 128, 0);
        const uint64_t dd = umma::sdesc(umma::smem_u32(sm + KV_SM_DOG + b * GBYTES), 128, (KV / 8) * 128, 0);
        if (!(a.dbg & 8)) {
          umma::mma_f16(t_dv, wd, dd, idesc_v, c > 0 ? 1u : 0u);
#pragma unroll
          for (int s = 1; s < MM; ++s) umma::mma_f16(t_dv, wd + (uint64_t)(16 * s), dd + (uint64_t)(16 * s), idesc_v, 1u);
        }
        umma::mma_commit(&wv_free[b]);
        KV_TRACE(true, 3, g);
      };
      int g0 = 0;
      for (int h = 0; h < 8; ++h) {
        umma::mbar_wait(k_ready, h & 1);
        KV_TRACE(true, 10, h);
        umma::mbar_wait(&vh_full[h & 1], (h >> 1) & 1);
        KV_TRACE(true, 10, 8 + h);
        issue_s(g0, nch == 1);
        issue_d(g0, h, nch == 1);
        for (int c = 0; c < nch; ++c) {
          if (c + 1 < nch) {
            issue_s(g0 + c + 1, c + 2 == nch);
            issue_d(g0 + c + 1, h, c + 2 == nch);
          }
          issue_v(g0 + c, c, h);
        }
        umma::mma_commit(acc_done);
        g0 += nch;
      }
    }
  } else if (is_row) {
    // ================= key rows: P, dP, dscores, Wt'; dv epilogue
    const int half = (warp - 2) >> 2;  // this warp's queries: quarters 2 half, 2 half + 1 of every chunk
    const int e0 = kin ? rev_ptr[kj] : 0;
    const int nvk = kin ? rev_ptr[kj + 1] - e0 : 0;
    const uint32_t* rl = rowlist + e0;
    int g0 = 0;
    for (int h = 0; h < 8; ++h) {
      int rp = 0, rbase = 0;
      uint32_t ent = nvk > 0 ? __ldg(rl) : 0xffff0000u;
      for (int c = 0; c < nch; ++c) {
        const int g = g0 + c, b = g & 1, sb_i = g % KV_NB;
        unsigned vmask = 0u;
        if ((int)(ent >> 16) == c) {
          vmask = ent & 0xffffu;
          ++rp;
          ent = rp < nvk ? __ldg(rl + rp) : 0xffff0000u;
        }
        if (a.dbg & 1) vmask = 0u;
        // the pair records of my 8 queries, issued before the barrier waits (their latency hides there)
        uint4 gr[2][4][2];
        {
          int eq = e0 + rbase + (half ? __popc(vmask & 0xffu) : 0);  // my first valid query's entry
          const unsigned hm = (vmask >> (8 * half)) & 0xffu;
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const uint4* src = reinterpret_cast<const uint4*>(geom + eq + __popc(hm & ((1u << t) - 1u)));
            if (hm >> t & 1) {
              gr[t >> 2][t & 3][0] = __ldg(src);
              gr[t >> 2][t & 3][1] = __ldg(src + 1);
            } else {
              gr[t >> 2][t & 3][0] = gr[t >> 2][t & 3][1] = make_uint4(0, 0, 0, 0);
            }
          }
        }
        rbase += __popc(vmask);
        umma::mbar_wait(&s_full[b], (g >> 1) & 1);
        umma::mbar_wait(d_full, g & 1);
        umma::mbar_wait(&full_b[sb_i], (g / KV_NB) & 1);
        umma::tc_fence_after();
        KV_TRACE(tid == 64, 4, g);
        const uint8_t* sb = sm + KV_SM_B + sb_i * KV_BSTAGE;
        uint8_t* wt = sm + KV_SM_WT;
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          const int quarter = 2 * half + qq;
          const unsigned qm = (vmask >> (4 * quarter)) & 0xfu;
          uint32_t r[40];  // [0, 4): S^T of the quarter's queries; [4, 40): D at 4 + 4 f + t
          umma::tmem_ld_4_36(t_s0 + 32 * b + 4 * quarter + lane_base, t_d + 36 * quarter + lane_base, r);
          if (qq == 1) {
            umma::tc_fence_before();
            umma::mbar_arrive(&s_free[b]);
            umma::mbar_arrive(d_free);
          }
          const float* ls = reinterpret_cast<const float*>(sb + KV_B_L) + 32 * quarter + h;
          const float* dl = reinterpret_cast<const float*>(sb + KV_B_D) + 32 * quarter + h;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            float y[MM];
            {
              const __half2* h2 = reinterpret_cast<const __half2*>(&gr[qq][t][0]);
              float2 f;
              f = __half22float2(h2[0]); y[0] = f.x; y[1] = f.y;
              f = __half22float2(h2[1]); y[2] = f.x; y[3] = f.y;
              f = __half22float2(h2[2]); y[4] = f.x; y[5] = f.y;
              f = __half22float2(h2[3]); y[6] = f.x; y[7] = f.y;
              y[8] = __low2float(*reinterpret_cast<const __half2*>(&gr[qq][t][1].x));
            }
            if (qm >> t & 1) {
              const float sc = fmaf(a.tau, __uint_as_float(r[t]), __uint_as_float(gr[qq][t][1].y));
              const float P = __expf(sc - ls[8 * t]);
              float dp = 0.f;
#pragma unroll
              for (int f = 0; f < MM; ++f) dp = fmaf(y[f], __uint_as_float(r[4 + 4 * f + t]), dp);
              dsbuf[(size_t)(int)gr[qq][t][1].z * 8 + h] = P * (dp - dl[8 * t]);
#pragma unroll
              for (int f = 0; f < MM; ++f) r[4 + 4 * f + t] = __float_as_uint(P * y[f]);
            } else {
#pragma unroll
              for (int f = 0; f < MM; ++f) r[4 + 4 * f + t] = 0u;
            }
          }
          if (qq == 0) KV_TRACE(tid == 64, 5, g);
          if (qq == 0 && g >= 1) umma::mbar_wait(&wv_free[(g - 1) & 1], ((g - 1) >> 1) & 1);  // Wt' free
          if (qq == 0) KV_TRACE(tid == 64, 6, g);
#pragma unroll
          for (int f = 0; f < MM; ++f) {
            const __nv_bfloat162 lo = __floats2bfloat162_rn(__uint_as_float(r[4 + 4 * f]), __uint_as_float(r[5 + 4 * f]));
            const __nv_bfloat162 hi = __floats2bfloat162_rn(__uint_as_float(r[6 + 4 * f]), __uint_as_float(r[7 + 4 * f]));
            uint2 u;
            u.x = *reinterpret_cast<const uint32_t*>(&lo);
            u.y = *reinterpret_cast<const uint32_t*>(&hi);
            *reinterpret_cast<uint2*>(wt + cm_off(row, 36 * quarter + 4 * f)) = u;
          }
        }
        umma::mbar_arrive(&empty_b[sb_i]);  // done with the stage's positions, lse and delta
        umma::fence_proxy_async();
        umma::mbar_arrive(wt_full);
        KV_TRACE(tid == 64, 7, g);
      }
      g0 += nch;
      KV_TRACE(tid == 64, 11, 16 + h);
      // ---- epilogue: dv_j of head h, the two halves each store half of the (i', c) columns
      KV_TRACE(tid == 64, 11, h);
      umma::mbar_wait(acc_done, h & 1);
      umma::tc_fence_after();
      KV_TRACE(tid == 64, 11, 8 + h);
      for (int cc = half ? 5 : 0; cc < (half ? MM : 5); ++cc) {
        uint32_t rr[16];
        umma::tmem_ld16(t_dv + lane_base + cc * 16, rr);
        float v[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) v[t] = __uint_as_float(rr[t]);
        if (kin) {
          uint4* dst = reinterpret_cast<uint4*>(dv + ((size_t)kj * MM + cc) * 128 + HD * h);
          dst[0] = pack8(v);
          dst[1] = pack8(v + 8);
        }
      }
      umma::tc_fence_before();
      umma::mbar_arrive(epi_done);
    }
  } else {
    // ================= query-side source coupling dOg (+ K_h rows 0-2 into TMEM) (warps 10-13)
    const int vt_id = tid - 320;
    const int vc = vt_id & 15, vjp = vt_id >> 4;  // channel, query pair (2 vjp, 2 vjp + 1)
    load_k(0);
    int g0 = 0;
    for (int h = 0; h < 8; ++h) {
      if (h + 1 < 8 && kin)  // next head's K rows into L2 while this head runs
        for (int m = 0; m < MM; ++m) asm volatile("prefetch.global.L2 [%0];" ::"l"(krow + m * 256 + DH * (h + 1)));
      for (int c = 0; c < nch; ++c) {
        const int g = g0 + c, b = g & 1, st = g % KV_NA;
        umma::mbar_wait(&full_a[st], (g / KV_NA) & 1);
        KV_TRACE(vt_id == 0, 8, g);
        const unsigned short* ost = reinterpret_cast<const unsigned short*>(sm + st * KV_ASTAGE + KV_QB);
        float d2[MM][2];
#pragma unroll
        for (int o = 0; o < MM; ++o)
#pragma unroll
          for (int t = 0; t < 2; ++t)
            d2[o][t] = __uint_as_float((uint32_t)ost[((2 * vjp + t) * MM + o) * HD + vc] << 16);
        umma::mbar_arrive(&empty_a[st]);
        if (g >= 2) umma::mbar_wait(&wv_free[b], ((g >> 1) - 1) & 1);  // dOg buffer b free
        uint8_t* dog = sm + KV_SM_DOG + b * GBYTES;
        if (!(a.dbg & 2))
          es_vgT_all(d2, [&](int ip, int f, float x0, float x1) {
            const __nv_bfloat162 pk = __floats2bfloat162_rn(x0, x1);
            *reinterpret_cast<uint32_t*>(dog + cm_off(ip * HD + vc, kv_k(f, 2 * vjp))) =
                *reinterpret_cast<const uint32_t*>(&pk);
          });
        umma::fence_proxy_async();
        umma::mbar_arrive(&dog_full[b]);
        KV_TRACE(vt_id == 0, 9, g);
      }
      g0 += nch;
      if (h + 1 < 8) {  // K_(h+1) rows 0-2 once the head's last S MMA is done (its dOg all produced: no cycle)
        KV_TRACE(vt_id == 0, 11, 32 + h);
        umma::mbar_wait(k_free, h & 1);
        KV_TRACE(vt_id == 0, 11, 40 + h);
        umma::tc_fence_after();
        if (a.dbg & 32) umma::mbar_arrive(k_ready);
        else load_k(h + 1);
        KV_TRACE(vt_id == 0, 11, 48 + h);
      }
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, 512);
#ifdef ES_TC_TRACE
  if (KTRACE && tid == 0) {
    const long long t0 = g_ktrace[0][0];
    printf("KTRACE nch=%d\n", nch);
    for (int g = 0; g < 8 * nch && g < 256; ++g)
      printf("KTRACE g=%d tmaA=%lld S=%lld D=%lld V=%lld rowW=%lld rowM=%lld rowWt=%lld rowE=%lld cpA=%lld cpE=%lld\n", g,
             g_ktrace[0][g] - t0, g_ktrace[1][g] - t0, g_ktrace[2][g] - t0, g_ktrace[3][g] - t0, g_ktrace[4][g] - t0,
             g_ktrace[5][g] - t0, g_ktrace[6][g] - t0, g_ktrace[7][g] - t0, g_ktrace[8][g] - t0, g_ktrace[9][g] - t0);
    for (int h = 0; h < 8; ++h)
      printf("KTRACE h=%d k_ready=%lld vh_full=%lld epi_wait=%lld epi_go=%lld rowK0=%lld rowK1=%lld cpVdone=%lld "
             "cpKfree=%lld cpK1=%lld\n", h, g_ktrace[10][h] - t0, g_ktrace[10][8 + h] - t0, g_ktrace[11][h] - t0,
             g_ktrace[11][8 + h] - t0, g_ktrace[11][16 + h] - t0, g_ktrace[11][24 + h] - t0, g_ktrace[11][32 + h] - t0,
             g_ktrace[11][40 + h] - t0, g_ktrace[11][48 + h] - t0);
  }
#endif
}
}  // namespace

bool attn_kv_tc_applicable(const AttnArgs& a) {
  const char* e = getenv("ES_KV_TC");  // read per call: the tests switch it
  if (e && e[0] == '0') return false;
  return attn_dq_tc_applicable(a) && a.N == a.Nk && a.row0 == 0;
}

size_t attn_kv_tc_geom_bytes(const AttnArgs& a) { return align256((size_t)a.N * a.K * sizeof(PairGeom)); }

es_status attn_kv_tc_launch(const AttnArgs& a, const void* q, const void* k, const void* v, const double* pos,
                            const int32_t* rev_ptr, const int32_t* rev_pair, const float* lse, const void* dout,
                            const float* delta, float* dsbuf, void* dv, void* geom_ws, cudaStream_t st) {
  if (a.N == 0) return ES_OK;
  if (!a.tiles) return fail(ES_INVALID_ARGUMENT, "attn_kv_tc: needs the key-side tile lists");
  if (!geom_ws) return fail(ES_INVALID_ARGUMENT, "attn_kv_tc: no pair-geometry workspace");
  es_status s = upload_tc_tables();
  if (s != ES_OK) return s;
  const TcScratch t = tc_scratch(key_side(a));
  const TcPtrs pp = tc_ptrs(const_cast<char*>(static_cast<const char*>(a.tiles)) + tiles_query_bytes(a), t);
  CUtensorMap mq, mo, mvh;
  if (!map3t(&mq, q, 256, MM, a.N, DH, KC, MM, CU_TENSOR_MAP_SWIZZLE_64B) ||
      !map3(&mo, dout, 128, MM, a.N, HD, MM, KC, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !map3t(&mvh, v, 128, MM, a.Nk, HD, TQ, MM, CU_TENSOR_MAP_SWIZZLE_32B))
    return fail(ES_CUDA_ERROR, "attn_kv_tc: tensor map encode failed");
  TcArgs ta{};
  ta.N = a.N; ta.K = a.K; ta.row0 = a.row0; ta.Nk = a.Nk;
  ta.tau = a.tau; ta.r_cut = a.r_cut; ta.inv_rcut = 1.f / a.r_cut;
  ta.phi_mode = a.phi_mode; ta.periodic = a.periodic;
  ta.bx = a.box[0]; ta.by = a.box[1]; ta.bz = a.box[2];
  ta.bias_mode = a.bias_mode; ta.b0 = a.bias[0]; ta.b1 = a.bias[1]; ta.b2 = a.bias[2];
  {  // profiling switches (ES_KV_DBG, outputs wrong): 1 no pair math, 2 no dOg math, 4 no D MMA,
     // 8 no dV MMA, 16 no S MMA, 32 no per-head K reload (coupling rows)
    const char* e = getenv("ES_KV_DBG");
    ta.dbg = e ? atoi(e) : 0;
  }
  PairGeom* geom = static_cast<PairGeom*>(geom_ws);
  attn_pair_geom_kernel<<<(unsigned)(((size_t)a.Nk * 4 + 255) / 256), 256, 0, st>>>(ta, pos, rev_ptr, rev_pair, geom);
  const int smem = KV_SM_TOTAL + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_kv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  attn_kv_tc_kernel<<<t.ntiles, TC_THREADS, smem, st>>>(mq, mo, mvh, ta, (const bf16*)k, pos, lse, delta, pp.cptr,
                                                        pp.clist, pp.rowlist, pp.tstart, rev_ptr, geom, dsbuf,
                                                        (bf16*)dv);
  return cuda_status(cudaGetLastError(), "attn_kv_tc_kernel");
}

}  // namespace es
