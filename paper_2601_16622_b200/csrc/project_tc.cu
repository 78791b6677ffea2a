// tcgen05 / TMEM / TMA projections for the bf16 path (north-star subsystem 1):
// Eq. (6) + W_H per degree l as UMMA GEMMs, operands staged by TMA with
// 128-byte swizzle, fp32 accumulators in tensor memory, epilogue from TMEM.
//
//   fwd : Y[(n,l,m), o]  = h[n,(l,m),:] . W[l][:, o]        A K-major (h rows), B MN-major (W as stored)
//   dh  : dh[(n,l,m), c] = G[n,(l,m),:] . W[l][c, :]        A K-major (dq|dk|dv rows), B K-major (W rows)
//   dW  : dW[l][c, o]   += sum_(n,m) h[.,c] G[., o]         A MN-major (h), B MN-major (G); split-K, fp32 red
// where G = [dq | dk | dv] along o.  The rows of degree l are the (n, m)
// pairs of the irreps layout -- a 3-D TMA box (C, M, N) picks them without
// any host-side re-layout.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>

#include "es_internal.h"
#include "umma.cuh"

namespace es {

namespace {

using bf16 = __nv_bfloat16;

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

// bf16 tensor map, dims innermost-first, 128B swizzle
bool make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
              const uint32_t* box, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn f = encode_fn();
  if (!f) return false;
  cuuint64_t gd[5], gs[4];
  cuuint32_t bd[5], es_[5];
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bd[i] = box[i];
    es_[i] = 1;
  }
  for (int i = 0; i < rank - 1; ++i) gs[i] = strides_bytes[i];
  return f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), gd, gs, bd, es_,
           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct TcP {
  int N, M, C, L;
};

__device__ __forceinline__ int degree_of_row(int mm) {
  int l = 0;
  while ((l + 1) * (l + 1) <= mm) ++l;
  return l;
}

__device__ __forceinline__ void store_row32(bf16* dst, const uint32_t (&r)[32]) {
  uint4 pk[4];
  uint32_t* w = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(r[2 * t]), __uint_as_float(r[2 * t + 1]));
    w[t] = *reinterpret_cast<const uint32_t*>(&b);
  }
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int t = 0; t < 4; ++t) d[t] = pk[t];
}

// ------------------------------------------------------------------ forward
// grid (ceil(N/128), M): tile = 128 atoms at one (l,m) row; the A tile
// (h rows, K = C = 128) is loaded ONCE and the five 128-column chunks of
// [Q1|Q2|K1|K2|H] stream through a double-buffered B stage and a
// double-buffered TMEM accumulator, so the epilogue of chunk c (TMEM ->
// bf16 rows, warps 0-3) overlaps the MMA of chunk c+1.  Warp 4 (one lane)
// issues TMA + MMA.
#ifndef ES_PF_NBUF
#define ES_PF_NBUF 1
#endif
constexpr int NBUF = ES_PF_NBUF;  // B stages = TMEM accumulators; 1: ~75 KB smem, 128 TMEM columns -> 3 CTAs per SM
__global__ void __launch_bounds__(160) proj_fwd_tc_kernel(const __grid_constant__ CUtensorMap mh,
                                                          const __grid_constant__ CUtensorMap mw, TcP p,
                                                          const __grid_constant__ CUtensorMap mq,
                                                          const __grid_constant__ CUtensorMap mk,
                                                          const __grid_constant__ CUtensorMap mv) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (umma::smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in .shared
  uint8_t* As = smem;                 // [2 kb][128 rows][64] bf16, 16 KB each
  uint8_t* Bs = smem + 32768;         // [NBUF stages][2 kb][2 nb][64 k-rows][64] bf16, 32 KB per stage
  uint8_t* Stg = smem + 32768 + NBUF * 32768;  // [4 warps][32 rows][64 B] epilogue staging (TMA-store SW64 box)
  uint64_t* bars = reinterpret_cast<uint64_t*>(Stg + 4 * 2048);
  uint64_t* a_full = bars + 0;
  uint64_t* b_full = bars + 1;        // [2]
  uint64_t* b_empty = bars + 3;       // [2] MMA done reading the stage
  uint64_t* acc_full = bars + 5;      // [2]
  uint64_t* acc_free = bars + 7;      // [2] epilogue read the accumulator (128)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 9);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid (M, tiles): the M rows of one atom tile run side by side -> their writes land on neighbouring DRAM rows
  const int n0 = blockIdx.y * 128, mm = blockIdx.x;
  const int l = degree_of_row(mm);
  constexpr int NCH = 5;
  if (threadIdx.x == 0) {
    umma::prefetch_tmap(&mh);
    umma::prefetch_tmap(&mw);
    umma::mbar_init(a_full, 1);
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&b_full[b], 1);
      umma::mbar_init(&b_empty[b], 1);
      umma::mbar_init(&acc_full[b], 1);
      umma::mbar_init(&acc_free[b], 128);
    }
    umma::fence_barrier_init();
  }
  if (warp == 0) umma::tmem_alloc(tslot, 128 * NBUF);
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t taddr = *tslot;
  if (warp == 4) {
    if (lane == 0) {
    auto load_b = [&](int c) {
      uint8_t* B = Bs + (c % NBUF) * 32768;
      umma::mbar_arrive_expect_tx(&b_full[c % NBUF], 32768);
#pragma unroll
      for (int kb = 0; kb < 2; ++kb)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
          umma::tma_load_2d(B + (kb * 2 + nb) * 8192, &mw, &b_full[c % NBUF], c * 128 + 64 * nb, l * p.C + 64 * kb);
    };
    umma::mbar_arrive_expect_tx(a_full, 32768);
    umma::tma_load_3d(As, &mh, a_full, 0, mm, n0);
    umma::tma_load_3d(As + 16384, &mh, a_full, 64, mm, n0);
    for (int c = 0; c < NBUF; ++c) load_b(c);
    umma::mbar_wait(a_full, 0);
    constexpr uint32_t idesc = umma::idesc_bf16(128, 128, 0, 1);
    for (int c = 0; c < NCH; ++c) {
      const int b = c % NBUF;
      umma::mbar_wait(&b_full[b], (c / NBUF) & 1);
      if (c >= NBUF) umma::mbar_wait(&acc_free[b], ((c / NBUF) - 1) & 1);
      umma::tc_fence_after();
      const uint8_t* B = Bs + b * 32768;
      // descriptors advance by (byte offset >> 4) from one base (no per-MMA descriptor arithmetic
      // on the single issuing thread)
      const uint64_t ad0 = umma::sdesc(umma::smem_u32(As), 16, 1024), bd0 = umma::sdesc(umma::smem_u32(B), 8192, 1024);
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int kb = s >> 2, ks = s & 3;
        umma::mma_f16(taddr + 128 * b, ad0 + (uint64_t)((kb * 16384 + ks * 32) >> 4),
                      bd0 + (uint64_t)((kb * 16384 + ks * 2048) >> 4), idesc, s > 0 ? 1u : 0u);
      }
      umma::mma_commit(&acc_full[b]);
      umma::mma_commit(&b_empty[b]);
      if (c + NBUF < NCH) {
        umma::mbar_wait(&b_empty[b], (c / NBUF) & 1);
        load_b(c + NBUF);
      }
    }
    }
  } else {
  for (int c = 0; c < NCH; ++c) {
    const int b = c % NBUF, o0 = c * 128;
    umma::mbar_wait(&acc_full[b], (c / NBUF) & 1);
    umma::tc_fence_after();
    // rows -> per-warp staging (32 rows x 32 columns, the 64-byte-swizzled layout of a TMA box:
    // conflict-free, lane = row) -> one TMA store per 32 x 32 block, clipped at N by the tensor map
    uint8_t* stg = Stg + warp * 2048;
    const CUtensorMap* om = o0 < 2 * p.C ? &mq : o0 < 4 * p.C ? &mk : &mv;
    const int oc = o0 < 2 * p.C ? o0 : o0 < 4 * p.C ? o0 - 2 * p.C : o0 - 4 * p.C;
#pragma unroll 1
    for (int cc = 0; cc < 4; ++cc) {
      uint32_t r[32];
      umma::tmem_ld32(taddr + 128 * b + ((uint32_t)(warp * 32) << 16) + cc * 32, r);
      uint4 pk[4];
      uint32_t* w = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(r[2 * t]), __uint_as_float(r[2 * t + 1]));
        w[t] = *reinterpret_cast<const uint32_t*>(&h2);
      }
      if (lane == 0) umma::bulk_wait_read0();  // the previous block's store has read the staging buffer
      __syncwarp();
#pragma unroll
      for (int t = 0; t < 4; ++t)
        *reinterpret_cast<uint4*>(stg + lane * 64 + ((t ^ ((lane >> 1) & 3)) << 4)) = pk[t];
      umma::fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        umma::tma_store_3d(om, stg, oc + cc * 32, mm, n0 + warp * 32);
        umma::bulk_commit();
      }
    }
    umma::tc_fence_before();
    umma::mbar_arrive(&acc_free[b]);
  }
  }
  if (warp < 4 && lane == 0) umma::bulk_wait0();  // stores complete before the CTA's shared memory goes
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(taddr, 128 * NBUF);
}

// ------------------------------------------------------------------ dh
// grid (ceil(N/128), M): tile = 128 atoms at (l,m) x 128 channels; K = 5C in 64-wide blocks.
#ifndef ES_DH_STAGES
#define ES_DH_STAGES 2
#endif
constexpr int kDhStages = ES_DH_STAGES;  // 2 x 32 KB: three CTAs per SM (short CTAs: residency beats depth)
__global__ void __launch_bounds__(128) proj_dh_tc_kernel(const __grid_constant__ CUtensorMap mdq,
                                                         const __grid_constant__ CUtensorMap mdk,
                                                         const __grid_constant__ CUtensorMap mdv,
                                                         const __grid_constant__ CUtensorMap mwk, TcP p,
                                                         bf16* __restrict__ dh) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (umma::smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in .shared
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kDhStages * 32768);
  uint64_t* empty = full + kDhStages;
  uint64_t* done = empty + kDhStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid (M, tiles): the M rows of one atom tile run side by side -> their writes land on neighbouring DRAM rows
  const int n0 = blockIdx.y * 128, mm = blockIdx.x;
  const int l = degree_of_row(mm);
  const int nkb = (5 * p.C) / 64, kq = (2 * p.C) / 64;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDhStages; ++s) {
      umma::mbar_init(&full[s], 1);
      umma::mbar_init(&empty[s], 1);
    }
    umma::mbar_init(done, 1);
    umma::fence_barrier_init();
  }
  if (warp == 0) umma::tmem_alloc(tslot, 128);
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t taddr = *tslot;
  if (warp == 0 && lane == 0) {  // TMA producer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kDhStages, round = kb / kDhStages;
      if (round > 0) umma::mbar_wait(&empty[s], (round - 1) & 1);
      uint8_t* A = smem + s * 32768;
      umma::mbar_arrive_expect_tx(&full[s], 32768);
      if (kb < kq) umma::tma_load_3d(A, &mdq, &full[s], kb * 64, mm, n0);
      else if (kb < 2 * kq) umma::tma_load_3d(A, &mdk, &full[s], (kb - kq) * 64, mm, n0);
      else umma::tma_load_3d(A, &mdv, &full[s], (kb - 2 * kq) * 64, mm, n0);
      umma::tma_load_2d(A + 16384, &mwk, &full[s], kb * 64, l * p.C);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    constexpr uint32_t idesc = umma::idesc_bf16(128, 128, 0, 0);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kDhStages, round = kb / kDhStages;
      umma::mbar_wait(&full[s], round & 1);
      umma::tc_fence_after();
      const uint32_t a0 = umma::smem_u32(smem + s * 32768);
      const uint64_t ad0 = umma::sdesc(a0, 16, 1024), bd0 = umma::sdesc(a0 + 16384, 16, 1024);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
        umma::mma_f16(taddr, ad0 + (uint64_t)(2 * ks), bd0 + (uint64_t)(2 * ks), idesc, (kb | ks) ? 1u : 0u);
      umma::mma_commit(&empty[s]);
    }
    umma::mma_commit(done);
  }
  umma::mbar_wait(done, 0);
  umma::tc_fence_after();
  // staged, coalesced epilogue (see proj_fwd_tc_kernel); staging reuses
  // pipeline stage 0, free once `done` fired
  uint8_t* stg = smem + warp * (32 * 80);
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) {
    uint32_t r[32];
    umma::tmem_ld32(taddr + ((uint32_t)(warp * 32) << 16) + cc * 32, r);
    uint4 pk[4];
    uint32_t* w = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(r[2 * t]), __uint_as_float(r[2 * t + 1]));
      w[t] = *reinterpret_cast<const uint32_t*>(&h2);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) *reinterpret_cast<uint4*>(stg + lane * 80 + t * 16) = pk[t];
    __syncwarp();
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int rr = it * 8 + (lane >> 2), part = lane & 3;
      const int nn = n0 + warp * 32 + rr;
      if (nn < p.N)
        *reinterpret_cast<uint4*>(dh + ((size_t)nn * p.M + mm) * p.C + cc * 32 + part * 8) =
            *reinterpret_cast<const uint4*>(stg + rr * 80 + part * 16);
    }
    __syncwarp();
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(taddr, 128);
}

// ------------------------------------------------------------------ dW
// grid (splits, 5): split-K over atoms for one degree l (R = (2l+1)*nb rows
// per stage); D = [c 128] x [o 128]; fp32 reduction into dW.
#ifndef ES_DW_STAGES
#define ES_DW_STAGES 2
#endif
constexpr int kDwStages = ES_DW_STAGES;
#ifndef ES_DW_SPLITS
#define ES_DW_SPLITS 60  // fallback atom splits per degree (x 5 column blocks); the launcher uses 2 x SMs / 5
#endif
__global__ void __launch_bounds__(128) proj_dw_tc_kernel(const __grid_constant__ CUtensorMap mh,
                                                         const __grid_constant__ CUtensorMap mdq,
                                                         const __grid_constant__ CUtensorMap mdk,
                                                         const __grid_constant__ CUtensorMap mdv, TcP p, int l,
                                                         int nb, int atoms_per_split, float* __restrict__ dW) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (umma::smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in .shared
  const int R = (2 * l + 1) * nb;
  const int half = R * 128;       // one 64-wide MN block: R rows x 128 B
  const int stage_bytes = 4 * half;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kDwStages * stage_bytes);
  uint64_t* empty = full + kDwStages;
  uint64_t* done = empty + kDwStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunk = blockIdx.y, o0 = chunk * 128;
  const int a_begin = blockIdx.x * atoms_per_split;
  const int a_end = min(p.N, a_begin + atoms_per_split);
  const int nst = a_end > a_begin ? (a_end - a_begin + nb - 1) / nb : 0;
  const CUtensorMap* mg = o0 < 2 * p.C ? &mdq : (o0 < 4 * p.C ? &mdk : &mdv);
  const int og = o0 < 2 * p.C ? o0 : (o0 < 4 * p.C ? o0 - 2 * p.C : o0 - 4 * p.C);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDwStages; ++s) {
      umma::mbar_init(&full[s], 1);
      umma::mbar_init(&empty[s], 1);
    }
    umma::mbar_init(done, 1);
    umma::fence_barrier_init();
  }
  if (warp == 0) umma::tmem_alloc(tslot, 128);
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t taddr = *tslot;
  if (nst > 0) {
    if (warp == 0 && lane == 0) {
      for (int it = 0; it < nst; ++it) {
        const int s = it % kDwStages, round = it / kDwStages;
        if (round > 0) umma::mbar_wait(&empty[s], (round - 1) & 1);
        uint8_t* st = smem + s * stage_bytes;
        const int na = a_begin + it * nb;
        umma::mbar_arrive_expect_tx(&full[s], stage_bytes);
        umma::tma_load_3d(st, &mh, &full[s], 0, l * l, na);
        umma::tma_load_3d(st + half, &mh, &full[s], 64, l * l, na);
        umma::tma_load_3d(st + 2 * half, mg, &full[s], og, l * l, na);
        umma::tma_load_3d(st + 3 * half, mg, &full[s], og + 64, l * l, na);
      }
    } else if (warp == 1 && lane == 0) {
      constexpr uint32_t idesc = umma::idesc_bf16(128, 128, 1, 1);
      for (int it = 0; it < nst; ++it) {
        const int s = it % kDwStages, round = it / kDwStages;
        umma::mbar_wait(&full[s], round & 1);
        umma::tc_fence_after();
        const uint32_t a0 = umma::smem_u32(smem + s * stage_bytes);
        const uint64_t ad0 = umma::sdesc(a0, half, 1024), bd0 = umma::sdesc(a0 + 2 * half, half, 1024);
#pragma unroll 4
        for (int ks = 0; ks < R / 16; ++ks)
          umma::mma_f16(taddr, ad0 + (uint64_t)(128 * ks), bd0 + (uint64_t)(128 * ks), idesc, (it | ks) ? 1u : 0u);
        umma::mma_commit(&empty[s]);
      }
      umma::mma_commit(done);
    }
    umma::mbar_wait(done, 0);
    umma::tc_fence_after();
    const int c = warp * 32 + lane;
    float* dst = dW + ((size_t)l * p.C + c) * (5 * p.C) + o0;
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      uint32_t r[32];
      umma::tmem_ld32(taddr + ((uint32_t)(warp * 32) << 16) + cc * 32, r);
#pragma unroll
      for (int t = 0; t < 32; t += 4)  // vector reductions (sm_90+): a quarter of the atomic instructions
        atomicAdd(reinterpret_cast<float4*>(dst + cc * 32 + t),
                  make_float4(__uint_as_float(r[t]), __uint_as_float(r[t + 1]), __uint_as_float(r[t + 2]),
                              __uint_as_float(r[t + 3])));
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(taddr, 128);
}

bool map3(CUtensorMap* m, const void* base, int inner, int M, int N, int box0, int box1, int box2,
          CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  const uint64_t dims[3] = {(uint64_t)inner, (uint64_t)M, (uint64_t)N};
  const uint64_t strides[2] = {(uint64_t)inner * 2, (uint64_t)inner * M * 2};
  const uint32_t box[3] = {(uint32_t)box0, (uint32_t)box1, (uint32_t)box2};
  return make_map(m, base, 3, dims, strides, box, sw);
}
bool map2(CUtensorMap* m, const void* base, int inner, int rows, int box0, int box1) {
  const uint64_t dims[2] = {(uint64_t)inner, (uint64_t)rows};
  const uint64_t strides[1] = {(uint64_t)inner * 2};
  const uint32_t box[2] = {(uint32_t)box0, (uint32_t)box1};
  return make_map(m, base, 2, dims, strides, box);
}

}  // namespace

bool proj_tc_supported(const ProjArgs& a) {
  return a.dtype == ES_BF16 && a.C == 128 && a.Dq == 2 * a.C && a.Cv == a.C && encode_fn() != nullptr;
}

es_status proj_fwd_tc_launch(const ProjArgs& a, const void* h, const void* W, void* q, void* k, void* v,
                             cudaStream_t st) {
  const int M = (a.L + 1) * (a.L + 1);
  CUtensorMap mh, mw;
  CUtensorMap mq, mk, mv;  // output boxes [32 rows][1 (l,m)][32 columns], 64-byte swizzle
  if (!map3(&mh, h, a.C, M, a.N, 64, 1, 128) || !map2(&mw, W, 5 * a.C, (a.L + 1) * a.C, 64, 64) ||
      !map3(&mq, q, 2 * a.C, M, a.N, 32, 1, 32, CU_TENSOR_MAP_SWIZZLE_64B) ||
      !map3(&mk, k, 2 * a.C, M, a.N, 32, 1, 32, CU_TENSOR_MAP_SWIZZLE_64B) ||
      !map3(&mv, v, a.C, M, a.N, 32, 1, 32, CU_TENSOR_MAP_SWIZZLE_64B))
    return fail(ES_CUDA_ERROR, "proj_fwd_tc: tensor map encode failed");
  const size_t smem = 32768 + NBUF * 32768 + 4 * 2048 + 1024 + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(proj_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  TcP p{a.N, M, a.C, a.L};
  dim3 grid(M, (a.N + 127) / 128);
  proj_fwd_tc_kernel<<<grid, 160, smem, st>>>(mh, mw, p, mq, mk, mv);
  return cuda_status(cudaGetLastError(), "proj_fwd_tc_kernel");
}

es_status proj_bwd_tc_launch(const ProjArgs& a, const void* h, const void* W, const void* dq, const void* dk,
                             const void* dv, void* dh, float* dW, cudaStream_t st) {
  const int M = (a.L + 1) * (a.L + 1);
  TcP p{a.N, M, a.C, a.L};
  CUtensorMap mdq, mdk, mdv, mwk;
  if (!map3(&mdq, dq, 2 * a.C, M, a.N, 64, 1, 128) || !map3(&mdk, dk, 2 * a.C, M, a.N, 64, 1, 128) ||
      !map3(&mdv, dv, a.C, M, a.N, 64, 1, 128) || !map2(&mwk, W, 5 * a.C, (a.L + 1) * a.C, 64, 128))
    return fail(ES_CUDA_ERROR, "proj_bwd_tc: tensor map encode failed");
  {
    const size_t smem = kDhStages * 32768 + 1024 + 1024;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(proj_dh_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    dim3 grid(M, (a.N + 127) / 128);
    proj_dh_tc_kernel<<<grid, 128, smem, st>>>(mdq, mdk, mdv, mwk, p, (bf16*)dh);
    es_status s = cuda_status(cudaGetLastError(), "proj_dh_tc_kernel");
    if (s != ES_OK) return s;
  }
  if (!dW) return ES_OK;
  cudaMemsetAsync(dW, 0, sizeof(float) * (size_t)(a.L + 1) * a.C * 5 * a.C, st);
  static bool attr_dw = false;
  if (!attr_dw) {
    cudaFuncSetAttribute(proj_dw_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_dw = true;
  }
  for (int l = 0; l <= a.L; ++l) {
    const int nb = l == 0 ? 64 : 16;
    const int R = (2 * l + 1) * nb;
    CUtensorMap mh, gq, gk, gv;
    if (!map3(&mh, h, a.C, M, a.N, 64, 2 * l + 1, nb) || !map3(&gq, dq, 2 * a.C, M, a.N, 64, 2 * l + 1, nb) ||
        !map3(&gk, dk, 2 * a.C, M, a.N, 64, 2 * l + 1, nb) || !map3(&gv, dv, a.C, M, a.N, 64, 2 * l + 1, nb))
      return fail(ES_CUDA_ERROR, "proj_dw_tc: tensor map encode failed");
    const size_t smem = (size_t)kDwStages * 4 * R * 128 + 1024 + 1024;
    // atom splits: at most two resident CTAs per SM, all in one wave (5 column blocks each) -- 60 splits
    // put 300 CTAs on 296 slots at l = 2 (a second, nearly empty wave: 0.59 -> 0.47 ms at 59); more
    // CTAs per SM (l = 0, 1 fit 3-4) measured slower (smaller splits, more fp32 atomics).
    // ES_DW_SPLITS overrides
    int splits = ES_DW_SPLITS;
    {
      static int nsm = 0;
      if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      }
      if (nsm > 0) splits = std::max(1, 2 * nsm / 5);  // two 82 KB CTAs per SM at l = 2
      const char* e = getenv("ES_DW_SPLITS");
      if (e && atoi(e) > 0) splits = atoi(e);
    }
    int per = (a.N + splits - 1) / splits;
    per = ((per + nb - 1) / nb) * nb;
    splits = (a.N + per - 1) / per;
    dim3 grid(splits, 5);
    proj_dw_tc_kernel<<<grid, 128, smem, st>>>(mh, gq, gk, gv, p, l, nb, per, dW);
    es_status s = cuda_status(cudaGetLastError(), "proj_dw_tc_kernel");
    if (s != ES_OK) return s;
  }
  return ES_OK;
}

}  // namespace es
