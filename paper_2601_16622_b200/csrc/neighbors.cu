// Neighbour index builder (build_neighbors) + transposed
// relation + tile-skip mask, sm_100a.
//
// Bit-exactness contract with the CPU oracle: every candidate's squared
// distance is ((dx*dx + dy*dy) + dz*dz) in double, each operation rounded
// to nearest with no FMA contraction (__dmul_rn / __dadd_rn), minimum image
// dx - box*rint(dx/box) under PBC; a pair is kept iff d2 < r_cut^2 (strict),
// j != i, same segment; the list is the K smallest by (d2, j).  Since the
// output is a pure function of that candidate set, the search structure
// (hashed cell grid or per-segment scan) cannot change a single bit.
//
// Search structures:
//  * segmented input (molecule batches): warp per atom over its segment,
//    slots by rank (nbr_segment_warp_kernel);
//  * one system: hashed uniform grid, cell edge >= r_cut, 27-cell stencil,
//    exact cell-coordinate filter against hash collisions; under PBC the grid
//    tiles the box (>= 3 cells per axis).
#include <cub/cub.cuh>

#include "es_internal.h"

namespace es {

constexpr int kMaxK = 128;

__device__ __forceinline__ double d2_exact(double xi, double yi, double zi, double xj, double yj, double zj,
                                           int periodic, double bx, double by, double bz) {
  double dx = __dsub_rn(xj, xi), dy = __dsub_rn(yj, yi), dz = __dsub_rn(zj, zi);
  if (periodic) {
    // |dx| < box/2 => rint(dx/box) == 0 exactly (a correctly rounded quotient can reach 0.5 at most,
    // which rounds to even 0): the fp64 divisions run only for pairs that actually wrap
    if (!(fabs(dx) < 0.5 * bx)) dx = __dsub_rn(dx, __dmul_rn(bx, rint(__ddiv_rn(dx, bx))));
    if (!(fabs(dy) < 0.5 * by)) dy = __dsub_rn(dy, __dmul_rn(by, rint(__ddiv_rn(dy, by))));
    if (!(fabs(dz) < 0.5 * bz)) dz = __dsub_rn(dz, __dmul_rn(bz, rint(__ddiv_rn(dz, bz))));
  }
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

struct TopK {
  double d2[kMaxK];
  int j[kMaxK];
  int n;
  __device__ void insert(double d, int jj, int K) {
    if (n == K) {
      if (d > d2[K - 1] || (d == d2[K - 1] && jj > j[K - 1])) return;
      --n;
    }
    int p = n;
    while (p > 0 && (d2[p - 1] > d || (d2[p - 1] == d && j[p - 1] > jj))) {
      d2[p] = d2[p - 1];
      j[p] = j[p - 1];
      --p;
    }
    d2[p] = d;
    j[p] = jj;
    ++n;
  }
};

struct NbrK {
  int N, K, nseg, periodic;
  int row0, nrows;  // query rows [row0, row0 + nrows) are searched; outputs are indexed by i - row0
  double rc2, bx, by, bz;
};

__device__ __forceinline__ void emit(const NbrK& p, int i, const TopK& t, int32_t* nbr, float* dist, int32_t* count) {
  i -= p.row0;
  for (int s = 0; s < p.K; ++s) {
    nbr[(size_t)i * p.K + s] = s < t.n ? t.j[s] : -1;
    if (dist) dist[(size_t)i * p.K + s] = s < t.n ? (float)sqrt(t.d2[s]) : 0.f;
  }
  count[i] = t.n;
}

// Warp per atom: the lanes evaluate candidates 32 at a time and compact the
// kept ones (d2 < r_cut^2, j != i) into shared memory; each kept candidate's
// slot is then its rank under (d2, j) -- the same order the sorted top-K
// produces -- so no per-thread sorted list (TopK lives in local memory).  The
// buffer bounds the KEPT candidates (an atom's neighbours within r_cut), not
// the segment or cell population; an atom with more falls back to lane 0's
// TopK scan of the same candidate set.
constexpr int SEG_WARP_MAX = 256;
constexpr int SEG_WARPS = 8;

struct WarpCand {  // one warp's kept-candidate buffer
  double* cd;
  int* cj;
  int n;
  // lanes offer (d, j, keep); the kept ones are appended in lane order
  __device__ __forceinline__ void offer(bool keep, double d, int j, int lane) {
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const int at = n + __popc(m & ((1u << lane) - 1u));
      if (at < SEG_WARP_MAX) {
        cd[at] = d;
        cj[at] = j;
      }
    }
    n += __popc(m);
  }
  // slots by rank under (d2, j); returns false when the buffer overflowed (caller falls back)
  __device__ __forceinline__ bool emit_ranked(const NbrK& p, int r, int lane, int32_t* nbr, float* dist,
                                              int32_t* count) const {
    if (n > SEG_WARP_MAX) return false;
    __syncwarp();
    const int K = p.K;
    int32_t* orow = nbr + (size_t)r * K;
    float* drow = dist ? dist + (size_t)r * K : nullptr;
    for (int c = lane; c < n; c += 32) {
      const double d = cd[c];
      const int j = cj[c];
      int rank = 0;
      for (int o = 0; o < n; ++o) {
        const double od = cd[o];
        rank += (od < d || (od == d && cj[o] < j)) ? 1 : 0;
      }
      if (rank < K) {
        orow[rank] = j;
        if (drow) drow[rank] = (float)sqrt(d);
      }
    }
    for (int s = min(n, K) + lane; s < K; s += 32) {
      orow[s] = -1;
      if (drow) drow[s] = 0.f;
    }
    if (lane == 0) count[r] = min(n, K);
    return true;
  }
};

__global__ void __launch_bounds__(SEG_WARPS * 32) nbr_segment_warp_kernel(NbrK p, const double* __restrict__ pos,
                                                                          const int32_t* __restrict__ seg_ptr,
                                                                          int32_t* __restrict__ nbr,
                                                                          float* __restrict__ dist,
                                                                          int32_t* __restrict__ count) {
  __shared__ double cd[SEG_WARPS][SEG_WARP_MAX];
  __shared__ int cj[SEG_WARPS][SEG_WARP_MAX];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * SEG_WARPS + warp;
  if (r >= p.nrows) return;
  const int i = p.row0 + r;
  int a0 = 0, a1 = p.N;
  if (seg_ptr) {
    int lo = 0, hi = p.nseg;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (seg_ptr[mid] <= i) lo = mid;
      else hi = mid;
    }
    a0 = seg_ptr[lo];
    a1 = seg_ptr[lo + 1];
  }
  const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
  WarpCand wc{cd[warp], cj[warp], 0};
  for (int j0 = a0; j0 < a1; j0 += 32) {
    const int j = j0 + lane;
    double d = 0.0;
    bool keep = false;
    if (j < a1 && j != i) {
      d = d2_exact(xi, yi, zi, pos[3 * j], pos[3 * j + 1], pos[3 * j + 2], p.periodic, p.bx, p.by, p.bz);
      keep = d < p.rc2;
    }
    wc.offer(keep, d, j, lane);
  }
  if (wc.emit_ranked(p, r, lane, nbr, dist, count)) return;
  if (lane == 0) {  // more than SEG_WARP_MAX atoms within r_cut: the sorted scan
    TopK t;
    t.n = 0;
    for (int j = a0; j < a1; ++j) {
      if (j == i) continue;
      const double d = d2_exact(xi, yi, zi, pos[3 * j], pos[3 * j + 1], pos[3 * j + 2], p.periodic, p.bx, p.by, p.bz);
      if (d < p.rc2) t.insert(d, j, p.K);
    }
    emit(p, i, t, nbr, dist, count);
  }
}

// ---------------------------------------------------------------- hashed grid
struct GridK {
  double cs[3];  // cell edge per axis
  int nc[3];     // cells per axis (PBC only)
  int periodic;
  unsigned mask;  // bucket count - 1
};

__device__ __forceinline__ unsigned cell_hash(int cx, int cy, int cz, unsigned mask) {
  return ((unsigned)cx * 73856093u ^ (unsigned)cy * 19349663u ^ (unsigned)cz * 83492791u) & mask;
}

__device__ __forceinline__ int4 cell_of(const GridK& g, double x, double y, double z, double bx, double by,
                                        double bz) {
  int4 c;
  if (g.periodic) {
    const double xw = x - bx * floor(x / bx), yw = y - by * floor(y / by), zw = z - bz * floor(z / bz);
    c.x = min(max((int)floor(xw / g.cs[0]), 0), g.nc[0] - 1);
    c.y = min(max((int)floor(yw / g.cs[1]), 0), g.nc[1] - 1);
    c.z = min(max((int)floor(zw / g.cs[2]), 0), g.nc[2] - 1);
  } else {
    c.x = (int)floor(x / g.cs[0]);
    c.y = (int)floor(y / g.cs[1]);
    c.z = (int)floor(z / g.cs[2]);
  }
  c.w = 0;
  return c;
}

__global__ void grid_key_kernel(int N, GridK g, NbrK p, const double* __restrict__ pos, unsigned* __restrict__ key,
                                int* __restrict__ idx, int4* __restrict__ cell) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int4 c = cell_of(g, pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], p.bx, p.by, p.bz);
  cell[i] = c;
  key[i] = cell_hash(c.x, c.y, c.z, g.mask);
  idx[i] = i;
}

__global__ void grid_bounds_kernel(int N, const unsigned* __restrict__ skey, int* __restrict__ start,
                                   int* __restrict__ end) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= N) return;
  const unsigned k = skey[s];
  if (s == 0 || skey[s - 1] != k) start[k] = s;
  if (s == N - 1 || skey[s + 1] != k) end[k] = s + 1;
}

// Warp per atom over the 27-cell stencil (the cell's candidates 32 at a time),
// compact + rank as in the segment kernel; lane 0's TopK scan on overflow.
__global__ void __launch_bounds__(SEG_WARPS * 32) nbr_grid_kernel(NbrK p, GridK g, const double* __restrict__ pos,
                                                                  const int4* __restrict__ cell,
                                                                  const int* __restrict__ sidx,
                                                                  const int* __restrict__ start,
                                                                  const int* __restrict__ end,
                                                                  int32_t* __restrict__ nbr, float* __restrict__ dist,
                                                                  int32_t* __restrict__ count) {
  __shared__ double cd[SEG_WARPS][SEG_WARP_MAX];
  __shared__ int cj[SEG_WARPS][SEG_WARP_MAX];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * SEG_WARPS + warp;
  if (r >= p.nrows) return;
  const int i = p.row0 + r;
  const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
  const int4 ci = cell[i];
  auto stencil = [&](auto&& visit) {
    for (int ox = -1; ox <= 1; ++ox)
      for (int oy = -1; oy <= 1; ++oy)
        for (int oz = -1; oz <= 1; ++oz) {
          int cx = ci.x + ox, cy = ci.y + oy, cz = ci.z + oz;
          if (g.periodic) {
            cx = (cx + g.nc[0]) % g.nc[0];
            cy = (cy + g.nc[1]) % g.nc[1];
            cz = (cz + g.nc[2]) % g.nc[2];
          }
          const unsigned h = cell_hash(cx, cy, cz, g.mask);
          visit(cx, cy, cz, start[h], end[h]);
        }
  };
  WarpCand wc{cd[warp], cj[warp], 0};
  stencil([&](int cx, int cy, int cz, int s0, int s1) {
    for (int b = s0; b < s1; b += 32) {
      const int s = b + lane;
      double d = 0.0;
      bool keep = false;
      int j = -1;
      if (s < s1) {
        j = sidx[s];
        const int4 cj4 = cell[j];
        if (cj4.x == cx && cj4.y == cy && cj4.z == cz && j != i) {  // hash collisions filtered exactly
          d = d2_exact(xi, yi, zi, pos[3 * j], pos[3 * j + 1], pos[3 * j + 2], p.periodic, p.bx, p.by, p.bz);
          keep = d < p.rc2;
        }
      }
      wc.offer(keep, d, j, lane);
    }
  });
  if (wc.emit_ranked(p, r, lane, nbr, dist, count)) return;
  if (lane == 0) {  // more than SEG_WARP_MAX atoms within r_cut: the sorted scan over the same stencil
    TopK t;
    t.n = 0;
    stencil([&](int cx, int cy, int cz, int s0, int s1) {
      for (int s = s0; s < s1; ++s) {
        const int j = sidx[s];
        const int4 cj4 = cell[j];
        if (cj4.x != cx || cj4.y != cy || cj4.z != cz || j == i) continue;
        const double d = d2_exact(xi, yi, zi, pos[3 * j], pos[3 * j + 1], pos[3 * j + 2], p.periodic, p.bx, p.by,
                                  p.bz);
        if (d < p.rc2) t.insert(d, j, p.K);
      }
    });
    emit(p, i, t, nbr, dist, count);
  }
}

namespace {
unsigned pow2_at_least(unsigned n) {
  unsigned b = 1024;
  while (b < n) b <<= 1;
  return b;
}
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct GridWs {
  size_t key, skey, idx, sidx, cell, start, end, cub, total;
  size_t cub_bytes;
};
GridWs grid_ws(int N) {
  GridWs w{};
  const unsigned nb = pow2_at_least(2u * (unsigned)N);
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (unsigned*)nullptr, (unsigned*)nullptr, (int*)nullptr,
                                  (int*)nullptr, N);
  size_t o = 0;
  w.key = o; o += align256(sizeof(unsigned) * N);
  w.skey = o; o += align256(sizeof(unsigned) * N);
  w.idx = o; o += align256(sizeof(int) * N);
  w.sidx = o; o += align256(sizeof(int) * N);
  w.cell = o; o += align256(sizeof(int4) * N);
  w.start = o; o += align256(sizeof(int) * nb);
  w.end = o; o += align256(sizeof(int) * nb);
  w.cub = o; o += align256(cub_bytes);
  w.cub_bytes = cub_bytes;
  w.total = o;
  return w;
}
bool use_grid(const NbrArgs& a) {
  if (a.nseg > 1) return false;
  if (a.N <= 1024) return false;
  if (a.periodic) {
    for (int d = 0; d < 3; ++d)
      if (a.box[d] / a.r_cut < 3.0) return false;
  }
  return true;
}
}  // namespace

size_t nbr_workspace_bytes(const NbrArgs& a) {
  if (!use_grid(a)) return 256;
  return grid_ws(a.N).total;
}

es_status nbr_build_launch(const NbrArgs& a, const double* pos, const int32_t* seg_ptr, int32_t* nbr, float* dist,
                           int32_t* count, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (a.K > kMaxK) return fail(ES_UNSUPPORTED, "neighbors: K > 128");
  if (a.N == 0 || a.nrows == 0) return ES_OK;
  NbrK p;
  p.N = a.N; p.K = a.K; p.nseg = a.nseg; p.periodic = a.periodic;
  p.row0 = a.row0; p.nrows = a.nrows;
  p.rc2 = a.r_cut * a.r_cut;
  p.bx = a.box[0]; p.by = a.box[1]; p.bz = a.box[2];
  const int tpb = 128, blocks = (a.N + tpb - 1) / tpb;
  if (!use_grid(a)) {
    const int32_t* sp = (seg_ptr && a.nseg >= 1) ? seg_ptr : nullptr;  // NULL: one segment [0, N)
    nbr_segment_warp_kernel<<<(a.nrows + SEG_WARPS - 1) / SEG_WARPS, SEG_WARPS * 32, 0, st>>>(p, pos, sp, nbr, dist,
                                                                                           count);
    return cuda_status(cudaGetLastError(), "nbr_segment_warp_kernel");
  }
  const GridWs w = grid_ws(a.N);
  if (ws_bytes < w.total) return fail(ES_INVALID_ARGUMENT, "neighbors: workspace too small");
  char* base = (char*)ws;
  GridK g;
  g.periodic = a.periodic;
  for (int d = 0; d < 3; ++d) {
    if (a.periodic) {
      g.nc[d] = (int)floor(a.box[d] / a.r_cut);
      g.cs[d] = a.box[d] / g.nc[d];
    } else {
      g.nc[d] = 0;
      g.cs[d] = a.r_cut * 1.000001;
    }
  }
  const unsigned nb = pow2_at_least(2u * (unsigned)a.N);
  g.mask = nb - 1;
  unsigned* key = (unsigned*)(base + w.key);
  unsigned* skey = (unsigned*)(base + w.skey);
  int* idx = (int*)(base + w.idx);
  int* sidx = (int*)(base + w.sidx);
  int4* cell = (int4*)(base + w.cell);
  int* start = (int*)(base + w.start);
  int* end = (int*)(base + w.end);
  grid_key_kernel<<<blocks, tpb, 0, st>>>(a.N, g, p, pos, key, idx, cell);
  size_t cb = w.cub_bytes;
  int bits = 1;
  while ((1u << bits) < nb) ++bits;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(base + w.cub, cb, key, skey, idx, sidx, a.N, 0, bits, st);
  if (e != cudaSuccess) return cuda_status(e, "neighbors: radix sort");
  cudaMemsetAsync(start, 0, sizeof(int) * nb, st);
  cudaMemsetAsync(end, 0, sizeof(int) * nb, st);
  grid_bounds_kernel<<<blocks, tpb, 0, st>>>(a.N, skey, start, end);
  nbr_grid_kernel<<<(a.nrows + SEG_WARPS - 1) / SEG_WARPS, SEG_WARPS * 32, 0, st>>>(p, g, pos, cell, sidx, start, end,
                                                                                   nbr, dist, count);
  return cuda_status(cudaGetLastError(), "nbr_grid_kernel");
}

// ---------------------------------------------------------------- transpose
// Counting-sort transpose (no radix sort of the N*K slots): count the
// pairs per key, exclusive-scan into rev_ptr, scatter each pair to its key's
// segment with an atomic cursor, then restore the stable order (ascending
// pair index i*K + s) per key -- segments hold the ~15-55 queries of one
// key, ranked by a warp in registers.
// vec: K % 4 == 0 and a 16-byte aligned table -> four slots per thread
__device__ __forceinline__ int tr_load4(const int32_t* __restrict__ nbr, size_t t, size_t n, bool vec, int (&js)[4]) {
  if (vec) {
    if (t * 4 >= n) return 0;
    const int4 v = __ldg(reinterpret_cast<const int4*>(nbr) + t);
    js[0] = v.x; js[1] = v.y; js[2] = v.z; js[3] = v.w;
    return 4;
  }
  if (t >= n) return 0;
  js[0] = nbr[t];
  return 1;
}

__global__ void tr_count_kernel(int N, int K, const int32_t* __restrict__ nbr, int* __restrict__ cnt, bool vec) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  int js[4];
  const int m = tr_load4(nbr, t, (size_t)N * K, vec, js);
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (e < m && js[e] >= 0) atomicAdd(&cnt[js[e]], 1);
}

__global__ void tr_fill_kernel(int N, int K, const int32_t* __restrict__ nbr, const int* __restrict__ rev_ptr,
                               int* __restrict__ cursor, int32_t* __restrict__ rev_pair, bool vec) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  int js[4];
  const int m = tr_load4(nbr, t, (size_t)N * K, vec, js);
  const size_t t0 = vec ? t * 4 : t;
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (e < m && js[e] >= 0) rev_pair[rev_ptr[js[e]] + atomicAdd(&cursor[js[e]], 1)] = (int32_t)(t0 + e);
}

// Restore ascending pair order per key: warp per key, each lane ranks its
// (<= 2) entries against the segment's by shuffles and stores them at their
// rank (pair indices are unique); segments over 64 pairs: lane 0 insertion sort.
__global__ void tr_sort_kernel(int Nk, const int* __restrict__ rev_ptr, int32_t* __restrict__ rev_pair) {
  const int j = (int)(((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= Nk) return;
  const int b = rev_ptr[j], n = rev_ptr[j + 1] - b;
  if (n <= 1) return;
  if (n <= 64) {
    constexpr int32_t BIG = 0x7fffffff;
    const int32_t v0 = lane < n ? rev_pair[b + lane] : BIG;
    const int32_t v1 = lane + 32 < n ? rev_pair[b + 32 + lane] : BIG;
    int r0 = 0, r1 = 0;
    for (int x = 0; x < n; ++x) {
      const int32_t w = __shfl_sync(0xffffffffu, x < 32 ? v0 : v1, x & 31);
      r0 += w < v0 ? 1 : 0;
      r1 += w < v1 ? 1 : 0;
    }
    if (lane < n) rev_pair[b + r0] = v0;
    if (lane + 32 < n) rev_pair[b + r1] = v1;
    return;
  }
  if (lane != 0) return;
  for (int x = b + 1; x < b + n; ++x) {
    const int32_t v = rev_pair[x];
    int y = x;
    while (y > b && rev_pair[y - 1] > v) {
      rev_pair[y] = rev_pair[y - 1];
      --y;
    }
    rev_pair[y] = v;
  }
}

namespace {
struct TrWs {
  size_t cnt, cursor, cub, total, cub_scan;
};
TrWs tr_ws(int N, int K, int Nk) {
  (void)N;
  (void)K;
  TrWs w{};
  size_t cc = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cc, (int*)nullptr, (int*)nullptr, Nk + 1);
  size_t o = 0;
  w.cnt = o; o += align256(sizeof(int) * (Nk + 1));
  w.cursor = o; o += align256(sizeof(int) * (Nk + 1));
  w.cub = o; o += align256(cc);
  w.cub_scan = cc;
  w.total = o;
  return w;
}
}  // namespace

size_t transpose_workspace_bytes(int N, int K, int Nk) { return tr_ws(N, K, Nk).total; }

es_status nbr_transpose_launch(int N, int K, int Nk, const int32_t* nbr, int32_t* rev_ptr, int32_t* rev_pair,
                               void* ws, size_t ws_bytes, cudaStream_t st) {
  const TrWs w = tr_ws(N, K, Nk);
  if (ws_bytes < w.total) return fail(ES_INVALID_ARGUMENT, "neighbors_transpose: workspace too small");
  if (N == 0 || Nk == 0) {
    if (Nk >= 0) cudaMemsetAsync(rev_ptr, 0, sizeof(int) * (Nk + 1), st);
    return ES_OK;
  }
  char* base = (char*)ws;
  int* cnt = (int*)(base + w.cnt);
  int* cursor = (int*)(base + w.cursor);
  const size_t n = (size_t)N * K;
  const bool vec = (K & 3) == 0 && ((uintptr_t)nbr & 15) == 0;
  const size_t nt = vec ? n / 4 : n;
  const unsigned blocks = (unsigned)((nt + 255) / 256);
  cudaMemsetAsync(cnt, 0, sizeof(int) * (Nk + 1), st);
  cudaMemsetAsync(cursor, 0, sizeof(int) * (Nk + 1), st);
  tr_count_kernel<<<blocks, 256, 0, st>>>(N, K, nbr, cnt, vec);
  size_t cb = w.cub_scan;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(base + w.cub, cb, cnt, (int*)rev_ptr, Nk + 1, st);
  if (e != cudaSuccess) return cuda_status(e, "neighbors_transpose: scan");
  tr_fill_kernel<<<blocks, 256, 0, st>>>(N, K, nbr, rev_ptr, cursor, rev_pair, vec);
  tr_sort_kernel<<<(unsigned)(((size_t)Nk * 32 + 255) / 256), 256, 0, st>>>(Nk, rev_ptr, rev_pair);
  return cuda_status(cudaGetLastError(), "neighbors_transpose");
}

// ---------------------------------------------------------------- tile mask
__global__ void tile_mask_kernel(int N, int K, const int32_t* __restrict__ nbr, int tq, int tk, int words,
                                 uint32_t* __restrict__ mask) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (size_t)N * K) return;
  const int j = nbr[t];
  if (j < 0) return;
  const int i = (int)(t / K);
  const int qb = i / tq, kb = j / tk;
  atomicOr(&mask[(size_t)qb * words + kb / 32], 1u << (kb % 32));
}

es_status tile_mask_launch(int N, int K, const int32_t* nbr, int tq, int tk, int nkb, uint32_t* mask,
                           cudaStream_t st) {
  if (tq <= 0 || tk <= 0) return fail(ES_INVALID_ARGUMENT, "tile_mask: tile sizes must be positive");
  if (N == 0) return ES_OK;
  const int words = (nkb + 31) / 32;
  const size_t n = (size_t)N * K;
  tile_mask_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(N, K, nbr, tq, tk, words, mask);
  return cuda_status(cudaGetLastError(), "tile_mask_kernel");
}

}  // namespace es
