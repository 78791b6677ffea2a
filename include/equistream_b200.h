/*
 * equistream_b200.h -- C ABI of libequistream_b200.so, the B200-native
 * (sm_100a) drop-in for the hot path of the reference `equistream` library
 * (/root/reference, arXiv 2601.16622 E2Former-V2): the fused on-the-fly
 * equivariant attention with per-pair EAAS, forward and recompute backward,
 * its neighbour/tile builder and its Q/K/V projections.
 *
 * Every entry point names the reference interface it replaces.  The
 * reference ships these as C++20 header-only library types and SPEC
 * operations (paths relative to /root/reference):
 *
 *   es_attn_fwd            <- stream_aggregate            SPEC.md:275-283 (Alg. 1)
 *   es_attn_bwd            <- stream_aggregate_backward
 *   es_neighbors_build     <- build_neighbors             SPEC.md:431-439 (NeighborIndex SPEC.md:237-242)
 *   es_neighbors_transpose <- (the scatter relation build_neighbors implies; used by es_attn_bwd)
 *   es_tile_mask           <- north-star tile-skip mask over NeighborIndex
 *   es_project_fwd         <- project_qk + W_H
 *   es_project_bwd         <- gradient of project_qk / W_H
 *   es_conventions_manifest<- so3::conventions_manifest() proj/include/equistream/so3/conventions.hpp:13-38
 *   es_cg_real / es_reindex_table / es_wigner_d_host
 *                          <- so3::cg_real clebsch.hpp:179, eaas build_reindex_rule SPEC.md:181,
 *                             so3::wigner_d wigner.hpp:70 (host-side tables the kernels use)
 *
 * Conventions (the reference's, restated): real orthonormal harmonics,
 * m = -l..l ascending, (-1)^m on positive-m components; feature blocks are
 * value vectors v -> D v; node features are "irreps layout" [N][M][C] with
 * M = (L+1)^2, row l*l + (m+l), channels innermost (the byte order of the
 * reference IrrepsFeature blocks, irreps.hpp:69-71).
 *
 * Rules of the ABI: plain C types, caller-owned device buffers (the library
 * never allocates or frees caller memory), `stream` is a cudaStream_t passed
 * as void* (NULL = legacy default stream), every call is stream-ordered and
 * returns an es_status; no exception crosses the boundary.  On failure,
 * es_last_error() returns a thread-local description.  There is no CPU
 * fallback: without an sm_100a device every compute call fails with
 * ES_CUDA_ERROR.
 */
#ifndef EQUISTREAM_B200_H
#define EQUISTREAM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ES_ABI_VERSION 9

typedef enum {
  ES_OK = 0,
  ES_INVALID_ARGUMENT = 1, /* maps to std::invalid_argument (reference errors, irreps.hpp:37-41) */
  ES_UNSUPPORTED = 2,      /* valid request outside the compiled kernel set */
  ES_CUDA_ERROR = 3,       /* maps to std::runtime_error */
  ES_NCCL_ERROR = 4
} es_status;

typedef enum { ES_F32 = 0, ES_BF16 = 1 } es_dtype;

typedef enum {
  ES_VALUE_PLAIN = 0, /* value = phi(r_ij) * v_j: SPEC stream_aggregate with precomputed h' */
  ES_VALUE_EAAS = 1   /* value = phi(r_ij) * sum_paths (v_j (x) R^lf(r_ij))^lo via per-pair EAAS
                         (north star; == edge_centric_message SPEC.md:342-350) */
} es_value_mode;

typedef enum {
  ES_BIAS_NONE = 0,  /* b == 0 */
  ES_BIAS_POLY2 = 1  /* b(r) = bias[0] + bias[1] r + bias[2] r^2 */
} es_bias_mode;

typedef enum {
  ES_PHI_COSINE = 0, /* phi = (cos(pi r / r_cut) + 1) / 2 for r < r_cut */
  ES_PHI_ONE = 1     /* phi == 1 */
} es_phi_mode;

/* Attention problem.  q, k: [N][M][2C]; v, out, dout: [N][M][C]
 * (dtype), lse: [N][H] float32, pos: [N][3] float64, nbr: [N][K] int32 with
 * sentinel -1 (NeighborIndex).  Head h owns q/k channels [h*2C/H, (h+1)*2C/H)
 * and value channels [h*C/H, (h+1)*C/H) at every (l, m) row; d_k = 2*M*C/H,
 * tau = 1/sqrt(d_k), b(r) == 0.  Attention weights softmax over the valid
 * neighbours of each atom; atoms without neighbours produce 0 and lse=-inf
 * (SPEC.md:311). */
typedef struct {
  int32_t N, K, H, L, C;
  int32_t value_mode; /* es_value_mode */
  int32_t phi_mode;   /* es_phi_mode */
  int32_t dtype;      /* es_dtype of q, k, v, out, dout, dq, dk, dv */
  double r_cut;
  int32_t periodic;   /* 1: minimum image in box[] */
  double box[3];
  /* Query-row sharding (one large system over several GPUs): the N query
   * rows are atoms row0 .. row0+N-1 of a system of Nk atoms; q, out, lse,
   * dout, dq and nbr hold the N local rows, k, v, pos, dk and dv all Nk atoms
   * (nbr entries index [0, Nk)).  Nk = 0 means Nk = N, row0 = 0. */
  int32_t row0, Nk;
  /* Radial score bias b(r_ij) of s_ij = tau q_i.k_j + b(r_ij) (RadialScalars,
   * SPEC.md:247-250, Eq. 18): the SPEC's callable as an enum + parameters.
   * ES_BIAS_NONE: b == 0 (the default); ES_BIAS_POLY2:
   * b(r) = bias[0] + bias[1] r + bias[2] r^2. */
  int32_t bias_mode;
  double bias[3];
  /* Segments of the neighbour index (molecule batches: the nseg given to
   * es_neighbors_build; 0 for one system).  Picks the kernel family: the
   * tensor-core tiles pay off where a 128-row tile's keys are its own few
   * molecules; one bulk system (~50 neighbours spread over ~150 key chunks
   * per tile) runs faster on the per-atom SIMT kernels. */
  int32_t nseg;
} es_attn_desc;

/* Compiled kernel set: L in [0, 4]; C a multiple of 32 up to 256; C/H in
 * {4, 8, 16, 32}.  bf16 + EAAS + L=2 + C=128 + H=8 + K<=64 runs on the
 * tcgen05 tensor-core kernel, everything else on the SIMT kernels. */
/* Tile structures of one neighbour index (north-star subsystem 3): query
 * tiles, the tile-skip mask, per-tile key-chunk lists, per-row (chunk, key
 * mask) lists and per-row slot order the tensor-core kernels walk.  Build
 * once per neighbour index with es_attn_tiles_build into a caller buffer of
 * es_attn_tiles_workspace_size(d) bytes (0: the kernels for d need none) and
 * pass it to every es_attn_fwd / es_attn_bwd (every layer) using that index;
 * tiles = NULL makes each call build uniform tiles in its workspace instead.
 * seg_ptr[nseg + 1] (molecule batches, the array given to
 * es_neighbors_build; NULL / 0 for one system): query tiles pack whole
 * segments, so a tile's key chunks cover only its own molecules. */
size_t es_attn_tiles_workspace_size(const es_attn_desc* d);
/* Byte offsets of the arrays inside a tile buffer (introspection and the
 * bit-exact tests; the kernels need nothing but the buffer).  ntiles is the
 * tile-count bound of the layout; a side that is absent has ntiles = 0. */
typedef struct {
  int64_t ntiles, words, nchunk_max;      /* tiles, mask words per tile, clist capacity */
  int64_t mask, cptr, clist, rowlist, tstart, rtile;
  int64_t slots, rank_of;                  /* query side only (-1 on the key side) */
} es_attn_tiles_side;
typedef struct {
  es_attn_tiles_side query, key;           /* key side: rows = key atoms, chunks of 16 queries */
} es_attn_tiles_layout;
es_status es_attn_tiles_layout_query(const es_attn_desc* d, es_attn_tiles_layout* out);
/* rev_ptr / rev_pair (optional, from es_neighbors_transpose on the same nbr):
 * also build the key-side lists (key tiles, their query-chunk lists and
 * per-key (chunk, query mask) entries) the tensor-core dk pass of the
 * backward walks; without them es_attn_bwd builds those in its workspace. */
es_status es_attn_tiles_build(const es_attn_desc* d, const int32_t* nbr, const int32_t* seg_ptr, int32_t nseg,
                              const int32_t* rev_ptr, const int32_t* rev_pair, void* tiles, size_t bytes,
                              void* stream);

/* Workspace: es_attn_fwd_workspace_size(d) bytes (the tile structures when
 * tiles == NULL; 256 bytes for the SIMT kernels).  Caller-owned, reusable
 * across calls on the same stream; the library allocates nothing. */
size_t es_attn_fwd_workspace_size(const es_attn_desc* d);
/* scores (optional, NULL = not kept): N*K*H float32 -- the scores s_ij =
 * tau q_i.k_j + b(r_ij) of the valid pairs, the O(N K H) scalars es_attn_bwd
 * can reuse instead of recomputing q_i.k_j (never O(N K C)).
 * Layout [H][N][K] with a row's valid pairs in its first count entries; their
 * order within the row is private to the library (pass the buffer back to
 * es_attn_bwd unchanged).  pos must be 16-byte aligned. */
es_status es_attn_fwd(const es_attn_desc* d, const void* q, const void* k, const void* v, const double* pos,
                      const int32_t* nbr, void* out, float* lse, float* scores, const void* tiles, void* workspace,
                      size_t workspace_bytes, void* stream);

/* Workspace: es_attn_bwd_workspace_size(d) bytes (per-pair-head dscore
 * buffer, O(N*K*H) scalars -- never O(N*K*C)). rev_ptr/rev_pair
 * come from es_neighbors_transpose on the same nbr.
 * dpos (optional, NULL = skip): [Nk][3] f64 gradient of sum <dout, out> with
 * respect to the atom positions (forces for the conservative mode, PAPER.md:
 * 786) through phi(r_ij), the solid harmonics of the value map
 * and the radial bias b(r_ij); every L.  Overwritten, not accumulated. */
size_t es_attn_bwd_workspace_size(const es_attn_desc* d);
/* scores (optional): the forward's scores output for the same inputs; NULL
 * recomputes them. */
es_status es_attn_bwd(const es_attn_desc* d, const void* q, const void* k, const void* v, const double* pos,
                      const int32_t* nbr, const int32_t* rev_ptr, const int32_t* rev_pair, const void* out,
                      const float* lse, const float* scores, const void* dout, void* dq, void* dk, void* dv,
                      double* dpos, const void* tiles, void* workspace, size_t workspace_bytes, void* stream);

/* Operation and memory accounting (OpCounters / the stats structure,
 * proj/include/equistream/core/counters.hpp:11-32) for one
 * layer of `n_pairs` valid pairs: algorithmic multiply-adds of the forward and
 * backward (score 2 d_k per pair-head ... counted as multiply-adds: d_k for
 * the score, C_h M^2 for the value operator; backward 3 d_k + 2 C_h M^2) and
 * the library's auxiliary device memory, split into floating-point
 * activations (what scales with C) and integer index structures (what scales
 * with the neighbour index, N K). */
typedef struct {
  uint64_t madds_fwd, madds_bwd;           /* attention (projections excluded) */
  uint64_t madds_proj_fwd, madds_proj_bwd;
  uint64_t aux_float_bytes_fwd;            /* floating-point scratch of es_attn_fwd (lse excluded: an output) */
  uint64_t aux_float_bytes_bwd;            /* floating-point scratch of es_attn_bwd: O(N K H) scalars */
  uint64_t aux_index_bytes;                /* tile lists / key-side lists (es_attn_tiles_workspace_size) */
  uint64_t workspace_fwd_bytes, workspace_bwd_bytes;
} es_attn_stats;
es_status es_attn_stats_query(const es_attn_desc* d, int64_t n_pairs, es_attn_stats* out);

/* Neighbour index: per atom the K nearest j != i with d^2 < r_cut^2, sorted
 * by (d^2, j), padded with -1, restricted to the atom's segment
 * (seg_ptr[nseg+1] contiguous molecule ranges, or NULL for one system) and,
 * if periodic, under the minimum image.  d^2 is evaluated in double with
 * round-to-nearest and no contraction, ((dx*dx + dy*dy) + dz*dz), so lists
 * are bit-identical to the CPU oracle.  dist (optional, may be NULL) gets
 * float(sqrt(d^2)); count[N] the filled slots. */
typedef struct {
  int32_t N, K, nseg;
  int32_t periodic;
  double r_cut;
  double box[3];
  /* Row range (query-row sharding, SURVEY 8 e): only atoms row0 .. row0 +
   * nrows - 1 are searched (against all N atoms); nbr, dist and count then
   * hold nrows rows.  nrows = 0 means all N rows (row0 must be 0). */
  int32_t row0, nrows;
} es_nbr_desc;
size_t es_neighbors_workspace_size(const es_nbr_desc* d);
es_status es_neighbors_build(const es_nbr_desc* d, const double* pos, const int32_t* seg_ptr, int32_t* nbr,
                             float* dist, int32_t* count, void* workspace, size_t workspace_bytes, void* stream);

/* Transposed (key-major) relation of nbr [N][K] over Nk key atoms (Nk = N
 * for one unsharded system): for key j, entries rev_pair[rev_ptr[j] ..
 * rev_ptr[j+1]) hold i*K + slot with nbr[i][slot] == j, ascending
 * (deterministic).  rev_ptr: [Nk+1], rev_pair: [N*K]. */
size_t es_neighbors_transpose_workspace_size(int32_t N, int32_t K, int32_t Nk);
es_status es_neighbors_transpose(int32_t N, int32_t K, int32_t Nk, const int32_t* nbr, int32_t* rev_ptr,
                                 int32_t* rev_pair, void* workspace, size_t workspace_bytes, void* stream);

/* Tile-skip mask: bit (qb, kb) of mask[qb * ceil(nkb/32) + kb/32] is set iff
 * some atom of query block qb (tq atoms) lists a neighbour in key block kb
 * (tk atoms).  mask must be zeroed by the caller. */
es_status es_tile_mask(int32_t N, int32_t K, const int32_t* nbr, int32_t tq, int32_t tk, uint32_t* mask,
                       void* stream);

/* Projections, Eq. (6) + W_H: per degree l a channel-mixing matrix
 * W[l] = [W_Q | W_K | W_V] of shape [C][2*Dq + C] (Dq = 2C: W_Q = [W_Q1 | W_Q2]).
 * h: [N][M][C] (dtype), W: [L+1][C][2Dq+C] (dtype), outputs q,k [N][M][Dq], v [N][M][C]. */
typedef struct {
  int32_t N, L, C;
  int32_t dtype;
} es_proj_desc;
es_status es_project_fwd(const es_proj_desc* d, const void* h, const void* W, void* q, void* k, void* v,
                         void* stream);
/* dh [N][M][C] (dtype, overwritten); dW [L+1][C][2Dq+C] float32 (overwritten) or NULL. */
es_status es_project_bwd(const es_proj_desc* d, const void* h, const void* W, const void* dq, const void* dk,
                         const void* dv, void* dh, float* dW, void* stream);

/* Node-centric factorized message (Eq. 5
 * PAPER.md:228-235; three-stage flow PAPER.md:299-322), fp64:
 *   m_i = sum_j alpha_ij sum_paths (h_j^li (x) R^lf(r_j - r_i))^lo
 * (== edge_centric_message SPEC.md:342-350 with the attention's path set)
 * evaluated as source term -> alpha aggregation -> target coupling through
 * the binomial translation identity R^lf(a+b) = sum_u w(lf,u)
 * (R^u(a) (x) R^{lf-u}(b))^lf (conventions.hpp:32-34) and the 6j recoupling,
 * so per edge only the scalar alpha_ij multiplies.  h, out: [N][M][C] f64;
 * alpha: [N][K][H] f64 (head h weights channels [h C/H, (h+1) C/H));
 * S, A (source terms, aggregates): [N][(L+1)^4][C] f64; origin: the
 * recentring point (SPEC ledger: the centroid), positions are absolute.
 * L <= 2 (SPEC ledger "degree budget"). */
typedef struct {
  int32_t N, K, H, L, C;
  double origin[3];
} es_msg_desc;
/* translation_coefficients: w[u], u = 0..l, solved from the identity (host) */
es_status es_translation_coefficients(int32_t l, double* w);
es_status es_source_term(const es_msg_desc* d, const double* pos, const double* h, double* S, void* stream);
es_status es_message_aggregate(const es_msg_desc* d, const int32_t* nbr, const double* alpha, const double* S,
                               double* A, void* stream);
es_status es_target_couple(const es_msg_desc* d, const double* pos, const double* A, double* out, void* stream);
size_t es_factorized_workspace_size(const es_msg_desc* d);
es_status es_factorized_message(const es_msg_desc* d, const double* pos, const double* h, const int32_t* nbr,
                                const double* alpha, double* out, void* workspace, size_t workspace_bytes,
                                void* stream);

/* Dense-CG vs EAAS tensor-product microbenchmark (run_tp_bench
 * SPEC.md:449-457, Figure 2): P independent pairs, x = sum over
 * the path set of (v^li (x) R^lf(r))^lo; v, x: [P][M][C] f32, r: [P][3] f32;
 * L in {2, 4}.  es_tp_madds: multiply-adds per pair-channel of each form. */
es_status es_tp_bench_dense(int32_t L, int32_t C, int32_t P, const float* v, const float* r, float* x, void* stream);
es_status es_tp_bench_eaas(int32_t L, int32_t C, int32_t P, const float* v, const float* r, float* x, void* stream);
es_status es_tp_madds(int32_t L, int64_t* dense_per_channel, int64_t* eaas_per_channel);

/* Host-side introspection of the tables the kernels use. */
const char* es_conventions_manifest(void);
double es_cg_real(int32_t l1, int32_t m1, int32_t l2, int32_t m2, int32_t lo, int32_t mo);
/* Aligned-frame re-index polynomial of entry (lo, li, m) for max degree L:
 * coefficient of source +m (a) and -m (b) as sum_lf coef[lf] r^lf, lf = 0..4. */
es_status es_reindex_table(int32_t L, int32_t lo, int32_t li, int32_t m, double* a5, double* b5);
/* D^l(R) by the kernels' harmonic-fit construction, in double (R row-major). */
es_status es_wigner_d_host(int32_t l, const double* R, double* D);

const char* es_last_error(void);
int32_t es_abi_version(void);
/* 1 if a CUDA device of compute capability 10.x is visible. */
int32_t es_device_ok(void);

#ifdef __cplusplus
}
#endif
#endif /* EQUISTREAM_B200_H */
