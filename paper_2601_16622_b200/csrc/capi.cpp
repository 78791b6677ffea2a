// C ABI of libequistream_b200.so (include/equistream_b200.h): argument
// validation with the reference's error taxonomy (std::invalid_argument ->
// ES_INVALID_ARGUMENT, internal/CUDA failures -> ES_CUDA_ERROR), the
// conventions manifest, and the launches.  No exception crosses the ABI.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>

#include "es_internal.h"

namespace es {

static thread_local std::string t_last_error;

void set_error(const std::string& msg) { t_last_error = msg; }

es_status fail(es_status st, const std::string& msg) {
  set_error(msg);
  return st;
}

es_status cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return ES_OK;
  return fail(ES_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

namespace {

es_status check_attn(const es_attn_desc* d) {
  if (!d) return fail(ES_INVALID_ARGUMENT, "attn: null descriptor");
  if (d->N < 0 || d->K < 1) return fail(ES_INVALID_ARGUMENT, "attn: N >= 0 and K >= 1 required");
  if (d->L < 0 || d->L > kMaxL) return fail(ES_UNSUPPORTED, "attn: L must be in [0, 4]");
  if (d->H < 1 || d->C < 1 || d->C % d->H != 0) return fail(ES_INVALID_ARGUMENT, "attn: C must be a multiple of H");
  if (!(d->r_cut > 0.0)) return fail(ES_INVALID_ARGUMENT, "attn: r_cut must be positive");
  if (d->value_mode != ES_VALUE_PLAIN && d->value_mode != ES_VALUE_EAAS)
    return fail(ES_INVALID_ARGUMENT, "attn: unknown value_mode");
  if (d->phi_mode != ES_PHI_COSINE && d->phi_mode != ES_PHI_ONE)
    return fail(ES_INVALID_ARGUMENT, "attn: unknown phi_mode");
  if (d->dtype != ES_F32 && d->dtype != ES_BF16) return fail(ES_INVALID_ARGUMENT, "attn: unknown dtype");
  if (d->periodic && !(d->box[0] > 0 && d->box[1] > 0 && d->box[2] > 0))
    return fail(ES_INVALID_ARGUMENT, "attn: periodic box must be positive");
  const int ch = d->C / d->H;
  if (d->C % 32 != 0 || d->C > 256) return fail(ES_UNSUPPORTED, "attn: C must be a multiple of 32 and <= 256");
  if (ch > 32 || 32 % ch != 0 || ch < 4) return fail(ES_UNSUPPORTED, "attn: C/H must be 4, 8, 16 or 32");
  if (d->H > 64) return fail(ES_UNSUPPORTED, "attn: H <= 64");
  if (d->Nk < 0 || d->row0 < 0) return fail(ES_INVALID_ARGUMENT, "attn: row0, Nk >= 0");
  if (d->Nk > 0 && d->row0 + d->N > d->Nk) return fail(ES_INVALID_ARGUMENT, "attn: row0 + N > Nk");
  if (d->bias_mode != ES_BIAS_NONE && d->bias_mode != ES_BIAS_POLY2)
    return fail(ES_INVALID_ARGUMENT, "attn: unknown bias_mode");
  if (d->bias_mode == ES_BIAS_POLY2 && !(std::isfinite(d->bias[0]) && std::isfinite(d->bias[1]) && std::isfinite(d->bias[2])))
    return fail(ES_INVALID_ARGUMENT, "attn: bias parameters must be finite");
  return ES_OK;
}

AttnArgs to_args(const es_attn_desc* d) {
  AttnArgs a;
  a.N = d->N; a.K = d->K; a.H = d->H; a.L = d->L; a.C = d->C; a.Dq = 2 * d->C;
  a.Nk = d->Nk > 0 ? d->Nk : d->N;
  a.row0 = d->Nk > 0 ? d->row0 : 0;
  a.value_mode = d->value_mode; a.phi_mode = d->phi_mode; a.dtype = d->dtype; a.periodic = d->periodic;
  const int M = (d->L + 1) * (d->L + 1);
  a.tau = (float)(1.0 / std::sqrt((double)M * (a.Dq / d->H)));
  a.r_cut = (float)d->r_cut;
  for (int x = 0; x < 3; ++x) a.box[x] = d->box[x];
  a.nseg = d->nseg > 0 ? d->nseg : 0;
  a.bias_mode = d->bias_mode;
  for (int x = 0; x < 3; ++x) a.bias[x] = d->bias_mode ? (float)d->bias[x] : 0.f;
  return a;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

template <class F>
es_status guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    return fail(ES_CUDA_ERROR, std::string("internal: ") + e.what());
  } catch (...) {
    return fail(ES_CUDA_ERROR, "internal: unknown exception");
  }
}

const char kManifest[] =
    "# equistream-b200 conventions manifest (keys of so3/conventions.hpp:16-36, plus the GPU path's)\n"
    "m_ordering=ascending_-l_to_l\n"
    "harmonic_normalization=orthonormal\n"
    "y00=0.28209479177387814\n"
    "complex_basis=condon_shortley\n"
    "real_basis_change=x_m = (i/sqrt2)(z_m - (-1)^m z_{-m}) [m<0]; z_0 [m=0]; (1/sqrt2)(z_m + (-1)^m z_{-m}) [m>0]\n"
    "l1_value_map=(m=-1,0,1) -> sqrt(3/4pi) * (y, z, -x)\n"
    "transformation_side=value_vectors_left: solid(l, R r) = D(l,R) solid(l, r); feature blocks right-multiply by "
    "D^T\n"
    "cg_source=complex_racah_conjugated_on_all_three_legs\n"
    "cg_frobenius_norm_sq_per_path=2*l_out+1\n"
    "cg_odd_path_phase=-i\n"
    "eaas_reindex_coefficients=m_f=0 slice of cg_real times Y_lf0(e_z) |r|^lf; the printed odd-branch factor "
    "-2(-1)^{m_o} of the source convention is absorbed by this basis normalization\n"
    "wigner_d=fit of solid(l, R p_k) = D solid(l, p_k) on 2l+1 fixed points (A^-1 precomputed); the reference "
    "generator build (wigner.hpp:43-53) has G_y sign-flipped and is not used\n"
    "alignment_gauge=R = R'(u') P, P = diag(1,-1,-1) iff u_z < 0, R' rows (e1, e2, u'); any gauge gives the same "
    "composite (SPEC.md:213)\n"
    "feature_layout=[N][M][C], row l*l+m+l, channels innermost (== IrrepsFeature column-major bytes)\n"
    "qk_layout=[N][M][2C]: per (l,m) row, W_Q = [W_Q1 | W_Q2]; head h owns channels [h*2C/H,(h+1)*2C/H)\n"
    "value_heads=head h owns value channels [h*C/H,(h+1)*C/H)\n"
    "path_set=all triangle-valid (l_i,l_f,l_o) with every degree <= L, weight 1\n"
    "score=tau * q_i.k_j + b, tau = 1/sqrt(d_k), d_k = 2*M*C/H, b == 0\n"
    "phi=0.5*(cos(pi r/r_cut)+1) for r < r_cut (cosine) | 1\n"
    "zero_neighbour_rows=output 0, lse -inf\n"
    "neighbor_order=(d2, j) ascending; d2 = ((dx*dx + dy*dy) + dz*dz) fp64 round-to-nearest, no FMA; strict "
    "d2 < r_cut^2\n"
    "max_degree_tables=4\n"
    "irreps_default_max_degree=4\n";

}  // namespace
}  // namespace es

using namespace es;

extern "C" {

const char* es_last_error(void) { return t_last_error.c_str(); }
int32_t es_abi_version(void) { return ES_ABI_VERSION; }
const char* es_conventions_manifest(void) { return kManifest; }

int32_t es_device_ok(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return 0;
  }
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  return major == 10 ? 1 : 0;
}

size_t es_attn_fwd_workspace_size(const es_attn_desc* d) {
  if (!d || check_attn(d) != ES_OK) return 256;
  const size_t n = attn_fwd_workspace(to_args(d));
  return n > 256 ? n : 256;
}

size_t es_attn_tiles_workspace_size(const es_attn_desc* d) {
  if (!d || check_attn(d) != ES_OK) return 0;
  const AttnArgs a = to_args(d);
  return attn_tc_tiles_used(a) ? attn_tc_tiles_bytes(a) : 0;
}

es_status es_attn_tiles_layout_query(const es_attn_desc* d, es_attn_tiles_layout* out) {
  return guarded([&] {
    es_status s = check_attn(d);
    if (s != ES_OK) return s;
    if (!out) return fail(ES_INVALID_ARGUMENT, "attn_tiles_layout: null output");
    attn_tc_tiles_layout(to_args(d), out);
    return ES_OK;
  });
}

es_status es_attn_tiles_build(const es_attn_desc* d, const int32_t* nbr, const int32_t* seg_ptr, int32_t nseg,
                              const int32_t* rev_ptr, const int32_t* rev_pair, void* tiles, size_t bytes,
                              void* stream) {
  return guarded([&] {
    es_status s = check_attn(d);
    if (s != ES_OK) return s;
    const AttnArgs a = to_args(d);
    if (!attn_tc_tiles_used(a)) return ES_OK;  // the SIMT kernels need no tile lists
    if (d->N > 0 && !nbr) return fail(ES_INVALID_ARGUMENT, "attn_tiles: null buffer");
    if (nseg < 0 || (nseg > 0 && !seg_ptr)) return fail(ES_INVALID_ARGUMENT, "attn_tiles: nseg > 0 needs seg_ptr");
    return attn_tc_tiles_build(a, nbr, nseg > 0 ? seg_ptr : nullptr, nseg, rev_ptr, rev_pair, tiles, bytes,
                               (cudaStream_t)stream);
  });
}

es_status es_attn_fwd(const es_attn_desc* d, const void* q, const void* k, const void* v, const double* pos,
                      const int32_t* nbr, void* out, float* lse, float* scores, const void* tiles, void* workspace,
                      size_t workspace_bytes, void* stream) {
  return guarded([&] {
    es_status s = check_attn(d);
    if (s != ES_OK) return s;
    if (d->N > 0 && (!q || !k || !v || !pos || !nbr || !out || !lse))
      return fail(ES_INVALID_ARGUMENT, "attn_fwd: null buffer");
    if (d->N > 0 && !tiles && (!workspace || workspace_bytes < es_attn_fwd_workspace_size(d)))
      return fail(ES_INVALID_ARGUMENT, "attn_fwd: workspace too small");
    if (d->N > 0 && ((uintptr_t)pos & 15) != 0)  // the tensor-core kernels bulk-copy key positions (16-byte units)
      return fail(ES_INVALID_ARGUMENT, "attn_fwd: pos must be 16-byte aligned");
    AttnArgs a = to_args(d);
    a.tiles = tiles;
    a.scores_out = scores;
    return attn_fwd_launch(a, q, k, v, pos, nbr, out, lse, workspace, workspace_bytes, (cudaStream_t)stream);
  });
}

static size_t bwd_base_bytes(const es_attn_desc* d) {
  return align256(sizeof(float) * (size_t)d->N * d->H) + align256(sizeof(float) * (size_t)d->N * d->K * d->H);
}

size_t es_attn_bwd_workspace_size(const es_attn_desc* d) {
  if (!d || d->N <= 0 || check_attn(d) != ES_OK) return 256;
  const AttnArgs a = to_args(d);
  // tensor-core passes without prebuilt tiles: the tile lists (query + key side) are built in the workspace
  // (+ the tensor-core key pass's per-pair geometry records after them)
  return bwd_base_bytes(d) + (attn_dq_tc_applicable(a) ? align256(attn_tc_tiles_bytes(a)) : 0) +
         (attn_kv_tc_applicable(a) ? attn_kv_tc_geom_bytes(a) : 0);
}

es_status es_attn_bwd(const es_attn_desc* d, const void* q, const void* k, const void* v, const double* pos,
                      const int32_t* nbr, const int32_t* rev_ptr, const int32_t* rev_pair, const void* out,
                      const float* lse, const float* scores, const void* dout, void* dq, void* dk, void* dv,
                      double* dpos, const void* tiles, void* workspace, size_t workspace_bytes, void* stream) {
  return guarded([&] {
    es_status s = check_attn(d);
    if (s != ES_OK) return s;
    if (d->N == 0) {
      // No query rows: dk / dv are still [Nk] outputs (a row shard with an empty slab contributes zeros to the
      // reduce-scatter), and dpos is overwritten.
      const AttnArgs a0 = to_args(d);
      const size_t es = d->dtype == ES_BF16 ? 2 : 4, M = (size_t)(d->L + 1) * (d->L + 1);
      const size_t nk = d->Nk > 0 ? (size_t)d->Nk : 0;
      if (nk > 0 && (!dk || !dv)) return fail(ES_INVALID_ARGUMENT, "attn_bwd: null dk/dv");
      if (nk > 0) {
        es_status z = cuda_status(cudaMemsetAsync(dk, 0, es * nk * M * 2 * d->C, (cudaStream_t)stream), "attn_bwd: dk");
        if (z == ES_OK)
          z = cuda_status(cudaMemsetAsync(dv, 0, es * nk * M * d->C, (cudaStream_t)stream), "attn_bwd: dv");
        if (z != ES_OK) return z;
      }
      return dpos ? attn_bwd_launch(a0, q, k, v, pos, nbr, rev_ptr, rev_pair, out, lse, dout, dq, dk, dv, nullptr,
                                    nullptr, dpos, nullptr, 0, (cudaStream_t)stream)
                  : ES_OK;
    }
    if (!q || !k || !v || !pos || !nbr || !rev_ptr || !rev_pair || !out || !lse || !dout || !dq || !dk || !dv)
      return fail(ES_INVALID_ARGUMENT, "attn_bwd: null buffer");
    if (!workspace || workspace_bytes < es_attn_bwd_workspace_size(d))
      return fail(ES_INVALID_ARGUMENT, "attn_bwd: workspace too small");
    float* delta = (float*)workspace;
    float* dsbuf = (float*)((char*)workspace + align256(sizeof(float) * (size_t)d->N * d->H));
    const size_t base = bwd_base_bytes(d);
    AttnArgs a = to_args(d);
    a.tiles = tiles;
    a.scores_in = scores;
    return attn_bwd_launch(a, q, k, v, pos, nbr, rev_ptr, rev_pair, out, lse, dout, dq, dk, dv, delta, dsbuf, dpos,
                           (char*)workspace + base, workspace_bytes - base, (cudaStream_t)stream);
  });
}

static es_status check_nbr(const es_nbr_desc* d) {
  if (!d) return fail(ES_INVALID_ARGUMENT, "neighbors: null descriptor");
  if (d->N < 0 || d->K < 1) return fail(ES_INVALID_ARGUMENT, "neighbors: K >= 1 required");
  if (!(d->r_cut > 0.0)) return fail(ES_INVALID_ARGUMENT, "neighbors: r_cut must be positive");
  if (d->periodic && !(d->box[0] > 0 && d->box[1] > 0 && d->box[2] > 0))
    return fail(ES_INVALID_ARGUMENT, "neighbors: periodic box must be positive");
  if (d->nseg < 0) return fail(ES_INVALID_ARGUMENT, "neighbors: nseg >= 0");
  if (d->row0 < 0 || d->nrows < 0 || (d->nrows > 0 && d->row0 + d->nrows > d->N) || (d->nrows == 0 && d->row0 != 0))
    return fail(ES_INVALID_ARGUMENT, "neighbors: rows [row0, row0 + nrows) must lie in [0, N)");
  return ES_OK;
}

static NbrArgs nbr_args(const es_nbr_desc* d) {
  NbrArgs a;
  a.N = d->N; a.K = d->K; a.nseg = d->nseg; a.periodic = d->periodic; a.r_cut = d->r_cut;
  a.row0 = d->nrows > 0 ? d->row0 : 0;
  a.nrows = d->nrows > 0 ? d->nrows : d->N;
  for (int x = 0; x < 3; ++x) a.box[x] = d->box[x];
  return a;
}

size_t es_neighbors_workspace_size(const es_nbr_desc* d) {
  if (check_nbr(d) != ES_OK) return 0;
  return nbr_workspace_bytes(nbr_args(d));
}

es_status es_neighbors_build(const es_nbr_desc* d, const double* pos, const int32_t* seg_ptr, int32_t* nbr,
                             float* dist, int32_t* count, void* workspace, size_t workspace_bytes, void* stream) {
  return guarded([&] {
    es_status s = check_nbr(d);
    if (s != ES_OK) return s;
    if (d->N > 0 && (!pos || !nbr || !count)) return fail(ES_INVALID_ARGUMENT, "neighbors: null buffer");
    if (d->nseg > 0 && !seg_ptr) return fail(ES_INVALID_ARGUMENT, "neighbors: nseg > 0 needs seg_ptr");
    if (workspace_bytes < es_neighbors_workspace_size(d) || !workspace)
      return fail(ES_INVALID_ARGUMENT, "neighbors: workspace too small");
    return nbr_build_launch(nbr_args(d), pos, seg_ptr, nbr, dist, count, workspace, workspace_bytes,
                            (cudaStream_t)stream);
  });
}

size_t es_neighbors_transpose_workspace_size(int32_t N, int32_t K, int32_t Nk) {
  if (N < 0 || K < 1 || Nk < 0) return 0;
  return transpose_workspace_bytes(N, K, Nk);
}

es_status es_neighbors_transpose(int32_t N, int32_t K, int32_t Nk, const int32_t* nbr, int32_t* rev_ptr,
                                 int32_t* rev_pair, void* workspace, size_t workspace_bytes, void* stream) {
  return guarded([&] {
    if (N < 0 || K < 1 || Nk < 0) return fail(ES_INVALID_ARGUMENT, "neighbors_transpose: N >= 0, K >= 1, Nk >= 0");
    if ((size_t)N * K >= (size_t)1 << 31) return fail(ES_UNSUPPORTED, "neighbors_transpose: N*K >= 2^31");
    if (N > 0 && (!nbr || !rev_ptr || !rev_pair || !workspace))
      return fail(ES_INVALID_ARGUMENT, "neighbors_transpose: null buffer");
    return nbr_transpose_launch(N, K, Nk, nbr, rev_ptr, rev_pair, workspace, workspace_bytes, (cudaStream_t)stream);
  });
}

es_status es_tile_mask(int32_t N, int32_t K, const int32_t* nbr, int32_t tq, int32_t tk, uint32_t* mask,
                       void* stream) {
  return guarded([&] {
    if (N < 0 || K < 1) return fail(ES_INVALID_ARGUMENT, "tile_mask: N >= 0, K >= 1");
    if (tq < 1 || tk < 1) return fail(ES_INVALID_ARGUMENT, "tile_mask: tq, tk >= 1");
    if (N > 0 && (!nbr || !mask)) return fail(ES_INVALID_ARGUMENT, "tile_mask: null buffer");
    return tile_mask_launch(N, K, nbr, tq, tk, (N + tk - 1) / tk, mask, (cudaStream_t)stream);
  });
}

static es_status check_proj(const es_proj_desc* d) {
  if (!d) return fail(ES_INVALID_ARGUMENT, "project: null descriptor");
  if (d->N < 0 || d->C < 1) return fail(ES_INVALID_ARGUMENT, "project: N >= 0, C >= 1");
  if (d->L < 0 || d->L > kMaxL) return fail(ES_UNSUPPORTED, "project: L must be in [0, 4]");
  if (d->dtype != ES_F32 && d->dtype != ES_BF16) return fail(ES_INVALID_ARGUMENT, "project: unknown dtype");
  return ES_OK;
}

es_status es_attn_stats_query(const es_attn_desc* d, int64_t n_pairs, es_attn_stats* out) {
  return guarded([&] {
    es_status s = check_attn(d);
    if (s != ES_OK) return s;
    if (!out || n_pairs < 0) return fail(ES_INVALID_ARGUMENT, "attn_stats: null output or negative pair count");
    const uint64_t M = (uint64_t)(d->L + 1) * (d->L + 1), H = d->H, C = d->C, ch = C / H;
    const uint64_t dk = 2 * M * C / H, E = (uint64_t)n_pairs, N = (uint64_t)d->N, K = (uint64_t)d->K;
    std::memset(out, 0, sizeof(*out));
    out->madds_fwd = E * H * (dk + ch * M * M);
    out->madds_bwd = E * H * (3 * dk + 2 * ch * M * M);
    out->madds_proj_fwd = N * M * C * 5 * C;
    out->madds_proj_bwd = 2 * out->madds_proj_fwd;
    // forward: (mu, z, A) live on chip (registers / TMEM), no floating-point scratch in HBM
    out->aux_float_bytes_fwd = 0;
    // backward: Delta [N][H] and the per-pair-head dscore [N][K][H] -- O(N K H), never O(N K C) -- plus,
    // with the tensor-core key pass, its head-independent per-pair geometry records (32 bytes per slot)
    out->aux_float_bytes_bwd = 4 * N * H + 4 * N * K * H;
    if (attn_kv_tc_applicable(to_args(d))) out->aux_float_bytes_bwd += 32 * N * K;
    out->aux_index_bytes = es_attn_tiles_workspace_size(d);
    out->workspace_fwd_bytes = es_attn_fwd_workspace_size(d);
    out->workspace_bwd_bytes = es_attn_bwd_workspace_size(d);
    return ES_OK;
  });
}

es_status es_project_fwd(const es_proj_desc* d, const void* h, const void* W, void* q, void* k, void* v,
                         void* stream) {
  return guarded([&] {
    es_status s = check_proj(d);
    if (s != ES_OK) return s;
    if (d->N > 0 && (!h || !W || !q || !k || !v)) return fail(ES_INVALID_ARGUMENT, "project_fwd: null buffer");
    ProjArgs a{d->N, d->L, d->C, 2 * d->C, d->C, d->dtype};
    return proj_fwd_launch(a, h, W, q, k, v, (cudaStream_t)stream);
  });
}

es_status es_project_bwd(const es_proj_desc* d, const void* h, const void* W, const void* dq, const void* dk,
                         const void* dv, void* dh, float* dW, void* stream) {
  return guarded([&] {
    es_status s = check_proj(d);
    if (s != ES_OK) return s;
    if (d->N > 0 && (!h || !W || !dq || !dk || !dv || !dh)) return fail(ES_INVALID_ARGUMENT, "project_bwd: null buffer");
    ProjArgs a{d->N, d->L, d->C, 2 * d->C, d->C, d->dtype};
    return proj_bwd_launch(a, h, W, dq, dk, dv, dh, dW, (cudaStream_t)stream);
  });
}

double es_cg_real(int32_t l1, int32_t m1, int32_t l2, int32_t m2, int32_t lo, int32_t mo) {
  return real_cg(l1, m1, l2, m2, lo, mo);
}

es_status es_reindex_table(int32_t L, int32_t lo, int32_t li, int32_t m, double* a5, double* b5) {
  if (L < 0 || L > kMaxL || lo < 0 || lo > L || li < 0 || li > L) return fail(ES_INVALID_ARGUMENT, "reindex: degree");
  const int mm = lo < li ? lo : li;
  if (m < -mm || m > mm) return fail(ES_INVALID_ARGUMENT, "reindex: |m| > min(lo, li)");
  const HostTables& t = host_tables();
  const int e = entry_index(lo, li, m);
  for (int f = 0; f <= kMaxL; ++f) {
    a5[f] = t.ca[L][e][f];
    b5[f] = t.cb[L][e][f];
  }
  return ES_OK;
}

es_status es_wigner_d_host(int32_t l, const double* R, double* D) {
  if (l < 0 || l > kMaxL) return fail(ES_INVALID_ARGUMENT, "wigner_d_host: l in [0, 4]");
  const HostTables& t = host_tables();
  const int d = 2 * l + 1;
  if (l == 0) {
    D[0] = 1.0;
    return ES_OK;
  }
  double y[9];
  for (int a = 0; a < d * d; ++a) D[a] = 0.0;
  for (int k = 0; k < d; ++k) {
    const double* p = t.fit_pts[k];
    const double q[3] = {R[0] * p[0] + R[1] * p[1] + R[2] * p[2], R[3] * p[0] + R[4] * p[1] + R[5] * p[2],
                         R[6] * p[0] + R[7] * p[1] + R[8] * p[2]};
    solid_harmonics_host(l, q, y);
    for (int m = 0; m < d; ++m)
      for (int mp = 0; mp < d; ++mp) D[m * d + mp] += y[m] * t.ainv[l][k * d + mp];
  }
  return ES_OK;
}

}  // extern "C"
