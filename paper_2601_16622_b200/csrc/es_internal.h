// Internal declarations shared by the CUDA translation units of
// libequistream_b200.so.  Not part of the C ABI (see include/equistream_b200.h).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <string>

#include "../../include/equistream_b200.h"

namespace es {

constexpr int kMaxL = 4;

// Thread-local last-error string behind es_last_error().
void set_error(const std::string& msg);
es_status fail(es_status st, const std::string& msg);
es_status cuda_status(cudaError_t e, const char* where);

// ---------------------------------------------------------------- so3 tables
// Host-built constants (double), uploaded to __constant__ memory as float.
// Reindex polynomial for the aligned frame: for entry e = (l_o, l_i, m), the
// per-pair coefficients are a_e(r) = sum_lf ca[e][lf] r^lf  (source  m) and
// b_e(r) = sum_lf cb[e][lf] r^lf (source -m); path set = all triangle-valid
// (l_i, l_f, l_o) with every degree <= L (weights 1).
struct HostTables {
  double fit_pts[2 * kMaxL + 1][3];
  double ainv[kMaxL + 1][(2 * kMaxL + 1) * (2 * kMaxL + 1)];  // [l][k*(2l+1)+m']
  double shnorm[kMaxL + 1][kMaxL + 1];                        // [l][mu] incl. sqrt2 for mu>0
  // entries of the canonical L=4 enumeration, coefficient sets per L
  double ca[kMaxL + 1][85][kMaxL + 1];
  double cb[kMaxL + 1][85][kMaxL + 1];
};
const HostTables& host_tables();
double real_cg(int l1, int m1, int l2, int m2, int lo, int mo);  // cg_real(l1,l2,lo)[mo](m1,m2)
void solid_harmonics_host(int l, const double* r, double* out);
// canonical entry index (l_o, l_i, m) for L = 4 enumeration
int entry_index(int lo, int li, int m);

// ---------------------------------------------------------------- launchers
struct AttnArgs {
  int N, K, H, L, C, Dq;
  int row0, Nk;
  int value_mode, phi_mode, dtype, periodic;
  float tau, r_cut;
  double box[3];
  int nseg = 0;                      // molecule segments of the index (0: one system)
  int bias_mode = 0;                 // es_bias_mode
  float bias[3] = {0.f, 0.f, 0.f};   // b(r) = bias[0] + bias[1] r + bias[2] r^2
  const void* tiles = nullptr;  // prebuilt tile lists (es_attn_tiles_build) or NULL
  float* scores_out = nullptr;       // es_attn_fwd: optional [N][K][H] scores
  const float* scores_in = nullptr;  // es_attn_bwd: optional saved scores
};

size_t attn_fwd_workspace(const AttnArgs& a);
es_status attn_fwd_launch(const AttnArgs& a, const void* q, const void* k, const void* v, const double* pos,
                          const int32_t* nbr, void* out, float* lse, void* ws, size_t ws_bytes, cudaStream_t st);
bool attn_tc_supported(const AttnArgs& a);
size_t attn_fwd_tc_workspace(const AttnArgs& a);
es_status attn_fwd_tc_launch(const AttnArgs& a, const void* q, const void* k, const void* v, const double* pos,
                             const int32_t* nbr, void* out, float* lse, void* ws, size_t ws_bytes,
                             cudaStream_t st);
es_status attn_bwd_launch(const AttnArgs& a, const void* q, const void* k, const void* v, const double* pos,
                          const int32_t* nbr, const int32_t* rev_ptr, const int32_t* rev_pair, const void* out,
                          const float* lse, const void* dout, void* dq, void* dk, void* dv, float* delta,
                          float* dsbuf, double* dpos, void* ws_tc, size_t ws_tc_bytes, cudaStream_t st);
bool attn_dq_tc_applicable(const AttnArgs& a);
bool attn_tc_tiles_used(const AttnArgs& a);    // the tcgen05 forward or dq would consume tile lists
size_t attn_tc_tiles_bytes(const AttnArgs& a);
es_status attn_tc_tiles_build(const AttnArgs& a, const int32_t* nbr, const int32_t* seg, int nseg,
                              const int32_t* rev_ptr, const int32_t* rev_pair, void* tiles, size_t bytes,
                              cudaStream_t st);
void attn_tc_tiles_layout(const AttnArgs& a, es_attn_tiles_layout* out);
// slot -> rank map inside a tile buffer (the tensor-core forward keeps scores in rank space)
const int* attn_tc_rank_of(const AttnArgs& a, const void* tiles);
// tensor-core dk = tau dS^T Q over key tiles (key-side lists in the tiles buffer or the workspace)
bool attn_dk_tc_applicable(const AttnArgs& a);
// the key pass (dv + dscores) on the tensor cores; dk / dq then follow on the tensor cores
bool attn_kv_tc_applicable(const AttnArgs& a);
es_status attn_kv_tc_launch(const AttnArgs& a, const void* q, const void* k, const void* v, const double* pos,
                            const int32_t* rev_ptr, const int32_t* rev_pair, const float* lse, const void* dout,
                            const float* delta, float* dsbuf, void* dv, void* geom_ws, cudaStream_t st);
size_t attn_kv_tc_geom_bytes(const AttnArgs& a);  // per-pair geometry records of the key pass
es_status attn_delta_launch(const AttnArgs& a, const void* out, const void* dout, float* delta, cudaStream_t st);
size_t attn_dk_tc_workspace(const AttnArgs& a);
es_status attn_dk_tc_launch(const AttnArgs& a, const void* q, const int32_t* nbr, const int32_t* rev_ptr,
                            const int32_t* rev_pair, const float* dsbuf, void* dk, void* ws, size_t ws_bytes,
                            cudaStream_t st);
size_t attn_dq_tc_workspace(const AttnArgs& a);
es_status attn_dq_tc_launch(const AttnArgs& a, const void* k, const int32_t* nbr, const float* dsbuf, void* dq,
                            void* ws, size_t ws_bytes, cudaStream_t st);


struct NbrArgs {
  int N, K, nseg, periodic;
  int row0, nrows;
  double r_cut;
  double box[3];
};
size_t nbr_workspace_bytes(const NbrArgs& a);
es_status nbr_build_launch(const NbrArgs& a, const double* pos, const int32_t* seg_ptr, int32_t* nbr, float* dist,
                           int32_t* count, void* ws, size_t ws_bytes, cudaStream_t st);
size_t transpose_workspace_bytes(int N, int K, int Nk);
es_status nbr_transpose_launch(int N, int K, int Nk, const int32_t* nbr, int32_t* rev_ptr, int32_t* rev_pair,
                               void* ws, size_t ws_bytes, cudaStream_t st);
es_status tile_mask_launch(int N, int K, const int32_t* nbr, int tq, int tk, int nkb, uint32_t* mask,
                           cudaStream_t st);

struct ProjArgs {
  int N, L, C, Dq, Cv, dtype;
};
es_status proj_fwd_launch(const ProjArgs& a, const void* h, const void* W, void* q, void* k, void* v,
                          cudaStream_t st);
bool proj_tc_supported(const ProjArgs& a);
es_status proj_fwd_tc_launch(const ProjArgs& a, const void* h, const void* W, void* q, void* k, void* v,
                             cudaStream_t st);
es_status proj_bwd_tc_launch(const ProjArgs& a, const void* h, const void* W, const void* dq, const void* dk,
                             const void* dv, void* dh, float* dW, cudaStream_t st);
es_status proj_bwd_launch(const ProjArgs& a, const void* h, const void* W, const void* dq, const void* dk,
                          const void* dv, void* dh, float* dW, cudaStream_t st);

}  // namespace es
