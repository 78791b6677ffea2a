// equistream/attention/stream_attention.hpp -- C++20 header-only front end
// of libequistream_b200.so, mirroring the reference operator interface of
// the stream_attention and bench modules the way
// the reference's own so3 headers are written (namespace equistream,
// value-semantic structs, std::invalid_argument for preconditions,
// std::runtime_error for internal/CUDA failures; proj/include/equistream).
//
// Device buffers are caller-owned raw pointers (CUDA device memory); every
// call is stream-ordered on `stream` (a cudaStream_t, or nullptr).  There is
// no CPU fallback.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "equistream_b200.h"

namespace equistream::attention {

inline void check(es_status s, const char* what) {
  if (s == ES_OK) return;
  const std::string msg = std::string(what) + ": " + es_last_error();
  if (s == ES_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

enum class ValueMode { Plain = ES_VALUE_PLAIN, EAAS = ES_VALUE_EAAS };
enum class Radial { CosineCutoff = ES_PHI_COSINE, One = ES_PHI_ONE };
enum class DType { F32 = ES_F32, BF16 = ES_BF16 };

// NeighborIndex: device table [N][K] int32, sentinel -1.
struct NeighborIndex {
  int32_t N = 0, K = 0;
  int32_t* table = nullptr;    // [N][K]
  float* distances = nullptr;  // [N][K] or nullptr
  int32_t* count = nullptr;    // [N]
  int32_t* rev_ptr = nullptr;  // [N+1]   (transposed relation, for the backward)
  int32_t* rev_pair = nullptr; // [N*K]
  const void* tiles = nullptr; // tile lists of the tensor-core kernels (build_tiles), optional
};

struct AttentionProblem {
  int32_t N = 0, K = 0, heads = 1, lmax = 2, channels = 64;
  ValueMode value = ValueMode::EAAS;
  Radial radial = Radial::CosineCutoff;
  DType dtype = DType::F32;
  double r_cut = 6.0;
  bool periodic = false;
  double box[3] = {0, 0, 0};
  int32_t row0 = 0, n_keys = 0;  // query-row sharding (0 = unsharded)
  // radial score bias b(r) = bias[0] + bias[1] r + bias[2] r^2 (RadialScalars b)
  bool has_bias = false;
  double bias[3] = {0, 0, 0};
  int32_t nseg = 0;  // molecule segments of the neighbour index (0: one system) -- picks the kernel family

  es_attn_desc desc() const {
    es_attn_desc d{};
    d.N = N; d.K = K; d.H = heads; d.L = lmax; d.C = channels;
    d.value_mode = static_cast<int32_t>(value);
    d.phi_mode = static_cast<int32_t>(radial);
    d.dtype = static_cast<int32_t>(dtype);
    d.r_cut = r_cut;
    d.periodic = periodic ? 1 : 0;
    for (int a = 0; a < 3; ++a) d.box[a] = box[a];
    d.row0 = row0;
    d.Nk = n_keys;
    d.bias_mode = has_bias ? ES_BIAS_POLY2 : ES_BIAS_NONE;
    for (int a = 0; a < 3; ++a) d.bias[a] = bias[a];
    d.nseg = nseg;
    return d;
  }
};

// build_neighbors: bit-identical to the CPU definition.
inline std::size_t neighbors_workspace_size(int32_t N, int32_t K, double r_cut, int32_t nseg = 0,
                                            const double* box = nullptr) {
  es_nbr_desc d{N, K, nseg, box ? 1 : 0, r_cut, {box ? box[0] : 0, box ? box[1] : 0, box ? box[2] : 0}};
  return es_neighbors_workspace_size(&d);
}
inline void build_neighbors(const double* pos, int32_t N, int32_t K, double r_cut, NeighborIndex& idx,
                            void* workspace, std::size_t ws_bytes, const int32_t* seg_ptr = nullptr,
                            int32_t nseg = 0, const double* box = nullptr, void* stream = nullptr) {
  es_nbr_desc d{N, K, nseg, box ? 1 : 0, r_cut, {box ? box[0] : 0, box ? box[1] : 0, box ? box[2] : 0}};
  idx.N = N;
  idx.K = K;
  check(es_neighbors_build(&d, pos, seg_ptr, idx.table, idx.distances, idx.count, workspace, ws_bytes, stream),
        "build_neighbors");
}
inline void transpose(NeighborIndex& idx, void* workspace, std::size_t ws_bytes, void* stream = nullptr,
                      int32_t n_keys = 0) {
  check(es_neighbors_transpose(idx.N, idx.K, n_keys > 0 ? n_keys : idx.N, idx.table, idx.rev_ptr, idx.rev_pair,
                               workspace, ws_bytes, stream),
        "neighbors_transpose");
}

// project_qk + W_H (Eq. 6)
inline void project_qk(const void* h, const void* W, int32_t N, int32_t lmax, int32_t channels, DType dt, void* q,
                       void* k, void* v, void* stream = nullptr) {
  es_proj_desc d{N, lmax, channels, static_cast<int32_t>(dt)};
  check(es_project_fwd(&d, h, W, q, k, v, stream), "project_qk");
}

// tile structures of a neighbour index, built once and reused by every call on it
inline std::size_t tiles_workspace_size(const AttentionProblem& p) {
  const es_attn_desc d = p.desc();
  return es_attn_tiles_workspace_size(&d);
}
inline void build_tiles(const AttentionProblem& p, NeighborIndex& idx, void* buf, std::size_t bytes,
                        void* stream = nullptr, const int32_t* seg_ptr = nullptr, int32_t nseg = 0) {
  const es_attn_desc d = p.desc();
  // the transposed relation (transpose()) lets the tiles carry the backward's key-side lists
  check(es_attn_tiles_build(&d, idx.table, seg_ptr, nseg, idx.rev_ptr, idx.rev_pair, buf, bytes, stream),
        "build_tiles");
  idx.tiles = bytes ? buf : nullptr;
}

// stream_aggregate: m [N][M][C], lse [N][H]
inline std::size_t forward_workspace_size(const AttentionProblem& p) {
  const es_attn_desc d = p.desc();
  return es_attn_fwd_workspace_size(&d);
}
// scores (optional): [N][K][H] float, kept for the backward (saves recomputing q.k)
inline void stream_aggregate(const AttentionProblem& p, const void* q, const void* k, const void* v,
                             const double* pos, const NeighborIndex& idx, void* m, float* lse, void* workspace,
                             std::size_t ws_bytes, void* stream = nullptr, float* scores = nullptr) {
  const es_attn_desc d = p.desc();
  check(es_attn_fwd(&d, q, k, v, pos, idx.table, m, lse, scores, idx.tiles, workspace, ws_bytes, stream),
        "stream_aggregate");
}

// stream_aggregate_backward
inline std::size_t backward_workspace_size(const AttentionProblem& p) {
  const es_attn_desc d = p.desc();
  return es_attn_bwd_workspace_size(&d);
}
inline void stream_aggregate_backward(const AttentionProblem& p, const void* grad_m, const void* q, const void* k,
                                      const void* v, const double* pos, const NeighborIndex& idx, const void* m,
                                      const float* lse, void* grad_q, void* grad_k, void* grad_v, void* workspace,
                                      std::size_t ws_bytes, void* stream = nullptr, double* grad_pos = nullptr,
                                      const float* scores = nullptr) {
  const es_attn_desc d = p.desc();
  check(es_attn_bwd(&d, q, k, v, pos, idx.table, idx.rev_ptr, idx.rev_pair, m, lse, scores, grad_m, grad_q, grad_k,
                    grad_v, grad_pos, idx.tiles, workspace, ws_bytes, stream),
        "stream_aggregate_backward");
}

// OpCounters / stats structure (counters.hpp:11-32)
inline es_attn_stats stats(const AttentionProblem& p, int64_t n_pairs) {
  const es_attn_desc d = p.desc();
  es_attn_stats st{};
  check(es_attn_stats_query(&d, n_pairs, &st), "stats");
  return st;
}

inline std::string conventions_manifest() { return es_conventions_manifest(); }

}  // namespace equistream::attention
