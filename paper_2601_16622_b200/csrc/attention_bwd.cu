// Launcher of the fused equivariant attention backward (es_attn_bwd): delta,
// key-centric dk/dv/dscore pass, dq (and optionally dk) on the tensor cores.
// The kernels of each degree L live in attention_bwd_l<L>.cu.
#include "attention_bwd.cuh"

namespace es {

es_status attn_bwd_launch(const AttnArgs& a, const void* q, const void* k, const void* v, const double* pos,
                          const int32_t* nbr, const int32_t* rev_ptr, const int32_t* rev_pair, const void* out,
                          const float* lse, const void* dout, void* dq, void* dk, void* dv, float* delta,
                          float* dsbuf, double* dpos, void* ws_tc, size_t ws_tc_bytes, cudaStream_t st) {
  es_status s = upload_tables_tu();
  if (s != ES_OK) return s;
  if (a.N == 0) {
    if (dpos) return cuda_status(cudaMemsetAsync(dpos, 0, sizeof(double) * 3 * (size_t)a.Nk, st), "attn_bwd: dpos");
    return ES_OK;
  }
  const bool tc_dq = attn_dq_tc_applicable(a), tc_dk = attn_dk_tc_applicable(a);
  AttnArgs at = a;
  if (tc_dq && !at.tiles) {  // no prebuilt tile lists: build query- and key-side lists in the workspace first
    s = attn_tc_tiles_build(at, nbr, nullptr, 0, rev_ptr, rev_pair, ws_tc, ws_tc_bytes, st);
    if (s != ES_OK) return s;
    at.tiles = ws_tc;
  }
  // the tensor-core forward keeps its scores in rank space
  const int* rank_of = (tc_dq && at.scores_in) ? attn_tc_rank_of(at, at.tiles) : nullptr;
  switch (at.L) {
#define ES_L(LL)                                                                                              \
  case LL:                                                                                                    \
    s = bwd_run_L<LL>(at, rank_of, q, k, v, pos, nbr, rev_ptr, rev_pair, out, lse, dout, dq, dk, dv, delta, dsbuf, dpos, \
                      tc_dq, tc_dk, st);                                                                      \
    break;
    ES_L(0) ES_L(1) ES_L(2) ES_L(3) ES_L(4)
#undef ES_L
    default:
      return fail(ES_UNSUPPORTED, "attention: no kernel for this L");
  }
  if (s != ES_OK) return s;
  if (tc_dq) {
    s = attn_dq_tc_launch(at, k, nbr, dsbuf, dq, nullptr, 0, st);
    if (s != ES_OK) return s;
  }
  if (tc_dk) s = attn_dk_tc_launch(at, q, nbr, rev_ptr, rev_pair, dsbuf, dk, nullptr, 0, st);
  return s;
}

}  // namespace es
