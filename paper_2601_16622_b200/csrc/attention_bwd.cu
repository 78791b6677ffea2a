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
  const bool tc_dq = attn_dq_tc_applicable(a);
  // forces stay on the SIMT key pass (any L); the tensor-core key pass bulk-copies query positions and
  // lse rows in 16-byte units (an unaligned caller buffer takes the SIMT pass)
  const bool tc_kv = !dpos && attn_kv_tc_applicable(a) && ((uintptr_t)pos & 15) == 0 && ((uintptr_t)lse & 15) == 0;
  const bool tc_dk = tc_kv || attn_dk_tc_applicable(a);
  AttnArgs at = a;
  if (tc_dq && !at.tiles) {  // no prebuilt tile lists: build query- and key-side lists in the workspace first
    s = attn_tc_tiles_build(at, nbr, nullptr, 0, rev_ptr, rev_pair, ws_tc, ws_tc_bytes, st);
    if (s != ES_OK) return s;
    at.tiles = ws_tc;
  }
  if (tc_kv) {  // delta, key pass (dv + dscores), dq, dk: every contraction on the tensor cores
    if ((s = attn_delta_launch(at, out, dout, delta, st)) != ES_OK) return s;
    // the pair-geometry records follow the (possibly unused) tile-list space of the workspace
    const size_t goff = (attn_tc_tiles_bytes(a) + 255) & ~size_t(255);
    if (!ws_tc || ws_tc_bytes < goff + attn_kv_tc_geom_bytes(a))
      return fail(ES_INVALID_ARGUMENT, "attn_bwd: workspace too small (key pass)");
    if ((s = attn_kv_tc_launch(at, q, k, v, pos, rev_ptr, rev_pair, lse, dout, delta, dsbuf, dv,
                               static_cast<char*>(ws_tc) + goff, st)) != ES_OK)
      return s;
    if ((s = attn_dq_tc_launch(at, k, nbr, dsbuf, dq, nullptr, 0, st)) != ES_OK) return s;
    return attn_dk_tc_launch(at, q, nbr, rev_ptr, rev_pair, dsbuf, dk, nullptr, 0, st);
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

es_status attn_delta_launch(const AttnArgs& a, const void* out, const void* dout, float* delta, cudaStream_t st) {
  // delta_i^h = dO_i^h . out_i^h (bf16, C = 128, H = 8: 16 threads per atom, 2 per head)
  if (a.dtype != ES_BF16 || a.C != 128 || a.H != 8) return fail(ES_UNSUPPORTED, "attn_delta: bf16 C=128 H=8 only");
  const int M = (a.L + 1) * (a.L + 1), apb = 256 / (a.C / 8);
  attn_delta_kernel<__nv_bfloat16, 8><<<(a.N + apb - 1) / apb, apb * (a.C / 8), 0, st>>>(
      a.N, M, a.C, a.H, (const __nv_bfloat16*)out, (const __nv_bfloat16*)dout, delta);
  return cuda_status(cudaGetLastError(), "attn_delta_kernel");
}

}  // namespace es
