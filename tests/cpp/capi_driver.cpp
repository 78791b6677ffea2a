// C++ drop-in driver: what a reference-side caller does through
// include/equistream/attention/stream_attention.hpp.  Built by
// tests/test_cpp_driver.py with g++ against libequistream_b200.so.
//
//   capi_driver <in.bin> <out.bin> <f32|bf16> N nseg L C H
//
// in.bin: pos [N][3] f64, seg_ptr [nseg+1] i32 (nseg > 0), q, k [N][M][2C]
// f32, v, dout [N][M][C] f32.  The driver runs the whole hot path --
// build_neighbors, transpose, build_tiles (with the key-side lists),
// stream_aggregate (keeping the scores), stream_aggregate_backward -- in the
// requested storage type and writes out, lse, dq, dk, dv (f32) to out.bin, so
// the test compares them elementwise with the CPU oracle.  Without a GPU it
// checks that an invalid problem surfaces as std::invalid_argument.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "equistream/attention/stream_attention.hpp"

namespace ea = equistream::attention;

namespace {
template <class T>
T* dalloc(size_t n) {
  void* p = nullptr;
  if (cudaMalloc(&p, n * sizeof(T) > 0 ? n * sizeof(T) : 16) != cudaSuccess) throw std::runtime_error("cudaMalloc");
  return static_cast<T*>(p);
}
// device copy of f32 host data in the storage type (bf16: round to nearest even)
void* upload(const std::vector<float>& h, bool bf) {
  if (!bf) {
    float* d = dalloc<float>(h.size());
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    return d;
  }
  std::vector<__nv_bfloat16> b(h.size());
  for (size_t i = 0; i < h.size(); ++i) b[i] = __float2bfloat16_rn(h[i]);
  __nv_bfloat16* d = dalloc<__nv_bfloat16>(h.size());
  cudaMemcpy(d, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  return d;
}
std::vector<float> download(const void* d, size_t n, bool bf) {
  std::vector<float> h(n);
  if (!bf) {
    cudaMemcpy(h.data(), d, n * 4, cudaMemcpyDeviceToHost);
    return h;
  }
  std::vector<__nv_bfloat16> b(n);
  cudaMemcpy(b.data(), d, n * 2, cudaMemcpyDeviceToHost);
  for (size_t i = 0; i < n; ++i) h[i] = __bfloat162float(b[i]);
  return h;
}
}  // namespace

int main(int argc, char** argv) {
  if (argc < 9) return 2;
  const bool bf = std::string(argv[3]) == "bf16";
  const int N = std::atoi(argv[4]), nseg = std::atoi(argv[5]), L = std::atoi(argv[6]), C = std::atoi(argv[7]),
            H = std::atoi(argv[8]);
  const int K = 64, M = (L + 1) * (L + 1);
  std::vector<double> pos((size_t)N * 3);
  std::vector<int32_t> seg(nseg > 0 ? nseg + 1 : 0);
  std::vector<float> q((size_t)N * M * 2 * C), k(q.size()), v((size_t)N * M * C), dout(v.size());
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 2;
  size_t got = std::fread(pos.data(), 8, pos.size(), f);
  got += seg.empty() ? 0 : std::fread(seg.data(), 4, seg.size(), f);
  for (auto* a : {&q, &k, &v, &dout}) got += std::fread(a->data(), 4, a->size(), f);
  std::fclose(f);
  if (got != pos.size() + seg.size() + 2 * q.size() + 2 * v.size()) return 2;
  if (!es_device_ok()) {
    try {  // invalid argument surfaces as std::invalid_argument, like the reference
      ea::AttentionProblem bad;
      bad.N = N; bad.K = K; bad.heads = 3; bad.channels = C;
      ea::stream_aggregate(bad, nullptr, nullptr, nullptr, nullptr, ea::NeighborIndex{}, nullptr, nullptr, nullptr, 0);
    } catch (const std::invalid_argument&) {
      std::printf("NOGPU invalid_argument ok\n");
      return 0;
    }
    return 1;
  }
  try {
    double* dpos = dalloc<double>(pos.size());
    cudaMemcpy(dpos, pos.data(), pos.size() * 8, cudaMemcpyHostToDevice);
    int32_t* dseg = nullptr;
    if (nseg > 0) {
      dseg = dalloc<int32_t>(seg.size());
      cudaMemcpy(dseg, seg.data(), seg.size() * 4, cudaMemcpyHostToDevice);
    }
    void *dq = upload(q, bf), *dk = upload(k, bf), *dv = upload(v, bf), *ddout = upload(dout, bf);
    const size_t es = bf ? 2 : 4;
    void* dout_m = dalloc<char>(v.size() * es);
    void* gq = dalloc<char>(q.size() * es);
    void* gk = dalloc<char>(q.size() * es);
    void* gv = dalloc<char>(v.size() * es);
    float* dlse = dalloc<float>((size_t)N * H);
    float* dscores = dalloc<float>((size_t)N * K * H);
    ea::NeighborIndex idx;
    idx.table = dalloc<int32_t>((size_t)N * K);
    idx.distances = dalloc<float>((size_t)N * K);
    idx.count = dalloc<int32_t>(N);
    idx.rev_ptr = dalloc<int32_t>(N + 1);
    idx.rev_pair = dalloc<int32_t>((size_t)N * K);
    size_t ws = ea::neighbors_workspace_size(N, K, 6.0, nseg);
    void* dws = dalloc<char>(ws);
    ea::build_neighbors(dpos, N, K, 6.0, idx, dws, ws, dseg, nseg);
    size_t tws = es_neighbors_transpose_workspace_size(N, K, N);
    void* dtws = dalloc<char>(tws);
    ea::transpose(idx, dtws, tws);
    ea::AttentionProblem p;
    p.N = N; p.K = K; p.heads = H; p.lmax = L; p.channels = C;
    p.dtype = bf ? ea::DType::BF16 : ea::DType::F32;
    p.nseg = nseg;
    const size_t tiles = ea::tiles_workspace_size(p);
    void* dtiles = tiles ? dalloc<char>(tiles) : nullptr;
    if (tiles) ea::build_tiles(p, idx, dtiles, tiles, nullptr, dseg, nseg);
    const size_t fws = ea::forward_workspace_size(p);
    void* dfws = dalloc<char>(fws);
    ea::stream_aggregate(p, dq, dk, dv, dpos, idx, dout_m, dlse, dfws, fws, nullptr, dscores);
    const size_t bws = ea::backward_workspace_size(p);
    void* dbws = dalloc<char>(bws);
    ea::stream_aggregate_backward(p, ddout, dq, dk, dv, dpos, idx, dout_m, dlse, gq, gk, gv, dbws, bws, nullptr,
                                  nullptr, dscores);
    if (cudaDeviceSynchronize() != cudaSuccess) throw std::runtime_error("device error");
    FILE* o = std::fopen(argv[2], "wb");
    if (!o) return 2;
    for (auto& a : {download(dout_m, v.size(), bf), download(gq, q.size(), bf), download(gk, q.size(), bf),
                    download(gv, v.size(), bf)})
      std::fwrite(a.data(), 4, a.size(), o);
    std::vector<float> lse((size_t)N * H);
    cudaMemcpy(lse.data(), dlse, lse.size() * 4, cudaMemcpyDeviceToHost);
    std::fwrite(lse.data(), 4, lse.size(), o);
    std::fclose(o);
    const es_attn_stats st = ea::stats(p, 0);
    std::printf("OK tiles=%zu fws=%zu bws=%zu madds_proj_fwd=%llu\n", tiles, fws, bws,
                (unsigned long long)st.madds_proj_fwd);
  } catch (const std::exception& e) {
    std::printf("ERROR %s\n", e.what());
    return 1;
  }
  return 0;
}
