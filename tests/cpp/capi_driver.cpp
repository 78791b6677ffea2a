// C++ drop-in driver: what a reference-side caller does through
// include/equistream/attention/stream_attention.hpp.  Built by
// tests/test_cpp_driver.py with g++ against libequistream_b200.so; on a GPU
// box it runs config 1 (N=64 FCC, L=2, C=64, H=8) and prints a checksum that
// the test compares with the oracle; without a GPU it checks the error path.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "equistream/attention/stream_attention.hpp"

namespace ea = equistream::attention;

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const int N = 64, K = 64, L = 2, C = 64, H = 8, M = (L + 1) * (L + 1);
  // inputs: positions / q / k / v from a binary blob written by the test
  std::vector<double> pos(N * 3);
  std::vector<float> q(N * M * 2 * C), k(N * M * 2 * C), v(N * M * C);
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 2;
  size_t got = std::fread(pos.data(), 8, pos.size(), f) + std::fread(q.data(), 4, q.size(), f) +
               std::fread(k.data(), 4, k.size(), f) + std::fread(v.data(), 4, v.size(), f);
  std::fclose(f);
  if (got != pos.size() + q.size() + k.size() + v.size()) return 2;
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
  double *dpos;
  float *dq, *dk, *dv, *dout, *dlse, *ddist;
  int32_t *dnbr, *dcnt;
  cudaMalloc(&dpos, pos.size() * 8);
  cudaMalloc(&dq, q.size() * 4);
  cudaMalloc(&dk, k.size() * 4);
  cudaMalloc(&dv, v.size() * 4);
  cudaMalloc(&dout, v.size() * 4);
  cudaMalloc(&dlse, N * H * 4);
  cudaMalloc(&dnbr, N * K * 4);
  cudaMalloc(&ddist, N * K * 4);
  cudaMalloc(&dcnt, N * 4);
  cudaMemcpy(dpos, pos.data(), pos.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dq, q.data(), q.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dk, k.data(), k.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, v.data(), v.size() * 4, cudaMemcpyHostToDevice);
  ea::NeighborIndex idx;
  idx.table = dnbr; idx.distances = ddist; idx.count = dcnt;
  const size_t ws = ea::neighbors_workspace_size(N, K, 6.0);
  void* dws;
  cudaMalloc(&dws, ws);
  ea::build_neighbors(dpos, N, K, 6.0, idx, dws, ws);
  ea::AttentionProblem p;
  p.N = N; p.K = K; p.heads = H; p.lmax = L; p.channels = C;
  const size_t fws = ea::forward_workspace_size(p);
  void* dfws;
  cudaMalloc(&dfws, fws);
  ea::stream_aggregate(p, dq, dk, dv, dpos, idx, dout, dlse, dfws, fws);
  std::vector<float> out(v.size());
  cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
  double s = 0, s2 = 0;
  for (float x : out) { s += x; s2 += (double)x * x; }
  std::printf("CHECKSUM %.9e %.9e\n", s, s2);
  return 0;
}
