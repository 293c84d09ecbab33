// slab_trace.cu — diagnostic harness: the slab TBMM kernel built with
// per-CTA globaltimer stamps (TCB_SLAB_TRACE); prints each phase's offset
// from the earliest CTA start (median / p90 / max over CTAs), cold operands
// (26 rotating sets). Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_SLAB_TRACE \
//        -I paper_1802_04730_b200/csrc profiles/slab_trace.cu -o /tmp/slab_trace && /tmp/slab_trace
#include "kernels/gemm.cu"

#include <algorithm>
#include <cstdio>
#include <vector>

using namespace tcb::k;

int main(int argc, char** argv) {
  const int variant = argc > 1 ? atoi(argv[1]) : 30;
  const int NS = 26, B = 500, N = 26, M = 72;
  std::vector<float*> X(NS), Y(NS), Z(NS);
  std::vector<float> h((size_t)B * N * M);
  for (auto& v : h) v = (rand() / (float)RAND_MAX) * 2 - 1;
  for (int i = 0; i < NS; ++i) {
    cudaMalloc(&X[i], h.size() * 4);
    cudaMalloc(&Y[i], h.size() * 4);
    cudaMalloc(&Z[i], (size_t)B * N * N * 4);
    cudaMemcpy(X[i], h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(Y[i], h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  }
  auto args = [&](int i) {
    GemmArgs a{};
    a.A = X[i]; a.B = Y[i]; a.C = Z[i];
    a.batch = B; a.M = N; a.N = N; a.K = M;
    a.lda = M; a.ldb = M; a.ldc = N; a.sA = N * M; a.sB = N * M; a.sC = N * N;
    return a;
  };
  for (int r = 0; r < 3; ++r)
    for (int i = 0; i < NS; ++i) launchGemm(args(i), variant, 0, 0);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 1; i < NS; ++i) launchGemm(args(i), variant, 0, 0);  // set 0 now cold
  cudaEventRecord(e0);
  launchGemm(args(0), variant, 0, 0);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  static unsigned long long tr[4096][10];
  cudaMemcpyFromSymbol(tr, g_slab_trace, sizeof(tr));
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < B; ++b) t0 = std::min(t0, tr[b][0]);
  printf("variant %d (%s): event time %.2f us (%s)\n", variant, gemmVariant(variant).name, ms * 1e3, cudaGetErrorString(err));
  const char* names[10] = {"entry", "copies issued", "chunk0 ready", "chunk1 ready", "chunk2 ready", "chunk3", "chunk4", "chunk5", "chains done", "stored"};
  for (int ev = 0; ev < 10; ++ev) {
    std::vector<double> v;
    for (int b = 0; b < B; ++b)
      if (tr[b][ev]) v.push_back((tr[b][ev] - t0) * 1e-3);
    if (v.empty()) continue;
    std::sort(v.begin(), v.end());
    printf("  %-14s min %6.2f  med %6.2f  p90 %6.2f  max %6.2f us\n", names[ev], v[0], v[v.size() / 2],
           v[v.size() * 9 / 10], v.back());
  }
  return 0;
}
