// wpair_trace.cu — diagnostic harness: the FFMA2 warp-tile TBMM kernel
// (gemm_chunk.cu) built with per-batch globaltimer stamps (TCB_WPAIR_TRACE);
// times it in a CUDA graph over 26 rotating (cold) input sets, then prints each
// phase's offset from the earliest warp start (min / med / p90 / max over
// batches) and how batches spread over SMs. Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_WPAIR_TRACE \
//        -I paper_1802_04730_b200/csrc profiles/wpair_trace.cu paper_1802_04730_b200/csrc/kernels/attr.cu \
//        -o /tmp/wpair_trace && /tmp/wpair_trace which warps
#include "kernels/gemm_chunk.cu"

#include <algorithm>
#include <cstdio>
#include <map>
#include <vector>

using namespace tcb::k;

int main(int argc, char** argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  const int warps = argc > 2 ? atoi(argv[2]) : 2;
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
    for (int i = 0; i < NS; ++i) launchGemmChunk(args(i), which, warps, 0, 0);
  cudaDeviceSynchronize();
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < NS; ++i) launchGemmChunk(args(i), which, warps, 0, s);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int r = 0; r < 20; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaError_t err = cudaStreamSynchronize(s);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("wpair which=%d warps=%d: %.3f us per launch in a graph (%s)\n", which, warps, ms * 1e3 / (20 * NS),
         cudaGetErrorString(err));
  for (int i = 1; i < NS; ++i) launchGemmChunk(args(i), which, warps, 0, 0);
  cudaDeviceSynchronize();
  launchGemmChunk(args(0), which, warps, 0, 0);
  err = cudaDeviceSynchronize();
  static unsigned long long tr[1024][8];
  cudaMemcpyFromSymbol(tr, g_wpair_trace, sizeof(tr));
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < B; ++b) t0 = std::min(t0, tr[b][0]);
  const char* names[6] = {"entry", "copies issued", "landed", "transposed", "chains done", "stored"};
  for (int ev = 0; ev < 6; ++ev) {
    std::vector<double> v;
    for (int b = 0; b < B; ++b)
      if (tr[b][ev] >= t0 && tr[b][ev] - t0 < 1000000000ull) v.push_back((tr[b][ev] - t0) * 1e-3);
    if (v.empty()) continue;
    std::sort(v.begin(), v.end());
    printf("  %-14s min %6.2f  med %6.2f  p90 %6.2f  max %6.2f us\n", names[ev], v[0], v[v.size() / 2],
           v[v.size() * 9 / 10], v.back());
  }
  std::map<int, int> perSm, hsm;
  for (int b = 0; b < B; ++b) perSm[(int)tr[b][6]]++;
  for (auto& kv : perSm) hsm[kv.second]++;
  printf("  SMs used %zu; batches per SM histogram:", perSm.size());
  for (auto& kv : hsm) printf(" %dx%d", kv.first, kv.second);
  printf("\n");
  return 0;
}
