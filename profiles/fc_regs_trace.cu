// fc_regs_trace.cu — diagnostic harness: the register FC chain (MLP3 paper
// shape) built with per-CTA globaltimer stamps (TCB_FCR_TRACE): entry,
// loads landed, each layer done; offsets from the earliest CTA entry.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_FCR_TRACE \
//        -I paper_1802_04730_b200/csrc profiles/fc_regs_trace.cu -o /tmp/fcr && /tmp/fcr [rows]
#include "kernels/fc_regs.cu"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

using namespace tcb::k;

int main(int argc, char** argv) {
  const int rows = argc > 1 ? atoi(argv[1]) : 2;
  const int NS = 16, B = 128;
  const int outs[3] = {64, 32, 2}, kreds[3] = {128, 64, 32};
  std::vector<FcChainArgs> sets(NS);
  for (int s = 0; s < NS; ++s) {
    FcChainArgs& a = sets[s];
    a = FcChainArgs{};
    float* I;
    cudaMalloc(&I, B * 128 * 4);
    cudaMemset(I, 0, B * 128 * 4);
    a.I = I;
    a.ldi = 128;
    a.batch = B;
    a.layers = 3;
    for (int l = 0; l < 3; ++l) {
      float *W, *b, *O;
      cudaMalloc(&W, outs[l] * kreds[l] * 4);
      cudaMalloc(&b, outs[l] * 4);
      cudaMalloc(&O, B * outs[l] * 4);
      cudaMemset(W, 0, outs[l] * kreds[l] * 4);
      cudaMemset(b, 0, outs[l] * 4);
      a.L[l].W = W;
      a.L[l].bias = b;
      a.L[l].O = O;
      a.L[l].out = outs[l];
      a.L[l].kred = kreds[l];
      a.L[l].ldw = kreds[l];
    }
  }
  for (int r = 0; r < 3; ++r)
    for (int s = 0; s < NS; ++s) launchFcRegs(sets[s], rows, 0);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaError_t le = launchFcRegs(sets[0], rows, 0);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  static unsigned long long tr[1024][8];
  cudaMemcpyFromSymbol(tr, g_fcr_trace, sizeof(tr));
  const int ctas = (B + rows - 1) / rows;
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < ctas; ++b) t0 = std::min(t0, tr[b][0]);
  printf("rows %d: %d CTAs, event %.2f us (launch %s, sync %s)\n", rows, ctas, ms * 1e3, cudaGetErrorString(le),
         cudaGetErrorString(err));
  const char* names[5] = {"entry", "loads landed", "layer 2 done", "layer 3 done", "layer 4 done"};
  for (int ev = 0; ev < 5; ++ev) {
    std::vector<double> v;
    for (int b = 0; b < ctas; ++b)
      if (tr[b][ev]) v.push_back((tr[b][ev] - t0) * 1e-3);
    if (v.empty()) continue;
    std::sort(v.begin(), v.end());
    printf("  %-14s min %6.2f  med %6.2f  p90 %6.2f  max %6.2f us\n", names[ev], v[0], v[v.size() / 2],
           v[v.size() * 9 / 10], v.back());
  }
  return 0;
}
