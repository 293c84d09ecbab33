// tcfc_trace.cu — phase stamps of the one-kernel tensor-core FC chain (MLP3
// paper shape): entry, operands landed, split done, per layer MMAs done /
// epilogue done. Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_TCFC_TRACE \
//        -I paper_1802_04730_b200/csrc profiles/tcfc_trace.cu paper_1802_04730_b200/csrc/kernels/attr.cu -o /tmp/tcfc -lcuda && /tmp/tcfc
#include "kernels/tc_fc_fused.cu"

#include <cstdio>

using namespace tcb::k;

int main() {
  const int B = 128, outs[3] = {64, 32, 2}, kreds[3] = {128, 64, 32};
  FcChainArgs a{};
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
    a.L[l] = FcLayer{W, b, O, outs[l], kreds[l], kreds[l]};
  }
  for (int math : {kMathTf32, kMath3xTf32}) {
    for (int r = 0; r < 3; ++r) launchTcFcFused(a, math, 0);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t le = launchTcFcFused(a, math, 0);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long tr[32];
    cudaMemcpyFromSymbol(tr, g_tcfc_trace, sizeof(tr));
    printf("%s: event %.2f us (%s / %s)\n", math == kMathTf32 ? "tf32" : "3xtf32", ms * 1e3, cudaGetErrorString(le),
           cudaGetErrorString(err));
    const char* nm[8] = {"entry", "landed", "split", "L1 mma", "L1 epi", "L2 mma", "L2 epi", "L3 mma"};
    for (int i = 1; i < 8; ++i) printf("  %-8s +%.2f us\n", nm[i], (tr[i] - tr[0]) * 1e-3);
    for (int i = 20; i < 23; ++i) printf("  L%d MMAs issued +%.2f us\n", i - 19, (tr[i] - tr[0]) * 1e-3);
  }
  return 0;
}
