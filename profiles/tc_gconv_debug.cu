// Diagnostic harness: the tcgen05 gconv kernel built with TCB_DEBUG_BARRIERS
// (a stuck mbarrier is recorded instead of trapping) on a small problem.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_DEBUG_BARRIERS \
//        -I paper_1802_04730_b200/csrc profiles/tc_gconv_debug.cu -o /tmp/tcg && /tmp/tcg
#include <cstdio>
#include <vector>

#include "kernels/tc_gconv.cu"

using namespace tcb::k;

int main(int argc, char** argv) {
  int N = 2, G = 3, C = 16, H = 10, W = 10, F = 16, KH = 3, KW = 3, Mb = 16;
  int x3 = argc > 1 ? atoi(argv[1]) : 0;
  size_t ni = (size_t)N * G * C * H * W, nw = (size_t)G * F * C * KH * KW, no = (size_t)N * G * F * (H - 2) * (W - 2);
  std::vector<float> hi(ni), hw(nw), hb(Mb, 0.f);
  for (size_t i = 0; i < ni; ++i) hi[i] = (i % 7) * 0.125f;
  for (size_t i = 0; i < nw; ++i) hw[i] = ((i % 5) - 2) * 0.25f;
  float *dI, *dW, *dB, *dO;
  cudaMalloc(&dI, ni * 4); cudaMalloc(&dW, nw * 4); cudaMalloc(&dB, Mb * 4); cudaMalloc(&dO, no * 4);
  cudaMemcpy(dI, hi.data(), ni * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, hw.data(), nw * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hb.data(), Mb * 4, cudaMemcpyHostToDevice);
  GconvArgs a{dI, dW, dB, dO, N, G, C, H, W, F, KH, KW, Mb};
  cudaError_t e = launchTcGconv(a, x3 ? kMath3xTf32 : kMathTf32, 0);
  printf("launch: %s\n", cudaGetErrorString(e));
  e = cudaDeviceSynchronize();
  printf("sync: %s\n", cudaGetErrorString(e));
  std::vector<float> ho(no);
  cudaMemcpy(ho.data(), dO, no * 4, cudaMemcpyDeviceToHost);
  // CPU reference for output (n=0,g=0,f=0..1, h=0, w=0..7)
  for (int f = 0; f < 2; ++f)
    for (int w = 0; w < 8; ++w) {
      double s = 0;
      for (int c = 0; c < C; ++c)
        for (int kh = 0; kh < 3; ++kh)
          for (int kw = 0; kw < 3; ++kw)
            s += hi[((size_t)c * H + kh) * W + w + kw] * hw[(((size_t)f * C + c) * 3 + kh) * 3 + kw];
      printf("f%d w%d gpu %.5f ref %.5f\n", f, w, ho[(size_t)f * 64 + w], s);
    }
  return 0;
}
