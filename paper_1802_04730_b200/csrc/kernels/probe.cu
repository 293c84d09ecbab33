// probe.cu — device peak probes for the roofline denominators that
// MEASURED_PEAKS.json does not hold: fp32 FFMA throughput (the bound of the
// FFMA-exact contractions: C3, gconv, MLP layers). Not on the hot path.
#include "kernels.cuh"

namespace tcb {
namespace k {
namespace {

constexpr int kChains = 8;

// Each thread runs kChains independent fma.rn.f32 chains (latency 4 cycles,
// 4 chains already saturate one SMSP's FMA pipe; 8 leaves slack).
__global__ void __launch_bounds__(256) ffma_probe(float* out, int iters, float a, float b) {
  float acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-7f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) acc[c] = __fmaf_rn(acc[c], a, b);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 123.456f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;  // defeat DCE
}

__global__ void empty_probe(int* p) {
  if (p && threadIdx.x == 1234567) *p = 0;
}

}  // namespace

// Device time per launch of back-to-back empty kernels replayed from a CUDA
// graph (the floor any launch-bound operator sits on): `ctas` CTAs of
// `threads` threads in clusters of `cluster` (1 = no cluster attribute).
cudaError_t probeLaunch(int ctas, int threads, int cluster, double* us) {
  cudaStream_t s;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e != cudaSuccess) return e;
  const int n = 64;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < n && e == cudaSuccess; ++i) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(threads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cluster > 1 ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, empty_probe, static_cast<int*>(nullptr));
  }
  cudaError_t e2 = cudaStreamEndCapture(s, &g);
  if (e == cudaSuccess) e = e2;
  if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, g, 0);
  float ms = 0.f;
  if (e == cudaSuccess) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    e = cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (ge) cudaGraphExecDestroy(ge);
  if (g) cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  *us = ms * 1e3 / (10.0 * n);
  return e;
}

cudaError_t probeFfma(int sms, double* tflops, float* ms_out) {
  float* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(float) * sms * 8 * 256);
  if (e != cudaSuccess) return e;
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ffma_probe<<<blocks, threads>>>(d, 64, 0.999f, 1e-3f);  // warm-up (clocks up)
  ffma_probe<<<blocks, threads>>>(d, iters, 0.999f, 1e-3f);
  cudaEventRecord(e0);
  ffma_probe<<<blocks, threads>>>(d, iters, 0.999f, 1e-3f);
  cudaEventRecord(e1);
  e = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (e != cudaSuccess) return e;
  e = cudaGetLastError();
  double flops = 2.0 * blocks * threads * double(iters) * 16 * kChains;
  *tflops = flops / (ms * 1e-3) / 1e12;
  if (ms_out) *ms_out = ms;
  return e;
}

}  // namespace k
}  // namespace tcb
