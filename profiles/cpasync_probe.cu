// Diagnostic: cycles from issuing to landing for per-thread 16-byte
// cp.async (LDGSTS) copies vs one bulk copy of the same bytes, 64-thread
// CTAs, 2 per SM, warm (L2) and cold (HBM) sources.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 profiles/cpasync_probe.cu -o /tmp/cpp && /tmp/cpp
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(64) lds_probe(const float* src, int n16, long long* out, int mode) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t bar;
  const float* s = src + (size_t)blockIdx.x * n16 * 4;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long t0 = clock64();
  if (mode == 0) {  // cp.async 16 B per thread, coalesced, padded destination rows of 256 floats
    for (int e = threadIdx.x; e < n16; e += blockDim.x) {
      const int row = e / 64, c = e % 64;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(sm + row * 260 + c * 4)), "l"(s + e * 4)
                   : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
  } else {  // one bulk copy
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(n16 * 16) : "memory");
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(sm)), "l"(s), "r"(n16 * 16), "r"(sa(&bar)) : "memory");
    }
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(sa(&bar)) : "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  float* src;
  cudaMalloc(&src, 256u << 20);
  cudaMemset(src, 0, 256u << 20);
  float* flush;
  cudaMalloc(&flush, 512u << 20);
  long long* out;
  cudaMalloc(&out, 4096 * 8);
  static long long h[4096];
  for (int mode : {0, 1})
    for (int kb : {4, 16, 64}) {
      const int n16 = kb * 1024 / 16;
      const size_t smem = (size_t)(n16 / 64 + 1) * 260 * 4 + 1024;
      cudaFuncSetAttribute(lds_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int pass = 0; pass < 3; ++pass) {
        if (pass == 0) cudaMemset(flush, 1, 512u << 20);
        lds_probe<<<296, 64, smem>>>(src, n16, out, mode);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, out, 296 * 8, cudaMemcpyDeviceToHost);
        long long mx = 0, sum = 0;
        for (int i = 0; i < 296; ++i) mx = h[i] > mx ? h[i] : mx, sum += h[i];
        printf("%-9s %3d KB per CTA (296 CTAs) %s: mean %6lld max %6lld cycles (%s)\n", mode ? "bulk" : "cp.async",
               kb, pass ? "warm" : "cold", sum / 296, mx, cudaGetErrorString(e));
      }
    }
  return 0;
}
