// Diagnostic: cycles a thread spends ISSUING cp.async.bulk copies (global ->
// shared, mbarrier complete_tx), and until they land, for several copy
// sizes, in a plain launch and a cluster launch, with warm and cold sources.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 profiles/bulk_probe.cu -o /tmp/bp && /tmp/bp
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void probe(const float* src, int ncopies, unsigned bytes, long long* out, int useCluster) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes * ncopies) : "memory");
    long long t1 = clock64();
    for (int i = 0; i < ncopies; ++i) {
      const float* s = src + (size_t)blockIdx.x * ncopies * (bytes / 4) + (size_t)i * (bytes / 4);
      if (useCluster)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         sa(sm + i * (bytes / 4))), "l"(s), "r"(bytes), "r"(sa(&bar)) : "memory");
      else
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         sa(sm + i * (bytes / 4))), "l"(s), "r"(bytes), "r"(sa(&bar)) : "memory");
    }
    long long t2 = clock64();
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(sa(&bar)) : "memory");
    long long t3 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t1;
      out[2] = t3 - t2;
    }
  }
}

int main() {
  float* src;
  size_t n = 256ull << 20;
  cudaMalloc(&src, n);
  cudaMemset(src, 0, n);
  long long* out;
  cudaMalloc(&out, 64);
  float* flush;
  cudaMalloc(&flush, 512ull << 20);
  for (int cl : {0, 1})
    for (unsigned bytes : {1024u, 8192u, 32768u})
      for (int nc : {1, 2, 4}) {
        if (bytes * nc > 200 * 1024) continue;
        size_t smem = bytes * nc;
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int pass = 0; pass < 3; ++pass) {  // 0: cold (after flush), 1-2: warm
          if (pass == 0) cudaMemset(flush, pass + 1, 512ull << 20);
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(128, 1, 1);
          cfg.blockDim = dim3(64, 1, 1);
          cfg.dynamicSmemBytes = smem;
          cudaLaunchAttribute attr[1];
          attr[0].id = cudaLaunchAttributeClusterDimension;
          attr[0].val.clusterDim.x = cl ? 4 : 1;
          attr[0].val.clusterDim.y = 1;
          attr[0].val.clusterDim.z = 1;
          cfg.attrs = attr;
          cfg.numAttrs = 1;
          cudaLaunchKernelEx(&cfg, probe, (const float*)src, nc, bytes, out, cl);
          cudaError_t e = cudaDeviceSynchronize();
          long long h[3];
          cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
          printf("cluster=%d bytes=%6u copies=%d %s: expect_tx %4lld  issue %5lld (%lld/copy)  land %6lld cycles (%s)\n",
                 cl, bytes, nc, pass == 0 ? "cold" : "warm", h[0], h[1], h[1] / nc, h[2], cudaGetErrorString(e));
        }
      }
  return 0;
}
