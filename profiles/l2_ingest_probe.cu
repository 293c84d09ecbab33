// l2_ingest_probe.cu — how many bytes per second can one SM pull when every
// SM streams operands at once? (1) L2-resident (a 4 MB buffer every CTA
// reads), (2) DRAM (a 1 GB buffer, disjoint per CTA). Loads by LDG.128
// (U float4 in flight per thread) and by 1-D bulk copies (S x 16 KB in
// flight per CTA). One CTA per SM, device time of back-to-back launches.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2p profiles/l2_ingest_probe.cu && /tmp/l2p
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void ldg_k(const float4* src, size_t n4, size_t perCta4, float* out) {
  const size_t base = (size_t)blockIdx.x * perCta4 % n4;
  float acc = 0.f;
  for (size_t i = threadIdx.x; i < perCta4; i += (size_t)blockDim.x * U) {
    float4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = __ldg(src + (base + i + (size_t)u * blockDim.x) % n4);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += r[u].x + r[u].y + r[u].z + r[u].w;
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void bulk_k(const char* src, size_t nbytes, size_t perCta, int S, float* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bars[16];
  const int chunk = 16384;
  const size_t base = (size_t)blockIdx.x * perCta % nbytes;
  const int nch = (int)(perCta / chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      unsigned b = (unsigned)__cvta_generic_to_shared(&bars[s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int c = 0; c < nch; ++c) {
      const int s = c % S;
      unsigned b = (unsigned)__cvta_generic_to_shared(&bars[s]);
      if (c >= S) {  // wait for the copy S chunks ago (its slot)
        unsigned done = 0, par = ((c / S) - 1) & 1;
        while (!done)
          asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                       : "=r"(done) : "r"(b), "r"(par) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(chunk) : "memory");
      const char* g = src + (base + (size_t)c * chunk) % nbytes;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (unsigned)__cvta_generic_to_shared(sm + s * chunk)), "l"(g), "r"(chunk), "r"(b) : "memory");
    }
    for (int c = (nch > S ? nch - S : 0); c < nch; ++c) {
      const int s = c % S;
      unsigned b = (unsigned)__cvta_generic_to_shared(&bars[s]);
      unsigned done = 0, par = (c / S) & 1;
      while (!done)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(b), "r"(par) : "memory");
    }
  }
  __syncthreads();
  if (sm[threadIdx.x] == 123) out[0] = 1.f;
}

int main() {
  const size_t big = (size_t)1 << 30, small = (size_t)4 << 20;
  char* buf;
  float* out;
  cudaMalloc(&buf, big);
  cudaMalloc(&out, 64);
  cudaMemset(buf, 0, big);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t perCta = (size_t)2 << 20;  // 2 MB per SM
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / 10;
    printf("%-40s %8.1f us  per SM %6.1f GB/s  total %7.1f GB/s  (%s)\n", name, us, perCta / us / 1e3,
           148.0 * perCta / us / 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  for (int pass = 0; pass < 2; ++pass) {
    const size_t n = pass ? big : small;
    printf("== %s\n", pass ? "DRAM (1 GB buffer, disjoint per SM)" : "L2-resident (4 MB buffer shared by all SMs)");
    run("ldg U4 x 1024 thr", [&] { ldg_k<4><<<148, 1024>>>((const float4*)buf, n / 16, perCta / 16, out); });
    run("ldg U8 x 1024 thr", [&] { ldg_k<8><<<148, 1024>>>((const float4*)buf, n / 16, perCta / 16, out); });
    run("ldg U8 x 512 thr", [&] { ldg_k<8><<<148, 512>>>((const float4*)buf, n / 16, perCta / 16, out); });
    for (int S : {2, 4, 8, 12}) {
      char nm[64];
      snprintf(nm, sizeof nm, "bulk 16 KB x %d in flight", S);
      cudaFuncSetAttribute(bulk_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
      run(nm, [&] { bulk_k<<<148, 128, S * 16384>>>(buf, n, perCta, S, out); });
    }
  }
  return 0;
}
