// bulk_issue_probe.cu — what does issuing a cp.async.bulk (global -> shared) cost
// the issuing thread? One CTA per SM, thread 0 issues N copies of B bytes from
// distinct 4 KB-aligned sources and reads clock64 before / after the issue
// loop and after the mbarrier completes. Sources L2-warm (second launch) or
// cold (a 512 MB sweep between launches).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 profiles/bulk_issue_probe.cu -o /tmp/bip && /tmp/bip
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// mode 0: one mbarrier, sources i*bytes apart; 1: one mbarrier per copy;
// 2: one mbarrier, sources 64 MB apart (distinct pages / allocations)
__global__ void probe(const char* src, int n, int bytes, long long* out, int stride, int mode) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t bars[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const char* s = src + (size_t)blockIdx.x * stride;
    long long t0 = clock64();
    if (mode == 1) {
      for (int i = 0; i < n; ++i)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[i])), "r"(bytes) : "memory");
    } else {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[0])), "r"(n * bytes) : "memory");
    }
    for (int i = 0; i < n; ++i) {
      const char* g = mode == 2 ? s + (size_t)i * (64ull << 20) : s + (size_t)i * bytes;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(sm + i * bytes)),
                   "l"(g), "r"(bytes), "r"(sa(&bars[mode == 1 ? i : 0]))
                   : "memory");
    }
    long long t1 = clock64();
    for (int i = 0; i < (mode == 1 ? n : 1); ++i) {
      unsigned done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(sa(&bars[i]))
                     : "memory");
    }
    long long t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
}

// copy sources / sizes read from a parameter struct spread over several
// 64-byte constant lines at issue time (as the FC chain kernel does)
struct Spread {
  const char* src[4];
  long long pad0[6];
  int bytes[4];
  long long pad1[7];
  int dst[4];
  long long pad2[7];
};
template <int TOUCH>
__global__ void probe_params(const __grid_constant__ Spread sp, int n, long long* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t bars[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long tt = clock64();
  if (TOUCH == 1)  // vector registers: LDC
    asm volatile("" ::"l"(sp.src[0]), "l"(sp.src[3]), "r"(sp.bytes[0]), "r"(sp.bytes[3]), "r"(sp.dst[0]), "r"(sp.dst[3]));
  if (TOUCH == 2 && (sp.src[0] == nullptr || sp.src[3] == nullptr || sp.bytes[0] == 7 || sp.bytes[3] == 7 ||
                     sp.dst[0] == 7 || sp.dst[3] == 7))  // warp-uniform branch: LDCU
    out[0] = -1;
  long long tt1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1000] = tt1 - tt;
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[i])), "r"(sp.bytes[i])
                   : "memory");
    for (int i = 0; i < n; ++i)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(sm + sp.dst[i])),
                   "l"(sp.src[i] + (size_t)blockIdx.x * (1 << 20)), "r"(sp.bytes[i]), "r"(sa(&bars[i]))
                   : "memory");
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) {
      unsigned done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(sa(&bars[i]))
                     : "memory");
    }
    long long t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
}

int main() {
  char* src;
  char* flush;
  long long* out;
  const size_t big = 512ull << 20;
  cudaMalloc(&src, 148ull * (1 << 20) + 5 * (64ull << 20));
  cudaMalloc(&flush, big);
  cudaMalloc(&out, 148 * 16 + 8008);
  cudaMemset(src, 1, 148ull * (1 << 20) + 5 * (64ull << 20));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  long long h[296];
  {
    Spread sp{};
    for (int i = 0; i < 4; ++i) sp.src[i] = src + (size_t)i * 8192, sp.bytes[i] = 8192, sp.dst[i] = i * 8192;
    void (*kk[3])(Spread, int, long long*) = {probe_params<0>, probe_params<1>, probe_params<2>};
    for (int t = 0; t < 3; ++t) {
      cudaFuncSetAttribute(kk[t], cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
      for (int n : {1, 4}) {
        kk[t]<<<148, 64, 100 * 1024>>>(sp, n, out);
        kk[t]<<<148, 64, 100 * 1024>>>(sp, n, out);
        cudaError_t e = cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        long long touch = 0;
        cudaMemcpy(&touch, out + 1000, 8, cudaMemcpyDeviceToHost);
        double iss = 0, land = 0;
        for (int b = 0; b < 148; ++b) iss += h[2 * b], land += h[2 * b + 1];
        printf("params spread over constant lines, touch %d (%lld cycles), warm %d x 8192 B: issue %7.0f cycles, "
               "landed %7.0f (%s)\n", t, touch, n, iss / 148, land / 148, cudaGetErrorString(e));
      }
    }
  }
  // cluster launches (the FC chain kernel's): does a cluster change the issue cost?
  for (int cl : {2, 4, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(144);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = 100 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    for (int n : {1, 2, 4}) {
      cudaLaunchKernelEx(&cfg, probe, (const char*)src, n, 8192, out, 1 << 20, 1);
      cudaLaunchKernelEx(&cfg, probe, (const char*)src, n, 8192, out, 1 << 20, 1);
      cudaError_t e = cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      double iss = 0, land = 0;
      for (int b = 0; b < 144; ++b) iss += h[2 * b], land += h[2 * b + 1];
      printf("cluster %d, mode 1 warm %3d x 8192 B: issue %7.0f cycles, landed %7.0f cycles (%s)\n", cl, n, iss / 144,
             land / 144, cudaGetErrorString(e));
    }
  }
  for (int mode = 0; mode < 3; ++mode)
  for (int cold = 0; cold < 2; ++cold)
    for (int bytes : {512, 8192})
      for (int n : {1, 2, 4}) {
        if (n * bytes > 200 * 1024) continue;
        probe<<<148, 64, 200 * 1024>>>(src, n, bytes, out, 1 << 20, mode);  // warm-up / L2 fill
        if (cold) cudaMemset(flush, cold, big);
        probe<<<148, 64, 200 * 1024>>>(src, n, bytes, out, 1 << 20, mode);
        cudaError_t e = cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        double iss = 0, land = 0;
        for (int b = 0; b < 148; ++b) iss += h[2 * b], land += h[2 * b + 1];
        printf("mode %d %s %3d x %6d B: issue %7.0f cycles, landed %7.0f cycles (mean over SMs) (%s)\n",
               mode, cold ? "cold" : "warm", n, bytes, iss / 148, land / 148, cudaGetErrorString(e));
      }
  return 0;
}
