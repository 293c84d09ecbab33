// read_floor.cu — how fast can one kernel pull TBMM's 7.49 MB of operands
// (cold in L2) and write its 1.35 MB result on a B200? Several load
// strategies, each a CUDA graph of back-to-back launches over 26 rotating
// buffer sets (> 2x L2), device time per launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/read_floor profiles/read_floor.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int NB = 500, ROWF = 26 * 72;     // per batch: X and Y 1872 floats each
constexpr int OUTF = 26 * 26;
constexpr int NSET = 26;

__global__ void empty_k(float*) {}

// one CTA per batch, every thread cp.async 16B, then write 676 floats
__global__ void cpasync_k(const float* X, const float* Y, float* Z) {
  __shared__ __align__(16) float s[2 * ROWF];
  const int b = blockIdx.x;
  for (int e = threadIdx.x; e < 2 * ROWF / 4; e += blockDim.x) {
    const float* src = e < ROWF / 4 ? X + (size_t)b * ROWF + 4 * e : Y + (size_t)b * ROWF + 4 * (e - ROWF / 4);
    unsigned d = (unsigned)__cvta_generic_to_shared(s + 4 * e);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src));
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  for (int e = threadIdx.x; e < OUTF; e += blockDim.x) Z[(size_t)b * OUTF + e] = s[e] + s[ROWF + e];
}

// one CTA per batch: thread 0 issues two bulk copies onto one mbarrier
__global__ void bulk_k(const float* X, const float* Y, float* Z) {
  __shared__ __align__(128) float s[2 * ROWF];
  __shared__ __align__(8) uint64_t bar;
  const int b = blockIdx.x;
  unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(2 * ROWF * 4) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(s)), "l"(X + (size_t)b * ROWF), "r"(ROWF * 4), "r"(sb) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(s + ROWF)), "l"(Y + (size_t)b * ROWF), "r"(ROWF * 4), "r"(sb) : "memory");
  }
  __syncthreads();
  unsigned done = 0;
  while (!done) {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(sb) : "memory");
  }
  for (int e = threadIdx.x; e < OUTF; e += blockDim.x) Z[(size_t)b * OUTF + e] = s[e] + s[ROWF + e];
}

// one CTA per batch, LDG.128 into registers (coalesced), reduce, write
__global__ void ldg_k(const float* X, const float* Y, float* Z) {
  const int b = blockIdx.x;
  const float4* x = reinterpret_cast<const float4*>(X + (size_t)b * ROWF);
  const float4* y = reinterpret_cast<const float4*>(Y + (size_t)b * ROWF);
  float acc = 0.f;
  float4 r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int e = threadIdx.x + i * blockDim.x;
    r[i] = e < ROWF / 4 ? __ldg(x + e) : e < ROWF / 2 ? __ldg(y + e - ROWF / 4) : make_float4(0, 0, 0, 0);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += r[i].x + r[i].y + r[i].z + r[i].w;
  for (int e = threadIdx.x; e < OUTF; e += blockDim.x) Z[(size_t)b * OUTF + e] = acc;
}

// grid-stride over all of X and Y as one flat stream, 148*k CTAs
template <int U>
__global__ void flat_k(const float4* X, const float4* Y, float* Z, int n4) {
  float acc = 0.f;
  const int T = gridDim.x * blockDim.x;
  for (int base = blockIdx.x * blockDim.x + threadIdx.x; base < 2 * n4; base += U * T) {
    float4 r[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      int e = base + i * T;
      r[i] = e < n4 ? __ldg(X + e) : e < 2 * n4 ? __ldg(Y + e - n4) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int i = 0; i < U; ++i) acc += r[i].x + r[i].y + r[i].z + r[i].w;
  }
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int e = tid; e < NB * OUTF; e += T) Z[e] = acc;
}


// the slab TBMM kernel (gemm.cu gemm_nt_slab<18,CH>) with stages switched
// off: mode 0 = loads only, 1 = loads + chains, 2 = chains without the
// B-row LDG (B from smem)
template <int CH>
__global__ void __launch_bounds__(256) slab_k(const float* X, const float* Y, float* Z, int mode) {
  __shared__ __align__(16) float sA[26 * 72];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ng = blockDim.x / 32, g = warp;
  const int b = blockIdx.x, n = lane, K4 = 18;
  const float* A = X + (size_t)b * ROWF;
  const float* B = Y + (size_t)b * ROWF;
  for (int e = tid; e < 26 * K4; e += blockDim.x) {
    unsigned d = (unsigned)__cvta_generic_to_shared(sA + 4 * e);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(A + 4 * e));
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  const float4* Brow = reinterpret_cast<const float4*>(B + (size_t)min(n, 25) * 72);
  float4 br[18];
#pragma unroll
  for (int q = 0; q < 18; ++q) br[q] = __ldg(Brow + q);
  float acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = 0.f;
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  if (mode == 1) {
    const unsigned aS = (unsigned)__cvta_generic_to_shared(sA);
    unsigned rowAddr[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) rowAddr[c] = aS + (unsigned)(min(g * CH + c, 25) * 72) * 4u;
#pragma unroll
    for (int q = 0; q < 18; ++q) {
      float4 av[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c)
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(av[c].x), "=f"(av[c].y), "=f"(av[c].z), "=f"(av[c].w) : "r"(rowAddr[c] + q * 16));
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = __fmaf_rn(av[c].x, br[q].x, acc[c]);
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = __fmaf_rn(av[c].y, br[q].y, acc[c]);
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = __fmaf_rn(av[c].z, br[q].z, acc[c]);
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = __fmaf_rn(av[c].w, br[q].w, acc[c]);
    }
  } else {
#pragma unroll
    for (int q = 0; q < 18; ++q) acc[0] += br[q].x + br[q].y + br[q].z + br[q].w + sA[q * 4 + lane];
  }
  if (n < 26) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int m = g * CH + c;
      if (m < 26) Z[(size_t)b * OUTF + m * 26 + n] = acc[c];
    }
  }
}

int main() {
  std::vector<float*> X(NSET), Y(NSET), Z(NSET);
  for (int i = 0; i < NSET; ++i) {
    CK(cudaMalloc(&X[i], (size_t)NB * ROWF * 4));
    CK(cudaMalloc(&Y[i], (size_t)NB * ROWF * 4));
    CK(cudaMalloc(&Z[i], (size_t)NB * OUTF * 4));
    cudaMemset(X[i], 0, (size_t)NB * ROWF * 4);
    cudaMemset(Y[i], 0, (size_t)NB * ROWF * 4);
  }
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  auto timeit = [&](const char* name, auto launch) -> int {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int r = 0; r < 4; ++r)
      for (int i = 0; i < NSET; ++i) launch(i);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaStreamSynchronize(s));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0, s);
      CK(cudaGraphLaunch(ge, s));
      cudaEventRecord(e1, s);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    double us = best * 1e3 / (4 * NSET);
    double bytes = (double)NB * (2 * ROWF + OUTF) * 4;
    printf("%-34s %8.3f us  %7.1f GB/s\n", name, us, bytes / us / 1e3);
    return 0;
  };
  timeit("empty 500x128", [&](int i) { empty_k<<<NB, 128, 0, s>>>(Z[i]); });
  timeit("cp.async 16B, 1 CTA/batch x128", [&](int i) { cpasync_k<<<NB, 128, 0, s>>>(X[i], Y[i], Z[i]); });
  timeit("cp.async 16B, 1 CTA/batch x256", [&](int i) { cpasync_k<<<NB, 256, 0, s>>>(X[i], Y[i], Z[i]); });
  timeit("bulk 2 copies, 1 CTA/batch x128", [&](int i) { bulk_k<<<NB, 128, 0, s>>>(X[i], Y[i], Z[i]); });
  timeit("ldg 8xf4/thread, 1 CTA/batch x128", [&](int i) { ldg_k<<<NB, 128, 0, s>>>(X[i], Y[i], Z[i]); });
  const int n4 = NB * ROWF / 4;
  timeit("flat U4 148x512", [&](int i) { flat_k<4><<<148, 512, 0, s>>>((float4*)X[i], (float4*)Y[i], Z[i], n4); });
  timeit("flat U8 148x512", [&](int i) { flat_k<8><<<148, 512, 0, s>>>((float4*)X[i], (float4*)Y[i], Z[i], n4); });
  timeit("flat U8 296x512", [&](int i) { flat_k<8><<<296, 512, 0, s>>>((float4*)X[i], (float4*)Y[i], Z[i], n4); });
  timeit("flat U4 592x256", [&](int i) { flat_k<4><<<592, 256, 0, s>>>((float4*)X[i], (float4*)Y[i], Z[i], n4); });
  timeit("flat U2 1184x256", [&](int i) { flat_k<2><<<1184, 256, 0, s>>>((float4*)X[i], (float4*)Y[i], Z[i], n4); });
  timeit("flat U1 2368x256", [&](int i) { flat_k<1><<<2368, 256, 0, s>>>((float4*)X[i], (float4*)Y[i], Z[i], n4); });
  timeit("slab c7 loads only", [&](int i) { slab_k<7><<<NB, 128, 0, s>>>(X[i], Y[i], Z[i], 0); });
  timeit("slab c7 full", [&](int i) { slab_k<7><<<NB, 128, 0, s>>>(X[i], Y[i], Z[i], 1); });
  timeit("slab c13 full", [&](int i) { slab_k<13><<<NB, 64, 0, s>>>(X[i], Y[i], Z[i], 1); });
  timeit("WARM slab c7 full", [&](int i) { slab_k<7><<<NB, 128, 0, s>>>(X[0], Y[0], Z[0], 1); });
  timeit("WARM slab c7 loads only", [&](int i) { slab_k<7><<<NB, 128, 0, s>>>(X[0], Y[0], Z[0], 0); });
  // same, warm (one set repeated: L2 resident)
  timeit("WARM cp.async 1 CTA/batch x128", [&](int i) { cpasync_k<<<NB, 128, 0, s>>>(X[0], Y[0], Z[0]); });
  timeit("WARM flat U8 296x512", [&](int i) { flat_k<8><<<296, 512, 0, s>>>((float4*)X[0], (float4*)Y[0], Z[0], n4); });
  return 0;
}
