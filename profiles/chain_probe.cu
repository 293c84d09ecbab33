// Diagnostic: cycles per step of one sequential FFMA chain (the FFMA-exact
// reduction order) with operands from registers, and from shared memory via
// the FC chain's double-buffered float4 loads, at 1..4 warps per SM sub-partition.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 profiles/chain_probe.cu -o /tmp/cp && /tmp/cp
#include <cstdio>

__device__ __forceinline__ float4 lds4(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float fma4(float4 x, float4 w, float acc) {
  acc = __fmaf_rn(x.x, w.x, acc);
  acc = __fmaf_rn(x.y, w.y, acc);
  acc = __fmaf_rn(x.z, w.z, acc);
  return __fmaf_rn(x.w, w.w, acc);
}

__global__ void chain_reg(float* out, long long* cyc, int n, float a, float b) {
  float acc = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) acc = __fmaf_rn(acc, a, b);
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// n steps, x and w rows in smem (row per lane), chunk of 16 prefetched one ahead
__global__ void chain_smem(float* out, long long* cyc, int n) {
  extern __shared__ float sm[];
  const int ld = n + 36;  // row stride ≡ 4 mod 32 when n % 32 == 0
  for (int e = threadIdx.x; e < 2 * blockDim.x * ld; e += blockDim.x) sm[e] = 1e-3f * (e % 97);
  __syncthreads();
  unsigned xa = (unsigned)__cvta_generic_to_shared(sm + threadIdx.x * ld);
  unsigned wa = (unsigned)__cvta_generic_to_shared(sm + (blockDim.x + threadIdx.x) * ld);
  float acc = 0.f;
  long long t0 = clock64();
  const int nch = n >> 4;
  float4 X0[4], W0[4], X1[4], W1[4];
  for (int i = 0; i < 4; ++i) { X0[i] = lds4(xa + i * 16); W0[i] = lds4(wa + i * 16); }
  for (int c = 0; c + 2 <= nch; c += 2) {
    const unsigned o = c * 64;
    for (int i = 0; i < 4; ++i) { X1[i] = lds4(xa + o + 64 + i * 16); W1[i] = lds4(wa + o + 64 + i * 16); }
    for (int i = 0; i < 4; ++i) acc = fma4(X0[i], W0[i], acc);
    for (int i = 0; i < 4; ++i) { X0[i] = lds4(xa + o + 128 + i * 16); W0[i] = lds4(wa + o + 128 + i * 16); }
    for (int i = 0; i < 4; ++i) acc = fma4(X1[i], W1[i], acc);
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void chain_reg_unrolled(float* out, long long* cyc, int n, float a, float b) {
  float acc = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) acc = __fmaf_rn(acc, a, b);
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// same loads as chain_smem, but each FFMA pairs components of different
// register-bank parity (x.y with w.x, ...): timing only, not the exact sum
__device__ __forceinline__ float fma4rot(float4 x, float4 w, float acc) {
  acc = __fmaf_rn(x.y, w.x, acc);
  acc = __fmaf_rn(x.z, w.y, acc);
  acc = __fmaf_rn(x.w, w.z, acc);
  return __fmaf_rn(x.x, w.w, acc);
}
template <bool ROT, bool BCAST>
__global__ void chain_smem_v(float* out, long long* cyc, int n) {
  extern __shared__ float sm[];
  const int ld = n + 36;
  for (int e = threadIdx.x; e < 2 * blockDim.x * ld; e += blockDim.x) sm[e] = 1e-3f * (e % 97);
  __syncthreads();
  unsigned xa = (unsigned)__cvta_generic_to_shared(sm + (BCAST ? 0 : threadIdx.x * ld));
  unsigned wa = (unsigned)__cvta_generic_to_shared(sm + (blockDim.x + threadIdx.x) * ld);
  float acc = 0.f;
  long long t0 = clock64();
  const int nch = n >> 4;
  float4 X0[4], W0[4], X1[4], W1[4];
  for (int i = 0; i < 4; ++i) { X0[i] = lds4(xa + i * 16); W0[i] = lds4(wa + i * 16); }
  for (int c = 0; c + 2 <= nch; c += 2) {
    const unsigned o = c * 64;
    for (int i = 0; i < 4; ++i) { X1[i] = lds4(xa + o + 64 + i * 16); W1[i] = lds4(wa + o + 64 + i * 16); }
    for (int i = 0; i < 4; ++i) acc = ROT ? fma4rot(X0[i], W0[i], acc) : fma4(X0[i], W0[i], acc);
    for (int i = 0; i < 4; ++i) { X0[i] = lds4(xa + o + 128 + i * 16); W0[i] = lds4(wa + o + 128 + i * 16); }
    for (int i = 0; i < 4; ++i) acc = ROT ? fma4rot(X1[i], W1[i], acc) : fma4(X1[i], W1[i], acc);
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// plain (non-volatile) loads: lets the compiler schedule and allocate freely
template <bool BCAST>
__global__ void chain_smem_plain(float* out, long long* cyc, int n) {
  extern __shared__ float sm[];
  const int ld = n + 36;
  for (int e = threadIdx.x; e < 2 * blockDim.x * ld; e += blockDim.x) sm[e] = 1e-3f * (e % 97);
  __syncthreads();
  const float4* x = reinterpret_cast<const float4*>(sm + (BCAST ? 0 : threadIdx.x * ld));
  const float4* w = reinterpret_cast<const float4*>(sm + (blockDim.x + threadIdx.x) * ld);
  float acc = 0.f;
  long long t0 = clock64();
#pragma unroll 8
  for (int c = 0; c < n / 4; ++c) acc = fma4(x[c], w[c], acc);
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K>
static void runSmem(const char* name, K kern, float* out, long long* cyc, int n) {
  long long h[1];
  for (int warps : {1, 2, 4, 8}) {
    size_t smem = 2ull * 32 * warps * (n + 36) * 4;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<148, 32 * warps, smem>>>(out, cyc, n);
    cudaDeviceSynchronize();
    kern<<<148, 32 * warps, smem>>>(out, cyc, n);
    cudaError_t e = cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %2d warps/SM: %.2f cycles/step (%s)\n", name, warps, (double)h[0] / n, cudaGetErrorString(e));
  }
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 22);
  cudaMalloc(&cyc, 1 << 16);
  long long h[4];
  const int n = 1024;
  for (int warps : {1, 4, 8, 16}) {
    chain_reg<<<148, 32 * warps>>>(out, cyc, n, 0.999f, 1e-3f);
    cudaDeviceSynchronize();
    chain_reg<<<148, 32 * warps>>>(out, cyc, n, 0.999f, 1e-3f);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("register chain, %2d warps/SM: %.2f cycles/step\n", warps, (double)h[0] / n);
  }
  for (int warps : {1, 2, 4, 8}) {
    size_t smem = 2ull * 32 * warps * (n + 36) * 4;
    cudaFuncSetAttribute(chain_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    chain_smem<<<148, 32 * warps, smem>>>(out, cyc, n);
    cudaDeviceSynchronize();
    chain_smem<<<148, 32 * warps, smem>>>(out, cyc, n);
    cudaError_t e = cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("smem chain,     %2d warps/SM: %.2f cycles/step (%s)\n", warps, (double)h[0] / n, cudaGetErrorString(e));
  }
  for (int warps : {1, 4}) {
    chain_reg_unrolled<<<148, 32 * warps>>>(out, cyc, n, 0.999f, 1e-3f);
    cudaDeviceSynchronize();
    chain_reg_unrolled<<<148, 32 * warps>>>(out, cyc, n, 0.999f, 1e-3f);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("register chain unrolled, %2d warps/SM: %.2f cycles/step\n", warps, (double)h[0] / n);
  }
  runSmem("smem volatile", chain_smem_v<false, false>, out, cyc, n);
  runSmem("smem volatile rotated", chain_smem_v<true, false>, out, cyc, n);
  runSmem("smem volatile bcast-x", chain_smem_v<false, true>, out, cyc, n);
  runSmem("smem volatile rot bcast-x", chain_smem_v<true, true>, out, cyc, n);
  runSmem("smem plain", chain_smem_plain<false>, out, cyc, n);
  runSmem("smem plain bcast-x", chain_smem_plain<true>, out, cyc, n);
  return 0;
}
