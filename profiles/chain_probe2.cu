// chain_probe2.cu — the FC cluster kernel's layer-1 chain in isolation, with
// its exact operand pattern: 64 threads per CTA, R = 4 input rows and 16
// weight rows of K = 1128 floats, dense in shared memory, thread idx -> row
// idx % 4, column idx / 4; chain variants: the kernel's chainSegment
// (double-buffered 16-step chunks) and deeper prefetch rings. Prints cycles
// per reduction step (thread 0, clock64), ~1.7 CTAs per SM like 2FCRelu.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 profiles/chain_probe2.cu -o /tmp/cp2 && /tmp/cp2
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

// the kernel's chain (fc_chain.cu chainSegment)
__device__ __noinline__ float chainA(unsigned xa, unsigned wa, int n, float acc) {
  const int nch = n >> 4;
  float4 X0[4], W0[4], X1[4], W1[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    X0[i] = lds4(xa + i * 16);
    W0[i] = lds4(wa + i * 16);
  }
  int c = 0;
  for (; c + 2 <= nch; c += 2) {
    const unsigned o = c * 64;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      X1[i] = lds4(xa + o + 64 + i * 16);
      W1[i] = lds4(wa + o + 64 + i * 16);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) acc = fma4(X0[i], W0[i], acc);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      X0[i] = lds4(xa + o + 128 + i * 16);
      W0[i] = lds4(wa + o + 128 + i * 16);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) acc = fma4(X1[i], W1[i], acc);
  }
  if (c < nch) {
#pragma unroll
    for (int i = 0; i < 4; ++i) acc = fma4(X0[i], W0[i], acc);
    ++c;
  }
  int kk = c * 16;
  for (; kk + 4 <= n; kk += 4) acc = fma4(lds4(xa + kk * 4), lds4(wa + kk * 4), acc);
  return acc;
}

// a ring of 4-step groups loaded D groups ahead (D = 4 / 8)
template <int D>
__device__ __noinline__ float chainRing(unsigned xa, unsigned wa, int n, float acc) {
  float4 X[D], W[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    X[i] = lds4(xa + i * 16);
    W[i] = lds4(wa + i * 16);
  }
  const int ng = n >> 2;
  int g = 0;
  for (; g + D <= ng; g += D) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const float4 x = X[i], w = W[i];
      const unsigned o = (unsigned)(g + i + D) * 16u;
      X[i] = lds4(xa + o);  // (reads up to D groups past n: the caller's slack)
      W[i] = lds4(wa + o);
      acc = fma4(x, w, acc);
    }
  }
  for (int i = 0; g + i < ng; ++i) acc = fma4(X[i], W[i], acc);
  return acc;
}

// WSEL: 0 = every warp runs chains; 1 = 4-warp CTAs, only the 2 warps on
// SMSPs {0,1} (first CTA of an SM slot pair) or {2,3} (second) run chains
template <int V, int WSEL = 0>
__global__ void probe(float* out, long long* cyc, int K) {
  extern __shared__ __align__(16) float sm[];
  const int R = 4, C = 16;
  if (WSEL == 1) {
    unsigned wid;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    // this warp's SMSP, and the SMSP pair this CTA should use (by its slot group)
    const unsigned pairWanted = ((wid / 4) & 1) ? 2u : 0u;
    const unsigned sub = wid % 4;
    if (sub != pairWanted && sub != pairWanted + 1) return;  // (no CTA barrier after this point)
  }
  float* X = sm;
  float* Wt = sm + R * K + 64;
  for (int e = threadIdx.x; e < (R + C) * K + 128; e += blockDim.x) sm[e] = 1e-3f * (e % 97);
  if (WSEL == 0) __syncthreads();
  else __syncwarp();
  const int lt = WSEL == 1 ? (threadIdx.x & 31) + 32 * (((threadIdx.x >> 5) & 1)) : threadIdx.x;
  const int r = lt % R, c = lt / R;
  const unsigned xa = (unsigned)__cvta_generic_to_shared(X + r * K);
  const unsigned wa = (unsigned)__cvta_generic_to_shared(Wt + c * K);
  float acc = 0.0f;
  long long t0 = clock64();
  if (V == 0) acc = chainA(xa, wa, K, acc);
  if (V == 1) acc = chainRing<4>(xa, wa, K, acc);
  if (V == 2) acc = chainRing<8>(xa, wa, K, acc);
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (lt == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 22);
  cudaMalloc(&cyc, 1 << 16);
  const int K = 1128;
  const size_t smem = ((4 + 16) * K + 256) * 4;
  void (*ks[3])(float*, long long*, int) = {probe<0>, probe<1>, probe<2>};
  const char* names[3] = {"kernel chainSegment", "ring of 4 groups", "ring of 8 groups"};
  for (int v = 0; v < 3; ++v) {
    cudaFuncSetAttribute(ks[v], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int ctas : {148, 256}) {
      ks[v]<<<ctas, 64, smem>>>(out, cyc, K);
      ks[v]<<<ctas, 64, smem>>>(out, cyc, K);
      long long h[256];
      cudaError_t e = cudaMemcpy(h, cyc, ctas * 8, cudaMemcpyDeviceToHost);
      double s = 0;
      for (int i = 0; i < ctas; ++i) s += h[i];
      printf("%-22s %3d CTAs x 64 thr: %.2f cycles/step (%s)\n", names[v], ctas, s / ctas / K, cudaGetErrorString(e));
    }
  }
  // placement: 2 CTAs per SM (296 x 64 threads) vs 4-warp CTAs whose chain warps pick an SMSP pair
  {
    cudaFuncSetAttribute(probe<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(probe<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long h[296];
    for (int w : {0, 1}) {
      for (int ctas : {148, 296}) {
        const int thr = w ? 128 : 64;
        if (w) { probe<0, 1><<<ctas, thr, smem>>>(out, cyc, K); probe<0, 1><<<ctas, thr, smem>>>(out, cyc, K); }
        else { probe<0, 0><<<ctas, thr, smem>>>(out, cyc, K); probe<0, 0><<<ctas, thr, smem>>>(out, cyc, K); }
        cudaError_t e = cudaMemcpy(h, cyc, ctas * 8, cudaMemcpyDeviceToHost);
        double s = 0;
        for (int i = 0; i < ctas; ++i) s += h[i];
        printf("chainSegment, %s, %3d CTAs: %.2f cycles/step (%s)\n", w ? "4-warp CTAs, SMSP-pair pick" : "2-warp CTAs",
               ctas, s / ctas / K, cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
