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

// 2 x 2 chains per thread: rows r, r+2 of X and columns c, c+8 of W share loads
__device__ __noinline__ void chain22(unsigned xa0, unsigned xa1, unsigned wa0, unsigned wa1, int n, float* acc) {
  float a00 = acc[0], a01 = acc[1], a10 = acc[2], a11 = acc[3];
  float4 X0 = lds4(xa0), X1 = lds4(xa1), W0 = lds4(wa0), W1 = lds4(wa1);
  for (int k = 4; k <= n; k += 4) {
    float4 x0 = X0, x1 = X1, w0 = W0, w1 = W1;
    if (k < n) {
      X0 = lds4(xa0 + k * 4); X1 = lds4(xa1 + k * 4); W0 = lds4(wa0 + k * 4); W1 = lds4(wa1 + k * 4);
    }
    a00 = fma4(x0, w0, a00); a01 = fma4(x0, w1, a01); a10 = fma4(x1, w0, a10); a11 = fma4(x1, w1, a11);
  }
  acc[0] = a00; acc[1] = a01; acc[2] = a10; acc[3] = a11;
}

// 1 x 2 chains per thread: one X row, columns c and c+8 of W (the X read shared)
__device__ __noinline__ void chain12(unsigned xa, unsigned wa0, unsigned wa1, int n, float* acc) {
  float a0 = acc[0], a1 = acc[1];
  const int nch = n >> 4;
  float4 X0[4], V0[4], U0[4], X1[4], V1[4], U1[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    X0[i] = lds4(xa + i * 16);
    V0[i] = lds4(wa0 + i * 16);
    U0[i] = lds4(wa1 + i * 16);
  }
  for (int c = 0; c + 2 <= nch; c += 2) {
    const unsigned o = c * 64;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      X1[i] = lds4(xa + o + 64 + i * 16);
      V1[i] = lds4(wa0 + o + 64 + i * 16);
      U1[i] = lds4(wa1 + o + 64 + i * 16);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a0 = fma4(X0[i], V0[i], a0);
      a1 = fma4(X0[i], U0[i], a1);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      X0[i] = lds4(xa + o + 128 + i * 16);
      V0[i] = lds4(wa0 + o + 128 + i * 16);
      U0[i] = lds4(wa1 + o + 128 + i * 16);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a0 = fma4(X1[i], V1[i], a0);
      a1 = fma4(X1[i], U1[i], a1);
    }
  }
  acc[0] = a0;
  acc[1] = a1;
}

__global__ void probe12(float* out, long long* cyc, int K) {
  extern __shared__ __align__(16) float sm[];
  const int R = 4, C = 16;
  float* X = sm;
  float* Wt = sm + R * K + 64;
  for (int e = threadIdx.x; e < (R + C) * K + 256; e += blockDim.x) sm[e] = 1e-3f * (e % 97);
  __syncthreads();
  const int r = threadIdx.x % R, c = threadIdx.x / R;  // 32 threads: c in 0..7, columns c and c+8
  float acc[2] = {0, 0};
  long long t0 = clock64();
  chain12((unsigned)__cvta_generic_to_shared(X + r * K), (unsigned)__cvta_generic_to_shared(Wt + c * K),
          (unsigned)__cvta_generic_to_shared(Wt + (c + 8) * K), K, acc);
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void probe22(float* out, long long* cyc, int K) {
  extern __shared__ __align__(16) float sm[];
  const int R = 4, C = 16;
  float* X = sm;
  float* Wt = sm + R * K + 64;
  for (int e = threadIdx.x; e < (R + C) * K + 128; e += blockDim.x) sm[e] = 1e-3f * (e % 97);
  __syncthreads();
  // 16 threads: r in {0,1} (+2), c in 0..7 (+8)
  const int r = threadIdx.x % 2, c = threadIdx.x / 2;
  float acc[4] = {0, 0, 0, 0};
  long long t0 = clock64();
  chain22((unsigned)__cvta_generic_to_shared(X + r * K), (unsigned)__cvta_generic_to_shared(X + (r + 2) * K),
          (unsigned)__cvta_generic_to_shared(Wt + c * K), (unsigned)__cvta_generic_to_shared(Wt + (c + 8) * K), K,
          acc);
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
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
  {
    cudaFuncSetAttribute(probe22, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long h[296];
    for (int ctas : {148, 256, 296}) {
      probe22<<<ctas, 16, smem>>>(out, cyc, K);
      probe22<<<ctas, 16, smem>>>(out, cyc, K);
      cudaError_t e = cudaMemcpy(h, cyc, ctas * 8, cudaMemcpyDeviceToHost);
      double s = 0;
      for (int i = 0; i < ctas; ++i) s += h[i];
      printf("chain22 (2x2 per thread, 16-thread CTAs), %3d CTAs: %.2f cycles/step (%s)\n", ctas, s / ctas / K,
             cudaGetErrorString(e));
    }
  }
  {
    cudaFuncSetAttribute(probe12, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long h[296];
    for (int ctas : {148, 256, 296}) {
      probe12<<<ctas, 32, smem>>>(out, cyc, K);
      probe12<<<ctas, 32, smem>>>(out, cyc, K);
      cudaError_t e = cudaMemcpy(h, cyc, ctas * 8, cudaMemcpyDeviceToHost);
      double s = 0;
      for (int i = 0; i < ctas; ++i) s += h[i];
      printf("chain12 (1 row x 2 columns per thread, 32-thread CTAs), %3d CTAs: %.2f cycles/step (%s)\n", ctas,
             s / ctas / K, cudaGetErrorString(e));
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
