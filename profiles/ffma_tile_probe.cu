// ffma_tile_probe.cu — throughput of the register-tiled exact chains that the
// TBMM kernels run: per lane an RM x RN tile of independent FFMA chains, each
// 4-step group fed by RM + RN float4 operands (from registers, or from shared
// memory as the kernels do). One CTA per SM, W warps per CTA; prints warp-FFMA
// instructions issued per cycle per SMSP. Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 profiles/ffma_tile_probe.cu -o /tmp/ftp && /tmp/ftp
#include <cstdio>
#include <cuda_runtime.h>

template <int RM, int RN, bool SMEM>
__global__ void probe(float* out, long long* cyc, int groups) {
  __shared__ float4 sm[2048];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(i * 1e-3f, 1.0f, -1.0f, 0.5f);
  __syncthreads();
  float acc[RM][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) acc[i][j] = 0.f;
  float4 x[RM], y[RN];
#pragma unroll
  for (int i = 0; i < RM; ++i) x[i] = sm[(lane >> 3) + 4 * i];
#pragma unroll
  for (int j = 0; j < RN; ++j) y[j] = sm[64 + (lane & 7) + 8 * j];
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  __syncthreads();
  long long t0 = clock64();
  for (int g = 0; g < groups; ++g) {
    if (SMEM) {
      const unsigned o = (unsigned)((g & 15) * 18 * 16);
#pragma unroll
      for (int i = 0; i < RM; ++i)
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x[i].x), "=f"(x[i].y), "=f"(x[i].z), "=f"(x[i].w)
                     : "r"(base + o + (unsigned)(((lane >> 3) + 4 * i) * 288)));
#pragma unroll
      for (int j = 0; j < RN; ++j)
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(y[j].x), "=f"(y[j].y), "=f"(y[j].z), "=f"(y[j].w)
                     : "r"(base + o + 16384u + (unsigned)(((lane & 7) + 8 * j) * 144)));
    }
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
      for (int j = 0; j < RN; ++j) acc[i][j] = __fmaf_rn(x[i].x, y[j].x, acc[i][j]);
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
      for (int j = 0; j < RN; ++j) acc[i][j] = __fmaf_rn(x[i].y, y[j].y, acc[i][j]);
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
      for (int j = 0; j < RN; ++j) acc[i][j] = __fmaf_rn(x[i].z, y[j].z, acc[i][j]);
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
      for (int j = 0; j < RN; ++j) acc[i][j] = __fmaf_rn(x[i].w, y[j].w, acc[i][j]);
    if (!SMEM) {  // keep the operands live and changing
#pragma unroll
      for (int i = 0; i < RM; ++i) x[i].x += 1e-7f;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) s += acc[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__device__ __forceinline__ void ffma2(unsigned long long& c, float a, unsigned long long b) {
  asm volatile("{\n.reg .b64 t;\nmov.b64 t, {%1, %1};\nfma.rn.f32x2 %0, t, %2, %0;\n}" : "+l"(c) : "f"(a), "l"(b));
}
// FFMA2 outer product: per k, RM broadcast A scalars x RN/2 column pairs of B
// (B stored k-major, so one LDS.128 gives 4 columns at one k)
template <int RM, int RN>
__global__ void probe2(float* out, long long* cyc, int groups) {
  __shared__ float4 sm[2048];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(i * 1e-3f, 1.0f, -1.0f, 0.5f);
  __syncthreads();
  unsigned long long acc[RM][RN / 2];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN / 2; ++j) acc[i][j] = 0ull;
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  __syncthreads();
  long long t0 = clock64();
  for (int g = 0; g < groups; ++g) {
    const unsigned o = (unsigned)((g & 15) * 18 * 16);
    float4 x[RM];
    ulonglong2 y[4][RN / 4];
#pragma unroll
    for (int i = 0; i < RM; ++i)
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x[i].x), "=f"(x[i].y), "=f"(x[i].z), "=f"(x[i].w)
                   : "r"(base + o + (unsigned)(((lane >> 3) + 4 * i) * 288)));
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int j = 0; j < RN / 4; ++j)
        asm volatile("ld.shared.v2.b64 {%0,%1}, [%2];" : "=l"(y[k][j].x), "=l"(y[k][j].y)
                     : "r"(base + o + 16384u + (unsigned)((k * 8 + j) * 128 + (lane & 7) * 16)));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
      for (int i = 0; i < RM; ++i) {
        const float xv = k == 0 ? x[i].x : k == 1 ? x[i].y : k == 2 ? x[i].z : x[i].w;
#pragma unroll
        for (int j = 0; j < RN / 4; ++j) {
          ffma2(acc[i][2 * j], xv, y[k][j].x);
          ffma2(acc[i][2 * j + 1], xv, y[k][j].y);
        }
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN / 2; ++j) s += __uint_as_float((unsigned)acc[i][j]) + __uint_as_float((unsigned)(acc[i][j] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int RM, int RN>
void run2(const char* name, int warps) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int groups = 2000;
  probe2<RM, RN><<<148, warps * 32>>>(out, cyc, groups);
  probe2<RM, RN><<<148, warps * 32>>>(out, cyc, groups);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double fma = (double)groups * 4 * RM * RN * warps;  // warp-level FMAs per SM (2 per FFMA2)
  printf("%-12s FFMA2 warps/SM %2d (%.1f/SMSP): %.3f warp-FMA per cycle per SMSP (%.3f FFMA2 instr) (%s)\n", name,
         warps, warps / 4.0, fma / mx / 4, fma / mx / 8, cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(cyc);
}

template <int RM, int RN, bool SMEM>
void run(const char* name, int warps) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int groups = 2000;
  probe<RM, RN, SMEM><<<148, warps * 32>>>(out, cyc, groups);
  probe<RM, RN, SMEM><<<148, warps * 32>>>(out, cyc, groups);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double ffma = (double)groups * 4 * RM * RN * warps;  // warp-FFMAs per SM
  printf("%-12s %s warps/SM %2d (%.1f/SMSP): %.3f warp-FFMA per cycle per SMSP (%s)\n", name,
         SMEM ? "smem" : "regs", warps, warps / 4.0, ffma / mx / 4, cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 12, 16}) {
    run<7, 4, false>("7x4", w);
    run<7, 4, true>("7x4", w);
    run<7, 2, true>("7x2", w);
    run<4, 4, true>("4x4", w);
    run<4, 2, true>("4x2", w);
    run<7, 1, true>("7x1", w);
    run2<7, 4>("7x4", w);
    run2<4, 4>("4x4", w);
    run2<4, 8>("4x8", w);
    run2<2, 4>("2x4", w);
  }
  return 0;
}
