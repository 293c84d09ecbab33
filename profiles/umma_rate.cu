// Diagnostic: tcgen05.mma kind::tf32 rate, M=128, K=8 per instruction, for
// N = 16/64/256, issued by one thread into 1 or 4 accumulators, operands in
// shared memory with K-major no-swizzle (small LBO vs a 4 KB LBO) or SW128.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1802_04730_b200/csrc/kernels profiles/umma_rate.cu -o /tmp/ur && /tmp/ur
#include <cstdio>
#include "sm100.cuh"
using namespace tcb::k::sm100;

__device__ __forceinline__ uint64_t dKI(uint32_t s, uint32_t lbo, uint32_t sbo) {
  return ((uint64_t)((s & 0x3FFFF) >> 4)) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
         ((uint64_t)1 << 46);
}

template <int N>
__global__ void __launch_bounds__(128, 1) rate(int iters, int nacc, int layout, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  fenceProxyAsyncSmem();
  if (threadIdx.x == 0) {
    mbarInit(&bar, 1);
    fenceBarrierInit();
  }
  if (threadIdx.x < 32) tmemAlloc<512>(&slot);
  tcFenceBefore();
  __syncthreads();
  tcFenceAfter();
  const uint32_t tmem = slot;
  __shared__ uint32_t offTab[18];
  if (threadIdx.x < 18) {  // the shifted-halo gconv's 9 taps x 2 channel steps (W = 58 pixels)
    const int tap = threadIdx.x / 2, c8 = threadIdx.x % 2, kh = tap / 3, kw = tap % 3;
    offTab[threadIdx.x] = (c8 * 2 * 248 * 16 + (kh * 58 + kw) * 16) >> 4;
  }
  __syncthreads();
  if (layout == 4 && threadIdx.x < 32) {  // gconv-like: plane LBO, table offsets, 18 MMAs per tile
    const uint32_t a = smem(sm), b = smem(sm + 64 * 1024);
    // nacc selects the variant: 1 = plane LBO + smem offset table (the kernel), 2 = plane LBO +
    // arithmetic offsets, 3 = LBO 128 + smem table
    const uint64_t ad0 = dKI(a, nacc == 3 ? 128 : 248 * 16, 128), bd0 = dKI(b, 16 * N, 128);
    constexpr uint32_t id = idescTf32(128, N);
    long long t0 = clock64();
    if (nacc == 4) {  // nested kh / kw / c8 loops, offsets from runtime W and HP (uniform arithmetic)
      const uint32_t Wd = 58u + (uint32_t)(iters >> 30), HP2 = 2u * 248u;  // runtime values
      for (int i = 0; i < iters; i += 18) {
        uint32_t ks = 0;
        for (uint32_t kh = 0; kh < 3; ++kh)
#pragma unroll
          for (uint32_t kw = 0; kw < 3; ++kw)
#pragma unroll
            for (uint32_t c8 = 0; c8 < 2; ++c8, ++ks) {
              const uint64_t ao = c8 * HP2 + kh * Wd + kw;
              const uint64_t bd = bd0 + (uint64_t)(ks * 2 * N);
              uint32_t pred;
              asm volatile("{ .reg .pred p; elect.sync _|p, 0xffffffff; selp.u32 %0, 1, 0, p; }" : "=r"(pred));
              if (pred) mmaTf32(tmem, ad0 + ao, bd, id, ks > 0);
            }
      }
    } else
    for (int i = 0; i < iters; i += 18) {
#pragma unroll 6
      for (int ks = 0; ks < 18; ++ks) {
        const uint64_t ao = nacc == 2 ? (uint64_t)(((ks & 1) * 2 * 248 * 16 + ((ks >> 1) / 3 * 58 + (ks >> 1) % 3) * 16) >> 4)
                                      : (uint64_t)offTab[ks];
        const uint64_t bd = bd0 + (uint64_t)(ks * 2 * N);
        uint32_t pred;
        asm volatile("{ .reg .pred p; elect.sync _|p, 0xffffffff; selp.u32 %0, 1, 0, p; }" : "=r"(pred));
        if (pred) mmaTf32(tmem, ad0 + ao, bd, id, ks > 0);
      }
    }
    if (threadIdx.x == 0) mmaCommit(&bar);
    __syncwarp();
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      unsigned done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem(&bar)) : "memory");
      long long t2 = clock64();
      if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
  } else
  if (layout == 3 && threadIdx.x < 32) {  // whole warp, elect.sync picks the issuing lane
    const uint32_t a = smem(sm), b = smem(sm + 64 * 1024);
    const uint64_t ad0 = dKI(a, 128, 256), bd0 = dKI(b, 128, 256);
    constexpr uint32_t id = idescTf32(128, N);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t pred;
        asm volatile("{ .reg .pred p; elect.sync _|p, 0xffffffff; selp.u32 %0, 1, 0, p; }" : "=r"(pred));
        // per-MMA operands vary (as in a real K loop): descriptor start + 32 B per step, accumulator j
        // per-MMA start offsets: multiples of 32 B (nacc <= 4) or of 16 B (nacc > 4: pixel-granular
        // shifts, as the shifted-halo gconv's taps)
        const uint64_t step = nacc > 4 ? 1 : 2;
        const uint64_t ad = ad0 + (uint64_t)(((i + j) & 7) * step), bd = bd0 + (uint64_t)(((i + j) & 7) * 2);
        if (pred) mmaTf32(tmem + (nacc > 1 ? (j % 4) * N : 0), ad, bd, id, 1);
      }
    }
    if (threadIdx.x == 0) mmaCommit(&bar);
    __syncwarp();
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      unsigned done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem(&bar)) : "memory");
      long long t2 = clock64();
      if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
  } else if (layout < 3 && threadIdx.x == 0) {
    const uint32_t a = smem(sm), b = smem(sm + 64 * 1024);
    uint64_t ad, bd;
    if (layout == 0) { ad = dKI(a, 128, 256); bd = dKI(b, 128, 256); }
    else if (layout == 1) { ad = dKI(a, 4096, 128); bd = dKI(b, 16 * N, 128); }
    else { ad = descSw128(a); bd = descSw128(b); }
    constexpr uint32_t id = idescTf32(128, N);
    long long t0 = clock64();
    if (nacc == 0) {  // loop-invariant operands: same accumulator, descriptors, accumulate flag
      for (int i = 0; i < iters; ++i) mmaTf32(tmem, ad, bd, id, 1);
    } else if (nacc < 0) {  // 4 accumulators, unrolled: every operand a loop invariant
      for (int i = 0; i < iters; i += 4) {
        mmaTf32(tmem, ad, bd, id, 1);
        mmaTf32(tmem + N, ad, bd, id, 1);
        mmaTf32(tmem + 2 * N, ad, bd, id, 1);
        mmaTf32(tmem + 3 * N, ad, bd, id, 1);
      }
    } else {
      for (int i = 0; i < iters; ++i) mmaTf32(tmem + (i % nacc) * N, ad, bd, id, i >= nacc);
    }
    mmaCommit(&bar);
    long long t1 = clock64();
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem(&bar)) : "memory");
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  tcFenceBefore();
  __syncthreads();
  if (threadIdx.x < 32) { tcFenceAfter(); tmemFree<512>(tmem); }
}

template <int N>
void runN(long long* d) {
  cudaFuncSetAttribute(rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int layout : {0, 2, 3, 4})
    for (int nacc : {1, 2, 3, 4, 0, -4, 8}) {
      if (layout >= 3 && nacc < 1) continue;
      if (layout == 4 && (nacc < 1 || nacc > 4 || N > 64)) continue;
      if (layout != 3 && nacc > 4) continue;
      if (layout < 4 && (nacc == 2 || nacc == 3)) continue;
      if (nacc * N > 512 || -nacc * N > 512) continue;
      const int iters = 2048;
      rate<N><<<148, 128, 100 * 1024>>>(iters, nacc, layout, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[2];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("N=%3d layout=%s acc=%d: issue %.1f, complete %.1f cycles/MMA (%.0f MAC/cycle) %s\n", N,
             layout == 0 ? "KI lbo128" : layout == 1 ? "KI lbo4K " : layout == 2 ? "SW128    " : layout == 3 ? "warp+elect" : "gconv-like", nacc, (double)h[0] / iters,
             (double)h[1] / iters, 128.0 * N * 8 * iters / h[1], cudaGetErrorString(e));
    }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  runN<16>(d);
  runN<64>(d);
  runN<256>(d);
  return 0;
}
