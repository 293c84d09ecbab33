// synccheck probe: does compute-sanitizer flag a __syncthreads that follows a
// lane-0-only loop of cp.async.bulk copies (the FC chain's prologue)?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 profiles/synccheck_probe.cu -o /tmp/scp
// compute-sanitizer --tool synccheck /tmp/scp <mode>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void probe(const float* src, float* out, int nrows, int mode) {
  __shared__ __align__(128) float buf[8][256];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (mode >= 1) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(nrows * 1024) : "memory");
      for (int r = 0; r < nrows; ++r)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         sa(&buf[r][0])), "l"(src + r * 256), "r"(1024), "r"(sa(&bar)) : "memory");
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar)) : "memory");
    }
  }
  if (mode == 2) __syncwarp();
  __syncthreads();
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(sa(&bar)) : "memory");
  if (mode >= 1) out[blockIdx.x * blockDim.x + tid] = buf[tid % nrows][tid];
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 1, nrows = argc > 2 ? atoi(argv[2]) : 8;
  float *src, *out;
  cudaMalloc(&src, 8 * 256 * 4);
  cudaMalloc(&out, 64 * 64 * 4);
  cudaMemset(src, 0, 8 * 256 * 4);
  probe<<<64, 64>>>(src, out, nrows, mode);
  printf("mode %d rows %d: %s\n", mode, nrows, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
