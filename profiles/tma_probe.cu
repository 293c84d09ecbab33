// Diagnostic: one 3-D TMA tile load with SWIZZLE_128B for several map shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1802_04730_b200/csrc profiles/tma_probe.cu -o /tmp/tp
#include <cuda.h>
#include <cstdio>
#include "kernels/sm100.cuh"
using namespace tcb::k::sm100;

__global__ void probe(const __grid_constant__ CUtensorMap tm, int c0, int c1, int c2, float* out) {
  __shared__ __align__(1024) uint8_t buf[8192];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbarInit(&bar, 1);
    fenceBarrierInit();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbarExpectTx(&bar, 32 * 8 * 4);
    tmaLoad3d(buf, &tm, c0, c1, c2, &bar);
  }
  mbarWait(&bar, 0, 0);
  out[threadIdx.x] = reinterpret_cast<float*>(buf)[threadIdx.x];
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

void run(const char* name, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b1, int c0) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  float* src;
  cudaMalloc(&src, d0 * d1 * d2 * 4 + 4096);
  float* out;
  cudaMalloc(&out, 4096);
  CUtensorMap tm;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * 4, d0 * d1 * 4};
  cuuint32_t box[3] = {32, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  probe<<<1, 256>>>(tm, c0, 0, 0, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%-28s encode=%d run=%s\n", name, (int)r, cudaGetErrorString(e));
  if (e != cudaSuccess) cudaDeviceReset();
}

int main() {
  run("gemm-like 1024x128x1 b128", 1024, 128, 1, 8, 0);
  run("100x16x6 box8 c0=0", 100, 16, 6, 8, 0);
  run("100x16x6 box8 c0=2", 100, 16, 6, 8, 2);
  run("128x16x6 box8 c0=0", 128, 16, 6, 8, 0);
  run("128x16x6 box8 c0=1", 128, 16, 6, 8, 1);
  run("128x16x6 box8 c0=4", 128, 16, 6, 8, 4);
  run("3364x16x1024 box8 c0=0", 3364, 16, 1024, 8, 0);
  run("3364x16x1024 box8 c0=3", 3364, 16, 1024, 8, 3);
  return 0;
}
