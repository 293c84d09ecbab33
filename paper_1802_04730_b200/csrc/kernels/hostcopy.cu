// hostcopy.cu — all of one call's small host<->device transfers in ONE
// launch. tcb_run with host tensors (the reference's ExecutionEngine::run
// on host DLTensors, execution_engine.h:93-101) otherwise issues one DMA per
// tensor, and a DMA costs a few µs of setup regardless of size: MLP3's 7
// inputs + 4 outputs took ~100 µs for 0.1 MB (profiles/e2e_probe.py). Pinned
// host memory is mapped into the device address space (UVA), so SM loads and
// stores can move it over PCIe directly: each thread keeps four 16-byte
// accesses in flight, the grid covers every SM.
#include <algorithm>

#include "kernels.cuh"

namespace tcb {
namespace k {

namespace {

constexpr int kUnroll = 4;

__device__ __forceinline__ int findSeg(const SegCopyArgs& a, int64_t u) {
  int s = 0;
  while (s + 1 < a.n && u >= a.start[s + 1]) ++s;
  return s;
}

__global__ void __launch_bounds__(256) seg_copy_kernel(const __grid_constant__ SegCopyArgs a) {
  const int64_t total = a.start[a.n];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < total; base += stride * kUnroll) {
    int4 v[kUnroll];
    int seg[kUnroll];
    int64_t off[kUnroll];
#pragma unroll
    for (int r = 0; r < kUnroll; ++r) {  // all loads first: four PCIe reads in flight per thread
      const int64_t u = base + r * stride;
      seg[r] = -1;
      if (u < total) {
        const int s = findSeg(a, u);
        seg[r] = s;
        off[r] = u - a.start[s];
        if (a.vec16[s])
          v[r] = static_cast<const int4*>(a.src[s])[off[r]];
        else
          v[r].x = static_cast<const int*>(a.src[s])[off[r]];
      }
    }
#pragma unroll
    for (int r = 0; r < kUnroll; ++r) {
      const int s = seg[r];
      if (s < 0) continue;
      if (a.vec16[s])
        static_cast<int4*>(a.dst[s])[off[r]] = v[r];
      else
        static_cast<int*>(a.dst[s])[off[r]] = v[r].x;
    }
  }
}

}  // namespace

void segCopyAdd(SegCopyArgs& a, void* dst, const void* src, int64_t bytes) {
  const int s = a.n++;
  a.dst[s] = dst;
  a.src[s] = src;
  const bool v = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | bytes) & 15) == 0;
  a.vec16[s] = v;
  a.start[s + 1] = a.start[s] + (v ? bytes / 16 : bytes / 4);
}

cudaError_t launchSegCopy(const SegCopyArgs& a, int sms, cudaStream_t s) {
  if (a.n == 0 || a.start[a.n] == 0) return cudaSuccess;
  const int64_t units = a.start[a.n];
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((units + 256 * kUnroll - 1) / (256 * kUnroll),
                                                                            (int64_t)sms * 4)));
  seg_copy_kernel<<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace k
}  // namespace tcb
