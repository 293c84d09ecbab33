// concat.cu — column concatenation of row-major matrices with a common row
// count: dst[r][off_s + c] = src_s[r][c]. The production model joins the
// 2LUT embeddings and the C3 output this way before MLP1 (PAPER.md:3026-3040,
// where `concat` is noted as not expressible in TC). A plain copy: exact.
#include <algorithm>

#include "kernels.cuh"

namespace tcb {
namespace k {

namespace {

__global__ void concat_kernel(const ConcatArgs a) {
  const int64_t total = a.rows * a.width;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / a.width;
    int c = static_cast<int>(i % a.width), s = 0;
    while (s + 1 < a.n && c >= a.off[s + 1]) ++s;
    a.dst[i] = a.src[s][r * (a.off[s + 1] - a.off[s]) + (c - a.off[s])];
  }
}

}  // namespace

cudaError_t launchConcat(const ConcatArgs& a, cudaStream_t s) {
  if (a.rows <= 0 || a.width <= 0) return cudaSuccess;
  const int64_t total = a.rows * a.width;
  int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 8));
  concat_kernel<<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace k
}  // namespace tcb
