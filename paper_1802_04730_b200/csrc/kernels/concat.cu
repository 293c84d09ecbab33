// concat.cu — column concatenation of row-major matrices with a common row
// count: dst[r][off_s + c] = src_s[r][c]. The production model joins the
// 2LUT embeddings and the C3 output this way before MLP1 (PAPER.md:3026-3040,
// where `concat` is noted as not expressible in TC). A plain copy: exact.
#include <algorithm>
#include <cstdint>

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

// every segment width and the sources/destination 16-byte aligned: one block
// per row, float4 copies (the production model's 64 + 64 + 1000 columns)
__global__ void concat_rows_v4(const ConcatArgs a) {
  const int64_t r = blockIdx.x;
  float4* dst = reinterpret_cast<float4*>(a.dst + r * a.width);
  for (int s = 0; s < a.n; ++s) {
    const int w4 = (a.off[s + 1] - a.off[s]) / 4;
    const float4* src = reinterpret_cast<const float4*>(a.src[s] + r * (a.off[s + 1] - a.off[s]));
    float4* d = dst + a.off[s] / 4;
    for (int j = threadIdx.x; j < w4; j += blockDim.x) d[j] = src[j];
  }
}

}  // namespace

cudaError_t launchConcat(const ConcatArgs& a, cudaStream_t s) {
  if (a.rows <= 0 || a.width <= 0) return cudaSuccess;
  const int64_t total = a.rows * a.width;
  bool v4 = (a.width % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.dst) & 15) == 0);
  for (int i = 0; i < a.n && v4; ++i)
    v4 = ((a.off[i + 1] - a.off[i]) % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.src[i]) & 15) == 0);
  if (v4 && a.rows <= (1 << 30)) {
    concat_rows_v4<<<static_cast<unsigned>(a.rows), 128, 0, s>>>(a);
    return cudaGetLastError();
  }
  int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 8));
  concat_kernel<<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace k
}  // namespace tcb
