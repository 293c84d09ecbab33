// kru.cu — the 3-factor Kronecker (3-KRU) layer as ONE fused kernel
// (PAPER.md:2902-2907):
//   XW2(m,n0,n1,d2) +=! X(m,n0,n1,r2)   * W2(d2,r2)
//   XW1(m,n0,d1,d2) +=! XW2(m,n0,r1,d2) * W1(d1,r1)
//   Y(m,d0,d1,d2)   +=! XW1(m,r0,d1,d2) * W0(d0,r0)
// The three contractions only couple along d2 trivially: every statement
// keeps d2 as a free index, so a CTA owning (m, a DC-wide chunk of d2) can
// run all three in shared memory: X[m] is staged once, XW2 and XW1 chunks
// stay on chip between steps, and all three returns are written exactly
// once. HBM traffic is the algorithmic minimum (X + W read once, XW2 +
// XW1 + Y written once) instead of the 3-kernel chain's extra XW2/XW1
// re-reads. Each output is one thread's sequential FFMA chain in
// ascending r, starting from 0 (the `+=!` neutral store).
#include "kernels.cuh"

namespace tcb {
namespace k {

namespace {

__global__ void kru3_kernel(const KruArgs a, const int DC) {
  extern __shared__ __align__(16) float sm[];
  const int T = blockDim.x, tid = threadIdx.x;
  const int m = blockIdx.y;
  const int d2_0 = blockIdx.x * DC;
  const int dc = min(DC, a.D2 - d2_0);
  const int N0 = a.N0, N1 = a.N1, N2 = a.N2, D0 = a.D0, D1 = a.D1, D2 = a.D2;

  float* Xs = sm;                      // [N0*N1][N2]
  float* W2t = Xs + N0 * N1 * N2;      // [N2][DC]    (transposed chunk)
  float* W1s = W2t + N2 * DC;          // [D1][N1]
  float* W0s = W1s + D1 * N1;          // [D0][N0]
  float* XW2s = W0s + D0 * N0;         // [N0][N1][DC]
  float* XW1s = XW2s + N0 * N1 * DC;   // [N0][D1][DC]

  const float* Xm = a.X + (int64_t)m * N0 * N1 * N2;
  const int nx = N0 * N1 * N2;
  if ((nx & 3) == 0 && ((reinterpret_cast<uintptr_t>(Xm) & 15) == 0)) {
    for (int e = tid; e < nx / 4; e += T)
      reinterpret_cast<float4*>(Xs)[e] = __ldg(reinterpret_cast<const float4*>(Xm) + e);
  } else {
    for (int e = tid; e < nx; e += T) Xs[e] = __ldg(Xm + e);
  }
  for (int e = tid; e < N2 * DC; e += T) {
    int r = e / DC, c = e % DC;
    W2t[e] = c < dc ? __ldg(a.W2 + (int64_t)(d2_0 + c) * N2 + r) : 0.0f;
  }
  for (int e = tid; e < D1 * N1; e += T) W1s[e] = __ldg(a.W1 + e);
  for (int e = tid; e < D0 * N0; e += T) W0s[e] = __ldg(a.W0 + e);
  __syncthreads();

  // step 1: XW2[n0][n1][c] = sum_r2 X[n0][n1][r2] * W2[d2][r2]
  {
    const int tot = N0 * N1 * dc;
    for (int e = tid; e < tot; e += T) {
      int c = e % dc, nn = e / dc;  // nn = n0*N1 + n1
      const float* x = Xs + nn * N2;
      float acc = 0.0f;
      for (int r = 0; r < N2; ++r) acc = __fmaf_rn(x[r], W2t[r * DC + c], acc);
      XW2s[nn * DC + c] = acc;
      a.XW2[((int64_t)m * N0 * N1 + nn) * D2 + d2_0 + c] = acc;
    }
  }
  __syncthreads();
  // step 2: XW1[n0][d1][c] = sum_r1 XW2[n0][r1][c] * W1[d1][r1]
  {
    const int tot = N0 * D1 * dc;
    for (int e = tid; e < tot; e += T) {
      int c = e % dc, t = e / dc;
      int d1 = t % D1, n0 = t / D1;
      const float* x = XW2s + n0 * N1 * DC + c;
      const float* w = W1s + d1 * N1;
      float acc = 0.0f;
      for (int r = 0; r < N1; ++r) acc = __fmaf_rn(x[r * DC], w[r], acc);
      XW1s[(n0 * D1 + d1) * DC + c] = acc;
      a.XW1[(((int64_t)m * N0 + n0) * D1 + d1) * D2 + d2_0 + c] = acc;
    }
  }
  __syncthreads();
  // step 3: Y[d0][d1][c] = sum_r0 XW1[r0][d1][c] * W0[d0][r0]
  {
    const int tot = D0 * D1 * dc;
    for (int e = tid; e < tot; e += T) {
      int c = e % dc, t = e / dc;
      int d1 = t % D1, d0 = t / D1;
      const float* x = XW1s + d1 * DC + c;
      const float* w = W0s + d0 * N0;
      float acc = 0.0f;
      for (int r = 0; r < N0; ++r) acc = __fmaf_rn(x[r * D1 * DC], w[r], acc);
      a.Y[(((int64_t)m * D0 + d0) * D1 + d1) * D2 + d2_0 + c] = acc;
    }
  }
}

}  // namespace

size_t kru3Smem(const KruArgs& a, int DC) {
  size_t f = (size_t)a.N0 * a.N1 * a.N2 + (size_t)a.N2 * DC + (size_t)a.D1 * a.N1 + (size_t)a.D0 * a.N0 +
             (size_t)a.N0 * a.N1 * DC + (size_t)a.N0 * a.D1 * DC;
  return f * sizeof(float);
}

cudaError_t launchKru3(const KruArgs& a, int DC, int threads, cudaStream_t s) {
  if (a.M <= 0) return cudaSuccess;
  size_t smem = kru3Smem(a, DC);
  if (smem > 227 * 1024 || DC < 1) return cudaErrorInvalidConfiguration;
  cudaFuncSetAttribute(kru3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((a.D2 + DC - 1) / DC, a.M);
  kru3_kernel<<<grid, threads, smem, s>>>(a, DC);
  return cudaGetLastError();
}

}  // namespace k
}  // namespace tcb
