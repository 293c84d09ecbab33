// kru.cu — the 3-factor Kronecker (3-KRU) layer as ONE fused kernel
// (PAPER.md:2902-2907):
//   XW2(m,n0,n1,d2) +=! X(m,n0,n1,r2)   * W2(d2,r2)
//   XW1(m,n0,d1,d2) +=! XW2(m,n0,r1,d2) * W1(d1,r1)
//   Y(m,d0,d1,d2)   +=! XW1(m,r0,d1,d2) * W0(d0,r0)
// Every statement keeps d2 as a free index, so a CTA owning (m, a DC-wide
// chunk of d2) runs all three contractions in shared memory: X[m] is
// staged once, the XW2 and XW1 chunks stay on chip between steps, and each
// return is written exactly once — HBM traffic is the algorithmic minimum
// (X + W read once, XW2 + XW1 + Y written once) instead of the 3-kernel
// chain's re-reads of XW2 and XW1.
//
// Register tiling: in each step a warp keeps one 4-wide group of the
// small weight factor (4 × N values) in registers for its whole share of
// the step, so the inner loop is one shared load (the activation) per 4
// FFMAs. Each output is still one thread's sequential chain in ascending
// r from 0 (the `+=!` neutral store) — the reference's order.
#include "kernels.cuh"

namespace tcb {
namespace k {

namespace {

// general shapes: one output per thread and step, weights read from smem
__device__ void kru3Generic(const KruArgs& a, float* sm, int m, int d2_0, int dc, int DC) {
  const int T = blockDim.x, tid = threadIdx.x;
  const int N0 = a.N0, N1 = a.N1, N2 = a.N2, D0 = a.D0, D1 = a.D1, D2 = a.D2;
  float* Xs = sm;
  float* W2t = Xs + N0 * N1 * N2;
  float* W1s = W2t + N2 * DC;
  float* W0s = W1s + D1 * N1;
  float* XW2s = W0s + D0 * N0;
  float* XW1s = XW2s + N0 * N1 * DC;
  for (int e = tid; e < N0 * N1 * dc; e += T) {
    int c = e % dc, nn = e / dc;
    float acc = 0.0f;
    for (int r = 0; r < N2; ++r) acc = __fmaf_rn(Xs[nn * N2 + r], W2t[r * DC + c], acc);
    XW2s[nn * DC + c] = acc;
    a.XW2[((int64_t)m * N0 * N1 + nn) * D2 + d2_0 + c] = acc;
  }
  __syncthreads();
  for (int e = tid; e < N0 * D1 * dc; e += T) {
    int c = e % dc, t = e / dc, d1 = t % D1, n0 = t / D1;
    float acc = 0.0f;
    for (int r = 0; r < N1; ++r) acc = __fmaf_rn(XW2s[(n0 * N1 + r) * DC + c], W1s[d1 * N1 + r], acc);
    XW1s[(n0 * D1 + d1) * DC + c] = acc;
    a.XW1[(((int64_t)m * N0 + n0) * D1 + d1) * D2 + d2_0 + c] = acc;
  }
  __syncthreads();
  for (int e = tid; e < D0 * D1 * dc; e += T) {
    int c = e % dc, t = e / dc, d1 = t % D1, d0 = t / D1;
    float acc = 0.0f;
    for (int r = 0; r < N0; ++r) acc = __fmaf_rn(XW1s[(r * D1 + d1) * DC + c], W0s[d0 * N0 + r], acc);
    a.Y[(((int64_t)m * D0 + d0) * D1 + d1) * D2 + d2_0 + c] = acc;
  }
}

// N0 = N1 = N2 = NR, D0 % 4 == D1 % 4 == 0, dc == DC, DC % 4 == 0.
// Xs rows are padded to XP floats (XP/4 odd) so float4 reads of 8
// different rows are conflict-free.
template <int NR>
__device__ void kru3Tiled(const KruArgs& a, float* sm, int m, int d2_0, int DC) {
  constexpr int XP = (NR % 8 == 0) ? NR + 4 : NR;
  const int T = blockDim.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = T >> 5;
  const int D0 = a.D0, D1 = a.D1, D2 = a.D2;
  float* Xs = sm;                 // [NR*NR][XP]
  float* W2t = Xs + NR * NR * XP;  // [NR][DC]
  float* W1s = W2t + NR * DC;      // [D1][NR]
  float* W0s = W1s + D1 * NR;      // [D0][NR]
  float* XW2s = W0s + D0 * NR;     // [NR][NR][DC]
  float* XW1s = XW2s + NR * NR * DC;  // [NR][D1][DC]

  // step 1: XW2[nn][c] — warp-uniform group of 4 consecutive c; lanes over nn
  // (warps beyond the group count split the lane range: `part` of `parts`)
  int G = DC / 4, parts = max(1, nw / G);
  for (int wi = warp; wi < G * parts; wi += nw) {
    const int grp = wi % G, part = wi / G;
    const int c = grp * 4;
    float w[NR][4];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      float4 v = *reinterpret_cast<const float4*>(W2t + r * DC + c);
      w[r][0] = v.x, w[r][1] = v.y, w[r][2] = v.z, w[r][3] = v.w;
    }
    for (int nn = part * 32 + lane; nn < NR * NR; nn += 32 * parts) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int r = 0; r < NR; r += 4) {
        float4 x = *reinterpret_cast<const float4*>(Xs + nn * XP + r);
        const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[j] = __fmaf_rn(xv[u], w[r + u][j], acc[j]);
      }
      float4 o = make_float4(acc[0], acc[1], acc[2], acc[3]);
      *reinterpret_cast<float4*>(XW2s + nn * DC + c) = o;
      *reinterpret_cast<float4*>(a.XW2 + ((int64_t)m * NR * NR + nn) * D2 + d2_0 + c) = o;
    }
  }
  __syncthreads();
  // step 2: XW1[n0][d1][c] — warp-uniform group of 4 d1; lanes over (n0, c)
  G = D1 / 4, parts = max(1, nw / G);
  for (int wi = warp; wi < G * parts; wi += nw) {
    const int grp = wi % G, part = wi / G;
    const int d1 = grp * 4;
    float w[4][NR];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < NR; r += 4) {
        float4 v = *reinterpret_cast<const float4*>(W1s + (d1 + j) * NR + r);
        w[j][r] = v.x, w[j][r + 1] = v.y, w[j][r + 2] = v.z, w[j][r + 3] = v.w;
      }
    for (int e = part * 32 + lane; e < NR * DC; e += 32 * parts) {
      const int c = e % DC, n0 = e / DC;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const float* x = XW2s + n0 * NR * DC + c;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const float xv = x[r * DC];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = __fmaf_rn(xv, w[j][r], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        XW1s[(n0 * D1 + d1 + j) * DC + c] = acc[j];
        a.XW1[(((int64_t)m * NR + n0) * D1 + d1 + j) * D2 + d2_0 + c] = acc[j];
      }
    }
  }
  __syncthreads();
  // step 3: Y[d0][d1][c] — warp-uniform group of 4 d0; lanes over (d1, c)
  G = D0 / 4, parts = max(1, nw / G);
  for (int wi = warp; wi < G * parts; wi += nw) {
    const int grp = wi % G, part = wi / G;
    const int d0 = grp * 4;
    float w[4][NR];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < NR; r += 4) {
        float4 v = *reinterpret_cast<const float4*>(W0s + (d0 + j) * NR + r);
        w[j][r] = v.x, w[j][r + 1] = v.y, w[j][r + 2] = v.z, w[j][r + 3] = v.w;
      }
    for (int e = part * 32 + lane; e < D1 * DC; e += 32 * parts) {
      const int c = e % DC, d1 = e / DC;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const float* x = XW1s + d1 * DC + c;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const float xv = x[r * D1 * DC];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = __fmaf_rn(xv, w[j][r], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) a.Y[(((int64_t)m * D0 + d0 + j) * D1 + d1) * D2 + d2_0 + c] = acc[j];
    }
  }
}

template <int NR>
__global__ void __launch_bounds__(512) kru3_kernel(const KruArgs a, const int DC, const int tiled) {
  extern __shared__ __align__(16) float sm[];
  const int T = blockDim.x, tid = threadIdx.x;
  const int m = blockIdx.y;
  const int d2_0 = blockIdx.x * DC;
  const int dc = min(DC, a.D2 - d2_0);
  const int N0 = a.N0, N1 = a.N1, N2 = a.N2, D0 = a.D0, D1 = a.D1;
  const int XP = tiled ? ((NR % 8 == 0) ? NR + 4 : NR) : N2;

  // stage X[m] (rows padded to XP), the d2 chunk of W2 (transposed), W1, W0
  float* Xs = sm;
  float* W2t = Xs + N0 * N1 * XP;
  float* W1s = W2t + N2 * DC;
  float* W0s = W1s + D1 * N1;
  const float* Xm = a.X + (int64_t)m * N0 * N1 * N2;
  if ((N2 & 3) == 0 && ((reinterpret_cast<uintptr_t>(Xm) & 15) == 0)) {
    const int q = N2 / 4;
    for (int e = tid; e < N0 * N1 * q; e += T) {
      int row = e / q, c = (e % q) * 4;
      *reinterpret_cast<float4*>(Xs + row * XP + c) = __ldg(reinterpret_cast<const float4*>(Xm + row * N2 + c));
    }
  } else {
    for (int e = tid; e < N0 * N1 * N2; e += T) Xs[(e / N2) * XP + e % N2] = __ldg(Xm + e);
  }
  for (int e = tid; e < N2 * DC; e += T) {
    int r = e / DC, c = e % DC;
    W2t[e] = c < dc ? __ldg(a.W2 + (int64_t)(d2_0 + c) * N2 + r) : 0.0f;
  }
  for (int e = tid; e < D1 * N1; e += T) W1s[e] = __ldg(a.W1 + e);
  for (int e = tid; e < D0 * N0; e += T) W0s[e] = __ldg(a.W0 + e);
  __syncthreads();
  if (tiled) kru3Tiled<NR>(a, sm, m, d2_0, DC);
  else kru3Generic(a, sm, m, d2_0, dc, DC);
}

bool tiledShape(const KruArgs& a, int DC) {
  return a.N0 == 16 && a.N1 == 16 && a.N2 == 16 && a.D0 % 4 == 0 && a.D1 % 4 == 0 && DC % 4 == 0 &&
         a.D2 % DC == 0 && (reinterpret_cast<uintptr_t>(a.XW2) & 15) == 0 && a.D2 % 4 == 0;
}

}  // namespace

size_t kru3Smem(const KruArgs& a, int DC) {
  const int XP = tiledShape(a, DC) ? 20 : a.N2;
  size_t f = (size_t)a.N0 * a.N1 * XP + (size_t)a.N2 * DC + (size_t)a.D1 * a.N1 + (size_t)a.D0 * a.N0 +
             (size_t)a.N0 * a.N1 * DC + (size_t)a.N0 * a.D1 * DC;
  return f * sizeof(float);
}

cudaError_t launchKru3(const KruArgs& a, int DC, int threads, cudaStream_t s) {
  if (a.M <= 0) return cudaSuccess;
  size_t smem = kru3Smem(a, DC);
  if (smem > 227 * 1024 || DC < 1 || threads > 512) return cudaErrorInvalidConfiguration;
  const int tiled = tiledShape(a, DC) ? 1 : 0;
  auto kfn = kru3_kernel<16>;
  {
    cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kfn), (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((a.D2 + DC - 1) / DC, a.M);
  kfn<<<grid, threads, smem, s>>>(a, DC, tiled);
  return cudaGetLastError();
}

}  // namespace k
}  // namespace tcb
