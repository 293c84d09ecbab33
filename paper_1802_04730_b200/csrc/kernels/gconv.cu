// gconv.cu — grouped convolution with the reference's sequential bias
// update (proj/kernels/gconv.tc:2-7):
//   O(n,g,o,h,w) +=! I(n,g,i,h+kh,w+kw) * W1(g,o,i,kh,kw)
//   O(n,g,o,h,w)  =  O(n,g,o,h,w) + B(m)      for m = 0..M-1, one by one
//
// Direct (implicit-GEMM-shaped) convolution on the FFMA pipe. A CTA owns
// one (image n, group g) pair and TH output rows: it stages the TH+KH-1
// input rows of all C channels of the group (the halo) and the group's
// weights — transposed to [c][kh][kw][f] so RF consecutive filters are one
// vector load — in shared memory. Each thread owns an RF×RW register tile
// (RF filters × RW adjacent output columns of one row) and walks c, kh,
// kw in ascending order, reusing each loaded input row segment across the
// KW taps: RF·RW·KW FFMAs per (RW+KW-1) scalar + KW vector smem loads.
// The chain order per output is exactly the reference's (i, kh, kw), and
// the bias loop adds B[0..M-1] sequentially (__fadd_rn, no contraction).
#include <algorithm>

#include "kernels.cuh"

namespace tcb {
namespace k {

namespace {

__device__ __forceinline__ void cpAsync4(float* dst, const float* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(ok ? 4 : 0)
               : "memory");
}

// One CTA per (n, g, run of RPB row blocks of TH output rows). The group's
// filters are staged once; the halo of row block b+1 streams in by cp.async
// while block b is computed (two halo buffers), so after the first block
// the global-load latency is hidden.
template <int RF, int RW, int KW>
__global__ void __launch_bounds__(512)
    gconv_kernel(const GconvArgs a, const int TH, const int TW, const int TF, const int RPB) {
  extern __shared__ __align__(16) float sm[];
  const int C = a.C, KH = a.KH, F = a.F;
  const int Ho = a.H - KH + 1, Wo = a.W - KW + 1;
  const int rows = TH + KH - 1;
  const int WP = TW * RW + KW - 1;
  const int FP = TF * RF;
  const int n = blockIdx.z, g = blockIdx.y;
  const int nblk = (Ho + TH - 1) / TH;
  const int b0 = blockIdx.x * RPB, b1 = min(nblk, b0 + RPB);
  const int tid = threadIdx.x, T = blockDim.x;
  const int haloF = C * rows * WP + (C * rows * WP) % 2;  // keep the second buffer 8-byte aligned

  float* Wt = sm;                      // [C][KH][KW][FP]
  float* Bs = Wt + C * KH * KW * FP;   // [Mb] (padded to 4)
  float* halo = Bs + ((a.Mb + 3) & ~3);  // [2][C][rows][WP]

  const float* Ig = a.I + ((int64_t)n * a.G + g) * C * a.H * a.W;
  // one halo row (c, r) per warp and pass, lanes along w: 8-byte copies when
  // the rows allow it (W and WP even: every pair is inside or outside the
  // image row, and 8-byte aligned on both sides), else 4-byte copies
  const bool pairs = (a.W % 2 == 0) && (WP % 2 == 0);
  const int lane = tid & 31, nw = T >> 5, wid = tid >> 5;
  auto loadHalo = [&](int blk, float* dst) {
    const int h0 = blk * TH;
    if (T % 32) {  // partial warps (tiny problems): one element per thread and pass
      for (int e = tid; e < C * rows * WP; e += T) {
        const int w = e % WP, t = e / WP, r = t % rows, c = t / rows, h = h0 + r;
        const bool ok = h < a.H && w < a.W;
        cpAsync4(dst + e, ok ? Ig + ((int64_t)c * a.H + h) * a.W + w : Ig, ok);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      return;
    }
    for (int row = wid; row < C * rows; row += nw) {
      const int c = row / rows, r = row - c * rows, h = h0 + r;
      const float* src = Ig + ((int64_t)c * a.H + (h < a.H ? h : 0)) * a.W;
      float* d = dst + row * WP;
      if (pairs) {
        for (int w = 2 * lane; w < WP; w += 64) {
          const bool ok = h < a.H && w < a.W;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                           static_cast<unsigned>(__cvta_generic_to_shared(d + w))),
                       "l"(ok ? src + w : Ig), "r"(ok ? 8 : 0)
                       : "memory");
        }
      } else {
        for (int w = lane; w < WP; w += 32) {
          const bool ok = h < a.H && w < a.W;
          cpAsync4(d + w, ok ? src + w : Ig, ok);
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (b0 < b1) loadHalo(b0, halo);
  const float* Wg = a.W1 + (int64_t)g * F * C * KH * KW;
  for (int e = tid; e < C * KH * KW * FP; e += T) {
    int f = e % FP, t = e / FP;  // t = (c*KH + kh)*KW + kw
    Wt[e] = f < F ? __ldg(Wg + (int64_t)f * C * KH * KW + t) : 0.0f;
  }
  for (int e = tid; e < a.Mb; e += T) Bs[e] = __ldg(a.B + e);

  const int wg = tid % TW;
  const int hl = (tid / TW) % TH;
  const int fg = tid / (TW * TH);
  const bool active = fg < TF;
  float* Og = a.O + ((int64_t)n * a.G + g) * F * Ho * Wo;

  for (int blk = b0; blk < b1; ++blk) {
    const float* In = halo + ((blk - b0) & 1) * haloF;
    if (blk + 1 < b1) {
      loadHalo(blk + 1, halo + ((blk + 1 - b0) & 1) * haloF);
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // this block's halo landed (this thread)
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();  // ... for every thread (and the filters are staged)
    if (active) {
      float acc[RF][RW];
#pragma unroll
      for (int f = 0; f < RF; ++f)
#pragma unroll
        for (int j = 0; j < RW; ++j) acc[f][j] = 0.0f;

      for (int c = 0; c < C; ++c) {
        for (int kh = 0; kh < KH; ++kh) {
          const float* row = In + (c * rows + hl + kh) * WP + wg * RW;
          float x[RW + KW - 1];
#pragma unroll
          for (int j = 0; j < RW + KW - 1; ++j) x[j] = row[j];
          const float* wp = Wt + ((c * KH + kh) * KW) * FP + fg * RF;
#pragma unroll
          for (int kw = 0; kw < KW; ++kw) {
            float wv[RF];
            if constexpr (RF % 4 == 0) {
#pragma unroll
              for (int f = 0; f < RF; f += 4) {
                float4 v = *reinterpret_cast<const float4*>(wp + kw * FP + f);
                wv[f] = v.x;
                wv[f + 1] = v.y;
                wv[f + 2] = v.z;
                wv[f + 3] = v.w;
              }
            } else {
#pragma unroll
              for (int f = 0; f < RF; ++f) wv[f] = wp[kw * FP + f];
            }
#pragma unroll
            for (int f = 0; f < RF; ++f)
#pragma unroll
              for (int j = 0; j < RW; ++j) acc[f][j] = __fmaf_rn(x[j + kw], wv[f], acc[f][j]);
          }
        }
      }

      const int h = blk * TH + hl;
      if (h < Ho) {
        for (int m = 0; m < a.Mb; ++m) {
          const float bm = Bs[m];
#pragma unroll
          for (int f = 0; f < RF; ++f)
#pragma unroll
            for (int j = 0; j < RW; ++j) acc[f][j] = __fadd_rn(acc[f][j], bm);
        }
#pragma unroll
        for (int f = 0; f < RF; ++f) {
          int o = fg * RF + f;
          if (o >= F) continue;
#pragma unroll
          for (int j = 0; j < RW; ++j) {
            int w = wg * RW + j;
            if (w < Wo) Og[((int64_t)o * Ho + h) * Wo + w] = acc[f][j];
          }
        }
      }
    }
    __syncthreads();  // the halo buffer of this block is free for block + 2
  }
}

const GconvVariant kGconvVariants[] = {
    {0, 4, 7, 3, "rf4_rw7_kw3"},  {1, 8, 7, 3, "rf8_rw7_kw3"},  {2, 4, 4, 3, "rf4_rw4_kw3"},
    {3, 4, 8, 3, "rf4_rw8_kw3"},  {4, 8, 4, 3, "rf8_rw4_kw3"},  {5, 2, 7, 3, "rf2_rw7_kw3"},
    {6, 4, 4, 1, "rf4_rw4_kw1"},  {7, 4, 4, 5, "rf4_rw4_kw5"},  {8, 1, 1, 3, "rf1_rw1_kw3"},
};

template <int RF, int RW, int KW>
cudaError_t launchV(const GconvArgs& a, int th, cudaStream_t s) {
  const int Ho = a.H - a.KH + 1, Wo = a.W - KW + 1;
  const int TW = (Wo + RW - 1) / RW, TF = (a.F + RF - 1) / RF;
  const int threads = TW * th * TF;
  if (threads > 512 || threads < 1) return cudaErrorInvalidConfiguration;
  size_t smem = gconvSmem(a, th, RW);
  smem += (size_t)a.C * a.KH * KW * (TF * RF - a.F) * sizeof(float);  // filter padding
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  // row blocks per CTA: enough CTAs for ~2 waves of 148 SMs, the rest
  // become a pipelined loop inside the CTA
  const int nblk = (Ho + th - 1) / th;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t pairs = (int64_t)a.G * a.N;
  const int want = static_cast<int>(std::max<int64_t>(1, (4 * sms + pairs - 1) / pairs));
  const int rpb = std::max(1, (nblk + want - 1) / want);
  auto kfn = gconv_kernel<RF, RW, KW>;
  {
    cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kfn), (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((nblk + rpb - 1) / rpb, a.G, a.N);
  kfn<<<grid, threads, smem, s>>>(a, th, TW, TF, rpb);
  return cudaGetLastError();
}

}  // namespace

int gconvVariantCount() { return sizeof(kGconvVariants) / sizeof(kGconvVariants[0]); }
const GconvVariant& gconvVariant(int i) { return kGconvVariants[i]; }

size_t gconvSmem(const GconvArgs& a, int th, int rw) {
  const int Wo = a.W - a.KW + 1;
  const int TW = (Wo + rw - 1) / rw;
  const int WP = TW * rw + a.KW - 1;
  // two halo buffers (double-buffered row blocks) + filters + bias
  return (2 * (size_t)a.C * (th + a.KH - 1) * WP + (size_t)a.C * a.KH * a.KW * a.F + ((a.Mb + 3) & ~3)) *
         sizeof(float);
}

int gconvThreads(const GconvArgs& a, int variant, int th) {
  const GconvVariant& v = kGconvVariants[variant];
  const int Wo = a.W - a.KW + 1;
  return ((Wo + v.rw - 1) / v.rw) * th * ((a.F + v.rf - 1) / v.rf);
}

cudaError_t launchGconv(const GconvArgs& a, int variant, int th, cudaStream_t s) {
  if (a.N <= 0 || a.G <= 0) return cudaSuccess;
  if (variant < 0 || variant >= gconvVariantCount()) return cudaErrorInvalidValue;
  if (kGconvVariants[variant].kw != a.KW || th < 1) return cudaErrorInvalidConfiguration;
  switch (variant) {
    case 0: return launchV<4, 7, 3>(a, th, s);
    case 1: return launchV<8, 7, 3>(a, th, s);
    case 2: return launchV<4, 4, 3>(a, th, s);
    case 3: return launchV<4, 8, 3>(a, th, s);
    case 4: return launchV<8, 4, 3>(a, th, s);
    case 5: return launchV<2, 7, 3>(a, th, s);
    case 6: return launchV<4, 4, 1>(a, th, s);
    case 7: return launchV<4, 4, 5>(a, th, s);
    case 8: return launchV<1, 1, 3>(a, th, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace k
}  // namespace tcb
