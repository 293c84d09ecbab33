// tc_gconv_tma.cu — tcgen05 grouped convolution from an NHWC staging copy
// (a tensor-core gconv variant, tile_sizes[2] == 2; the default is the
// on-chip im2col kernel in tc_gconv.cu).
//
//   1. nchw_to_nhwc: the input I[n][g][c][h][w] is transposed once per call
//      into S[n*g][h][w][c] (one HBM read + write of the input).
//   2. tc_gconv_nhwc_kernel: per group g, D[p][f] = sum_{kh,kw,c} S[h+kh][w+kw][c]
//      * W1[g][f][c][kh][kw] on tcgen05 (M = 128 virtual pixels, N = F, K = 8
//      channels per step), then O = D + B(0) + ... + B(Mb-1) in order
//      (gconv.tc:6).
//
// In NHWC every pixel's 8-channel vector is 32 contiguous, 32-byte aligned
// bytes, so a K step's A operand (128 pixels x 8 channels at tap (kh, kw))
// is 256 independent 16-byte copies into the K-major SWIZZLE_32B layout —
// one cp.async per loader thread, zero-filled past the image. (A 4-D TMA box
// {8 c, VW w, 128/VW h, 1} at origin (c0, kw, h0 + kh, ng) describes the
// same tile and was tried first; its 32-byte rows move at ~1 TB/s through
// the TMA unit, slower still.) Measured on B200: correct, but ~3 ms at the
// paper shape: a 4-KB K step per pipeline stage keeps too few bytes in
// flight per SM to cover the L2/HBM latency (Little's law), see
// profiles/README.md. Roles (512 threads): warp 1 MMA issuer, warp 2 TMEM
// allocator, warps 4-7 epilogue, warps 8-15 loaders (3xTF32: each loader
// splits its own chunk into hi/lo). Not FFMA-exact.
#include <algorithm>
#include <mutex>

#include "kernels.cuh"
#include "sm100.cuh"

namespace tcb {
namespace k {

namespace {

using namespace sm100;

constexpr int kThreads = 512;  // warp 1 MMA, warp 2 TMEM alloc, 4-7 epilogue, 8-15 loaders
constexpr int kLoaders = 256;
constexpr int kStages = 12;
constexpr int kAhead = 8;     // K steps each loader keeps in flight
constexpr int kStep = 4096;  // A per K step: 128 pixels x 8 channels fp32
constexpr int kAcc = 4;      // independent accumulators, K steps dealt round-robin
constexpr int kMaxBias = 16;

// ------------------------------------------------------------ transpose
// S[ng][h][w][c] = I[ng][c][h][w]; one CTA per (ng, h), coalesced both ways
__global__ void nchw_to_nhwc(const float* __restrict__ I, float* __restrict__ S, int C, int H, int W) {
  extern __shared__ float tile[];  // [C][W + 1]
  const int ng = blockIdx.y, h = blockIdx.x;
  const float* src = I + ((int64_t)ng * C * H + h) * W;
  for (int e = threadIdx.x; e < C * W; e += blockDim.x) {
    const int c = e / W, w = e % W;
    tile[c * (W + 1) + w] = __ldg(src + (int64_t)c * H * W + w);
  }
  __syncthreads();
  float* dst = S + ((int64_t)ng * H + h) * W * C;
  for (int e = threadIdx.x; e < C * W; e += blockDim.x) {
    const int w = e / C, c = e % C;
    dst[e] = tile[c * (W + 1) + w];
  }
}

struct Params {
  const float* S;  // NHWC staging copy of the input
  float* O;
  const float* W1;
  const float* bias;
  int N, G, C, H, W, F, KH, KW, Mb;
  int Ho, Wo, VW, tilesPerImg, ctasPerGroup, kSteps, kAtoms;
};

// K-major SWIZZLE_32B operand: 32-byte rows, 8-row atoms 256 B apart
__device__ __forceinline__ uint64_t descSw32K(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>(1) << 16;           // LBO (unused: K fits one atom)
  d |= static_cast<uint64_t>(256 >> 4) << 32;    // SBO: next 8-row atom
  d |= static_cast<uint64_t>(1) << 46;           // version
  d |= static_cast<uint64_t>(6) << 61;           // SWIZZLE_32B
  return d;
}

template <int F, bool X3>
struct Cfg {
  static constexpr int kCols = 2 * kAcc * F;
  static constexpr int kTmemCols = kCols <= 32 ? 32 : kCols <= 64 ? 64 : kCols <= 128 ? 128 : kCols <= 256 ? 256 : 512;
  static constexpr int kStageBytes = kStep * (X3 ? 2 : 1);
  __host__ __device__ static int bBytes(int kAtoms) { return kAtoms * F * 128; }
  __host__ __device__ static int smem(int kAtoms, int Mb) {
    return 1024 + kStages * kStageBytes + bBytes(kAtoms) * (X3 ? 2 : 1) + 512 + 4 * Mb;
  }
};

template <int F, bool X3>
__global__ void __launch_bounds__(kThreads, 1) tc_gconv_nhwc_kernel(const Params p) {
  using C_ = Cfg<F, X3>;
  constexpr int S = kStages;
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const int bBytes = C_::bBytes(p.kAtoms);
  uint8_t* aSt = sm;                           // stage s: [4 KB hi][4 KB lo (3xTF32)]
  uint8_t* bHi = sm + S * C_::kStageBytes;     // [kAtoms][F][128 B]
  uint8_t* bLo = bHi + bBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(bHi + bBytes * (X3 ? 2 : 1));
  uint64_t* empty = full + S;
  uint64_t* tFull = empty + S;
  uint64_t* tEmpty = tFull + 2;
  uint32_t* tmemSlot = reinterpret_cast<uint32_t*>(tEmpty + 2);
  float* sBias = reinterpret_cast<float*>(tmemSlot + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x % p.G, part = blockIdx.x / p.G;
  const int tilesG = p.N * p.tilesPerImg;
  const int t0 = static_cast<int>((int64_t)part * tilesG / p.ctasPerGroup);
  const int t1 = static_cast<int>((int64_t)(part + 1) * tilesG / p.ctasPerGroup);
  const int cb = p.C / 8, rowsPerTile = 128 / p.VW;

  // ---- B: the group's filters, K-major SW128, k = (kh*KW + kw)*C + c; zero past K
  {
    const int K = p.KH * p.KW * p.C;
    const float* Wg = p.W1 + (int64_t)g * p.F * p.C * p.KH * p.KW;
    for (int e = threadIdx.x; e < p.kAtoms * 32 * F; e += blockDim.x) {
      const int f = e / (p.kAtoms * 32), k = e % (p.kAtoms * 32);
      float v = 0.f;
      if (k < K) {
        const int tap = k / p.C, c = k % p.C, kh = tap / p.KW, kw = tap % p.KW;
        v = __ldg(Wg + (((int64_t)f * p.C + c) * p.KH + kh) * p.KW + kw);
      }
      const int atom = k >> 5, j = (k & 31) >> 2, el = k & 3, rg = f >> 3, r = f & 7;
      const int off = atom * F * 128 + rg * 1024 + r * 128 + ((j ^ r) << 4) + el * 4;
      if constexpr (X3) {
        const float h = rzTf32(v);
        *reinterpret_cast<float*>(bHi + off) = h;
        *reinterpret_cast<float*>(bLo + off) = toTf32(v - h);
      } else {
        *reinterpret_cast<float*>(bHi + off) = v;
      }
    }
    for (int e = threadIdx.x; e < p.Mb; e += blockDim.x) sBias[e] = __ldg(p.bias + e);
  }
  fenceProxyAsyncSmem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbarInit(&full[s], kLoaders);
      mbarInit(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbarInit(&tFull[b], 1);
      mbarInit(&tEmpty[b], 128);
    }
    fenceBarrierInit();
  }
  if (warp == 2) tmemAlloc<C_::kTmemCols>(tmemSlot);
  tcFenceBefore();
  __syncthreads();
  tcFenceAfter();
  const uint32_t tmem = *tmemSlot;

  if (warp >= 8) {
    // ---- loaders: each K step's A (128 pixels x 8 channels, K-major SW32)
    // comes straight from the NHWC staging copy: thread b moves pixel m's
    // channel quad kq (16 bytes) with one cp.async, zero-filled past the
    // image. kAhead steps stay in flight; when a step's copy has landed the
    // thread (3xTF32: splits its own chunk into hi/lo,) fences it to the async
    // proxy and arrives on the stage barrier.
    const int b = threadIdx.x - 256, m = b & 127, kq = b >> 7;
    const int r = m / p.VW, w = m % p.VW;
    const uint32_t chunk = m * 32 + ((kq ^ ((m >> 2) & 1)) << 4);  // SW32: 16-B chunk bit ^= row bit 2
    auto publish = [&](int j) {
      const int st = j % S;
      if constexpr (X3) {
        float4* hp = reinterpret_cast<float4*>(aSt + st * C_::kStageBytes + chunk);
        float4 x = *hp, hh, ll;
        hh.x = rzTf32(x.x); hh.y = rzTf32(x.y); hh.z = rzTf32(x.z); hh.w = rzTf32(x.w);
        ll.x = toTf32(x.x - hh.x); ll.y = toTf32(x.y - hh.y); ll.z = toTf32(x.z - hh.z); ll.w = toTf32(x.w - hh.w);
        *hp = hh;
        *reinterpret_cast<float4*>(aSt + st * C_::kStageBytes + kStep + chunk) = ll;
      }
      fenceProxyAsyncSmem();
      mbarArrive(&full[st]);
    };
    int it = 0;
    for (int t = t0; t < t1; ++t) {
      const int n = t / p.tilesPerImg, h0 = (t % p.tilesPerImg) * rowsPerTile;
      const float* Sg = p.S + (int64_t)(n * p.G + g) * p.H * p.W * p.C;
      for (int s = 0; s < p.kSteps; ++s, ++it) {
        const int st = it % S;
        if (it >= S) mbarWait(&empty[st], ((it / S) - 1) & 1, 1);
        const int tap = s / cb, c0 = (s % cb) * 8, kh = tap / p.KW, kw = tap % p.KW;
        const int h = h0 + r + kh, x = w + kw;
        const bool ok = h < p.H && x < p.W;
        const float* src = ok ? Sg + ((int64_t)h * p.W + x) * p.C + c0 + kq * 4 : Sg;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem(aSt + st * C_::kStageBytes) + chunk),
                     "l"(src), "r"(ok ? 16 : 0)
                     : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (it >= kAhead - 1) {
          asm volatile("cp.async.wait_group %0;" ::"n"(kAhead - 1) : "memory");
          publish(it - (kAhead - 1));
        }
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    for (int j = max(0, it - (kAhead - 1)); j < it; ++j) publish(j);
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idesc = idescTf32(128, F);
      const uint32_t bh = smem(bHi), bl = smem(bLo);
      int it = 0, lt = 0;
      for (int t = t0; t < t1; ++t, ++lt) {
        const int buf = lt & 1;
        if (lt >= 2) mbarWait(&tEmpty[buf], ((lt >> 1) - 1) & 1, 2);
        tcFenceAfter();
        const uint32_t d0 = tmem + buf * kAcc * F;
        for (int s = 0; s < p.kSteps; ++s, ++it) {
          const int st = it % S;
          mbarWait(&full[st], (it / S) & 1, 3);
          tcFenceAfter();
          const uint32_t a = smem(aSt + st * C_::kStageBytes);
          const uint32_t boff = (s >> 2) * F * 128 + (s & 3) * 32;
          const uint32_t d = d0 + (s % kAcc) * F, acc = s >= kAcc;
          if constexpr (X3) {
            mmaTf32(d, descSw32K(a + kStep), descSw128(bh + boff), idesc, acc);
            mmaTf32(d, descSw32K(a), descSw128(bl + boff), idesc, 1);
            mmaTf32(d, descSw32K(a), descSw128(bh + boff), idesc, 1);
          } else {
            mmaTf32(d, descSw32K(a), descSw128(bh + boff), idesc, acc);
          }
          mmaCommit(&empty[st]);
        }
        mmaCommit(&tFull[buf]);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---- epilogue: partial accumulators in fixed order, bias chain, stores
    const int q = warp - 4, pix = q * 32 + lane;
    const int r = pix / p.VW, w = pix % p.VW;
    float bR[kMaxBias];
#pragma unroll
    for (int m = 0; m < kMaxBias; ++m) bR[m] = m < p.Mb ? sBias[m] : 0.0f;
    const int nacc = min(kAcc, p.kSteps);
    int lt = 0;
    for (int t = t0; t < t1; ++t, ++lt) {
      const int buf = lt & 1;
      mbarWait(&tFull[buf], (lt >> 1) & 1, 4);
      __syncwarp();
      tcFenceAfter();
      const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16) + buf * kAcc * F;
      float v[F];
#pragma unroll
      for (int c = 0; c < F; c += 16) tmemLoad16(trow + c, v + c);
      tmemLoadWait();
      for (int j = 1; j < nacc; ++j) {
        float u[F];
#pragma unroll
        for (int c = 0; c < F; c += 16) tmemLoad16(trow + j * F + c, u + c);
        tmemLoadWait();
#pragma unroll
        for (int c = 0; c < F; ++c) v[c] += u[c];
      }
      tcFenceBefore();
      mbarArrive(&tEmpty[buf]);
      const int n = t / p.tilesPerImg, h = (t % p.tilesPerImg) * rowsPerTile + r;
      if (w < p.Wo && h < p.Ho) {
        float* o = p.O + (((int64_t)n * p.G + g) * p.F) * p.Ho * p.Wo + (int64_t)h * p.Wo + w;
#pragma unroll
        for (int f = 0; f < F; ++f) {
          float x = v[f];
#pragma unroll
          for (int m = 0; m < kMaxBias; ++m)
            if (m < p.Mb) x = __fadd_rn(x, bR[m]);  // B(0), B(1), ... in order
          for (int m = kMaxBias; m < p.Mb; ++m) x = __fadd_rn(x, sBias[m]);
          o[(int64_t)f * p.Ho * p.Wo] = x;
        }
      }
    }
  }
  tcFenceBefore();
  __syncthreads();
  if (warp == 2) {
    tcFenceAfter();
    tmemFree<C_::kTmemCols>(tmem);
  }
}

// NHWC staging buffer, grown on demand (never inside stream capture: the
// first call of a shape, e.g. a warm-up, allocates it)
struct Staging {
  std::mutex mu;
  float* ptr = nullptr;
  size_t bytes = 0;
};
Staging& staging() {
  static Staging s;
  return s;
}

template <int F, bool X3>
cudaError_t launchT(const Params& p, cudaStream_t s) {
  using C_ = Cfg<F, X3>;
  auto kern = tc_gconv_nhwc_kernel<F, X3>;
  const int smemBytes = C_::smem(p.kAtoms, p.Mb);
  if (smemBytes > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kern), smemBytes);
  if (e != cudaSuccess) return e;
  kern<<<p.G * p.ctasPerGroup, kThreads, smemBytes, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launchTcGconvTma(const GconvArgs& a, int math, cudaStream_t s) {
  if (!tcGconvSupported(a, nullptr)) return cudaErrorInvalidValue;
  const size_t bytes = (size_t)a.N * a.G * a.C * a.H * a.W * 4;
  float* S = nullptr;
  {
    Staging& st = staging();
    std::lock_guard<std::mutex> g(st.mu);
    if (st.bytes < bytes) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(s, &cs);
      if (cs != cudaStreamCaptureStatusNone) return cudaErrorStreamCaptureUnsupported;
      if (st.ptr) cudaFree(st.ptr);
      st.ptr = nullptr;
      st.bytes = 0;
      cudaError_t e = cudaMalloc(&st.ptr, bytes);
      if (e != cudaSuccess) return e;
      st.bytes = bytes;
    }
    S = st.ptr;
  }
  nchw_to_nhwc<<<dim3(a.H, a.N * a.G), 256, (size_t)a.C * (a.W + 1) * 4, s>>>(a.I, S, a.C, a.H, a.W);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;

  Params p{};
  p.S = S;
  p.O = a.O;
  p.W1 = a.W1;
  p.bias = a.B;
  p.N = a.N;
  p.G = a.G;
  p.C = a.C;
  p.H = a.H;
  p.W = a.W;
  p.F = a.F;
  p.KH = a.KH;
  p.KW = a.KW;
  p.Mb = a.Mb;
  p.Ho = a.H - a.KH + 1;
  p.Wo = a.W - a.KW + 1;
  p.VW = p.Wo <= 32 ? 32 : p.Wo <= 64 ? 64 : 128;
  p.tilesPerImg = (p.Ho + 128 / p.VW - 1) / (128 / p.VW);
  p.kSteps = a.KH * a.KW * a.C / 8;
  p.kAtoms = (a.KH * a.KW * a.C + 31) / 32;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  p.ctasPerGroup = std::max(1, std::min((sms + a.G - 1) / a.G, a.N * p.tilesPerImg));

  const bool x3 = math == kMath3xTf32;
  switch (a.F) {
    case 16: return x3 ? launchT<16, true>(p, s) : launchT<16, false>(p, s);
    case 32: return x3 ? launchT<32, true>(p, s) : launchT<32, false>(p, s);
    case 64: return x3 ? launchT<64, true>(p, s) : launchT<64, false>(p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace k
}  // namespace tcb
