// tc_gconv.cu — tensor-core (tcgen05, TF32 / 3xTF32) grouped convolution
// (proj/kernels/gconv.tc:2-7) as an implicit GEMM per group g:
//   D[p][f] = sum_{kh,kw,c} X[c][h+kh][w+kw] * W1[g][f][c][kh][kw]
//   O(n,g,f,h,w) = D + B(0) + B(1) + ... + B(Mb-1)   (sequential, gconv.tc:6)
// with p = a virtual output pixel (h, w), w in [0, VW), VW = Wo rounded up to
// 32/64/128 so one 128-pixel UMMA M tile is 128/VW whole output rows.
//
// The A operand (128 pixels x 8 channels per K step, K-major 8x16-byte core
// matrices) is built on chip by 8 builder warps from a 3-deep ring of halo
// tiles of the group's input rows, prefetched two tiles ahead by 4-byte
// cp.async: for tap (kh, kw) and channel group cg, every pixel's 4-channel
// quad is read from the halo at the (kh, kw)-shifted position and stored as
// one 16-byte core-matrix row. (A TMA box cannot do this: the tile
// mode needs 16-byte aligned box starts, and a kw tap or a 58-float input
// row is not; profiles/tma_probe.cu.) Measured: correct within the stated
// tolerance, but 1.18 ms at the paper shape, slower than the FFMA kernel
// (703 us): the builders are bound by the halo loads and the per-element
// im2col expansion (9 A values built per output pixel-channel), ncu in
// profiles/README.md. The fix is an NHWC staging copy so TMA can fetch each
// tap's 16-byte channel vectors directly. The B operand (the group's filters,
// K-major, k = (kh, kw, c)) is built once per CTA; every CTA serves a single
// group. Columns past the input row read zero-padded halo and only feed
// virtual pixels w >= Wo, which are never stored.
//
// Roles (512 threads): warp 1 = MMA issuer (one lane), warp 2 = TMEM
// allocator, warps 4-7 = epilogue (TMEM lane quarter = warp % 4), warps 8-15
// = builders (3xTF32: they write hi = tf32(x) and lo = tf32(x - hi)). The
// accumulator is double-buffered in TMEM so tile t's epilogue overlaps tile
// t+1's MMAs.
// Not FFMA-exact: selected by tensor-core math.
#include <algorithm>

#include "kernels.cuh"
#include "sm100.cuh"

namespace tcb {
namespace k {

namespace {

using namespace sm100;

constexpr int kThreadsTc = 512;  // warps 0-3: MMA (1), TMEM alloc (2); 4-7 epilogue; 8-15 builders
constexpr int kBuilders = 256;
constexpr int kStagesConv = 2;     // a stage is a whole chunk of K steps: few hand-offs per tile
constexpr int kAStep = 4 * 1024;   // one K step of A: 128 pixels x 8 channels fp32
constexpr int kMaxSteps = 256;
constexpr int kMaxBias = 16;
// Successive MMAs into one accumulator are dependent; with N = F = 16 each is
// short, so K steps are dealt round-robin to kAcc independent accumulators
// (summed in fixed order by the epilogue) to keep several MMAs in flight.
constexpr int kAcc = 4;
constexpr int kHalos = 3;  // halo ring: loads run two tiles ahead of the build  // bias terms held in registers by the epilogue (more are read from smem)

struct TcConvParams {
  const float* I;
  float* O;
  const float* W1;
  const float* bias;
  int N, G, C, H, W, F, KH, KW, Mb;
  int Ho, Wo, VW, tilesPerImg, ctasPerGroup;
  int kSteps;  // KH * KW * C / 8
  int kAtoms;  // ceil(KH * KW * C / 32): B is [kAtoms][F rows][128 B]
  int HWP;     // halo row pitch (floats): covers every column a virtual pixel's taps read
  int kc;      // K steps per pipeline stage (a stage holds kc x 4 KB of A)
};

__device__ __forceinline__ void sts4(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
template <int F, bool X3>
struct ConvCfg {
  // 2 accumulator buffers x kAcc independent partial accumulators of F columns
  static constexpr int kCols = 2 * kAcc * F;
  static constexpr int kTmemCols = kCols <= 32 ? 32 : kCols <= 64 ? 64 : kCols <= 128 ? 128 : kCols <= 256 ? 256 : 512;
  __host__ __device__ static int stageBytes(int kc) { return kc * kAStep * (X3 ? 2 : 1); }
  __host__ __device__ static int bBytes(int kAtoms) { return kAtoms * F * 128; }
  __host__ __device__ static int smem(int kAtoms, int haloFloats, int kc) {
    return 1024 + kStagesConv * stageBytes(kc) + bBytes(kAtoms) * (X3 ? 2 : 1) + kHalos * haloFloats * 4 + 512 +
           4 * kMaxSteps;
  }
};

template <int F, bool X3>
__global__ void __launch_bounds__(kThreadsTc, 1) tc_gconv_kernel(const TcConvParams p) {
  using Cfg = ConvCfg<F, X3>;
  constexpr int S = kStagesConv;
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const int bBytes = Cfg::bBytes(p.kAtoms);
  const int HR = 128 / p.VW + p.KH - 1;   // halo rows per tile
  const int haloF = p.C * HR * p.HWP;     // floats per halo buffer
  const int stB = Cfg::stageBytes(p.kc);
  uint8_t* aHi = sm;                          // stage st: [kc][4 KB] hi, then (3xTF32) [kc][4 KB] lo
  uint8_t* bHi = sm + S * stB;                // [kAtoms][F][128 B]
  uint8_t* bLo = bHi + bBytes;
  float* halo = reinterpret_cast<float*>(bHi + bBytes * (X3 ? 2 : 1));  // [kHalos][C][HR][HWP]
  uint64_t* full = reinterpret_cast<uint64_t*>(halo + kHalos * haloF);
  uint64_t* empty = full + S;
  uint64_t* tFull = empty + S;   // [2]
  uint64_t* tEmpty = tFull + 2;  // [2]

  uint32_t* tmemSlot = reinterpret_cast<uint32_t*>(tEmpty + 2);
  int* stepOff = reinterpret_cast<int*>(tmemSlot + 4);  // [kSteps] halo offset of K step s's tap/channels
  float* sBias = reinterpret_cast<float*>(stepOff + kMaxSteps);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x % p.G, part = blockIdx.x / p.G;
  const int tilesG = p.N * p.tilesPerImg;
  const int t0 = static_cast<int>((int64_t)part * tilesG / p.ctasPerGroup);
  const int t1 = static_cast<int>((int64_t)(part + 1) * tilesG / p.ctasPerGroup);
  const int cb = p.C / 8;
  const int rowsPerTile = 128 / p.VW;

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
    for (int st = threadIdx.x; st < p.kSteps; st += blockDim.x) {
      const int tap = st / cb, c0 = (st % cb) * 8, kh = tap / p.KW, kw = tap % p.KW;
      stepOff[st] = (c0 * HR + kh) * p.HWP + kw;
    }
    for (int e = threadIdx.x; e < kHalos * haloF; e += blockDim.x) halo[e] = 0.0f;  // pad columns stay zero
  }
  fenceProxyAsyncSmem();  // generic writes of B visible to the tensor core
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbarInit(&full[s], kBuilders);
      mbarInit(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbarInit(&tFull[b], 1);
      mbarInit(&tEmpty[b], 128);
    }

    fenceBarrierInit();
  }
  if (warp == 2) tmemAlloc<Cfg::kTmemCols>(tmemSlot);
  tcFenceBefore();
  __syncthreads();
  tcFenceAfter();
  const uint32_t tmem = *tmemSlot;

  if (warp >= 8) {
    // ---- builders: halo rows -> K-major A stages (implicit im2col)
    // K-major, no swizzle: 8-pixel x 4-channel core matrices (128 B), the two
    // channel quads of a K step LBO = 128 B apart, 8-pixel groups SBO = 256 B
    // apart. Thread b writes pixel m's channel quad kq as one 16-byte store.
    const int b = threadIdx.x - 256;
    const int m = b & 127, kq = b >> 7;
    const int r = m / p.VW, w = m % p.VW;
    const uint32_t dstOff = (m >> 3) * 256 + kq * 128 + (m & 7) * 16;
    const float* Ig = p.I + (int64_t)g * p.C * p.H * p.W;
    // halo of tile t -> ring slot (t - t0) % kHalos by 4-byte cp.async (input
    // rows are only 8-byte aligned), rows past the image zero-filled; every
    // builder warp loads its share, kHalos - 1 tiles ahead of the build
    auto haloLoad = [&](int t) {
      const int n = t / p.tilesPerImg, h0 = (t % p.tilesPerImg) * rowsPerTile;
      float* hbuf = halo + ((t - t0) % kHalos) * haloF;
      const float* In = Ig + (int64_t)n * p.G * p.C * p.H * p.W;
      const int bw = b >> 5, bl = b & 31;
      for (int row = bw; row < p.C * HR; row += kBuilders / 32) {
        const int c = row / HR, rr = row - c * HR, h = h0 + rr;
        const bool okRow = h < p.H;
        const float* srow = In + ((int64_t)c * p.H + (okRow ? h : 0)) * p.W;
        const uint32_t drow = smem(hbuf + row * p.HWP);
        for (int x = bl; x < p.W; x += 32)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(drow + 4 * x), "l"(srow + x),
                       "r"(okRow ? 4 : 0)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int k = 0; k < kHalos - 1; ++k)  // always commit kHalos-1 groups (empty past t1)
      if (t0 + k < t1) haloLoad(t0 + k);
      else asm volatile("cp.async.commit_group;" ::: "memory");
    int it = 0, lt = 0;
    for (int t = t0; t < t1; ++t, ++lt) {
      asm volatile("cp.async.wait_group %0;" ::"n"(kHalos - 2) : "memory");  // halo t landed (this thread)
      asm volatile("bar.sync 1, %0;" ::"n"(kBuilders) : "memory");  // ... for every builder; tile t-1 built
      if (t + kHalos - 1 < t1) haloLoad(t + kHalos - 1);
      else asm volatile("cp.async.commit_group;" ::: "memory");
      const float* hb = halo + (lt % kHalos) * haloF;
      const float* base = hb + (kq * 4 * HR + r) * p.HWP + w;
      const int cs = HR * p.HWP;
      for (int s0 = 0; s0 < p.kSteps; s0 += p.kc, ++it) {
        const int st = it % S, s1 = min(p.kSteps, s0 + p.kc);
        if (it >= S) mbarWait(&empty[st], ((it / S) - 1) & 1, 1);
        const uint32_t hiA = smem(aHi + st * stB) + dstOff, loA = hiA + p.kc * kAStep;
        for (int s = s0; s < s1; ++s) {
          const float* src = base + stepOff[s];
          float4 x = make_float4(src[0], src[cs], src[2 * cs], src[3 * cs]);
          const uint32_t o = (s - s0) * kAStep;
          if constexpr (X3) {
            float4 hh, ll;
            hh.x = rzTf32(x.x); hh.y = rzTf32(x.y); hh.z = rzTf32(x.z); hh.w = rzTf32(x.w);
            ll.x = toTf32(x.x - hh.x); ll.y = toTf32(x.y - hh.y); ll.z = toTf32(x.z - hh.z); ll.w = toTf32(x.w - hh.w);
            sts4(hiA + o, hh);
            sts4(loA + o, ll);
          } else {
            sts4(hiA + o, x);
          }
        }
        fenceProxyAsyncSmem();
        mbarArrive(&full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idescTf32(128, F);  // both operands K-major
      const uint32_t bh = smem(bHi), bl = smem(bLo);
      int it = 0, lt = 0;
      for (int t = t0; t < t1; ++t, ++lt) {
        const int buf = lt & 1;
        if (lt >= 2) mbarWait(&tEmpty[buf], ((lt >> 1) - 1) & 1, 2);
        tcFenceAfter();
        const uint32_t d0 = tmem + buf * kAcc * F;
        for (int s0 = 0; s0 < p.kSteps; s0 += p.kc, ++it) {
          const int st = it % S, s1 = min(p.kSteps, s0 + p.kc);
          mbarWait(&full[st], (it / S) & 1, 3);
          tcFenceAfter();
          const uint32_t hiA = smem(aHi + st * stB), loA = hiA + p.kc * kAStep;
          for (int s = s0; s < s1; ++s) {
            const uint32_t boff = (s >> 2) * F * 128 + (s & 3) * 32, o = (s - s0) * kAStep;
            const uint64_t ah = descKInterleave(hiA + o, 128, 256);
            const uint64_t bhd = descSw128(bh + boff);
            const uint32_t d = d0 + (s % kAcc) * F, first = s >= kAcc;
            if constexpr (X3) {
              const uint64_t al = descKInterleave(loA + o, 128, 256);
              const uint64_t bld = descSw128(bl + boff);
              mmaTf32(d, al, bhd, idesc, first);
              mmaTf32(d, ah, bld, idesc, 1);
              mmaTf32(d, ah, bhd, idesc, 1);
            } else {
              mmaTf32(d, ah, bhd, idesc, first);
            }
          }
          mmaCommit(&empty[st]);
        }
        mmaCommit(&tFull[buf]);
      }
    }
  } else if (warp >= 4) {
    // ---- epilogue: TMEM -> registers -> bias chain -> coalesced stores
    const int q = warp - 4, pix = q * 32 + lane;
    const int r = pix / p.VW, w = pix % p.VW;
    float bR[kMaxBias];
#pragma unroll
    for (int m = 0; m < kMaxBias; ++m) bR[m] = m < p.Mb ? sBias[m] : 0.0f;
    int lt = 0;
    for (int t = t0; t < t1; ++t, ++lt) {
      const int buf = lt & 1;
      mbarWait(&tFull[buf], (lt >> 1) & 1, 4);
      __syncwarp();
      tcFenceAfter();
      float v[F];
      const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16) + buf * kAcc * F;
#pragma unroll
      for (int c = 0; c < F; c += 16) tmemLoad16(trow + c, v + c);
      const int nacc = min(kAcc, p.kSteps);
      for (int j = 1; j < nacc; ++j) {  // partial accumulators in fixed order
        float u[F];
#pragma unroll
        for (int c = 0; c < F; c += 16) tmemLoad16(trow + j * F + c, u + c);
        tmemLoadWait();
#pragma unroll
        for (int c = 0; c < F; ++c) v[c] += u[c];
      }
      tmemLoadWait();
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
            if (m < p.Mb) x = __fadd_rn(x, bR[m]);  // B(0), B(1), ... in order (gconv.tc:6)
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
    tmemFree<Cfg::kTmemCols>(tmem);
  }
}

template <int F, bool X3>
cudaError_t launchT(const TcConvParams& p, cudaStream_t s) {
  using Cfg = ConvCfg<F, X3>;
  auto kern = tc_gconv_kernel<F, X3>;
  const int HR = 128 / p.VW + p.KH - 1;
  const int fixed = Cfg::smem(p.kAtoms, p.C * HR * p.HWP, 0) + 4 * p.Mb;
  TcConvParams q = p;  // K steps per stage: as many as fit two stages in ~220 KB
  const int kcMax = std::min(p.kSteps, (220 * 1024 - fixed) / (2 * Cfg::stageBytes(1)));
  if (kcMax < 1) return cudaErrorInvalidValue;
  const int chunks = (p.kSteps + kcMax - 1) / kcMax;
  q.kc = (p.kSteps + chunks - 1) / chunks;  // balanced chunks
  const int smemBytes = fixed + kStagesConv * Cfg::stageBytes(q.kc);
  if (smemBytes > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kern), smemBytes);
  if (e != cudaSuccess) return e;
  kern<<<p.G * p.ctasPerGroup, kThreadsTc, smemBytes, s>>>(q);
  return cudaGetLastError();
}

}  // namespace

bool tcGconvSupported(const GconvArgs& a, const char** why) {
  auto no = [&](const char* w) {
    if (why) *why = w;
    return false;
  };
  const int Wo = a.W - a.KW + 1;
  if (a.C % 8) return no("tensor-core gconv needs input channels per group that are a multiple of 8");
  if (a.F != 16 && a.F != 32 && a.F != 64) return no("tensor-core gconv needs 16, 32 or 64 filters per group");
  if ((static_cast<int64_t>(a.H) * a.W) % 4) return no("tensor-core gconv needs H*W to be a multiple of 4");
  if (Wo > 128) return no("tensor-core gconv supports output rows up to 128 wide");
  if (reinterpret_cast<uintptr_t>(a.I) & 15) return no("tensor-core gconv needs a 16-byte aligned input");
  return true;
}

cudaError_t launchTcGconv(const GconvArgs& a, int math, cudaStream_t s) {
  if (!tcGconvSupported(a, nullptr)) return cudaErrorInvalidValue;
  TcConvParams p{};
  p.I = a.I;
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
  p.HWP = ((std::max(a.W, p.VW + a.KW - 1) + 3) / 4) * 4 + 4;  // reads up to VW-1+3+KW-1
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  p.ctasPerGroup = std::max(1, std::min((2 * sms + a.G - 1) / a.G, a.N * p.tilesPerImg));
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
