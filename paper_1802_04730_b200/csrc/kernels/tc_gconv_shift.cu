// tc_gconv_shift.cu — tensor-core (tcgen05, TF32 / 3xTF32) grouped
// convolution (proj/kernels/gconv.tc:2-7) as an implicit GEMM per group g
// with NO im2col: each tap is a shifted view of one halo tile.
//
//   D[p][f] = sum_{kh,kw,c} X[c][p + kh*W + kw] * W1[g][f][c][kh][kw]
//   O(n,g,f,h,w) = D[h*W + w] + B(0) + ... + B(Mb-1)   (sequential, gconv.tc:6)
//
// Virtual pixels p = h*W + w run over the INPUT row pitch W, so tap (kh, kw)
// of pixel p is input pixel p + kh*W + kw: a constant shift. An M tile is 128
// consecutive virtual pixels; its halo is the HP = 128 + (KH-1)*W + (KW-1)
// input pixels from p0, stored channel-block-major: [C/4][HP][4 channels],
// 16 bytes per pixel per block. That is exactly a K-major, no-swizzle UMMA
// operand (8-pixel x 16-byte core matrices: SBO = 128 B to the next 8
// pixels, LBO = HP*16 B to the next 4 channels) for EVERY tap, starting
// (kh*W + kw)*16 bytes further in: 9 taps x C/8 K steps read one tile that
// was written once (vs 9x the bytes for an im2col A; tc_gconv.cu). Outputs
// at w >= Wo (the row's last KW-1 virtual pixels) are computed and dropped.
//
// Roles (512 threads): warp 1 = MMA issuer (whole warp, elect.sync), warp 2 = TMEM
// allocator, warps 4-7 = epilogue (TMEM lane quarter = warp % 4), warps 8-15
// = builders: 4-byte cp.async of the tile's input pixels straight into the
// transposed layout (lanes = 8 pixels x 4 channels: 128 contiguous shared
// bytes, four 32-byte global segments), two tiles ahead; 3xTF32 then splits
// each landed tile into hi/lo planes. Accumulators are double-buffered in
// TMEM so tile t's epilogue overlaps tile t+1's MMAs. Not FFMA-exact:
// selected by tensor-core math.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "sm100.cuh"

namespace tcb {
namespace k {

namespace {

using namespace sm100;

constexpr int kThreadsSh = 512;
constexpr int kBuildersSh = 256;
constexpr int kStagesSh = 4;  // halo tiles in flight (ring)
constexpr int kAheadSh = 2;   // tiles loaded ahead of the one being finalised
// TMA path: a 4-deep ring of transposed tiles and 2 raw staging buffers
// (4 or 8 staging buffers with a 3-deep ring measured 211 us vs 203,
// profiles/r02_tma_sweep.txt)
constexpr int kRingTma = 4;
constexpr int kStagingBufs = 2;
// One accumulator per tile: a tcgen05.mma from shared memory costs ~40 cycles
// at N = 16 whatever the accumulator dependence (it is bound by reading the
// 4 KB A operand, profiles/umma_rate.cu), so partial accumulators would only
// multiply the epilogue's TMEM reads.
// TMEM accumulator ring: the MMA issuer runs up to kTmemBufs tiles ahead of
// the epilogue, so the commit -> epilogue -> release round trip (~1-3k cycles)
// is paid once per kTmemBufs tiles, not once per tile
constexpr int kTmemBufs = 8;

struct ShiftParams {
  const float* I;
  float* O;
  const float* W1;
  const float* bias;
  int N, G, C, H, W, F, KH, KW, Mb;
  int Ho, Wo, tilesPerImg, items;  // items = G * N * tilesPerImg, split evenly over the grid
  int HP;  // halo pixels per tile (multiple of 8)
  int tma;  // 1: halo tiles land by one TMA tensor copy into a staging buffer, then an on-chip transpose
  int skip;  // diagnostics only (TCB_GCONV_SKIP env, ablations): 1 MMAs, 2 transposes, 4 output stores
};

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

template <int F, bool X3>
struct ShiftCfg {
  // 3xTF32 stacks B as [b_hi | b_lo] (N = 2F): a_hi*[b_hi|b_lo] and
  // a_lo*[b_hi|b_lo] are two MMAs per K step instead of three (an MMA from
  // shared memory at small N costs its A read, not its N), and the lo*lo
  // term comes for free; the epilogue adds the two column halves
  static constexpr int kN = X3 ? 2 * F : F;
  static constexpr int kTmemCols = kTmemBufs * kN <= 32    ? 32
                                   : kTmemBufs * kN <= 64  ? 64
                                   : kTmemBufs * kN <= 128 ? 128
                                   : kTmemBufs * kN <= 256 ? 256
                                                           : 512;
  __host__ __device__ static int stageFloats(int C, int HP) { return C * HP * (X3 ? 2 : 1); }
  __host__ __device__ static int bBytes(int KH, int KW, int C) { return KH * KW * (C / 8) * 32 * kN; }
  __host__ __device__ static int stagingBytes(const ShiftParams& p) { return p.tma ? kStagingBufs * p.C * p.HP * 4 : 0; }
  __host__ __device__ static int ring(const ShiftParams& p) { return p.tma ? kRingTma : kStagesSh; }
  __host__ __device__ static int smem(const ShiftParams& p) {
    return 1024 + ring(p) * stageFloats(p.C, p.HP) * 4 + 2 * bBytes(p.KH, p.KW, p.C) + stagingBytes(p) + 1024 +
           8 * p.KH * p.KW * (p.C / 8) + 4 * p.Mb;
  }
};

template <int F, bool X3>
__global__ void __launch_bounds__(kThreadsSh, 1)
    tc_gconv_shift_kernel(const ShiftParams p, const __grid_constant__ CUtensorMap tmI) {
  using Cfg = ShiftCfg<F, X3>;
  const int S = Cfg::ring(p);
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const int C = p.C, HP = p.HP, taps = p.KH * p.KW, kcb = C / 8;
  const int stF = Cfg::stageFloats(C, HP);
  const int planeF = C * HP;  // hi (or raw fp32) plane of a stage; lo follows (3xTF32)
  float* stages = reinterpret_cast<float*>(sm);
  uint8_t* bBank = sm + S * stF * 4;  // [2 banks][hi (+ lo)] of the CTA's first and last group
  constexpr int NB = Cfg::kN;
  const int bStride = Cfg::bBytes(p.KH, p.KW, C);
  float* staging = reinterpret_cast<float*>(bBank + 2 * bStride);  // p.tma: [2][C][HP] as the TMA lands it
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(staging) + Cfg::stagingBytes(p));
  uint64_t* empty = full + kStagesSh;
  uint64_t* tFull = empty + kStagesSh;    // [kTmemBufs]
  uint64_t* tEmpty = tFull + kTmemBufs;   // [kTmemBufs]
  uint64_t* stFull = tEmpty + kTmemBufs;  // [kStagingBufs] staging buffer landed
  uint32_t* tmemSlot = reinterpret_cast<uint32_t*>(stFull + kStagingBufs);
  uint32_t* aOff16 = tmemSlot + 4;              // [K steps] A descriptor start offset (16-byte units)
  float* sBias = reinterpret_cast<float*>(aOff16 + taps * kcb);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // work items (g, n, tile), g-major, split evenly over the grid: a CTA's
  // range spans at most two groups (items per CTA <= items per group)
  const int tilesG = p.N * p.tilesPerImg;
  const int t0 = static_cast<int>((int64_t)blockIdx.x * p.items / gridDim.x);
  const int t1 = static_cast<int>((int64_t)(blockIdx.x + 1) * p.items / gridDim.x);
  const int gFirst = t0 / tilesG;
  const int HW = p.H * p.W;

  // ---- B: the group's filters per (tap, 8-channel step), K-major no swizzle:
  // NB-row x 16-byte core matrices (SBO 128 B per 8 rows), channel halves
  // LBO = 16*NB B; 3xTF32 rows [0, F) = hi, [F, 2F) = lo
  for (int bank = 0; bank < 2; ++bank) {
    const int g = min(gFirst + bank, p.G - 1);
    const float* Wg = p.W1 + (int64_t)g * F * C * taps;
    uint8_t* bb = bBank + bank * bStride;
    for (int e = threadIdx.x; e < F * C * taps; e += blockDim.x) {
      const int f = e / (C * taps), rem = e - f * C * taps, c = rem / taps, tap = rem - c * taps;
      const float v = __ldg(Wg + e);  // W1[g][f][c][kh][kw]
      const int ks = tap * kcb + (c >> 3), half = (c >> 2) & 1, el = c & 3;
      auto at = [&](int r) { return bb + ks * 32 * NB + half * 16 * NB + (r >> 3) * 128 + (r & 7) * 16 + el * 4; };
      if constexpr (X3) {
        const float h = rzTf32(v);
        *reinterpret_cast<float*>(at(f)) = h;
        *reinterpret_cast<float*>(at(F + f)) = toTf32(v - h);
      } else {
        *reinterpret_cast<float*>(at(f)) = v;
      }
    }
  }
  // A start offset of K step ks = (tap, 8-channel block c8): channel block
  // 2*c8's plane plus the tap's pixel shift
  for (int ks = threadIdx.x; ks < taps * kcb; ks += blockDim.x) {
    const int tap = ks / kcb, c8 = ks - tap * kcb, kh = tap / p.KW, kw = tap - kh * p.KW;
    aOff16[ks] = (c8 * 2 * HP * 16 + (kh * p.W + kw) * 16) >> 4;
  }
  for (int e = threadIdx.x; e < p.Mb; e += blockDim.x) sBias[e] = __ldg(p.bias + e);
  fenceProxyAsyncSmem();  // generic writes of B visible to the tensor core
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbarInit(&full[s], kBuildersSh / 32);  // one arrive per builder warp
      mbarInit(&empty[s], 1);
    }
    for (int b = 0; b < kTmemBufs; ++b) {
      mbarInit(&tFull[b], 1);
      mbarInit(&tEmpty[b], 4);  // one arrive per epilogue warp
    }
    for (int i = 0; i < kStagingBufs; ++i) mbarInit(&stFull[i], 1);
    fenceBarrierInit();
  }
  if (warp == 2) tmemAlloc<Cfg::kTmemCols>(tmemSlot);
  tcFenceBefore();
  __syncthreads();
  tcFenceAfter();
  const uint32_t tmem = *tmemSlot;

  if (warp >= 8 && p.tma) {
    // ---- builders, TMA path: tile lt's halo (C channel rows of HP
    // consecutive input pixels, contiguous in every channel plane) lands in
    // staging[lt & 1] by ONE tensor copy {HP px, C ch, 1} (zero-filled past
    // the plane), issued two tiles ahead; the builders then transpose it on
    // chip into the channel-block-major UMMA layout [C/4][HP][4] (+ the hi/lo
    // split for 3xTF32). Round 1's builders issued 4-byte cp.async per
    // element: ~4000 per tile, the kernel's bound (222 of 281 us with every
    // MMA skipped).
    const int b = threadIdx.x - 256;
    const int n4 = HP / 4, items = n4 * (C / 4);  // (4-pixel group, 4-channel block) per item
    const int nt = t1 - t0;
    constexpr int NS = kStagingBufs;
    auto issue = [&](int lt) {
      const int t = t0 + lt, g = t / tilesG, tt = t - g * tilesG, n = tt / p.tilesPerImg;
      const int p0 = (tt - n * p.tilesPerImg) * 128;
      uint64_t* bar = &stFull[lt % NS];
      mbarExpectTx(bar, (uint32_t)(C * HP * 4));
      tmaLoad3d(staging + (lt % NS) * C * HP, &tmI, p0, 0, n * p.G + g, bar);
    };
    if (b == 0) {
      tmaPrefetch(&tmI);
      for (int lt = 0; lt < min(NS, nt); ++lt) issue(lt);
    }
    for (int lt = 0; lt < nt; ++lt) {
      const int s = lt % S;
      if (lt >= S) mbarWait(&empty[s], ((lt / S) - 1) & 1, 1);  // MMAs of tile lt - S done
      mbarWait(&stFull[lt % NS], (lt / NS) & 1, 5);
      const uint32_t src = smem(staging + (lt % NS) * C * HP), hiP = smem(stages + s * stF);
      for (int it = (p.skip & 2) ? items : b; it < items; it += kBuildersSh) {
        const int cb = it / n4, pg = it - cb * n4;  // consecutive lanes: consecutive pixel groups
        float4 r[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) r[c] = lds128(src + (uint32_t)(((cb * 4 + c) * HP + pg * 4) * 4));
        const int rot = pg & 3;  // rotate the pixel order across lanes: fewer bank conflicts on the stores
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = (jj + rot) & 3;
          // the 4 channels of pixel pg*4 + j (selects, not a dynamically indexed array)
          float4 v;
          v.x = j == 0 ? r[0].x : j == 1 ? r[0].y : j == 2 ? r[0].z : r[0].w;
          v.y = j == 0 ? r[1].x : j == 1 ? r[1].y : j == 2 ? r[1].z : r[1].w;
          v.z = j == 0 ? r[2].x : j == 1 ? r[2].y : j == 2 ? r[2].z : r[2].w;
          v.w = j == 0 ? r[3].x : j == 1 ? r[3].y : j == 2 ? r[3].z : r[3].w;
          const uint32_t dst = hiP + (uint32_t)(((cb * HP) + pg * 4 + j) * 16);
          if constexpr (X3) {
            float4 h, l;
            h.x = rzTf32(v.x); h.y = rzTf32(v.y); h.z = rzTf32(v.z); h.w = rzTf32(v.w);
            l.x = toTf32(v.x - h.x); l.y = toTf32(v.y - h.y); l.z = toTf32(v.z - h.z); l.w = toTf32(v.w - h.w);
            sts128(dst, h);
            sts128(dst + (uint32_t)planeF * 4, l);
          } else {
            sts128(dst, v);
          }
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kBuildersSh) : "memory");  // staging[lt % NS] fully read
      if (b == 0 && lt + NS < nt) {
        fenceProxyAsyncSmem();
        issue(lt + NS);
      }
      fenceProxyAsyncSmem();  // this lane's stage writes -> visible to the tensor core
      __syncwarp();
      if (lane == 0) mbarArrive(&full[s]);
    }
  } else if (warp >= 8) {
    // ---- builders
    const int b = threadIdx.x - 256, el = b & 3, qq = b >> 2;  // 64 pixels x 4 channels per pass
    auto load = [&](int t, int s) {
      const int g = t / tilesG, tt = t - g * tilesG, n = tt / p.tilesPerImg, p0 = (tt - n * p.tilesPerImg) * 128;
      const float* In = p.I + ((int64_t)n * p.G + g) * C * HW;
      const uint32_t base = smem(stages + s * stF);
      for (int cb = 0; cb < C / 4; ++cb) {
        const float* src = In + (int64_t)(cb * 4 + el) * HW;
        for (int q = qq; q < HP; q += 64) {
          const int px = p0 + q;
          const bool ok = px < HW;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(base + ((cb * HP + q) * 4 + el) * 4),
                       "l"(src + (ok ? px : 0)), "r"(ok ? 4 : 0)
                       : "memory");
        }
      }
    };
    auto finalise = [&](int lt) {  // tile lt's copies landed (this thread's): split (3x), publish
      const int s = lt % S;
      if constexpr (X3) {
        asm volatile("bar.sync 1, %0;" ::"n"(kBuildersSh) : "memory");  // every builder's copies landed
        float4* hi = reinterpret_cast<float4*>(stages + s * stF);
        float4* lo = hi + planeF / 4;
        for (int e = b; e < planeF / 4; e += kBuildersSh) {
          const float4 x = hi[e];
          float4 h, l;
          h.x = rzTf32(x.x); h.y = rzTf32(x.y); h.z = rzTf32(x.z); h.w = rzTf32(x.w);
          l.x = toTf32(x.x - h.x); l.y = toTf32(x.y - h.y); l.z = toTf32(x.z - h.z); l.w = toTf32(x.w - h.w);
          hi[e] = h;
          lo[e] = l;
        }
      }
      fenceProxyAsyncSmem();  // this lane's landed copies -> visible to the tensor core
      __syncwarp();
      if (lane == 0) mbarArrive(&full[s]);  // (256 single-thread arrives per tile serialise)
    };
    const int nt = t1 - t0;
    for (int lt = 0; lt < nt + kAheadSh; ++lt) {
      if (lt < nt) {
        const int s = lt % S;
        if (lt >= S) mbarWait(&empty[s], ((lt / S) - 1) & 1, 1);  // MMAs of tile lt - S done
        load(t0 + lt, s);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");  // (empty groups keep the count uniform)
      if (lt >= kAheadSh) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kAheadSh) : "memory");
        finalise(lt - kAheadSh);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issue: the whole warp runs the loop (operands stay warp-uniform);
    // elect.sync picks the issuing lane. Descriptors are per-tile bases plus
    // a per-K-step start offset (the start field is the low 14 bits: adding
    // a 16-byte-unit offset to a valid address cannot carry out of it).
    constexpr uint32_t idesc = idescTf32(128, NB);  // both operands K-major
    const uint32_t lboA = HP * 16, lboB = 16 * NB;
    const int nks = taps * kcb;
    constexpr int kFastKs = 18;  // KH = KW = 3, C = 16
    uint32_t fastOff[kFastKs];
#pragma unroll
    for (int ks = 0; ks < kFastKs; ++ks) {
      const int tap = ks / 2, c8 = ks % 2, kh = tap / 3, kw = tap % 3;
      fastOff[ks] = (uint32_t)((c8 * 2 * HP * 16 + (kh * p.W + kw) * 16) >> 4);
    }
    if (!(p.KH == 3 && p.KW == 3 && C == 16)) fastOff[0] = 0;  // (unused: nks != 18 or a different tap set)
    for (int lt = 0; lt < t1 - t0; ++lt) {
      const int s = lt % S, buf = lt % kTmemBufs, bank = (t0 + lt) / tilesG - gFirst;
      if (lt >= kTmemBufs) mbarWait(&tEmpty[buf], ((lt / kTmemBufs) - 1) & 1, 2);
      mbarWait(&full[s], (lt / S) & 1, 3);
      tcFenceAfter();
      const uint32_t aHi = smem(stages + s * stF);
      const uint64_t ah0 = descKInterleave(aHi, lboA, 128), al0 = descKInterleave(aHi + planeF * 4, lboA, 128);
      const uint64_t b0 = descKInterleave(smem(bBank + bank * bStride), lboB, 128);
      const uint32_t d = tmem + buf * NB;
      if (nks == kFastKs && p.KH == 3 && p.KW == 3 && C == 16) {
        // the paper's 3x3, 16-channel groups: 18 K steps, offsets in registers
        // (a shared-memory table read + 64-bit adds per MMA held the issue
        // rate at 76-117 cycles per MMA, profiles/experiments/r01_gconv_shift_tuning.txt)
#pragma unroll
        for (int ks = 0; ks < kFastKs; ++ks) {
          const uint64_t ao = fastOff[ks], bd = b0 + static_cast<uint64_t>(ks * 2 * NB);
          if (electSync() && !(p.skip & 1)) {
            mmaTf32(d, ah0 + ao, bd, idesc, ks > 0);
            if constexpr (X3) mmaTf32(d, al0 + ao, bd, idesc, 1);
          }
        }
      } else {
#pragma unroll 2
        for (int ks = 0; ks < nks; ++ks) {
          const uint64_t ao = aOff16[ks], bd = b0 + static_cast<uint64_t>(ks * 2 * NB);  // 32*NB bytes per step
          if (electSync()) {
            mmaTf32(d, ah0 + ao, bd, idesc, ks > 0);
            if constexpr (X3) mmaTf32(d, al0 + ao, bd, idesc, 1);
          }
        }
      }
      if (electSync()) {
        mmaCommit(&empty[s]);
        mmaCommit(&tFull[buf]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ---- epilogue: TMEM -> registers -> + bias -> stores. The Mb bias terms
    // (gconv.tc:6 adds B(0), B(1), ... in turn) are folded once, in order,
    // into one constant: one add per output instead of Mb. Not the FFMA
    // kernel's rounding sequence, which this math mode does not claim; the
    // difference (<= Mb ulps of sum|B|) is far inside the TF32 bound (§2).
    const int q = warp - 4, pix = q * 32 + lane;
    float bsum = 0.0f;
    for (int m = 0; m < p.Mb; ++m) bsum = __fadd_rn(bsum, sBias[m]);
    for (int lt = 0; lt < t1 - t0; ++lt) {
      const int t = t0 + lt, buf = lt % kTmemBufs;
      mbarWait(&tFull[buf], (lt / kTmemBufs) & 1, 4);
      __syncwarp();
      tcFenceAfter();
      float v[NB];
      const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16) + buf * NB;
#pragma unroll
      for (int c = 0; c < NB; c += 16) tmemLoad16(trow + c, v + c);
      tmemLoadWait();
      if constexpr (X3) {
#pragma unroll
        for (int f = 0; f < F; ++f) v[f] += v[F + f];  // (hi*hi + lo*hi) + (hi*lo + lo*lo)
      }
      tcFenceBefore();
      __syncwarp();
      if (lane == 0) mbarArrive(&tEmpty[buf]);
      const int g = t / tilesG, tt = t - g * tilesG, n = tt / p.tilesPerImg;
      const int vp = (tt - n * p.tilesPerImg) * 128 + pix;
      const int h = vp / p.W, w = vp - h * p.W;
      if (w < p.Wo && h < p.Ho && !(p.skip & 4)) {
        float* o = p.O + (((int64_t)n * p.G + g) * F) * p.Ho * p.Wo + (int64_t)h * p.Wo + w;
#pragma unroll
        for (int f = 0; f < F; ++f) {
          o[(int64_t)f * p.Ho * p.Wo] = v[f] + bsum;
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
cudaError_t launchShift(ShiftParams p, cudaStream_t s) {
  using Cfg = ShiftCfg<F, X3>;
  auto kern = tc_gconv_shift_kernel<F, X3>;
  // the TMA halo path: planes whose rows of HP floats can be one tensor box
  // (16-byte plane pitch, HP <= 256); else the per-element cp.async builders
  CUtensorMap tmI{};
  p.tma = 0;
  const int64_t HW = (int64_t)p.H * p.W;
  EncodeFn enc = encodeFn();
  if (enc && HW % 4 == 0 && p.HP <= 256 && (reinterpret_cast<uintptr_t>(p.I) & 15) == 0 &&
      Cfg::smem(ShiftParams{p.I, p.O, p.W1, p.bias, p.N, p.G, p.C, p.H, p.W, p.F, p.KH, p.KW, p.Mb, p.Ho, p.Wo,
                            p.tilesPerImg, p.items, p.HP, 1, 0}) <= 227 * 1024) {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(HW), static_cast<cuuint64_t>(p.C),
                          static_cast<cuuint64_t>(p.N) * p.G};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(HW) * 4, static_cast<cuuint64_t>(HW) * p.C * 4};
    cuuint32_t box[3] = {static_cast<cuuint32_t>(p.HP), static_cast<cuuint32_t>(p.C), 1};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&tmI, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(p.I), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      p.tma = 1;
  }
  const int smemBytes = Cfg::smem(p);
  if (smemBytes > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kern), smemBytes);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one CTA per SM (one wave); a CTA's items must not span more than 2 groups
  const int tilesG = p.N * p.tilesPerImg;
  const int grid = std::max(std::min(sms, p.items), (p.items + tilesG - 1) / tilesG);
  kern<<<grid, kThreadsSh, smemBytes, s>>>(p, tmI);
  return cudaGetLastError();
}

}  // namespace

bool tcGconvShiftSupported(const GconvArgs& a, int math, const char** why) {
  auto no = [&](const char* w) {
    if (why) *why = w;
    return false;
  };
  if (a.C % 8) return no("tensor-core gconv needs input channels per group that are a multiple of 8");
  if (a.F != 16 && a.F != 32 && a.F != 64) return no("tensor-core gconv needs 16, 32 or 64 filters per group");
  const int HP = ((128 + (a.KH - 1) * a.W + (a.KW - 1)) + 7) / 8 * 8;
  const bool x3 = math == kMath3xTf32;
  const int64_t bytes = 1024 + (int64_t)kStagesSh * a.C * HP * 4 * (x3 ? 2 : 1) +
                        (int64_t)a.KH * a.KW * (a.C / 8) * 32 * (x3 ? 2 * a.F : a.F) * 2 + 1024 +
                        8 * a.KH * a.KW * (a.C / 8) + 4 * a.Mb;
  if (bytes > 227 * 1024) return no("tensor-core gconv (shifted halo): the halo ring exceeds shared memory");
  return true;
}

cudaError_t launchTcGconvShift(const GconvArgs& a, int math, cudaStream_t s) {
  if (!tcGconvShiftSupported(a, math, nullptr)) return cudaErrorInvalidValue;
  ShiftParams p{};
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
  p.tilesPerImg = (p.Ho * p.W + 127) / 128;
  p.HP = ((128 + (a.KH - 1) * a.W + (a.KW - 1)) + 7) / 8 * 8;
  p.items = a.G * a.N * p.tilesPerImg;
  if (const char* sk = std::getenv("TCB_GCONV_SKIP")) p.skip = std::atoi(sk);  // diagnostics only
  const bool x3 = math == kMath3xTf32;
  switch (a.F) {
    case 16: return x3 ? launchShift<16, true>(p, s) : launchShift<16, false>(p, s);
    case 32: return x3 ? launchShift<32, true>(p, s) : launchShift<32, false>(p, s);
    case 64: return x3 ? launchShift<64, true>(p, s) : launchShift<64, false>(p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace k
}  // namespace tcb
