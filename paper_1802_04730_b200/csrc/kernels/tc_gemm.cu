// tc_gemm.cu — tensor-core (tcgen05, TF32) variant of the GEMM-NT family:
//   C[b][m][n] = epi(init + sum_k A[b][m][k] * B[b][n][k])
// for TMM (tmm.tc), C3, TBMM (tbmm.tc) and the FC layers
// of MLP1/2FCRelu/MLP3 when the caller asks for tensor-core math
// (TCB_MATH_TF32 / TCB_MATH_3XTF32). The exact FFMA kernels (gemm.cu) stay
// the default: a tensor-core reduction cannot reproduce the reference's
// per-step fp32 chain (interpreter.cc:218-233), so these variants carry a
// stated tolerance instead of bit equality.
//
// Structure (one CTA = one 128 x BN output tile of one K split):
//   warp 0       TMA producer: 128x32 A and BNx32 B fp32 boxes, SWIZZLE_128B,
//                into an S-stage shared-memory ring (mbarrier full/empty);
//   warps 4..7   (3xTF32 only) split each landed fp32 k-block: A's hi =
//                rz(x) and lo = tf32(x - rz(x)) go to TMEM (the MMA's A
//                operand, so the tensor core re-reads only B from shared
//                memory); B's hi is the landed tile itself (the MMA uses the
//                top 19 bits of fp32 operands, rzTf32), its lo goes to a
//                second buffer;
//   warp 1       one elected lane issues tcgen05.mma.kind::tf32 (M=128,
//                N=BN, K=8 per instruction; 3xTF32: lo*hi + hi*lo + hi*hi,
//                A from TMEM)
//                into a TMEM accumulator, tcgen05.commit frees the stage;
//   warp 2       allocates / frees the TMEM columns;
//   warps 4..7   epilogue: tcgen05.ld the accumulator (lane = row) into a
//                shared-memory partial tile.
// Split-K: the `splits` CTAs of one output tile form a thread-block
// cluster along z. After a cluster barrier, CTA r reduces rows
// [r*128/splits, (r+1)*128/splits) of the tile by reading every CTA's
// partial over DSMEM in fixed rank order (deterministic), adds the init
// (bias / incoming C), applies ReLU and stores coalesced rows.
#include <atomic>
#include <cuda.h>

#include <mutex>

#include "kernels.cuh"
#include "sm100.cuh"

namespace tcb {
namespace k {

namespace {

using namespace sm100;

constexpr int kBM = 128;   // UMMA M (one TMEM lane per output row)
constexpr int kBK = 32;    // fp32 elements per 128-byte swizzle row
constexpr int kThreads = 256;

struct TcParams {
  float* C;
  const float* bias;
  int M, N, K;
  int64_t ldc, sC;
  int init, relu;
  int splits, kbPerSplit, nkb;
  int aBatched, bBatched;
  // block-diagonal packing of many small batches (TBMM): CTA tile t holds
  // batches [t*packP, t*packP + packP) stacked along M (rows of M each) and
  // along N; only the diagonal blocks are stored. 0 = no packing.
  int packP, batch;
};

template <int BN, bool X3>
struct TcCfg {
  static constexpr int kABytes = kBM * kBK * 4;
  static constexpr int kBBytes = BN * kBK * 4;
  // a stage: the landed fp32 A and B k-blocks (+ B's lo half for 3xTF32;
  // A's hi and lo halves go to TMEM, the MMA's A operand there)
  static constexpr int kStage = kABytes + kBBytes + (X3 ? kBBytes : 0);
  static constexpr int kPartLd = BN + 4;  // partial tile row stride (floats)
  static constexpr int kPartBytes = kBM * kPartLd * 4;
  static constexpr int kBudget = 200 * 1024;
  static constexpr int kAccCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr int kStagesSm = kBudget / kStage;
  // 3xTF32: every stage owns 2 x 32 TMEM columns (A hi | A lo) after the accumulator
  static constexpr int kStagesTm = X3 ? (512 - kAccCols) / (2 * kBK) : 8;
  static constexpr int kStagesRaw = kStagesSm < kStagesTm ? kStagesSm : kStagesTm;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kRing = kStages * kStage > kPartBytes ? kStages * kStage : kPartBytes;
  static constexpr int kSmem = 1024 + kRing + 256;
  static constexpr int kTmemCols = X3 ? 512 : kAccCols;
  static_assert(kStages >= 2, "stage ring too small");
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128 is a multiple of 16 in [16, 256]");
};

// the low part of the 3xTF32 split (sm100.cuh rzTf32): the MMA takes hi from
// the raw fp32 tile itself
__device__ __forceinline__ float lo1(float x) { return toTf32(x - rzTf32(x)); }
__device__ __forceinline__ float4 loPart(float4 x) { return make_float4(lo1(x.x), lo1(x.y), lo1(x.z), lo1(x.w)); }

template <int BN, bool X3>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcParams p) {
  using Cfg = TcCfg<BN, X3>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  auto aBig = [&](int s) { return sm + s * Cfg::kStage; };
  auto bBig = [&](int s) { return sm + s * Cfg::kStage + Cfg::kABytes; };
  auto bLo = [&](int s) { return sm + s * Cfg::kStage + Cfg::kABytes + Cfg::kBBytes; };
  // 3xTF32: TMEM columns of stage s's A operand, hi at +0, lo at +kBK
  auto aCol = [&](int s) { return static_cast<uint32_t>(Cfg::kAccCols + s * 2 * kBK); };
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + Cfg::kRing);
  uint64_t* conv = full + S;
  uint64_t* empty = conv + S;
  uint64_t* tmemFull = empty + S;
  uint32_t* tmemSlot = reinterpret_cast<uint32_t*>(tmemFull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = blockIdx.x, mt = blockIdx.y;
  const int split = blockIdx.z % p.splits, b = blockIdx.z / p.splits;
  const int kb0 = split * p.kbPerSplit;
  const int nk = min(p.nkb, kb0 + p.kbPerSplit) - kb0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbarInit(&full[s], 1);
      mbarInit(&conv[s], 128);
      mbarInit(&empty[s], 1);
    }
    mbarInit(tmemFull, 1);
    fenceBarrierInit();
  }
  if (warp == 0 && lane == 0) {
    tmaPrefetch(&tmA);
    tmaPrefetch(&tmB);
  }
  if (warp == 2) tmemAlloc<Cfg::kTmemCols>(tmemSlot);
  tcFenceBefore();
  __syncthreads();
  tcFenceAfter();
  const uint32_t tmem = *tmemSlot;

  if (warp == 0) {
    if (lane == 0) {
      const int ba = p.aBatched ? b : 0, bb = p.bBatched ? b : 0;
      // packed: the maps view A, B as [batch * M][K] and [batch * N][K]
      const int arow = p.packP ? mt * p.packP * p.M : mt * kBM;
      const int brow = p.packP ? mt * p.packP * p.N : nt * BN;
      for (int i = 0; i < nk; ++i) {
        const int s = i % S;
        if (i >= S) mbarWait(&empty[s], ((i / S) - 1) & 1, 1);
        mbarExpectTx(&full[s], Cfg::kABytes + Cfg::kBBytes);
        const int kc = (kb0 + i) * kBK;
        tmaLoad3d(aBig(s), &tmA, kc, arow, ba, &full[s]);
        tmaLoad3d(bBig(s), &tmB, kc, brow, bb, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idescTf32(kBM, BN);
      for (int i = 0; i < nk; ++i) {
        const int s = i % S;
        mbarWait(X3 ? &conv[s] : &full[s], (i / S) & 1, 2);
        tcFenceAfter();
        const uint32_t ab = smem(aBig(s)), bbg = smem(bBig(s));
#pragma unroll
        for (int kk = 0; kk < kBK / 8; ++kk) {
          const uint32_t off = kk * 32;  // 8 tf32 = 32 bytes along K inside the swizzle row
          const uint32_t acc = (i | kk) != 0;
          if constexpr (X3) {
            // A from TMEM (lane = row, column = k): the tensor core re-reads
            // only B from shared memory for the three products
            const uint32_t bl = smem(bLo(s)), ahi = tmem + aCol(s) + kk * 8, alo = ahi + kBK;
            mmaTf32Tmem(tmem, alo, descSw128(bbg + off), idesc, acc);
            mmaTf32Tmem(tmem, ahi, descSw128(bl + off), idesc, 1);
            mmaTf32Tmem(tmem, ahi, descSw128(bbg + off), idesc, 1);
          } else {
            mmaTf32(tmem, descSw128(ab + off), descSw128(bbg + off), idesc, acc);
          }
        }
        mmaCommit(&empty[s]);
      }
      mmaCommit(tmemFull);
    }
  } else if (warp >= 4) {
    const int et = threadIdx.x - 128;
    if constexpr (X3) {
      for (int i = 0; i < nk; ++i) {
        const int s = i % S;
        mbarWait(&full[s], (i / S) & 1, 4);
        // A: thread `row` reads its landed fp32 row of the k-block (128-byte
        // swizzled: 16-byte unit j at j ^ (row & 7)) and writes hi = rz(x)
        // and lo = tf32(x - rz(x)) into its TMEM lane (warp w % 4 owns lanes
        // 32(w % 4)..+31); x - rz(x) is exact in fp32
        {
          const int row = et;
          const float4* ar = reinterpret_cast<const float4*>(aBig(s) + row * 128);
          float hi[kBK], lo[kBK];
#pragma unroll
          for (int j = 0; j < kBK / 4; ++j) {
            const float4 x = ar[j ^ (row & 7)];
            const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              hi[4 * j + e] = rzTf32(xs[e]);
              lo[4 * j + e] = toTf32(xs[e] - hi[4 * j + e]);
            }
          }
          const uint32_t tl = tmem + (static_cast<uint32_t>((warp - 4) * 32) << 16) + aCol(s);
          tmemStore32(tl, hi);
          tmemStore32(tl + kBK, lo);
        }
        // B: hi is the landed tile itself (the MMA reads rzTf32 of it); lo to
        // the stage's second buffer
        const float4* bv = reinterpret_cast<const float4*>(bBig(s));
        float4* bl = reinterpret_cast<float4*>(bLo(s));
        for (int j = et; j < Cfg::kBBytes / 16; j += 128) bl[j] = loPart(bv[j]);
        tmemStoreWait();
        tcFenceBefore();
        fenceProxyAsyncSmem();
        mbarArrive(&conv[s]);
      }
    }
    // accumulator → shared partial tile (the ring is idle once tmemFull fires)
    mbarWait(tmemFull, 0, 3);
    tcFenceAfter();
    const int q = warp - 4, row = q * 32 + lane;
    float* part = reinterpret_cast<float*>(sm) + row * Cfg::kPartLd;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    if constexpr (BN % 32 == 0) {
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        float v[32];
        tmemLoad32(trow + c, v);
        tmemLoadWait();
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(part + c + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    } else {
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        float v[16];
        tmemLoad16(trow + c, v);
        tmemLoadWait();
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(part + c + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    }
    tcFenceBefore();
  }
  __syncthreads();
  if (p.splits > 1) clusterSync();

  // split-K reduction + epilogue: this CTA's slice of rows, columns coalesced
  {
    const int R = kBM / p.splits;
    const uint32_t base = smem(sm);
    const int64_t cb = static_cast<int64_t>(b) * p.sC;
    if (p.packP) {
      // diagonal blocks only: row r = (batch i, m), column c = (batch j, n), i == j
      for (int idx = threadIdx.x; idx < kBM * BN; idx += kThreads) {
        const int row = idx / BN, col = idx % BN;
        const int i = row / p.M, j = col / p.N;
        const int bq = mt * p.packP + i;
        if (i != j || i >= p.packP || bq >= p.batch) continue;
        const int m = row - i * p.M, n = col - j * p.N;
        float v = *reinterpret_cast<const float*>(sm + (row * Cfg::kPartLd + col) * 4);
        float* cp = p.C + static_cast<int64_t>(bq) * p.sC + static_cast<int64_t>(m) * p.ldc + n;
        if (p.init == kInitInout) v = *cp + v;
        else if (p.init == kInitBias) v = p.bias[n] + v;
        if (p.relu) v = fmaxf(v, 0.f);
        *cp = v;
      }
    }
    constexpr int Q = BN / 4;  // float4 column groups per row
    for (int idx = threadIdx.x; !p.packP && idx < R * Q; idx += kThreads) {
      const int row = split * R + idx / Q, col = (idx % Q) * 4;
      const int m = mt * kBM + row, n0 = nt * BN + col;
      if (m >= p.M || n0 >= p.N) continue;
      const uint32_t off = base + (row * Cfg::kPartLd + col) * 4;
      float4 acc;
      if (p.splits == 1) {
        acc = *reinterpret_cast<const float4*>(sm + (row * Cfg::kPartLd + col) * 4);
      } else {
        // every rank's partial in flight at once, then summed in rank order
        float4 part[16];
#pragma unroll
        for (int r = 0; r < 16; ++r)
          if (r < p.splits) part[r] = ldsCluster4(mapa(off, r));
        acc = part[0];
#pragma unroll
        for (int r = 1; r < 16; ++r)
          if (r < p.splits) {
            acc.x += part[r].x;
            acc.y += part[r].y;
            acc.z += part[r].z;
            acc.w += part[r].w;
          }
      }
      const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
      float* cp = p.C + cb + static_cast<int64_t>(m) * p.ldc + n0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (n0 + j >= p.N) break;
        float v = a4[j];
        if (p.init == kInitInout) v = cp[j] + v;
        else if (p.init == kInitBias) v = p.bias[n0 + j] + v;
        if (p.relu) v = fmaxf(v, 0.f);
        cp[j] = v;
      }
    }
  }
  if (p.splits > 1) clusterSync();  // peers may still be reading this CTA's partial
  if (warp == 2) {
    tcFenceAfter();
    tmemFree<Cfg::kTmemCols>(tmem);
  }
}

// ----------------------------------------------------------------- host
// 3-D map {K, rows, batch} of a row-major fp32 operand; box {32, boxRows, 1}
bool makeMap(CUtensorMap* m, const float* base, int K, int rows, int batch, int64_t ld, int64_t sBatch,
             int boxRows) {
  sm100::EncodeFn enc = sm100::encodeFn();
  if (!enc) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(batch)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 4,
                           static_cast<cuuint64_t>(batch > 1 ? sBatch : ld * rows) * 4};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(boxRows), 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, bool X3>
cudaError_t launchT(const CUtensorMap& ta, const CUtensorMap& tb, const TcParams& p, int tilesN, int tilesM,
                    int batch, cudaStream_t s) {
  using Cfg = TcCfg<BN, X3>;
  auto kern = tc_gemm_kernel<BN, X3>;
  // function attributes belong to a device context: set once per device
  // (bit d of `done`), never once per process
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(done.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    done.fetch_or(bit, std::memory_order_release);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tilesN, tilesM, batch * p.splits);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = p.splits;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, p);
}

template <bool X3>
cudaError_t dispatchBn(int bn, const CUtensorMap& ta, const CUtensorMap& tb, const TcParams& p, int tilesN,
                       int tilesM, int batch, cudaStream_t s) {
  switch (bn) {
    case 16: return launchT<16, X3>(ta, tb, p, tilesN, tilesM, batch, s);
    case 32: return launchT<32, X3>(ta, tb, p, tilesN, tilesM, batch, s);
    case 64: return launchT<64, X3>(ta, tb, p, tilesN, tilesM, batch, s);
    case 128: return launchT<128, X3>(ta, tb, p, tilesN, tilesM, batch, s);
    case 256: return launchT<256, X3>(ta, tb, p, tilesN, tilesM, batch, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

bool tcGemmSupported(const GemmArgs& a, const char** why) {
  auto no = [&](const char* w) {
    if (why) *why = w;
    return false;
  };
  if (a.lda % 4 || a.ldb % 4) return no("tensor-core GEMM needs operand rows that are multiples of 16 bytes");
  if (a.batch > 1 && ((a.sA && a.sA % 4) || (a.sB && a.sB % 4)))
    return no("tensor-core GEMM needs batch strides that are multiples of 16 bytes");
  if ((reinterpret_cast<uintptr_t>(a.A) | reinterpret_cast<uintptr_t>(a.B)) & 15)
    return no("tensor-core GEMM needs 16-byte aligned operands");
  if (a.K < 1 || a.M < 1 || a.N < 1) return no("empty GEMM");
  return true;
}

TcPlan tcGemmPlan(int batch, int M, int N, int K, int sms) {
  // Measured on B200 (profiles/r01_tc_plan_sweep.txt): 128-wide N tiles,
  // K split across a cluster of <= 8 CTAs until the grid is ~one wave —
  // wider tiles or 16-way splits lose more to the DSMEM reduction and the
  // per-CTA pipeline fill than they gain. Narrow the tile only when even
  // 8-way splitting leaves most SMs idle.
  const int tilesM = (M + kBM - 1) / kBM;
  const int nkb = (K + kBK - 1) / kBK;
  auto ctas = [&](int b) { return static_cast<int64_t>(batch) * tilesM * ((N + b - 1) / b); };
  auto splitsFor = [&](int b) {
    int s = 1;
    while (s < 8 && ctas(b) * s * 5 < sms * 4 && s * 4 <= nkb) s *= 2;  // >= 2 k-blocks per split
    return s;
  };
  if (batch > 1 && M <= 64 && N <= 128) {
    // many small batches: stack P of them per 128-row tile, block-diagonally
    int P = std::min(kBM / M, 256 / N);
    int bn = 16;
    while (bn < P * N) bn *= 2;
    if (P > 1 && bn <= 256) {
      TcPlan pl;
      pl.bn = bn;
      pl.splits = 1;
      pl.packP = P;
      return pl;
    }
  }
  int bn = 16;
  while (bn < 128 && bn < N) bn *= 2;
  while (bn > 32 && ctas(bn) * splitsFor(bn) * 4 < sms) bn /= 2;
  TcPlan pl;
  pl.bn = bn;
  pl.splits = splitsFor(bn);
  return pl;
}

cudaError_t launchTcGemm(const GemmArgs& a, int math, const TcPlan& pl, cudaStream_t s) {
  const char* why = nullptr;
  if (!tcGemmSupported(a, &why)) return cudaErrorInvalidValue;
  if (math != kMathTf32 && math != kMath3xTf32) return cudaErrorInvalidValue;
  const int bn = pl.bn, splits = pl.splits;
  if (splits < 1 || splits > 16 || (splits & (splits - 1))) return cudaErrorInvalidValue;
  CUtensorMap ta, tb;
  if (!makeMap(&ta, a.A, a.K, a.M, a.sA ? a.batch : 1, a.lda, a.sA, kBM)) return cudaErrorInvalidValue;
  if (!makeMap(&tb, a.B, a.K, a.N, a.sB ? a.batch : 1, a.ldb, a.sB, bn)) return cudaErrorInvalidValue;
  TcParams p;
  p.C = a.C;
  p.bias = a.bias;
  p.M = a.M;
  p.N = a.N;
  p.K = a.K;
  p.ldc = a.ldc;
  p.sC = a.sC;
  p.init = a.init;
  p.relu = a.relu;
  p.nkb = (a.K + kBK - 1) / kBK;
  p.splits = std::min(splits, p.nkb);
  while (p.splits & (p.splits - 1)) --p.splits;  // keep a power of two
  p.kbPerSplit = (p.nkb + p.splits - 1) / p.splits;
  // every split must own at least one k-block
  while (p.splits > 1 && (p.splits - 1) * p.kbPerSplit >= p.nkb) {
    p.splits /= 2;
    p.kbPerSplit = (p.nkb + p.splits - 1) / p.splits;
  }
  p.aBatched = a.sA != 0 && a.batch > 1;
  p.bBatched = a.sB != 0 && a.batch > 1;
  p.packP = 0;
  p.batch = a.batch;
  int tilesN = (a.N + bn - 1) / bn, tilesM = (a.M + kBM - 1) / kBM;
  const bool contiguous = a.batch > 1 && a.sA == (int64_t)a.M * a.lda && a.sB == (int64_t)a.N * a.ldb &&
                          a.lda == a.K && a.ldb == a.K;
  if (pl.packP > 1 && contiguous) {
    // block-diagonal packing: 2-D views of the contiguous batches
    p.packP = pl.packP;
    p.splits = 1;
    p.kbPerSplit = p.nkb;
    p.aBatched = p.bBatched = 0;
    if (!makeMap(&ta, a.A, a.K, a.batch * a.M, 1, a.lda, 0, kBM)) return cudaErrorInvalidValue;
    if (!makeMap(&tb, a.B, a.K, a.batch * a.N, 1, a.ldb, 0, bn)) return cudaErrorInvalidValue;
    tilesN = 1;
    tilesM = (a.batch + p.packP - 1) / p.packP;
    return math == kMath3xTf32 ? dispatchBn<true>(bn, ta, tb, p, tilesN, tilesM, 1, s)
                               : dispatchBn<false>(bn, ta, tb, p, tilesN, tilesM, 1, s);
  }
  return math == kMath3xTf32 ? dispatchBn<true>(bn, ta, tb, p, tilesN, tilesM, a.batch, s)
                             : dispatchBn<false>(bn, ta, tb, p, tilesN, tilesM, a.batch, s);
}

}  // namespace k
}  // namespace tcb
