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
  // fused second FC layer (tcFc2): O2 = relu(O1 . W2^T + bias2), O1 being this
  // GEMM's bias + ReLU output; N2p = N2 rounded up to 16, K2p = K2 = N (a
  // multiple of 32)
  float* O2;
  const float* bias2;
  int N2, N2p, K2p;
};

template <int BN, bool X3, bool L2 = false>
struct TcCfg {
  static constexpr int kABytes = kBM * kBK * 4;
  static constexpr int kBBytes = BN * kBK * 4;
  // a stage: the landed fp32 A and B k-blocks (+ B's lo half for 3xTF32;
  // A's hi and lo halves go to TMEM, the MMA's A operand there). With B no
  // wider than A, B's lo half overwrites the landed A once it is in TMEM
  // (kLoInA): 32 KB stages, a 6-deep ring at BN = 128 instead of 4
  static constexpr bool kLoInA = X3 && BN <= kBM;
  static constexpr int kStage = kABytes + kBBytes + (X3 && !kLoInA ? kBBytes : 0);
  static constexpr int kPartLd = BN + 4;  // partial tile row stride (floats)
  static constexpr int kPartBytes = kBM * kPartLd * 4;
  static constexpr int kBudget = 200 * 1024;
  static constexpr int kAccCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr int kStagesSm = kBudget / kStage;
  // 3xTF32: every stage owns 2 x 32 TMEM columns (A hi | A lo) after the accumulator
  static constexpr int kStagesTm = X3 ? (512 - kAccCols) / (2 * kBK) : 8;
  static constexpr int kStagesRaw = kStagesSm < kStagesTm ? kStagesSm : kStagesTm;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kRingRaw = kStages * kStage > kPartBytes ? kStages * kStage : kPartBytes;
  // L2: the partial tile, A2 (K2p <= 128) and W2 (N2p <= 128 TF32 / 64 3xTF32, + its lo plane)
  static constexpr int kL2Bytes = 69632 + 65536 + 65536;
  static constexpr int kRing = L2 && kL2Bytes > kRingRaw ? kL2Bytes : kRingRaw;
  static constexpr int kSmem = 1024 + kRing + 256;
  // L2 (fused second layer, BN <= 128): layer 2's A operand hi / lo (3xTF32)
  // at TMEM columns 128 / 256, its accumulator at 384
  static constexpr int kTmemCols = (X3 || L2) ? 512 : kAccCols;
  static constexpr int kA2Off = (kPartBytes + 1023) / 1024 * 1024;  // L2: layer 2's A (rank 0), after the partial tile
  static_assert(kStages >= 2, "stage ring too small");
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128 is a multiple of 16 in [16, 256]");
};

// the low part of the 3xTF32 split (sm100.cuh rzTf32): the MMA takes hi from
// the raw fp32 tile itself
__device__ __forceinline__ float lo1(float x) { return toTf32(x - rzTf32(x)); }
__device__ __forceinline__ float4 loPart(float4 x) { return make_float4(lo1(x.x), lo1(x.y), lo1(x.z), lo1(x.w)); }

// swizzled K-major SW128 offset of element (row, k) of a 128-row operand
// (k-blocks of 32 fp32, 128-byte rows, 16-byte unit j of row r at j ^ (r & 7))
__device__ __forceinline__ uint32_t swOff128(int row, int k) {
  return (uint32_t)((k >> 5) * (kBM * 128) + row * 128 + ((((k & 31) >> 2) ^ (row & 7)) << 4) + ((k & 3) << 2));
}

template <int BN, bool X3, bool L2 = false>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmW2, TcParams p) {
  using Cfg = TcCfg<BN, X3, L2>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  auto aBig = [&](int s) { return sm + s * Cfg::kStage; };
  auto bBig = [&](int s) { return sm + s * Cfg::kStage + Cfg::kABytes; };
  auto bLo = [&](int s) { return Cfg::kLoInA ? aBig(s) : sm + s * Cfg::kStage + Cfg::kABytes + Cfg::kBBytes; };
  // 3xTF32: TMEM columns of stage s's A operand, hi at +0, lo at +kBK
  auto aCol = [&](int s) { return static_cast<uint32_t>(Cfg::kAccCols + s * 2 * kBK); };
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + Cfg::kRing);
  uint64_t* conv = full + S;
  uint64_t* empty = conv + S;
  uint64_t* tmemFull = empty + S;
  uint64_t* b2Full = tmemFull + 1;  // L2: W2 landed (rank 0)
  uint64_t* l2Done = tmemFull + 2;  // L2: layer-2 MMAs complete (rank 0)
  uint64_t* a2Full = tmemFull + 3;  // L2: every peer's O1 rows landed in rank 0's A2
  uint32_t* tmemSlot = reinterpret_cast<uint32_t*>(tmemFull + 4);

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
    mbarInit(b2Full, 1);
    mbarInit(l2Done, 1);
    mbarInit(a2Full, 1);
    // rank 0's A2 receives every other rank's rows by bulk copy
    if (L2 && split == 0)
      mbarExpectTx(a2Full, (unsigned)((kBM - kBM / p.splits) * p.K2p * 4));
    fenceBarrierInit();
  }
  if (warp == 0 && lane == 0) {
    tmaPrefetch(&tmA);
    tmaPrefetch(&tmB);
    if (L2) tmaPrefetch(&tmW2);
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
        // B's lo half lands where A was: every conversion thread has its A row
        // in registers first
        if constexpr (Cfg::kLoInA) asm volatile("bar.sync 1, 128;" ::: "memory");
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
    if (L2 && split == 0 && warp == 4 && lane == 0) {
      // layer 2's weights land behind layer 1's epilogue, after A2 (the
      // partial tile and A2 sit below them; the ring is idle)
      const int nkb2 = p.K2p / kBK;
      uint8_t* b2 = sm + Cfg::kA2Off + nkb2 * kBM * 128;
      mbarExpectTx(b2Full, (unsigned)(nkb2 * p.N2p * 128));
      for (int kb = 0; kb < nkb2; ++kb) tmaLoad3d(b2 + kb * p.N2p * 128, &tmW2, kb * kBK, 0, 0, b2Full);
    }
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
        if (L2)  // layer 2's A operand, K-major SW128: this CTA's rows, locally
          *reinterpret_cast<float*>(sm + Cfg::kA2Off + swOff128(m, n0 + j)) = v;
      }
    }
  }
  if constexpr (L2) {
    // this CTA's O1 rows go to rank 0's A2 by one bulk copy per 32-column
    // block (16 rows x 128 B, contiguous under the swizzle): 4-byte remote
    // stores from every rank queued ~1 per cycle at rank 0 (6.4 us)
    if (split > 0) {
      fenceProxyAsyncSmem();
      __syncthreads();
      if (threadIdx.x == 0) {
        const int R = kBM / p.splits;
        const uint32_t src = smem(sm + Cfg::kA2Off) + split * R * 128;
        const uint32_t bar0 = mapa(smem(a2Full), 0);
        for (int kb = 0; kb < p.K2p / kBK; ++kb)
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  mapa(src + kb * kBM * 128, 0)),
              "r"(src + kb * kBM * 128), "r"((unsigned)(R * 128)), "r"(bar0)
              : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    }
  }
  if (p.splits > 1) clusterSync();  // peers may still be reading this CTA's partial
  if constexpr (L2) {
    if (p.splits == 1) __syncthreads();
    if (split == 0) {
      // ---- the fused second layer, in rank 0: M = 128 rows of O1 (A2, every
      // rank's reduced rows), N = N2p, K = K2p
      const int nkb2 = p.K2p / kBK;
      uint8_t* a2 = sm + Cfg::kA2Off;
      uint8_t* b2 = a2 + nkb2 * kBM * 128;
      uint8_t* b2lo = b2 + nkb2 * p.N2p * 128;
      const uint32_t acc2 = tmem + 384u;
      mbarWait(b2Full, 0, 8);
      if (p.splits > 1) mbarWait(a2Full, 0, 10);
      {
        // (3xTF32) B2's lo plane (all threads); A2's hi (/ lo) into TMEM
        // (warps 4-7: lane = row): the MMA reads A from TMEM, so the O1 rows
        // the ranks stored into this CTA's shared memory are only ever read
        // by the generic proxy
        if (X3) {
          const float4* bv = reinterpret_cast<const float4*>(b2);
          float4* bl = reinterpret_cast<float4*>(b2lo);
          for (int j = threadIdx.x; j < nkb2 * p.N2p * 8; j += kThreads) bl[j] = loPart(bv[j]);
        }
        if (warp >= 4) {
          const int row = (warp - 4) * 32 + lane;
          const uint32_t tl = tmem + (static_cast<uint32_t>((warp - 4) * 32) << 16);
          for (int kb = 0; kb < nkb2; ++kb) {
            const float4* ar = reinterpret_cast<const float4*>(a2 + kb * kBM * 128 + row * 128);
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
            tmemStore32(tl + 128 + kb * kBK, hi);
            if (X3) tmemStore32(tl + 256 + kb * kBK, lo);
          }
          tmemStoreWait();
        }
        if (X3) fenceProxyAsyncSmem();
      }
      tcFenceBefore();
      __syncthreads();
      tcFenceAfter();
      if (warp == 1 && lane == 0) {
        const uint32_t idesc2 = idescTf32(kBM, p.N2p);
        for (int kb = 0; kb < nkb2; ++kb) {
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk) {
            const uint32_t acc = (kb | kk) != 0;
            const uint32_t bhi = smem(b2 + kb * p.N2p * 128) + kk * 32;
            const uint32_t ahi = tmem + 128 + kb * kBK + kk * 8;
            if constexpr (X3) {
              const uint32_t alo = tmem + 256 + kb * kBK + kk * 8;
              const uint32_t blo = smem(b2lo + kb * p.N2p * 128) + kk * 32;
              mmaTf32Tmem(acc2, alo, descSw128(bhi), idesc2, acc);
              mmaTf32Tmem(acc2, ahi, descSw128(blo), idesc2, 1);
              mmaTf32Tmem(acc2, ahi, descSw128(bhi), idesc2, 1);
            } else {
              mmaTf32Tmem(acc2, ahi, descSw128(bhi), idesc2, acc);
            }
          }
        }
        mmaCommit(l2Done);
      }
      // layer-2 epilogue: accumulator rows -> shared memory (the A2 region is
      // free once the MMAs completed) -> bias + ReLU, coalesced row stores
      // (per-lane row stores cost ~8.7 us)
      float* o2s = reinterpret_cast<float*>(a2);  // [128][N2p + 4]
      const int ld2 = p.N2p + 4;
      if (warp >= 4) {
        mbarWait(l2Done, 0, 9);
        tcFenceAfter();
        const int row = (warp - 4) * 32 + lane;
        const uint32_t trow = acc2 + (static_cast<uint32_t>((warp - 4) * 32) << 16);
        for (int c = 0; c < p.N2p; c += 16) {
          float v[16];
          tmemLoad16(trow + c, v);
          tmemLoadWait();
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<float4*>(o2s + row * ld2 + c + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
        tcFenceBefore();
      }
      __syncthreads();
      for (int e = threadIdx.x; e < p.M * p.N2; e += kThreads) {
        const int r = e / p.N2, c = e - r * p.N2;
        p.O2[e] = fmaxf(p.bias2[c] + o2s[r * ld2 + c], 0.f);
      }
    }
  }
  if (warp == 2) {
    tcFenceAfter();
    tmemFree<Cfg::kTmemCols>(tmem);
  }
}

// ----------------------------------------------------------------- host
// 3-D map {K, rows, batch} of a row-major fp32 operand; box {32, boxRows, 1}
bool makeMap(CUtensorMap* m, const float* base, int K, int rows, int batch, int64_t ld, int64_t sBatch,
             int boxRows) {
  return cachedMapF32Sw128(m, base, K, rows, batch, ld, sBatch, kBK, boxRows);  // (sm100.cuh: cached per geometry)
}

template <int BN, bool X3, bool L2 = false>
cudaError_t launchT(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tw2, const TcParams& p,
                    int tilesN, int tilesM, int batch, cudaStream_t s) {
  using Cfg = TcCfg<BN, X3, L2>;
  auto kern = tc_gemm_kernel<BN, X3, L2>;
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
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, tw2, p);
}

template <bool X3>
cudaError_t dispatchBn(int bn, const CUtensorMap& ta, const CUtensorMap& tb, const TcParams& p, int tilesN,
                       int tilesM, int batch, cudaStream_t s) {
  switch (bn) {
    case 16: return launchT<16, X3>(ta, tb, ta, p, tilesN, tilesM, batch, s);
    case 32: return launchT<32, X3>(ta, tb, ta, p, tilesN, tilesM, batch, s);
    case 64: return launchT<64, X3>(ta, tb, ta, p, tilesN, tilesM, batch, s);
    case 128: return launchT<128, X3>(ta, tb, ta, p, tilesN, tilesM, batch, s);
    case 256: return launchT<256, X3>(ta, tb, ta, p, tilesN, tilesM, batch, s);
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
  TcParams p{};
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

// ---- two FC layers in one launch (2FCRelu in tensor-core math): layer 1 is
// the split-K cluster GEMM above (bias + ReLU epilogue, O1 stored); every
// rank also writes its reduced O1 rows into rank 0's shared memory as layer
// 2's K-major A operand, and rank 0 then runs layer 2 (M = 128, N = N2, K =
// N1) on the tensor cores with W2 landed by TMA behind layer 1's epilogue.
bool tcFc2Supported(const FcChainArgs& a, int math, const char** why) {
  auto no = [&](const char* w) {
    if (why) *why = w;
    return false;
  };
  if (math != kMathTf32 && math != kMath3xTf32) return no("fused 2-layer FC: tensor-core math only");
  if (a.layers != 2) return no("fused 2-layer FC: exactly two layers");
  const FcLayer &L1 = a.L[0], &L2 = a.L[1];
  if (a.batch < 1 || a.batch > kBM) return no("fused 2-layer FC: at most 128 rows");
  if (L1.out < 1 || L1.out > 128 || L1.out % 32) return no("fused 2-layer FC: layer 1 width a multiple of 32, <= 128");
  if (L2.kred != L1.out) return no("fused 2-layer FC: layer 2 reduces over layer 1's width");
  if (L2.out < 1 || L2.out > (math == kMath3xTf32 ? 64 : 128)) return no("fused 2-layer FC: layer 2 too wide");
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (a.ldi % 4 || L1.ldw % 4 || L2.ldw % 4 || !al16(a.I) || !al16(L1.W) || !al16(L2.W))
    return no("fused 2-layer FC: 16-byte operand rows");
  return true;
}

cudaError_t launchTcFc2(const FcChainArgs& a, int math, int sms, cudaStream_t s) {
  if (!tcFc2Supported(a, math, nullptr)) return cudaErrorInvalidValue;
  const FcLayer &L1 = a.L[0], &L2 = a.L[1];
  const int bn = L1.out <= 32 ? 32 : L1.out <= 64 ? 64 : 128;
  TcParams p{};
  p.C = L1.O;
  p.bias = L1.bias;
  p.M = a.batch;
  p.N = L1.out;
  p.K = L1.kred;
  p.ldc = L1.out;
  p.sC = 0;
  p.init = kInitBias;
  p.relu = 1;
  p.nkb = (L1.kred + kBK - 1) / kBK;
  p.splits = tcGemmPlan(1, a.batch, L1.out, L1.kred, sms).splits;
  p.splits = std::min(std::max(1, p.splits), std::min(8, p.nkb));
  while (p.splits & (p.splits - 1)) --p.splits;
  p.kbPerSplit = (p.nkb + p.splits - 1) / p.splits;
  while (p.splits > 1 && (p.splits - 1) * p.kbPerSplit >= p.nkb) {
    p.splits /= 2;
    p.kbPerSplit = (p.nkb + p.splits - 1) / p.splits;
  }
  p.aBatched = p.bBatched = 0;
  p.packP = 0;
  p.batch = 1;
  p.O2 = L2.O;
  p.bias2 = L2.bias;
  p.N2 = L2.out;
  p.N2p = (L2.out + 15) / 16 * 16;
  p.K2p = L1.out;
  CUtensorMap ta, tb, tw;
  if (!makeMap(&ta, a.I, L1.kred, a.batch, 1, a.ldi, 0, kBM)) return cudaErrorInvalidValue;
  if (!makeMap(&tb, L1.W, L1.kred, L1.out, 1, L1.ldw, 0, bn)) return cudaErrorInvalidValue;
  if (!makeMap(&tw, L2.W, L2.kred, L2.out, 1, L2.ldw, 0, p.N2p)) return cudaErrorInvalidValue;
  const bool x3 = math == kMath3xTf32;
  switch (bn) {
    case 32: return x3 ? launchT<32, true, true>(ta, tb, tw, p, 1, 1, 1, s) : launchT<32, false, true>(ta, tb, tw, p, 1, 1, 1, s);
    case 64: return x3 ? launchT<64, true, true>(ta, tb, tw, p, 1, 1, 1, s) : launchT<64, false, true>(ta, tb, tw, p, 1, 1, 1, s);
    default: return x3 ? launchT<128, true, true>(ta, tb, tw, p, 1, 1, 1, s) : launchT<128, false, true>(ta, tb, tw, p, 1, 1, 1, s);
  }
}

}  // namespace k
}  // namespace tcb
