// gemm_tma.cu — exact fp32 NT-GEMM fed by TMA (TMM, TBMM, C3, FC layers).
//
// Same arithmetic as gemm_nt_tiled (gemm.cu): every output is one thread's
// sequential FFMA chain in ascending k from its init value (the reference
// interpreter's per-step order, interpreter.cc:218-233), bit-identical. What
// changes is how operands reach shared memory. The tiled kernel fills its
// ring with 16-byte cp.async from every thread, and an SM keeps too few of
// those in flight: C3 (128 x 1024 -> 1000) streams 256 KB per CTA and ran at
// 17% of the FFMA peak (r01). Here one producer warp issues two TMA tensor
// copies per 32-deep k stage (an A box {32 k, TM rows} and a B box {32 k,
// TN rows}, 128-byte swizzled), S stages deep on full/empty mbarriers, so
// the copy engine keeps S x (TM + TN) x 128 bytes in flight per CTA while
// the consumer warps run their chains. Consumers own RM x RN micro-tiles and
// read float4 groups at the swizzled position (16-byte chunk q of row r sits
// at chunk q ^ (r & 7)), so eight consecutive rows hit eight bank groups.
// Rows past M / N arrive as zeros (TMA out-of-bounds fill) and are never
// stored; the last k stage runs only its K - 32*kt valid steps.
#include <cuda.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "kernels.cuh"
#include "sm100.cuh"

namespace tcb {
namespace k {

namespace {

using namespace sm100;

constexpr int kTK = 32;  // k steps per stage (one 128-byte swizzle row)

__device__ __forceinline__ float4 ldsSw(uint32_t rowBase, int r, int q) {
  float4 v;
  const uint32_t addr = rowBase + (uint32_t)((q ^ (r & 7)) << 4);
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float ldsSw1(uint32_t rowBase, int r, int k) {
  float v;
  const uint32_t addr = rowBase + (uint32_t)((((k >> 2) ^ (r & 7)) << 4) + ((k & 3) << 2));
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

// arrive on the mbarrier at the same offset in cluster CTA `rank`
__device__ __forceinline__ void mbarArriveRemote(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n.reg .b32 ra;\nmapa.shared::cluster.u32 ra, %0, %1;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}" ::"r"(smem(bar)),
      "r"(rank)
      : "memory");
}

__device__ __forceinline__ float initOf(const GemmArgs& a, const float* C, int m, int n) {
  if (a.init == kInitInout) return C[(int64_t)m * a.ldc + n];
  if (a.init == kInitBias) return a.bias[n];
  return 0.0f;
}

// CN > 1: the CN CTAs of a cluster along N share their A tile (same rows
// m0.., different column tiles): each loads TM / CN of its rows and
// multicasts them to all CN, so every A line leaves L2 once per cluster
// instead of once per CTA (C3's I3 rows were read by 32 CTAs at once). A
// stage is refilled only when every consumer warp of every cluster CTA has
// released it (remote arrivals on each CTA's empty barrier).
template <int TM, int TN, int RM, int RN, int S, int CN>
__global__ void __launch_bounds__((TM / RM) * (TN / RN) + 32)
    gemm_nt_tma(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, const GemmArgs a) {
  constexpr int TX = TN / RN, TY = TM / RM, CT = TX * TY, CW = CT / 32;
  constexpr int ABYTES = TM * 128, SBYTES = (TM + TN) * 128;
  static_assert(CT % 32 == 0 && TM % 8 == 0 && TN % 8 == 0, "tile");
  static_assert(CN == 1 || (TM / CN) % 8 == 0, "multicast slices are whole 8-row swizzle atoms");
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * SBYTES);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.x * TN, m0 = blockIdx.y * TM, b = blockIdx.z;
  const int nk = (a.K + kTK - 1) / kTK;
  const uint32_t rank = CN > 1 ? clusterRank() : 0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbarInit(&full[s], 1);
      mbarInit(&empty[s], CW * CN);
    }
    fenceBarrierInit();
  }
  if (CN > 1) clusterSync();  // every CTA's barriers exist before any multicast lands
  else __syncthreads();

  if (warp == CW) {  // ---- producer: one elected lane issues every TMA copy
    if (lane == 0) {
      tmaPrefetch(&ta);
      tmaPrefetch(&tb);
      const int bA = a.sA ? b : 0, bB = a.sB ? b : 0;
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % S;
        if (kt >= S) mbarWait(&empty[s], ((kt / S) - 1) & 1, 1);
        mbarExpectTx(&full[s], SBYTES);
        if (CN > 1) {
          constexpr int SL = TM / CN;
          tmaLoad3dMc(sm + s * SBYTES + rank * SL * 128, &ta, kt * kTK, m0 + rank * SL, bA, &full[s],
                      (uint16_t)((1u << CN) - 1));
        } else {
          tmaLoad3d(sm + s * SBYTES, &ta, kt * kTK, m0, bA, &full[s]);
        }
        tmaLoad3d(sm + s * SBYTES + ABYTES, &tb, kt * kTK, n0, bB, &full[s]);
      }
    }
    if (CN > 1) clusterSync();  // stay until no peer can still multicast into this CTA
    return;
  }

  // ---- consumers: RM x RN chains per thread
  const int tx = tid % TX, ty = tid / TX;
  float* C = a.C + (int64_t)b * a.sC;
  float acc[RM][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int m = m0 + ty + i * TY, n = n0 + tx + j * TX;
      acc[i][j] = (m < a.M && n < a.N) ? initOf(a, C, m, n) : 0.0f;
    }
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % S;
    mbarWait(&full[s], (kt / S) & 1, 0);
    const uint32_t aBase = smem(sm + s * SBYTES), bBase = aBase + ABYTES;
    uint32_t ra[RM], rb[RN];
#pragma unroll
    for (int i = 0; i < RM; ++i) ra[i] = aBase + (uint32_t)((ty + i * TY) * 128);
#pragma unroll
    for (int j = 0; j < RN; ++j) rb[j] = bBase + (uint32_t)((tx + j * TX) * 128);
    const int klim = min(kTK, a.K - kt * kTK);
    if (klim == kTK) {
      float4 av[2][RM], bv[2][RN];
#pragma unroll
      for (int i = 0; i < RM; ++i) av[0][i] = ldsSw(ra[i], ty + i * TY, 0);
#pragma unroll
      for (int j = 0; j < RN; ++j) bv[0][j] = ldsSw(rb[j], tx + j * TX, 0);
#pragma unroll
      for (int q = 0; q < kTK / 4; ++q) {
        if (q + 1 < kTK / 4) {  // next group's operands before this group's FFMAs
#pragma unroll
          for (int i = 0; i < RM; ++i) av[(q + 1) & 1][i] = ldsSw(ra[i], ty + i * TY, q + 1);
#pragma unroll
          for (int j = 0; j < RN; ++j) bv[(q + 1) & 1][j] = ldsSw(rb[j], tx + j * TX, q + 1);
        }
        const float4* x = av[q & 1];
        const float4* y = bv[q & 1];
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) acc[i][j] = __fmaf_rn(x[i].x, y[j].x, acc[i][j]);
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) acc[i][j] = __fmaf_rn(x[i].y, y[j].y, acc[i][j]);
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) acc[i][j] = __fmaf_rn(x[i].z, y[j].z, acc[i][j]);
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) acc[i][j] = __fmaf_rn(x[i].w, y[j].w, acc[i][j]);
      }
    } else {  // the last, partial stage: exactly K - 32*kt steps
      for (int kk = 0; kk < klim; ++kk)
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j)
            acc[i][j] = __fmaf_rn(ldsSw1(ra[i], ty + i * TY, kk), ldsSw1(rb[j], tx + j * TX, kk), acc[i][j]);
    }
    __syncwarp();
    if (lane == 0) {  // this warp is done with stage s (in every cluster CTA: they share its A slice)
      if (CN > 1)
        for (uint32_t r = 0; r < CN; ++r) mbarArriveRemote(&empty[s], r);
      else
        mbarArrive(&empty[s]);
    }
  }
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int m = m0 + ty + i * TY, n = n0 + tx + j * TX;
      if (m < a.M && n < a.N) {
        float v = acc[i][j];
        if (a.relu) v = fmaxf(v, 0.0f);
        C[(int64_t)m * a.ldc + n] = v;
      }
    }
  // every wait and arrival on the ring is behind us (the producer warp has
  // left; peers stop arriving at the cluster barrier): end the barriers
  if (CN > 1) clusterSync();
  else asm volatile("bar.sync 1, %0;" ::"r"(CT) : "memory");
  if (tid == 0)
    for (int s = 0; s < S; ++s) {
      mbarInval(&full[s]);
      mbarInval(&empty[s]);
    }
}

// ------------------------------------------------------------------ host
// operand maps: sm100::cachedMapF32Sw128 (cached by pointer and geometry)
bool mapOf(CUtensorMap* m, const float* base, int K, int rows, int batch, int64_t ld, int64_t sBatch, int boxRows) {
  return cachedMapF32Sw128(m, base, K, rows, batch, ld, sBatch, kTK, boxRows);
}

template <int TM, int TN, int RM, int RN, int S, int CN = 1>
cudaError_t launchT(const GemmArgs& a, cudaStream_t s) {
  CUtensorMap ta, tb;
  const int batched = a.batch > 1;
  if (!mapOf(&ta, a.A, a.K, a.M, batched && a.sA ? a.batch : 1, a.lda, a.sA, CN > 1 ? TM / CN : TM))
    return cudaErrorInvalidValue;
  if (!mapOf(&tb, a.B, a.K, a.N, batched && a.sB ? a.batch : 1, a.ldb, a.sB, TN)) return cudaErrorInvalidValue;
  auto kfn = gemm_nt_tma<TM, TN, RM, RN, S, CN>;
  const int smem = S * (TM + TN) * 128 + 2 * S * 8 + 1024;
  cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kfn), smem);
  if (e != cudaSuccess) return e;
  const int tilesN = (a.N + TN - 1) / TN;
  // the grid's N extent rounded up to whole clusters (CTAs past N load and
  // share their A slice, store nothing)
  dim3 grid((tilesN + CN - 1) / CN * CN, (a.M + TM - 1) / TM, a.batch);
  if (CN == 1) {
    kfn<<<grid, (TM / RM) * (TN / RN) + 32, smem, s>>>(ta, tb, a);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3((TM / RM) * (TN / RN) + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CN;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kfn, ta, tb, a);
}

}  // namespace

bool gemmTmaOk(const GemmArgs& a) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  // TMA: 16-byte aligned base and row / batch strides; rows of >= 1 float
  return a.K > 0 && a.lda % 4 == 0 && a.ldb % 4 == 0 && a.sA % 4 == 0 && a.sB % 4 == 0 && al16(a.A) && al16(a.B) &&
         a.batch <= 65535 && sm100::encodeFn() != nullptr;
}

// (TM, TN, RM, RN[, A multicast over CN]): 0 (32,32,4,4)  1 (32,32,4,2)
// 2 (32,64,4,4)  3 (16,32,2,4)  4 (32,16,4,2)  5 (64,32,4,4)  6 (32,32,2,2)
// 7 (32,32,2,2 CN 4)  8 (32,32,4,2 CN 4)  9 (32,16,2,2 CN 4)  10 (32,32,2,2 CN 2)
cudaError_t launchGemmTma(const GemmArgs& a, int which, cudaStream_t s) {
  if (!gemmTmaOk(a)) return cudaErrorInvalidValue;
  switch (which) {
    case 0: return launchT<32, 32, 4, 4, 8>(a, s);
    case 1: return launchT<32, 32, 4, 2, 8>(a, s);
    case 2: return launchT<32, 64, 4, 4, 6>(a, s);
    case 3: return launchT<16, 32, 2, 4, 8>(a, s);
    case 4: return launchT<32, 16, 4, 2, 8>(a, s);
    case 5: return launchT<64, 32, 4, 4, 6>(a, s);
    case 6: return launchT<32, 32, 2, 2, 8>(a, s);
    case 7: return launchT<32, 32, 2, 2, 8, 4>(a, s);
    case 8: return launchT<32, 32, 4, 2, 8, 4>(a, s);
    case 9: return launchT<32, 16, 2, 2, 8, 4>(a, s);
    case 10: return launchT<32, 32, 2, 2, 8, 2>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace k
}  // namespace tcb
