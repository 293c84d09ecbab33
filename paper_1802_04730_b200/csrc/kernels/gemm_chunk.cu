// gemm_chunk.cu — exact fp32 batched NT-GEMM for many small batches whose
// whole output fits one warp tile (TBMM: 500 x Z(26x26) = X(26x72) . Y(26x72)^T,
// proj/kernels/tbmm.tc:2-4), on packed FFMA2.
//
// One warp (or S warps) owns one batch. The batch's two dense operand blocks
// land by one bulk copy each (issued first thing by one lane; whole
// contiguous blocks keep the DRAM streams long: the k-chunked TMA boxes of
// the first version of this kernel landed the same bytes ~60% slower,
// profiles/r02_wchunk/trace.txt), then the batch's warps transpose B into
// k-major rows Bt[k][32] in shared memory, so that one LDS.128 gives four
// adjacent output columns at one k. Each lane owns RM rows x 4 adjacent
// columns and advances them with `fma.rn.f32x2`: per k, each row's A value
// (a scalar broadcast operand of the FFMA2) times two column pairs. One
// FFMA2 does the two FMAs two FFMAs did, with fewer register-file reads
// (the measured 3-register FFMA rate is ~0.5-0.6 warp-FFMA per cycle per
// SMSP, FFMA2 ~0.6-0.75 FMA, profiles/r02_ffma_tile_probe.txt).
//
// Rows: lane = rg * 8 + cg, warp s of the batch's S: rows S*(rg + 4i) + s
// (i < RM), columns 4cg..4cg+3. 7 x 4 with S = 1 is a 28 x 32 warp tile; 4 x 4
// with S = 2 splits a 26-row batch 13 / 13 over two SMSPs.
//
// Exactness: fma.rn.f32x2 is two independent fma.rn.f32 (one rounding
// each); each output is one lane's sequential chain in ascending k from its
// init value (0, bias[n] or the in/out value), the reference interpreter's
// per-step order (interpreter.cc:218-233).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "sm100.cuh"

namespace tcb {
namespace k {

#ifdef TCB_WPAIR_TRACE
// diagnostic build only (profiles/wpair_trace.cu): per-batch globaltimer stamps
// [0] entry [1] copies issued [2] landed [3] transposed [4] chains done
// [5] stored [6] SM id [7] warp slot
__device__ unsigned long long g_wpair_trace[1024][8];
#define WP_STAMP(ev, dep)                                                          \
  do {                                                                             \
    unsigned long long t_;                                                         \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_) : "l"(dep) : "memory"); \
    if (lane == 0 && s == 0 && b < 1024) g_wpair_trace[b][ev] = t_;                \
  } while (0)
#else
#define WP_STAMP(ev, dep) \
  do {                    \
  } while (0)
#endif

namespace {

using namespace sm100;

constexpr int kBtLd = 32;  // transposed B row: 32 columns (N <= 32)

__device__ __forceinline__ float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ ulonglong2 lds4u(uint32_t addr) {
  ulonglong2 v;
  asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts1(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
// c = {x * b.lo + c.lo, x * b.hi + c.hi}, each rounded once (fma.rn.f32)
__device__ __forceinline__ void ffma2(unsigned long long& c, float x, unsigned long long b) {
  asm volatile("{\n.reg .b64 t;\nmov.b64 t, {%1, %1};\nfma.rn.f32x2 %0, t, %2, %0;\n}"
               : "+l"(c)
               : "f"(x), "l"(b));
}
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo32(unsigned long long v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float hi32(unsigned long long v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ void bulkLoad(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem(dst)),
      "l"(src), "r"(bytes), "r"(smem(bar))
      : "memory");
}
__device__ __forceinline__ void cpAsync16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ float initOf(const GemmArgs& a, const float* C, int m, int n) {
  if (a.init == kInitInout) return C[(int64_t)m * a.ldc + n];
  if (a.init == kInitBias) return a.bias[n];
  return 0.0f;
}

// one 4-step group: RM A rows (4 k each) x 4 k-major B rows (4 columns each)
template <int RM>
__device__ __forceinline__ void group(unsigned long long (&acc)[RM][2], const float4 (&x)[RM],
                                      const ulonglong2 (&y)[4]) {
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    ffma2(acc[i][0], x[i].x, y[0].x);
    ffma2(acc[i][1], x[i].x, y[0].y);
  }
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    ffma2(acc[i][0], x[i].y, y[1].x);
    ffma2(acc[i][1], x[i].y, y[1].y);
  }
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    ffma2(acc[i][0], x[i].z, y[2].x);
    ffma2(acc[i][1], x[i].z, y[2].y);
  }
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    ffma2(acc[i][0], x[i].w, y[3].x);
    ffma2(acc[i][1], x[i].w, y[3].y);
  }
}

// smem per batch: A [M][K] | B [N][K] (landed) | Bt [K][32] (transposed) |
// Z [M][N] (the output tile, stored by one bulk copy when C is dense)
struct PairLayout {
  int offB, offBt, offZ, bytes;  // per-batch byte offsets / size (16-aligned)
};
__host__ __device__ inline PairLayout pairLayout(int M, int N, int K) {
  PairLayout L;
  const int a = (M * K * 4 + 15) & ~15, b = (N * K * 4 + 15) & ~15;
  L.offB = a;
  L.offBt = a + b;
  L.offZ = a + b + K * kBtLd * 4;
  L.bytes = L.offZ + ((M * N * 4 + 15) & ~15);
  return L;
}

template <int RM, int S>
__global__ void __launch_bounds__(256) gemm_nt_wpair(const GemmArgs a, const int dense, const int bulkOut) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int s = warp % S, slot = warp / S, P = (blockDim.x >> 5) / S;  // batch slots per CTA
  const int b = blockIdx.x * P + slot;
  const PairLayout L = pairLayout(a.M, a.N, a.K);
  unsigned char* base = sm + slot * L.bytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + P * L.bytes) + slot;
  const bool live = b < a.batch;
  WP_STAMP(0, 0ull);
#ifdef TCB_WPAIR_TRACE
  if (lane == 0 && s == 0 && b < 1024) {
    unsigned smid, wid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    g_wpair_trace[b][6] = smid;
    g_wpair_trace[b][7] = wid;
  }
#endif
  const float* A = a.A + (int64_t)b * a.sA;
  const float* B = a.B + (int64_t)b * a.sB;
  const uint32_t sA = smem(base), sB = sA + L.offB, sBt = sA + L.offBt;
  const int K4 = a.K >> 2;
  if (live) {
    if (dense) {
      if (s == 0 && lane == 0) {
        mbarInit(bar, 1);
        fenceBarrierInit();
        mbarExpectTx(bar, (unsigned)((a.M + a.N) * a.K * 4));
        bulkLoad(base, A, (unsigned)(a.M * a.K * 4), bar);
        bulkLoad(base + L.offB, B, (unsigned)(a.N * a.K * 4), bar);
      }
    } else {  // strided rows: 16-byte cp.async by the batch's warps
      for (int e = s * 32 + lane; e < (a.M + a.N) * K4; e += S * 32) {
        const int r = e / K4, q = e - r * K4;
        if (r < a.M)
          cpAsync16(sA + (uint32_t)(r * a.K + 4 * q) * 4u, A + (int64_t)r * a.lda + 4 * q);
        else
          cpAsync16(sB + (uint32_t)((r - a.M) * a.K + 4 * q) * 4u, B + (int64_t)(r - a.M) * a.ldb + 4 * q);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  }
  WP_STAMP(1, 0ull);
  // init values (in flight behind the copies)
  const int rg = lane >> 3, cg = lane & 7, n0 = 4 * cg;
  const float* C = a.C + (int64_t)b * a.sC;
  unsigned long long acc[RM][2];
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    const int m = S * (rg + 4 * i) + s;
    float v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = (live && m < a.M && n0 + q < a.N) ? initOf(a, C, m, n0 + q) : 0.0f;
    acc[i][0] = pack2(v[0], v[1]);
    acc[i][1] = pack2(v[2], v[3]);
  }
  // the barrier init is visible to the batch's other warps / lanes
  if (S > 1) __syncthreads();
  else __syncwarp();
  if (live) {
    if (dense) mbarWait(bar, 0, 0);
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  if (!dense) {
    if (S > 1) __syncthreads();
    else __syncwarp();
  }
  WP_STAMP(2, 0ull);
  // transpose B [N][K] -> Bt [K][32]: the batch's S warps split the (n, 4k) units
  if (live) {
    for (int e = s * 32 + lane; e < a.N * K4; e += S * 32) {
      const int n = e % a.N, q = e / a.N;
      const float4 v = lds4(sB + (uint32_t)(n * a.K + 4 * q) * 4u);
      const uint32_t d = sBt + (uint32_t)(4 * q * kBtLd + n) * 4u;
      sts1(d, v.x);
      sts1(d + kBtLd * 4, v.y);
      sts1(d + 2 * kBtLd * 4, v.z);
      sts1(d + 3 * kBtLd * 4, v.w);
    }
  }
  if (S > 1) __syncthreads();
  else __syncwarp();
  WP_STAMP(3, 0ull);
  if (live) {
    uint32_t ra[RM];
#pragma unroll
    for (int i = 0; i < RM; ++i) ra[i] = sA + (uint32_t)(min(S * (rg + 4 * i) + s, a.M - 1) * a.K) * 4u;
    const uint32_t rb = sBt + (uint32_t)n0 * 4u;
    float4 x[2][RM];
    ulonglong2 y[2][4];
#pragma unroll
    for (int i = 0; i < RM; ++i) x[0][i] = lds4(ra[i]);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) y[0][kk] = lds4u(rb + (uint32_t)(kk * kBtLd) * 4u);
    int q = 0;
    for (; q + 2 <= K4; q += 2) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (q + h + 1 < K4) {
          const uint32_t o = (uint32_t)(q + h + 1) * 16u;
#pragma unroll
          for (int i = 0; i < RM; ++i) x[h ^ 1][i] = lds4(ra[i] + o);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            y[h ^ 1][kk] = lds4u(rb + (uint32_t)((4 * (q + h + 1) + kk) * kBtLd) * 4u);
        }
        group<RM>(acc, x[h], y[h]);
      }
    }
    if (q < K4) group<RM>(acc, x[0], y[0]);
    WP_STAMP(4, acc[RM - 1][1]);
    float* Cb = a.C + (int64_t)b * a.sC;
    const uint32_t sZ = sA + L.offZ;
#pragma unroll
    for (int i = 0; i < RM; ++i) {
      const int m = S * (rg + 4 * i) + s;
      if (m >= a.M) continue;
      float v[4] = {lo32(acc[i][0]), hi32(acc[i][0]), lo32(acc[i][1]), hi32(acc[i][1])};
#pragma unroll
      for (int q2 = 0; q2 < 4; ++q2) {
        if (n0 + q2 < a.N) {
          float o = v[q2];
          if (a.relu) o = fmaxf(o, 0.0f);
          if (bulkOut) sts1(sZ + (uint32_t)(m * a.N + n0 + q2) * 4u, o);
          else Cb[(int64_t)m * a.ldc + n0 + q2] = o;
        }
      }
    }
  }
  if (bulkOut) {
    // the batch's whole output block leaves by one bulk copy (full sectors,
    // one request) instead of 4-byte stores scattered over 104-byte rows
    fenceProxyAsyncSmem();
    if (S > 1) __syncthreads();
    else __syncwarp();
    if (live && s == 0 && lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a.C + (int64_t)b * a.sC),
                   "r"(sA + L.offZ), "r"((unsigned)(a.M * a.N * 4))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  }
  if (live) {
    WP_STAMP(5, 0ull);
  }
  if (S > 1) __syncthreads();  // the batch's waits on its barrier are behind us
  else __syncwarp();
  if (live && dense && s == 0 && lane == 0) mbarInval(bar);
}

template <int RM, int S>
cudaError_t launchT(const GemmArgs& a, int warps, cudaStream_t st) {
  if (a.M > 4 * RM * S || a.N > kBtLd) return cudaErrorInvalidValue;
  const PairLayout L = pairLayout(a.M, a.N, a.K);
  warps = std::max(S, std::min(8, warps / S * S));
  const int P = std::max(1, std::min(warps / S, (int)((227 * 1024 - 64) / (L.bytes + 8))));
  warps = P * S;
  const size_t smemBytes = (size_t)P * L.bytes + 8 * P;
  if (smemBytes > 227 * 1024) return cudaErrorInvalidValue;
  const int dense = a.lda == a.K && a.ldb == a.K;
  // dense 16-byte-aligned output blocks leave by one bulk copy per batch
  // (plain stores for ReLU-free and ReLU epilogues alike; in/out C included)
  const int bulkOut = a.ldc == a.N && (a.batch == 1 || a.sC == (int64_t)a.M * a.N) && (a.M * a.N) % 4 == 0 &&
                      (reinterpret_cast<uintptr_t>(a.C) & 15) == 0 && getenv("TCB_WPAIR_STG") == nullptr;
  auto kfn = gemm_nt_wpair<RM, S>;
  cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kfn), (int)smemBytes);
  if (e != cudaSuccess) return e;
  kfn<<<(a.batch + P - 1) / P, warps * 32, smemBytes, st>>>(a, dense, bulkOut);
  return cudaGetLastError();
}

}  // namespace

bool gemmChunkOk(const GemmArgs& a) {
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  // bulk copies / 16-byte cp.async: aligned bases, row and batch strides
  return a.batch >= 1 && a.K > 0 && a.K % 4 == 0 && a.lda % 4 == 0 && a.ldb % 4 == 0 && a.sA % 4 == 0 &&
         a.sB % 4 == 0 && al16(a.A) && al16(a.B) && a.N <= kBtLd && a.batch <= (1 << 30) &&
         pairLayout(a.M, a.N, a.K).bytes <= 200 * 1024;
}

// which: 0 = 7 rows x 4 columns per lane, one warp per batch (M <= 28);
//        1 = 4 x 4, two warps per batch (M <= 32)
cudaError_t launchGemmChunk(const GemmArgs& a, int which, int warps, int, cudaStream_t s) {
  if (a.batch <= 0 || a.M <= 0 || a.N <= 0) return cudaSuccess;
  if (!gemmChunkOk(a)) return cudaErrorInvalidValue;
  switch (which) {
    case 0: return launchT<7, 1>(a, warps, s);
    case 1: return launchT<4, 2>(a, warps, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace k
}  // namespace tcb
