// gemm_chunk.cu — exact fp32 batched NT-GEMM for many small batches whose
// whole output fits one warp tile (TBMM: 500 x Z(26x26) = X(26x72) . Y(26x72)^T,
// proj/kernels/tbmm.tc:2-4).
//
// One warp owns one batch. Its two operand blocks land by TMA tensor copies
// in NCH reduction chunks (a box {w k-steps, rows, 1 batch} per operand and
// chunk, each chunk on its own mbarrier), issued by the warp's lane 0 before
// anything else, so the copy engine streams every chunk of every batch while
// the warps start their chains on chunk 0 and follow the data in. The loads
// never pass through the LSU pipe: the cp.async-filled slab kernels shared it
// with their chains' shared-memory reads and slowed both.
//
// Lane = rg * 8 + cg owns the RM x RN outputs at rows rg + 4i, columns
// cg + 8j (7 x 4 per lane: a 28 x 32 warp tile holds a 26 x 26 batch). Each
// 4-step group reads RM + RN float4s from shared memory for 4*RM*RN FFMAs.
// A chunk lands dense ([rows][w]); full chunks are w = 20 or 36 floats wide at
// the paper shape so that the 8 B rows one load instruction touches (80 or
// 144 bytes apart) fall in 8 distinct 16-byte bank groups.
//
// Exactness: each output is one lane's sequential FFMA chain in ascending k
// from its init value (0, bias[n] or the in/out value), the reference
// interpreter's per-step order (interpreter.cc:218-233); the chunking only
// changes when operands arrive, never the order they are consumed in.
#include <cuda.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "kernels.cuh"
#include "sm100.cuh"

namespace tcb {
namespace k {

#ifdef TCB_WCHUNK_TRACE
// diagnostic build only (profiles/wchunk_trace.cu): per-warp globaltimer stamps
// [0] entry [1] copies issued [2..7] chunk c landed [8] chains done [9] stored
// [10] SM id [11] SMSP (warp slot % 4)
__device__ unsigned long long g_wchunk_trace[1024][12];
#define WC_STAMP(ev)                                                          \
  do {                                                                        \
    unsigned long long t_;                                                    \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
    if (lane == 0 && b < 1024) g_wchunk_trace[b][ev] = t_;                    \
  } while (0)
#else
#define WC_STAMP(ev) \
  do {               \
  } while (0)
#endif

namespace {

using namespace sm100;

constexpr int kMaxChunks = 6;

struct ChunkPlan {
  int nch;                  // reduction chunks
  int cw, tw;               // floats per full chunk, floats in the last chunk
  int slot;                 // bytes of one warp's operand slot (multiple of 128)
  int offA[kMaxChunks];     // byte offset of chunk c's A box [M][w] in the slot
  int offB[kMaxChunks];     // ... and of its B box [N][w]
};

__device__ __forceinline__ float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

__device__ __forceinline__ float initOf(const GemmArgs& a, const float* C, int m, int n) {
  if (a.init == kInitInout) return C[(int64_t)m * a.ldc + n];
  if (a.init == kInitBias) return a.bias[n];
  return 0.0f;
}

template <int RM, int RN>
__device__ __forceinline__ void group4(float (&acc)[RM][RN], const float4* x, const float4* y) {
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

// the chains over one landed chunk of G 4-step groups: register double
// buffer, the next group's float4s loaded before this group's FFMAs
template <int RM, int RN>
__device__ __forceinline__ void chunkChains(float (&acc)[RM][RN], const uint32_t (&ra)[RM],
                                            const uint32_t (&rb)[RN], int G) {
  float4 av[2][RM], bv[2][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i) av[0][i] = lds4(ra[i]);
#pragma unroll
  for (int j = 0; j < RN; ++j) bv[0][j] = lds4(rb[j]);
  int q = 0;
  for (; q + 2 <= G; q += 2) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (q + h + 1 < G) {
        const uint32_t o = (uint32_t)(q + h + 1) * 16u;
#pragma unroll
        for (int i = 0; i < RM; ++i) av[h ^ 1][i] = lds4(ra[i] + o);
#pragma unroll
        for (int j = 0; j < RN; ++j) bv[h ^ 1][j] = lds4(rb[j] + o);
      }
      group4<RM, RN>(acc, av[h], bv[h]);
    }
  }
  if (q < G) group4<RM, RN>(acc, av[0], bv[0]);  // odd group count: the last sits in buffer 0
}

template <int RM, int RN>
__global__ void __launch_bounds__(256) gemm_nt_wchunk(const __grid_constant__ CUtensorMap mA,
                                                      const __grid_constant__ CUtensorMap mAt,
                                                      const __grid_constant__ CUtensorMap mB,
                                                      const __grid_constant__ CUtensorMap mBt, const GemmArgs a,
                                                      const ChunkPlan p) {
  extern __shared__ __align__(128) unsigned char smRaw[];
  unsigned char* sm = smRaw + ((128u - (smem(smRaw) & 127u)) & 127u);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int b = blockIdx.x * W + warp;
  unsigned char* slot = sm + warp * p.slot;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + W * p.slot) + warp * kMaxChunks;
  if (b >= a.batch) return;  // (no CTA-wide barrier below)
  WC_STAMP(0);
#ifdef TCB_WCHUNK_TRACE
  if (lane == 0 && b < 1024) {
    unsigned smid, wid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    g_wchunk_trace[b][10] = smid;
    g_wchunk_trace[b][11] = wid;
  }
#endif
  if (lane == 0) {
    for (int c = 0; c < p.nch; ++c) mbarInit(&bars[c], 1);
    fenceBarrierInit();
    for (int c = 0; c < p.nch; ++c) {
      const bool last = c + 1 == p.nch;
      mbarExpectTx(&bars[c], (unsigned)((a.M + a.N) * (last ? p.tw : p.cw) * 4));
      tmaLoad3d(slot + p.offA[c], last ? &mAt : &mA, c * p.cw, 0, b, &bars[c]);
      tmaLoad3d(slot + p.offB[c], last ? &mBt : &mB, c * p.cw, 0, b, &bars[c]);
    }
  }
  WC_STAMP(1);
  const float* C = a.C + (int64_t)b * a.sC;
  const int rg = lane >> 3, cg = lane & 7;
  float acc[RM][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int m = rg + 4 * i, n = cg + 8 * j;
      acc[i][j] = (m < a.M && n < a.N) ? initOf(a, C, m, n) : 0.0f;
    }
  __syncwarp();  // lane 0's barrier init before the others poll
  const uint32_t sBase = smem(slot);
  for (int c = 0; c < p.nch; ++c) {
    const int w = c + 1 == p.nch ? p.tw : p.cw;
    uint32_t ra[RM], rb[RN];
#pragma unroll
    for (int i = 0; i < RM; ++i) ra[i] = sBase + p.offA[c] + (uint32_t)(min(rg + 4 * i, a.M - 1) * w) * 4u;
#pragma unroll
    for (int j = 0; j < RN; ++j) rb[j] = sBase + p.offB[c] + (uint32_t)(min(cg + 8 * j, a.N - 1) * w) * 4u;
    mbarWait(&bars[c], 0, c);
    WC_STAMP(2 + min(c, 5));
    chunkChains<RM, RN>(acc, ra, rb, w >> 2);
  }
  WC_STAMP(8);
  float* Cb = a.C + (int64_t)b * a.sC;
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    const int m = rg + 4 * i;
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int n = cg + 8 * j;
      if (m < a.M && n < a.N) {
        float v = acc[i][j];
        if (a.relu) v = fmaxf(v, 0.0f);
        Cb[(int64_t)m * a.ldc + n] = v;
      }
    }
  }
  WC_STAMP(9);
}

// ------------------------------------------------------------------ host
// 3-D map {K, rows, batch} of a row-major fp32 operand, box {w, rows, 1},
// no swizzle (the box lands dense, [rows][w]); cached by (pointer, geometry)
struct WcKey {
  const void* p;
  int64_t K, rows, batch, ld, sb;
  int w, dev;
  bool operator==(const WcKey& o) const {
    return p == o.p && K == o.K && rows == o.rows && batch == o.batch && ld == o.ld && sb == o.sb && w == o.w &&
           dev == o.dev;
  }
};
std::mutex g_wcMu;
std::vector<std::pair<WcKey, CUtensorMap>> g_wcMaps;  // most recent last, <= 128

bool wcMap(CUtensorMap* m, const float* base, int K, int rows, int batch, int64_t ld, int64_t sb, int w) {
  int dev = 0;
  cudaGetDevice(&dev);
  WcKey key{base, K, rows, batch, ld, sb, w, dev};
  {
    std::lock_guard<std::mutex> g(g_wcMu);
    for (size_t i = g_wcMaps.size(); i-- > 0;)
      if (g_wcMaps[i].first == key) {
        *m = g_wcMaps[i].second;
        return true;
      }
  }
  EncodeFn enc = encodeFn();
  if (!enc) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(batch)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 4, static_cast<cuuint64_t>(sb) * 4};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(w), static_cast<cuuint32_t>(rows), 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  std::lock_guard<std::mutex> g(g_wcMu);
  if (g_wcMaps.size() >= 128) g_wcMaps.erase(g_wcMaps.begin());
  g_wcMaps.push_back({key, *m});
  return true;
}

int up128(int x) { return (x + 127) & ~127; }

// chunk widths: full chunks of cw floats (a multiple of 4), the last one the
// remainder; nch requested chunks
bool planChunks(const GemmArgs& a, int nch, ChunkPlan& p) {
  p = ChunkPlan{};
  const int K4 = a.K / 4;
  nch = std::max(1, std::min(nch, std::min(kMaxChunks, K4)));
  p.cw = 4 * ((K4 + nch - 1) / nch);
  p.nch = (a.K + p.cw - 1) / p.cw;
  p.tw = a.K - (p.nch - 1) * p.cw;
  int off = 0;
  for (int c = 0; c < p.nch; ++c) {
    const int w = c + 1 == p.nch ? p.tw : p.cw;
    p.offA[c] = off;
    off += up128(a.M * w * 4);
    p.offB[c] = off;
    off += up128(a.N * w * 4);
  }
  p.slot = off;
  return true;
}

template <int RM, int RN>
cudaError_t launchT(const GemmArgs& a, int warps, int nch, cudaStream_t s) {
  if (a.M > 4 * RM || a.N > 8 * RN) return cudaErrorInvalidValue;
  ChunkPlan p;
  planChunks(a, nch, p);
  warps = std::max(1, std::min(8, warps));
  const size_t smemBytes = (size_t)warps * p.slot + (size_t)warps * kMaxChunks * 8 + 128;
  if (smemBytes > 227 * 1024) return cudaErrorInvalidValue;
  CUtensorMap mA, mAt, mB, mBt;
  if (!wcMap(&mA, a.A, a.K, a.M, a.batch, a.lda, a.sA, p.cw)) return cudaErrorInvalidValue;
  if (!wcMap(&mB, a.B, a.K, a.N, a.batch, a.ldb, a.sB, p.cw)) return cudaErrorInvalidValue;
  mAt = mA;
  mBt = mB;
  if (p.tw != p.cw) {
    if (!wcMap(&mAt, a.A, a.K, a.M, a.batch, a.lda, a.sA, p.tw)) return cudaErrorInvalidValue;
    if (!wcMap(&mBt, a.B, a.K, a.N, a.batch, a.ldb, a.sB, p.tw)) return cudaErrorInvalidValue;
  }
  auto kfn = gemm_nt_wchunk<RM, RN>;
  cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kfn), (int)smemBytes);
  if (e != cudaSuccess) return e;
  kfn<<<(a.batch + warps - 1) / warps, warps * 32, smemBytes, s>>>(mA, mAt, mB, mBt, a, p);
  return cudaGetLastError();
}

}  // namespace

bool gemmChunkOk(const GemmArgs& a) {
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  // TMA boxes: 16-byte aligned bases, row and batch strides, chunk widths;
  // a real batch stride for both operands (broadcast operands take the slab)
  return a.batch > 1 && a.K > 0 && a.K % 4 == 0 && a.lda % 4 == 0 && a.ldb % 4 == 0 && a.sA > 0 && a.sB > 0 &&
         a.sA % 4 == 0 && a.sB % 4 == 0 && al16(a.A) && al16(a.B) && a.M <= 256 && a.N <= 256 &&
         a.batch <= (1 << 30) && sm100::encodeFn() != nullptr;
}

// which: 0 = 7x4 per lane (28 x 32 warp tile), 1 = 4x4 (16 x 32)
cudaError_t launchGemmChunk(const GemmArgs& a, int which, int warps, int nch, cudaStream_t s) {
  if (a.batch <= 0 || a.M <= 0 || a.N <= 0) return cudaSuccess;
  if (!gemmChunkOk(a)) return cudaErrorInvalidValue;
  switch (which) {
    case 0: return launchT<7, 4>(a, warps, nch, s);
    case 1: return launchT<4, 4>(a, warps, nch, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace k
}  // namespace tcb
