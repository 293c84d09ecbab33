// tc_fc_fused.cu — an FC+bias+ReLU chain (MLP3, proj/kernels/mlp3.tc:4-16:
// the paper's single-kernel MLP3) as ONE tcgen05 kernel,
// TF32 / 3xTF32. Tensor-core math mode: not FFMA-exact.
//
// One CTA owns 128 batch rows (the UMMA M) and runs every layer:
//   - at entry one thread lands every operand by TMA tensor copies on one
//     mbarrier: the input rows as 32-wide K chunks {32 k, 128 rows} and
//     each layer's weights {32 k, N_l rows} (rows past N_l zero-filled),
//     all 128-byte swizzled (K-major SW128 UMMA layout);
//   - 3xTF32: the landed operands are split in place into hi (tf32 rna) and
//     lo planes; each K step issues lo*hi + hi*lo + hi*hi (tc_gemm.cu's
//     order; the tensor-core emulation in tests/tc_emulate.py);
//   - layer l: one elected lane issues K_l / 8 MMAs (M = 128, N = N_l
//     padded to 16) into its TMEM columns and commits; the four warps read
//     their 32 TMEM lanes (= rows), add the bias, apply ReLU, store the
//     layer's return, and write the activations straight into shared memory
//     as layer l+1's A operand, in the same swizzled K-major layout (the
//     input's region is free once layer l's MMAs completed).
// So the activations never leave the chip and the chain costs one launch
// (round 1 ran one tc_gemm launch per layer: MLP3 3xTF32 16.6 us).
// Requirements (tcFcFusedSupported): every K_l % 32 == 0, N_l <= 256, the
// operands fit shared memory; B any (one CTA per 128 rows).
#include <cuda.h>

#include <mutex>
#include <vector>

#include "kernels.cuh"
#include "sm100.cuh"

namespace tcb {
namespace k {

namespace {

using namespace sm100;

constexpr int kFcMaxL = 3;
constexpr int kRowsTc = 128;

struct FusedPlan {
  int layers, batch;
  int K[kFcMaxL], N[kFcMaxL], Np[kFcMaxL];  // reduction, outputs, outputs padded to 16
  int aBytes;                               // one plane of the A region (max over layers)
  int bOff[kFcMaxL];                        // weight regions (bytes from the base)
  int bBytes[kFcMaxL];                      // one plane of each weight region
  int tcol[kFcMaxL];                        // TMEM column of each layer's accumulator
  int total;                                // bytes of the TMA landing (hi planes)
  int tmaOut[kFcMaxL];                      // 1: layer l's return leaves by TMA tensor stores from its
                                            // swizzled tile in the A hi plane (the next layer's A)
  const float* bias[kFcMaxL];
  float* O[kFcMaxL];
};

__host__ __device__ inline int up16(int x) { return (x + 15) & ~15; }

// fp32 value into the swizzled K-major SW128 layout: chunk of 32 k, 128-byte
// rows, 16-byte unit j of row r at j ^ (r & 7)
__device__ __forceinline__ uint32_t swOff(int row, int k) {
  return (uint32_t)((k >> 5) * (kRowsTc * 128) + row * 128 + ((((k & 31) >> 2) ^ (row & 7)) << 4) + ((k & 3) << 2));
}

__device__ __forceinline__ void splitPlane(float* hi, float* lo, int bytes, int tid, int nthreads) {
  float4* h4 = reinterpret_cast<float4*>(hi);
  float4* l4 = reinterpret_cast<float4*>(lo);
  // hi stays the landed fp32 plane (the MMA reads its top 19 bits = rzTf32)
  for (int j = tid; j < bytes / 16; j += nthreads) {
    const float4 x = h4[j];
    float4 l;
    l.x = toTf32(x.x - rzTf32(x.x)); l.y = toTf32(x.y - rzTf32(x.y));
    l.z = toTf32(x.z - rzTf32(x.z)); l.w = toTf32(x.w - rzTf32(x.w));
    l4[j] = l;
  }
}

#ifdef TCB_TCFC_TRACE
// diagnostic build only (profiles/tcfc_trace.cu): globaltimer stamps of CTA 0
__device__ unsigned long long g_tcfc_trace[32];
#define TCFC_STAMP(ev)                                              \
  do {                                                              \
    unsigned long long t_;                                          \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));         \
    if (threadIdx.x == 0 && blockIdx.x == 0) g_tcfc_trace[ev] = t_; \
  } while (0)
#else
#define TCFC_STAMP(ev) \
  do {                 \
  } while (0)
#endif

constexpr int kThreadsFc = 512;  // 16 warps: elementwise passes and the epilogues use all of them

template <int NL, bool X3>
__global__ void __launch_bounds__(kThreadsFc, 1)
    tc_fc_fused_kernel(const __grid_constant__ CUtensorMap tIn, const __grid_constant__ CUtensorMap tW0,
                       const __grid_constant__ CUtensorMap tW1, const __grid_constant__ CUtensorMap tW2,
                       const __grid_constant__ CUtensorMap tO0, const __grid_constant__ CUtensorMap tO1,
                       const __grid_constant__ CUtensorMap tO2,
                       const __grid_constant__ FusedPlan p) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row0 = blockIdx.x * kRowsTc;
  TCFC_STAMP(0);
  // regions: A hi [, A lo], then per layer B hi [, B lo]
  uint8_t* aHi = sm;
  uint8_t* aLo = sm + p.aBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + p.bOff[NL - 1] + p.bBytes[NL - 1] * (X3 ? 2 : 1));
  uint64_t* landed = bars;
  uint64_t* mmaDone = bars + 1;
  uint32_t* tmemSlot = reinterpret_cast<uint32_t*>(bars + 2);
  float* sBias = reinterpret_cast<float*>(bars + 4);  // [NL][256]: every layer's bias, zero past N_l
  constexpr int kCols = 256;  // all layers' accumulators side by side: sum of N_l padded to 16 (<= 256, checked)
  if (tid == 0) {
    mbarInit(landed, 1);
    mbarInit(mmaDone, 1);
    fenceBarrierInit();
  }
  if (warp == 0) tmemAlloc<kCols>(tmemSlot);
#pragma unroll
  for (int l = 0; l < NL; ++l)
    for (int n = tid; n < 256; n += kThreadsFc) sBias[l * 256 + n] = n < p.N[l] ? __ldg(p.bias[l] + n) : 0.0f;
  tcFenceBefore();
  __syncthreads();
  tcFenceAfter();
  const uint32_t tmem = *tmemSlot;

  // ---- every operand by TMA, one barrier
  if (tid == 0) {
    tmaPrefetch(&tIn);
    mbarExpectTx(landed, (uint32_t)p.total);
    for (int c = 0; c < p.K[0] / 32; ++c) tmaLoad3d(aHi + c * kRowsTc * 128, &tIn, c * 32, row0, 0, landed);
    const CUtensorMap* tw[3] = {&tW0, &tW1, &tW2};
#pragma unroll
    for (int l = 0; l < NL; ++l)
      for (int c = 0; c < p.K[l] / 32; ++c)
        tmaLoad3d(sm + p.bOff[l] + c * p.Np[l] * 128, tw[l], c * 32, 0, 0, landed);
  }
  mbarWait(landed, 0, 0);
  TCFC_STAMP(1);
  if constexpr (X3) {
    splitPlane(reinterpret_cast<float*>(aHi), reinterpret_cast<float*>(aLo), p.K[0] / 32 * kRowsTc * 128, tid,
               kThreadsFc);
#pragma unroll
    for (int l = 0; l < NL; ++l)
      splitPlane(reinterpret_cast<float*>(sm + p.bOff[l]), reinterpret_cast<float*>(sm + p.bOff[l] + p.bBytes[l]),
                 p.bBytes[l], tid, kThreadsFc);
    fenceProxyAsyncSmem();
    __syncthreads();
  }
  TCFC_STAMP(2);

#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const int Np = p.Np[l];
    // ---- MMAs of layer l (one elected lane of warp 0)
    if (warp == 0) {
      tcFenceAfter();
      const uint32_t idesc = idescTf32(128, Np);
      const uint32_t ah = smem(aHi), al = smem(aLo), bh = smem(sm + p.bOff[l]),
                     bl = smem(sm + p.bOff[l] + p.bBytes[l]);
      const uint32_t d = tmem + p.tcol[l];
      const int nks = p.K[l] / 8;
      const int nks2 = nks;
      if constexpr (!X3) {
        // TF32: one lane issues the layer's MMAs back to back, then commits
        // (an elect + warp sync per K step: ~150 cycles an MMA; MLP3 7.6 ->
        // 6.9 us). 3xTF32 keeps the per-step elect: its three MMAs a step
        // issued back to back from one lane measured slower (10.6 vs 10.0 us)
        if (lane == 0) {
          for (int ks = 0; ks < nks2; ++ks) {
            const uint32_t oa = (ks >> 2) * kRowsTc * 128 + (ks & 3) * 32, ob = (ks >> 2) * Np * 128 + (ks & 3) * 32;
            mmaTf32(d, descSw128(ah + oa), descSw128(bh + ob), idesc, ks > 0);
          }
          mmaCommit(mmaDone);
        }
        __syncwarp();
      } else {
        for (int ks = 0; ks < nks2; ++ks) {
          // chunk ks / 4; 8 tf32 = 32 bytes along K inside the swizzle row
          const uint32_t oa = (ks >> 2) * kRowsTc * 128 + (ks & 3) * 32, ob = (ks >> 2) * Np * 128 + (ks & 3) * 32;
          if (electSync()) {
            mmaTf32(d, descSw128(al + oa), descSw128(bh + ob), idesc, ks > 0);
            mmaTf32(d, descSw128(ah + oa), descSw128(bl + ob), idesc, 1);
            mmaTf32(d, descSw128(ah + oa), descSw128(bh + ob), idesc, 1);
          }
          __syncwarp();
        }
        if (electSync()) mmaCommit(mmaDone);
        __syncwarp();
      }
      if (l < 3) TCFC_STAMP(20 + l);  // (trace build) this layer's MMAs issued
    }
    if (l > 0 && p.tmaOut[l - 1]) {  // layer l-1's tile stays in place until its stores have read it
      if (tid == 0) tmaStoreWaitRead();
      __syncthreads();
    }
    mbarWait(mmaDone, l & 1, 1);
    TCFC_STAMP(3 + 2 * l);
    tcFenceAfter();
    // ---- epilogue: warp w reads TMEM lane quarter w % 4 (rows) and the
    // 16-column groups w / 4, w / 4 + 4, ...; + bias, ReLU, store, next A
    const int q4 = warp & 3, row = q4 * 32 + lane, grow = row0 + row;
    const bool last = l + 1 == NL;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q4 * 32) << 16) + p.tcol[l];
    const float* bl = sBias + l * 256;
    for (int c0 = (warp >> 2) * 16; c0 < Np; c0 += (kThreadsFc / 128) * 16) {
      float v[16];
      tmemLoad16(trow + c0, v);
      tmemLoadWait();
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        float4 o;
        float* op = &o.x;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int n = c0 + j + q;
          op[q] = n < p.N[l] ? fmaxf(v[j + q] + bl[n], 0.0f) : 0.0f;
        }
        const int n = c0 + j;
        if (p.tmaOut[l]) {
          // the return leaves by TMA from the swizzled tile (below); for the
          // last layer the dead A plane holds it
          if (last || n >= p.K[l + 1]) *reinterpret_cast<float4*>(aHi + swOff(row, n)) = o;
        } else if (grow < p.batch && n < p.N[l]) {
          float* dst = p.O[l] + (int64_t)grow * p.N[l] + n;
          if (n + 4 <= p.N[l] && (p.N[l] & 3) == 0) {
            *reinterpret_cast<float4*>(dst) = o;
          } else {
            for (int q = 0; q < 4 && n + q < p.N[l]; ++q) dst[q] = op[q];
          }
        }
        if (!last && n < p.K[l + 1]) {  // layer l+1's A operand (its K = this N)
          const uint32_t off = swOff(row, n);
          if constexpr (X3) {
            float4 lo;  // hi: o itself (the MMA reads rzTf32(o))
            lo.x = toTf32(o.x - rzTf32(o.x)); lo.y = toTf32(o.y - rzTf32(o.y));
            lo.z = toTf32(o.z - rzTf32(o.z)); lo.w = toTf32(o.w - rzTf32(o.w));
            *reinterpret_cast<float4*>(aHi + off) = o;
            *reinterpret_cast<float4*>(aLo + off) = lo;
          } else {
            *reinterpret_cast<float4*>(aHi + off) = o;
          }
        }
      }
    }
    fenceProxyAsyncSmem();  // the next layer's A, written by the generic proxy, for the tensor core
    tcFenceBefore();
    __syncthreads();
    TCFC_STAMP(4 + 2 * l);
    if (p.tmaOut[l] && tid == 0) {
      // coalesced by the TMA engine: lane-per-row stores put 32 separate
      // 16-byte L2 writes in every warp store (~1.4 us of layer 1's epilogue)
      const CUtensorMap* to[3] = {&tO0, &tO1, &tO2};
      for (int c = 0; c * 32 < p.N[l]; ++c) tmaStore3d(to[l], aHi + c * kRowsTc * 128, c * 32, row0, 0);
      tmaStoreCommit();
    }
  }
  if (tid == 0) tmaStoreWaitAll();  // (no-op without TMA stores) the tiles are read before the CTA exits
  if (warp == 0) {
    tcFenceAfter();
    tmemFree<kCols>(tmem);
  }
}

// cached 3-D {K, rows, 1} maps, box {32, boxRows, 1}, SW128
std::mutex g_fmu;
std::vector<std::pair<std::vector<int64_t>, CUtensorMap>> g_fmaps;

bool mapFc(CUtensorMap* m, const float* base, int K, int rows, int64_t ld, int boxRows) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::vector<int64_t> key{(int64_t)reinterpret_cast<uintptr_t>(base), K, rows, ld, boxRows, dev};
  {
    std::lock_guard<std::mutex> g(g_fmu);
    for (size_t i = g_fmaps.size(); i-- > 0;)
      if (g_fmaps[i].first == key) {
        *m = g_fmaps[i].second;
        return true;
      }
  }
  EncodeFn enc = encodeFn();
  if (!enc) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows), 1};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 4, static_cast<cuuint64_t>(ld) * rows * 4};
  cuuint32_t box[3] = {32, static_cast<cuuint32_t>(boxRows), 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  std::lock_guard<std::mutex> g(g_fmu);
  if (g_fmaps.size() >= 128) g_fmaps.erase(g_fmaps.begin());
  g_fmaps.push_back({key, *m});
  return true;
}

int planFused(const FcChainArgs& a, bool x3, FusedPlan& p) {
  p = FusedPlan{};
  p.layers = a.layers;
  p.batch = a.batch;
  int aMax = 0, off = 0, col = 0;
  for (int l = 0; l < a.layers; ++l) {
    p.K[l] = a.L[l].kred;
    p.N[l] = a.L[l].out;
    p.Np[l] = up16(a.L[l].out);
    aMax = std::max(aMax, p.K[l] / 32 * kRowsTc * 128);
    p.bias[l] = a.L[l].bias;
    p.O[l] = a.L[l].O;
  }
  p.aBytes = aMax;
  // TMA-stored returns: 16-byte rows, the whole padded tile inside the A plane,
  // and (not last) the next layer's A covering every column of it
  for (int l = 0; l < a.layers; ++l)
    p.tmaOut[l] = p.N[l] % 4 == 0 && (reinterpret_cast<uintptr_t>(p.O[l]) & 15) == 0 &&
                  (p.N[l] + 31) / 32 * kRowsTc * 128 <= aMax;
  off = aMax * (x3 ? 2 : 1);
  p.total = p.K[0] / 32 * kRowsTc * 128;
  for (int l = 0; l < a.layers; ++l) {
    off = (off + 1023) & ~1023;
    p.bOff[l] = off;
    p.bBytes[l] = ((p.K[l] / 32 * p.Np[l] * 128) + 1023) & ~1023;
    off += p.bBytes[l] * (x3 ? 2 : 1);
    p.total += p.K[l] / 32 * p.Np[l] * 128;
    p.tcol[l] = col;
    col += x3 ? p.Np[l] : p.Np[l];
  }
  return off + 64 + 4 * kFcMaxL * 256 + 1024;  // + barriers/slot, biases, alignment slack
}

template <int NL, bool X3>
cudaError_t launchFusedT(const FcChainArgs& a, cudaStream_t s) {
  FusedPlan p;
  const int smemBytes = planFused(a, X3, p);
  CUtensorMap tIn{}, tw[3]{};
  if (!mapFc(&tIn, a.I, a.L[0].kred, a.batch, a.ldi, kRowsTc)) return cudaErrorInvalidValue;
  for (int l = 0; l < NL; ++l)
    if (!mapFc(&tw[l], a.L[l].W, a.L[l].kred, a.L[l].out, a.L[l].ldw, up16(a.L[l].out))) return cudaErrorInvalidValue;
  CUtensorMap to[3]{};
  for (int l = 0; l < NL; ++l)  // {N, rows} returns, box {32, 128}: the epilogue's swizzled tile
    if (p.tmaOut[l] && !mapFc(&to[l], a.L[l].O, a.L[l].out, a.batch, a.L[l].out, kRowsTc)) p.tmaOut[l] = 0;
  auto kern = tc_fc_fused_kernel<NL, X3>;
  cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kern), smemBytes);
  if (e != cudaSuccess) return e;
  kern<<<(a.batch + kRowsTc - 1) / kRowsTc, kThreadsFc, smemBytes, s>>>(tIn, tw[0], tw[1], tw[2], to[0], to[1],
                                                                        to[2], p);
  return cudaGetLastError();
}

}  // namespace

bool tcFcFusedSupported(const FcChainArgs& a, int math, const char** why) {
  auto no = [&](const char* m) {
    if (why) *why = m;
    return false;
  };
  if (math != kMathTf32 && math != kMath3xTf32) return no("fused tensor-core FC chain: tf32 or 3xtf32 only");
  if (a.layers < 1 || a.layers > kFcMaxL) return no("fused tensor-core FC chain: 1 to 3 layers");
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  int cols = 0;
  for (int l = 0; l < a.layers; ++l) {
    const FcLayer& L = a.L[l];
    if (L.kred % 32) return no("fused tensor-core FC chain: every reduction a multiple of 32");
    if (L.out > 256 || L.out < 1) return no("fused tensor-core FC chain: at most 256 outputs per layer");
    if (L.ldw % 4 || !al16(L.W)) return no("fused tensor-core FC chain: 16-byte weight rows");
    if (l + 1 < a.layers && a.L[l + 1].kred > up16(L.out)) return no("fused tensor-core FC chain: layer widths");
    if (L.out % 4 == 0 && !al16(L.O)) return no("fused tensor-core FC chain: 16-byte aligned outputs");
    cols += up16(L.out);
  }
  if (a.ldi % 4 || !al16(a.I)) return no("fused tensor-core FC chain: 16-byte input rows");
  if (cols > 256) return no("fused tensor-core FC chain: TMEM columns");
  FusedPlan p;
  if (planFused(a, math == kMath3xTf32, p) > 227 * 1024) return no("fused tensor-core FC chain: shared memory");
  if (!sm100::encodeFn()) return no("fused tensor-core FC chain: no tensor-map encoder");
  return true;
}

cudaError_t launchTcFcFused(const FcChainArgs& a, int math, cudaStream_t s) {
  if (a.batch <= 0) return cudaSuccess;
  if (!tcFcFusedSupported(a, math, nullptr)) return cudaErrorInvalidValue;
  const bool x3 = math == kMath3xTf32;
  switch (a.layers) {
    case 1: return x3 ? launchFusedT<1, true>(a, s) : launchFusedT<1, false>(a, s);
    case 2: return x3 ? launchFusedT<2, true>(a, s) : launchFusedT<2, false>(a, s);
    default: return x3 ? launchFusedT<3, true>(a, s) : launchFusedT<3, false>(a, s);
  }
}

}  // namespace k
}  // namespace tcb
