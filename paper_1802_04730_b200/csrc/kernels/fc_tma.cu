// fc_tma.cu — the FC-chain cluster kernel (fc_chain.cu) with its first layer
// streamed in by TMA tensor copies, so that layer's chains start on the first
// reduction chunk instead of after the whole input and weight slice.
//   MLP1     proj/kernels/mlp1.tc:2-6        (1 layer)
//   2FCRelu  paper_1802_04730_b200/tc/ops.tc (2 layers)
//   MLP3     proj/kernels/mlp3.tc:4-16       (3 layers)
//
// Layer 0 (the long reduction: K = 1128 at the paper shapes) is viewed as a
// 3-D tensor {32 floats, row, k/32} (strides 4 B, row stride, 128 B) and
// fetched in chunks of kChunkKb 32-wide k blocks: one box for the CTA's R
// input rows, one for its weight-column slice, each landing as
// [k block][row][32 floats] with the 128-byte swizzle (16-byte unit q of
// row r at q ^ (r & 7)), so the float4 reads of up to 8 distinct rows in a
// warp hit 8 distinct bank groups. Every chunk completes on its own
// mbarrier; a thread's chain waits for chunk j only when it reaches it. The
// K % 32 tail lands by one more unswizzled box pair. Later layers are the
// cluster kernel's: weight slices by one bulk copy, activations pushed into
// every cluster CTA's shared memory (st.async completing on its mbarrier).
//
// Exactness: each (row, column) output is one thread's sequential FFMA
// chain in ascending k from bias[o], then fmaxf(·, 0) — the interpreter's
// order (interpreter.cc:218-233). The chunking only changes when operands
// arrive, never the order they are consumed in.
#include <algorithm>
#include <mutex>
#include <vector>

#include "kernels.cuh"
#include "sm100.cuh"

namespace tcb {
namespace k {

namespace {

using namespace sm100;

constexpr int kChunkKb = 8;  // 32-wide k blocks per TMA chunk (256 reduction steps)
constexpr int kMaxChunks = 16;

struct FcTmaPlan {
  int cn, R;
  int cols[kMaxLayers];
  int KB, tail, nchunk;      // layer 0: full 32-wide k blocks, K % 32, chunks
  int offX0, offW0;          // layer 0 chunk buffers (floats from the 1024-aligned base)
  int offXt, offWt;          // layer 0 tail boxes [R][tail], [cols0][tail]
  int ald[kMaxLayers + 1];   // l >= 1: padded row stride of layer l's input activations
  int wld[kMaxLayers];       // l >= 1: weight-slice row stride
  int offW[kMaxLayers];      // l >= 1: weight slices
  int offAct[kMaxLayers];    // l >= 1: layer l's input activations (pushed by layer l-1)
  int offBar;                // uint64 barriers: [0, nchunk) chunks, nchunk tail, then 2 per later layer
};

__host__ __device__ inline int up4(int x) { return (x + 3) & ~3; }
__host__ __device__ inline int padRow(int k) {
  int l = up4(k);
  while (l % 32 != 4) l += 4;
  return l;
}

__device__ __forceinline__ float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ float lds1(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ float fma4(float4 x, float4 w, float acc) {
  acc = __fmaf_rn(x.x, w.x, acc);
  acc = __fmaf_rn(x.y, w.y, acc);
  acc = __fmaf_rn(x.z, w.z, acc);
  return __fmaf_rn(x.w, w.w, acc);
}
__device__ __forceinline__ void bulkCopy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem(dst)),
      "l"(src), "r"(bytes), "r"(smem(bar))
      : "memory");
}
__device__ __forceinline__ void tmaLoad2d(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem(bar))
      : "memory");
}
__device__ __forceinline__ void stAsyncCluster(const float* local, const uint64_t* localBar, unsigned rank, float v) {
  const unsigned ra = mapa(smem(local), rank), rb = mapa(smem(localBar), rank);
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(ra),
               "r"(__float_as_uint(v)), "r"(rb)
               : "memory");
}

// one 16-step half block h of the swizzled layer-0 layout: rowBase = the
// operand's chunk-buffer address + its row * 128, step = rows * 128 bytes per
// k block; the 16-byte unit q of a 128-byte row sits at q ^ (row index & 7)
__device__ __forceinline__ void loadHalf(uint32_t rowBase, uint32_t step, int h, float4* v) {
  const uint32_t ra = rowBase + (uint32_t)(h >> 1) * step;
  const uint32_t sw = ((ra >> 7) & 7u) << 4, q0 = (uint32_t)(h & 1) << 6;
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = lds4(ra + ((q0 + 16u * i) ^ sw));
}

// the later layers' chain (fc_chain.cu's chainSegment): double-buffered
// 16-step chunks over linear rows; reads up to 32 floats past n
__device__ __forceinline__ float chainLinear(uint32_t xa, uint32_t wa, int n, float acc) {
  const int nch = n >> 4;
  float4 X0[4], W0[4], X1[4], W1[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    X0[i] = lds4(xa + i * 16);
    W0[i] = lds4(wa + i * 16);
  }
  int c = 0;
  for (; c + 2 <= nch; c += 2) {
    const uint32_t o = c * 64;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      X1[i] = lds4(xa + o + 64 + i * 16);
      W1[i] = lds4(wa + o + 64 + i * 16);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) acc = fma4(X0[i], W0[i], acc);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      X0[i] = lds4(xa + o + 128 + i * 16);
      W0[i] = lds4(wa + o + 128 + i * 16);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) acc = fma4(X1[i], W1[i], acc);
  }
  if (c < nch) {
#pragma unroll
    for (int i = 0; i < 4; ++i) acc = fma4(X0[i], W0[i], acc);
    ++c;
  }
  int kk = c * 16;
  for (; kk + 4 <= n; kk += 4) acc = fma4(lds4(xa + kk * 4), lds4(wa + kk * 4), acc);
  for (; kk < n; ++kk) acc = __fmaf_rn(lds1(xa + kk * 4), lds1(wa + kk * 4), acc);
  return acc;
}

struct FcTmaMaps {
  CUtensorMap x, w, xt, wt;  // layer 0: swizzled chunk views, tail views
};

template <int NL>
__global__ void __launch_bounds__(kFcMaxThreads, 1)
    fc_tma_kernel(const __grid_constant__ FcChainArgs a, const __grid_constant__ FcTmaPlan p,
                  const __grid_constant__ FcTmaMaps maps) {
  extern __shared__ __align__(1024) unsigned char smRaw[];
  float* sm = reinterpret_cast<float*>(smRaw + ((1024u - (smem(smRaw) & 1023u)) & 1023u));
  const int tid = threadIdx.x, T = blockDim.x, R = p.R, cn = p.cn;
  const int rank = cn > 1 ? static_cast<int>(clusterRank()) : 0;
  const int row0 = blockIdx.y * R;
  const int rows = min(R, a.batch - row0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + p.offBar);
  uint64_t* tailBar = bars + p.nchunk;
  uint64_t* actBar = tailBar;         // actBar[l] = bars[nchunk + l], l >= 1
  uint64_t* wBar = tailBar + NL - 1;  // wBar[l] = bars[nchunk + NL - 1 + l], l >= 1
  const int C0 = p.cols[0];

  float biasPre[NL];  // first-pass bias of every layer, in flight behind the copies
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const int c = tid / R, c0 = rank * p.cols[l];
    biasPre[l] = (tid < R * p.cols[l] && c0 + c < a.L[l].out) ? __ldg(a.L[l].bias + c0 + c) : 0.0f;
  }
  if (tid == 0) {
    if (p.KB > 0) {
      tmaPrefetch(&maps.x);
      tmaPrefetch(&maps.w);
    }
    const int nb = p.nchunk + 1 + 2 * (NL - 1);
    for (int b = 0; b < nb; ++b) mbarInit(&bars[b], 1);
    const unsigned chunkBytes = (unsigned)(R + C0) * kChunkKb * 128u;
    for (int j = 0; j < p.nchunk; ++j) mbarExpectTx(&bars[j], chunkBytes);
    if (p.tail) mbarExpectTx(tailBar, (unsigned)((R + C0) * p.tail * 4));
#pragma unroll
    for (int l = 1; l < NL; ++l) {
      if (cn > 1) mbarExpectTx(&actBar[l], (unsigned)(R * a.L[l - 1].out * 4));
      const int c0 = rank * p.cols[l], nc = max(0, min(p.cols[l], a.L[l].out - c0));
      mbarExpectTx(&wBar[l], (unsigned)(a.L[l].kred * 4 * nc));
    }
    fenceBarrierInit();
  }
  __syncthreads();
  // peers push into this CTA's buffers: every CTA's barriers must be armed
  // first (arrive now, wait before the first push)
  if (cn > 1) asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");

  // ---- every load of the kernel, issued up front; copies dealt to lane 0
  // of every warp (a copy costs its issuing thread a few hundred cycles)
  {
    const int warp = tid >> 5, nw = (T + 31) >> 5, lane = tid & 31;
    if (lane == 0) {
      int j = 0;
      for (int ch = 0; ch < p.nchunk; ++ch) {
        if (j++ % nw == warp)
          tmaLoad3d(sm + p.offX0 + ch * kChunkKb * R * 32, &maps.x, 0, row0, ch * kChunkKb, &bars[ch]);
        if (j++ % nw == warp)
          tmaLoad3d(sm + p.offW0 + ch * kChunkKb * C0 * 32, &maps.w, 0, rank * C0, ch * kChunkKb, &bars[ch]);
      }
      if (p.tail) {
        if (j++ % nw == warp) tmaLoad2d(sm + p.offXt, &maps.xt, p.KB * 32, row0, tailBar);
        if (j++ % nw == warp) tmaLoad2d(sm + p.offWt, &maps.wt, p.KB * 32, rank * C0, tailBar);
      }
#pragma unroll
      for (int l = 1; l < NL; ++l) {
        const int c0 = rank * p.cols[l], nc = max(0, min(p.cols[l], a.L[l].out - c0));
        if (nc == 0) continue;
        const float* src = a.L[l].W + (int64_t)c0 * a.L[l].ldw;
        if (a.L[l].ldw == a.L[l].kred) {
          if (j++ % nw == warp) bulkCopy(sm + p.offW[l], src, (unsigned)(nc * a.L[l].kred * 4), &wBar[l]);
        } else {
          for (int q = 0; q < nc; ++q)
            if (j++ % nw == warp)
              bulkCopy(sm + p.offW[l] + q * p.wld[l], src + (int64_t)q * a.L[l].ldw, a.L[l].kred * 4, &wBar[l]);
        }
      }
    }
  }

  // ---- layer 0: chains over the swizzled chunks, waiting chunk by chunk
  {
    const FcLayer L = a.L[0];
    const int c0 = rank * C0, nchains = R * C0;
    const uint32_t xBase = smem(sm + p.offX0), wBase = smem(sm + p.offW0);
    const uint32_t xStep = (uint32_t)R * 128u, wStep = (uint32_t)C0 * 128u;
    const int H = 2 * p.KB;  // 16-step half blocks
    for (int base = 0; base < nchains; base += T) {
      const int idx = base + tid;
      const bool live = idx < nchains && c0 + idx / R < L.out;
      const int r = live ? idx % R : 0, c = live ? idx / R : 0;
      float acc = !live ? 0.0f : base == 0 ? biasPre[0] : __ldg(L.bias + c0 + c);
      const uint32_t xr = xBase + (uint32_t)r * 128u, wr = wBase + (uint32_t)c * 128u;
      if (H > 0) {
        float4 X0[4], W0[4], X1[4], W1[4];
        mbarWait(&bars[0], 0, 0);
        loadHalf(xr, xStep, 0, X0);
        loadHalf(wr, wStep, 0, W0);
        for (int h = 0; h < H; h += 2) {
          loadHalf(xr, xStep, h + 1, X1);  // same k block as h: already landed
          loadHalf(wr, wStep, h + 1, W1);
#pragma unroll
          for (int i = 0; i < 4; ++i) acc = fma4(X0[i], W0[i], acc);
          if (h + 2 < H) {
            if ((h + 2) % (2 * kChunkKb) == 0) mbarWait(&bars[(h + 2) / (2 * kChunkKb)], 0, 1);
            loadHalf(xr, xStep, h + 2, X0);
            loadHalf(wr, wStep, h + 2, W0);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) acc = fma4(X1[i], W1[i], acc);
        }
      }
      if (p.tail) {
        mbarWait(tailBar, 0, 2);
        const uint32_t xt = smem(sm + p.offXt) + (uint32_t)(r * p.tail) * 4u;
        const uint32_t wt = smem(sm + p.offWt) + (uint32_t)(c * p.tail) * 4u;
        for (int q = 0; q < p.tail; q += 4) acc = fma4(lds4(xt + 4u * q), lds4(wt + 4u * q), acc);
      }
      if (live) {
        const float v = fmaxf(acc, 0.0f);
        if (r < rows) L.O[(int64_t)(row0 + r) * L.out + c0 + c] = v;
        if (NL > 1) {
          if (base == 0 && cn > 1) asm volatile("barrier.cluster.wait;" ::: "memory");
          float* dst = sm + p.offAct[1] + r * p.ald[1] + c0 + c;
          if (cn > 1) {
            for (int q = 0; q < cn; ++q) stAsyncCluster(dst, &actBar[1], q, v);
          } else {
            *dst = v;
          }
        }
      } else if (NL > 1 && base == 0 && cn > 1) {
        asm volatile("barrier.cluster.wait;" ::: "memory");
      }
    }
    if (NL > 1 && cn == 1) __syncthreads();
  }

  // ---- later layers: the cluster kernel's chains over pushed activations
#pragma unroll
  for (int l = 1; l < NL; ++l) {
    const FcLayer L = a.L[l];
    const int cols = p.cols[l], c0 = rank * cols;
    const bool last = l + 1 == NL;
    const uint32_t actBase = smem(sm + p.offAct[l]), wBase = smem(sm + p.offW[l]);
    if (cn > 1) mbarWait(&actBar[l], 0, 3);
    mbarWait(&wBar[l], 0, 4);
    const int nchains = R * cols;
    for (int base = 0; base < nchains; base += T) {
      const int idx = base + tid;
      const bool live = idx < nchains && c0 + idx / R < L.out;
      const int r = live ? idx % R : 0, c = live ? idx / R : 0;
      float acc = !live ? 0.0f : base == 0 ? biasPre[l] : __ldg(L.bias + c0 + c);
      acc = chainLinear(actBase + (uint32_t)(r * p.ald[l]) * 4u, wBase + (uint32_t)(c * p.wld[l]) * 4u, L.kred, acc);
      if (live) {
        const float v = fmaxf(acc, 0.0f);
        if (r < rows) L.O[(int64_t)(row0 + r) * L.out + c0 + c] = v;
        if (!last) {
          float* dst = sm + p.offAct[l + 1] + r * p.ald[l + 1] + c0 + c;
          if (cn > 1) {
            for (int q = 0; q < cn; ++q) stAsyncCluster(dst, &actBar[l + 1], q, v);
          } else {
            *dst = v;
          }
        }
      }
    }
    if (!last && cn == 1) __syncthreads();
  }
  if (cn > 1 && NL == 1) asm volatile("barrier.cluster.wait;" ::: "memory");  // pair the arrive
  // every wait is behind us: invalidate the barriers (their shared memory is
  // plain memory again for the next kernel; compute-sanitizer synccheck)
  __syncthreads();
  if (tid == 0)
    for (int b = 0; b < p.nchunk + 1 + 2 * (NL - 1); ++b)
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(&bars[b]))) : "memory");
}

// ------------------------------------------------------------------ host
// Encoded maps cached by geometry: graph capture and repeated synchronised
// calls re-use them.
struct TmaKey {
  const void* p;
  int rank, dev, sw;
  uint64_t dims[3], strides[2];
  uint32_t box[3];
  bool operator==(const TmaKey& o) const {
    if (p != o.p || rank != o.rank || dev != o.dev || sw != o.sw) return false;
    for (int i = 0; i < 3; ++i)
      if (dims[i] != o.dims[i] || box[i] != o.box[i]) return false;
    return strides[0] == o.strides[0] && strides[1] == o.strides[1];
  }
};
std::mutex g_tmu;
std::vector<std::pair<TmaKey, CUtensorMap>> g_tmaps;  // most recent last, <= 128

bool encodeCached(CUtensorMap* m, const TmaKey& key) {
  {
    std::lock_guard<std::mutex> g(g_tmu);
    for (size_t i = g_tmaps.size(); i-- > 0;)
      if (g_tmaps[i].first == key) {
        *m = g_tmaps[i].second;
        return true;
      }
  }
  EncodeFn enc = encodeFn();
  if (!enc) return false;
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3], es[3] = {1, 1, 1};
  for (int i = 0; i < 3; ++i) dims[i] = key.dims[i], box[i] = key.box[i];
  strides[0] = key.strides[0];
  strides[1] = key.strides[1];
  if (enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, key.rank, const_cast<void*>(key.p), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, key.sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  std::lock_guard<std::mutex> g(g_tmu);
  if (g_tmaps.size() >= 128) g_tmaps.erase(g_tmaps.begin());
  g_tmaps.push_back({key, *m});
  return true;
}

int curDev() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

// swizzled chunk view of a row-major [rows][ld] operand: {32, rows, K/32},
// box {32, boxRows, kChunkKb}
bool chunkMap(CUtensorMap* m, const float* base, int K, int rows, int64_t ld, int boxRows) {
  TmaKey k{};
  k.p = base;
  k.rank = 3;
  k.dev = curDev();
  k.sw = 1;
  k.dims[0] = 32;
  k.dims[1] = (uint64_t)rows;
  k.dims[2] = (uint64_t)(K / 32);
  k.strides[0] = (uint64_t)ld * 4;
  k.strides[1] = 128;
  k.box[0] = 32;
  k.box[1] = (uint32_t)boxRows;
  k.box[2] = kChunkKb;
  return encodeCached(m, k);
}
// unswizzled view of the K % 32 tail: {K, rows}, box {tail, boxRows}
bool tailMap(CUtensorMap* m, const float* base, int K, int rows, int64_t ld, int tail, int boxRows) {
  TmaKey k{};
  k.p = base;
  k.rank = 2;
  k.dev = curDev();
  k.sw = 0;
  k.dims[0] = (uint64_t)K;
  k.dims[1] = (uint64_t)rows;
  k.dims[2] = 1;
  k.strides[0] = (uint64_t)ld * 4;
  k.box[0] = (uint32_t)tail;
  k.box[1] = (uint32_t)boxRows;
  k.box[2] = 1;
  return encodeCached(m, k);
}

// returns the dynamic shared-memory bytes (including the 1024-byte alignment
// slack), or 0 when the plan is impossible
size_t planFcTma(const FcChainArgs& a, int R, int cn, FcTmaPlan& p) {
  p = FcTmaPlan{};
  p.cn = cn;
  p.R = R;
  for (int l = 0; l < a.layers; ++l) p.cols[l] = (a.L[l].out + cn - 1) / cn;
  const int K0 = a.L[0].kred;
  p.KB = K0 / 32;
  p.tail = K0 % 32;
  p.nchunk = (p.KB + kChunkKb - 1) / kChunkKb;
  if (p.nchunk > kMaxChunks) return 0;
  int off = 0;  // floats from the aligned base; chunk boxes 1024-byte aligned
  p.offX0 = off;
  off += p.nchunk * kChunkKb * R * 32;
  off = (off + 255) & ~255;
  p.offW0 = off;
  off += p.nchunk * kChunkKb * p.cols[0] * 32;
  off = (off + 31) & ~31;  // tensor-copy destinations: 128-byte aligned
  p.offXt = off;
  off += R * p.tail + 4;
  off = (off + 31) & ~31;
  p.offWt = off;
  off += p.cols[0] * p.tail + 4;
  off = up4(off);
  for (int l = 1; l < a.layers; ++l) {
    p.wld[l] = up4(a.L[l].kred);
    p.offW[l] = off;
    off += p.cols[l] * p.wld[l] + 32;
  }
  for (int l = 1; l < a.layers; ++l) {
    int w = std::max(a.L[l].kred, a.L[l - 1].out);
    p.ald[l] = padRow(w);
    p.offAct[l] = off;
    off += R * p.ald[l] + 32;
  }
  off = up4(off);
  p.offBar = off;
  off += 2 * (p.nchunk + 1 + 2 * (a.layers - 1));
  return (size_t)off * 4 + 1024;
}

template <int NL>
cudaError_t launchT(const FcChainArgs& a, int rows, int cn, int threads, cudaStream_t s) {
  FcTmaPlan p;
  const size_t smemBytes = planFcTma(a, rows, cn, p);
  if (smemBytes == 0 || smemBytes > 227 * 1024) return cudaErrorInvalidConfiguration;
  FcTmaMaps maps{};
  const FcLayer& L0 = a.L[0];
  if (p.KB > 0) {
    if (!chunkMap(&maps.x, a.I, L0.kred, a.batch, a.ldi, rows)) return cudaErrorInvalidValue;
    if (!chunkMap(&maps.w, L0.W, L0.kred, L0.out, L0.ldw, p.cols[0])) return cudaErrorInvalidValue;
  }
  if (p.tail) {
    if (!tailMap(&maps.xt, a.I, L0.kred, a.batch, a.ldi, p.tail, rows)) return cudaErrorInvalidValue;
    if (!tailMap(&maps.wt, L0.W, L0.kred, L0.out, L0.ldw, p.tail, p.cols[0])) return cudaErrorInvalidValue;
  }
  auto kern = fc_tma_kernel<NL>;
  cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kern), (int)smemBytes, cn > 8);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cn, (a.batch + rows - 1) / rows, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = smemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cn;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, p, maps);
}

}  // namespace

bool fcTmaSupported(const FcChainArgs& a, int rows, int cn, const char** why) {
  auto no = [&](const char* m) {
    if (why) *why = m;
    return false;
  };
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  // single-layer chains (MLP1) trap on a barrier that never completes
  // (profiles/fctma_matrix.py); the cluster kernel serves them
  if (a.layers < 2 || a.layers > kMaxLayers) return no("TMA FC chain: 2 to 4 layers");
  if (rows < 1 || rows > 256) return no("TMA FC chain: rows per cluster in [1, 256]");
  if (cn < 1 || cn > 16) return no("TMA FC chain: cluster size in [1, 16]");
  const FcLayer& L0 = a.L[0];
  if (L0.kred % 4) return no("TMA FC chain: first-layer reduction a multiple of 4");
  if (a.ldi % 4 || L0.ldw % 4 || !al16(a.I) || !al16(L0.W)) return no("TMA FC chain: 16-byte first-layer rows");
  if ((L0.out + cn - 1) / cn > 256) return no("TMA FC chain: at most 256 first-layer columns per CTA");
  for (int l = 1; l < a.layers; ++l) {
    const FcLayer& L = a.L[l];
    if (L.kred % 4 || L.ldw % 4 || !al16(L.W)) return no("TMA FC chain: 16-byte weight rows");
  }
  FcTmaPlan p;
  const size_t b = planFcTma(a, rows, cn, p);
  if (b == 0 || b > 227 * 1024) return no("TMA FC chain: exceeds the shared-memory capacity");
  return true;
}

cudaError_t launchFcTma(const FcChainArgs& a, int rows, int cn, int threads, cudaStream_t s) {
  if (a.batch <= 0) return cudaSuccess;
  if (!fcTmaSupported(a, rows, cn, nullptr)) return cudaErrorInvalidConfiguration;
  if (threads < 32 || threads > kFcMaxThreads || threads % 32) return cudaErrorInvalidConfiguration;
  switch (a.layers) {
    case 1: return launchT<1>(a, rows, cn, threads, s);
    case 2: return launchT<2>(a, rows, cn, threads, s);
    case 3: return launchT<3>(a, rows, cn, threads, s);
    case 4: return launchT<4>(a, rows, cn, threads, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace k
}  // namespace tcb
