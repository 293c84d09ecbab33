// fc_chain.cu — chains of FC+bias+ReLU layers in ONE kernel, split across a
// thread-block cluster:
//   MLP1     proj/kernels/mlp1.tc:2-6        (1 layer)
//   2FCRelu  paper_1802_04730_b200/tc/ops.tc (2 layers)
//   MLP3     proj/kernels/mlp3.tc:4-16       (3 layers; the paper's single-
//            kernel claim)
//
// A cluster of CN CTAs owns R batch rows. Layer l's output features are
// split across the cluster (CTA c owns columns [c*cols_l, (c+1)*cols_l)),
// so each CTA streams only its slice of every weight matrix. At kernel
// start one warp issues EVERY bulk async copy the CTA will need — one
// cp.async.bulk per row: the R input rows and the weight-slice rows of all
// layers, completing on mbarriers (one per first-layer operand row, so a
// thread starts its chain as soon as its two rows landed; one per later
// layer). After a layer, each CTA publishes its output slice in shared
// memory, the cluster synchronises, and every CTA gathers the full next-
// layer input from its peers over DSMEM (mapa + ld.shared::cluster): the
// activations never touch HBM except as the layer's own return tensor.
//
// Exactness: each (row, column) output is one thread's sequential FFMA
// chain in ascending k from bias[o], then fmaxf(·, 0) — the interpreter's
// order (interpreter.cc:218-233; builtin fmaxf → std::fmax, :22-24).
#include <cstdio>

#include "kernels.cuh"

namespace tcb {
namespace k {

namespace {


struct FcPlan {
  int cn, R;
  int cols[kMaxLayers];      // columns per CTA
  int wld[kMaxLayers];       // padded row stride of the weight slice (floats)
  int ald[kMaxLayers + 1];   // padded row stride of layer l's input activations
  int offW[kMaxLayers];      // smem float offsets
  int offAct, offSlice0, offSlice1, offBar;
  int kc, nchunk0;           // (unused: first layer loads one copy per row)
  int bulk;                  // 1: cp.async.bulk path, 0: cooperative loads
};

__host__ __device__ inline int up4(int x) { return (x + 3) & ~3; }
// row stride ≡ 4 (mod 32) floats: float4 reads of 8 consecutive rows hit 8
// distinct 16-byte bank groups
__host__ __device__ inline int padRow(int k) {
  int l = up4(k);
  while (l % 32 != 4) l += 4;
  return l;
}

__device__ __forceinline__ unsigned smemAddr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbarInit(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smemAddr(bar)), "r"(count));
}
__device__ __forceinline__ void mbarExpectTx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smemAddr(bar)), "r"(bytes)
               : "memory");
}
// Waits for the barrier phase; traps (a launch error the host reports as
// ErrorKind::Cuda) instead of hanging if the phase never completes.
__device__ __forceinline__ void mbarWait(uint64_t* bar, unsigned parity, int tag = -1) {
  const unsigned addr = smemAddr(bar);
  for (unsigned spin = 0;; ++spin) {
    unsigned done;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
    if (spin > (1u << 22)) {
      if ((threadIdx.x & 31) == 0)
        printf("tc-b200: mbarrier %d never completed (block %d,%d thread %d)\n", tag, blockIdx.x, blockIdx.y,
               threadIdx.x);
      __trap();
    }
  }
}
__device__ __forceinline__ void bulkCopy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smemAddr(dst)),
      "l"(src), "r"(bytes), "r"(smemAddr(bar))
      : "memory");
}
// Non-.aligned form: callers may reach it with a warp that diverged in an
// mbarrier spin (lanes waiting on different barriers); we also __syncwarp().
__device__ __forceinline__ void clusterSync() {
  __syncwarp();
  asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;\n" ::: "memory");
}
__device__ __forceinline__ unsigned clusterRank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ float ldCluster(const float* local, unsigned rank) {
  unsigned remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smemAddr(local)), "r"(rank));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
  return v;
}

__device__ __forceinline__ float4 lds4(unsigned addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ float lds1(unsigned addr) {
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

// acc = chain over k in [k0, k1) of act[k] * w[k]; operands addressed as
// 32-bit shared-window byte addresses. Three register sets rotate by code
// position (no moves): the loads of 4-k group g+2 are in flight while the
// dependent FFMAs of group g run.
__device__ __forceinline__ float chainSegment(unsigned xa, unsigned wa, int k0, int k1, float acc) {
  const int ng = (k1 - k0) >> 2;
  const unsigned x0 = xa + k0 * 4, w0 = wa + k0 * 4;
  float4 xA, wA, xB, wB, xC, wC;
  if (ng > 0) {
    xA = lds4(x0);
    wA = lds4(w0);
  }
  if (ng > 1) {
    xB = lds4(x0 + 16);
    wB = lds4(w0 + 16);
  }
  int g = 0;
  for (; g + 3 <= ng; g += 3) {
    const unsigned o = g * 16;
    xC = lds4(x0 + o + 32);
    wC = lds4(w0 + o + 32);
    acc = fma4(xA, wA, acc);
    if (g + 3 < ng) {
      xA = lds4(x0 + o + 48);
      wA = lds4(w0 + o + 48);
    }
    acc = fma4(xB, wB, acc);
    if (g + 4 < ng) {
      xB = lds4(x0 + o + 64);
      wB = lds4(w0 + o + 64);
    }
    acc = fma4(xC, wC, acc);
  }
  if (g < ng) acc = fma4(xA, wA, acc);
  if (g + 1 < ng) acc = fma4(xB, wB, acc);
  for (int kk = k0 + 4 * ng; kk < k1; ++kk) acc = __fmaf_rn(lds1(xa + kk * 4), lds1(wa + kk * 4), acc);
  return acc;
}

__global__ void fc_cluster_kernel(const FcChainArgs a, const FcPlan p) {
  extern __shared__ __align__(128) float sm[];
  const int tid = threadIdx.x, T = blockDim.x, R = p.R;
  const int rank = p.cn > 1 ? static_cast<int>(clusterRank()) : 0;
  const int row0 = blockIdx.y * R;
  const int rows = min(R, a.batch - row0);
  float* act = sm + p.offAct;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + p.offBar);  // [nchunk0 + layers]
  const int nbar = R + p.cols[0] + a.layers;

  // ---- issue every load of the kernel up front: one bulk copy per operand
  // row (layer-0 activation rows and weight rows each complete on their own
  // mbarrier; each later layer's weight slice on one barrier)
  uint64_t* rowBar = bars;                 // [R]
  uint64_t* wBar0 = bars + R;              // [cols0]
  uint64_t* layerBar = bars + R + p.cols[0];  // [layers] (slot 0 unused)
  if (p.bulk) {
    if (tid == 0) {
      for (int b = 0; b < nbar; ++b) mbarInit(&bars[b], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid < 32) {
      const int lane = tid;
      const int kb0 = a.L[0].kred * 4;
      const int c00 = rank * p.cols[0], nc0 = max(0, min(p.cols[0], a.L[0].out - c00));
      // expected bytes first (one lane per barrier), then the copies
      for (int r = lane; r < R; r += 32) mbarExpectTx(&rowBar[r], r < rows ? kb0 : 0);
      for (int j = lane; j < p.cols[0]; j += 32) mbarExpectTx(&wBar0[j], j < nc0 ? kb0 : 0);
      for (int l = lane; l < a.layers; l += 32) {
        int nc = l == 0 ? 0 : max(0, min(p.cols[l], a.L[l].out - rank * p.cols[l]));
        mbarExpectTx(&layerBar[l], (unsigned)(a.L[l].kred * 4 * nc));
      }
      __syncwarp();
      for (int r = lane; r < rows; r += 32)
        bulkCopy(act + r * p.ald[0], a.I + (int64_t)(row0 + r) * a.ldi, kb0, &rowBar[r]);
      for (int j = lane; j < nc0; j += 32)
        bulkCopy(sm + p.offW[0] + j * p.wld[0], a.L[0].W + (int64_t)(c00 + j) * a.L[0].ldw, kb0, &wBar0[j]);
      for (int l = 1; l < a.layers; ++l) {
        const int c0 = rank * p.cols[l], nc = max(0, min(p.cols[l], a.L[l].out - c0));
        for (int j = lane; j < nc; j += 32)
          bulkCopy(sm + p.offW[l] + j * p.wld[l], a.L[l].W + (int64_t)(c0 + j) * a.L[l].ldw,
                   a.L[l].kred * 4, &layerBar[l]);
      }
    }
    // rows past the batch end are zero
    for (int e = tid; e < (R - rows) * p.ald[0]; e += T) act[rows * p.ald[0] + e] = 0.0f;
    __syncthreads();
  } else {
    for (int e = tid; e < R * p.ald[0]; e += T) {
      int r = e / p.ald[0], kk = e % p.ald[0];
      act[e] = (r < rows && kk < a.L[0].kred) ? a.I[(int64_t)(row0 + r) * a.ldi + kk] : 0.0f;
    }
    for (int l = 0; l < a.layers; ++l) {
      const int c0 = rank * p.cols[l];
      for (int e = tid; e < p.cols[l] * a.L[l].kred; e += T) {
        int j = e / a.L[l].kred, kk = e % a.L[l].kred;
        sm[p.offW[l] + j * p.wld[l] + kk] =
            (c0 + j < a.L[l].out) ? a.L[l].W[(int64_t)(c0 + j) * a.L[l].ldw + kk] : 0.0f;
      }
    }
    __syncthreads();
  }

#pragma unroll 1
  for (int l = 0; l < a.layers; ++l) {
    const FcLayer L = a.L[l];
    const int cols = p.cols[l], c0 = rank * cols;
    const float* W = sm + p.offW[l];
    const int wld = p.wld[l], ald = p.ald[l];
    float* slice = sm + ((l & 1) ? p.offSlice1 : p.offSlice0);  // [R][cols]
    const unsigned actBase = smemAddr(act), wBase = smemAddr(W);
    const int nchains = R * cols;
    for (int base = 0; base < nchains; base += T) {
      // one (row, column) chain per thread and pass; idle lanes run a dummy
      // chain on row 0 / column 0 (no branches inside the reduction)
      const int idx = base + tid;
      const bool live = idx < nchains && c0 + idx / R < L.out;
      const int r = live ? idx % R : 0, c = live ? idx / R : 0;
      const unsigned xa = actBase + (unsigned)(r * ald) * 4u, wa = wBase + (unsigned)(c * wld) * 4u;
      float acc = live ? __ldg(L.bias + c0 + c) : 0.0f;
      if (p.bulk) {
        if (l == 0) {  // lanes wait on different barriers: reconverge after
          mbarWait(&rowBar[r], 0, r);
          mbarWait(&wBar0[c], 0, 100 + c);
        } else {
          mbarWait(&layerBar[l], 0, 1000 + l);
        }
        __syncwarp();
      }
      acc = chainSegment(xa, wa, 0, L.kred, acc);
      if (live) {
        float v = fmaxf(acc, 0.0f);
        slice[r * cols + c] = v;
        if (r < rows) L.O[(int64_t)(row0 + r) * L.out + c0 + c] = v;
      }
    }
    if (l + 1 < a.layers) {
      // publish the slice to the cluster, then gather the next layer's input
      if (p.cn > 1) clusterSync();
      else __syncthreads();
      const int ldn = p.ald[l + 1];
      for (int e = tid; e < R * L.out; e += T) {
        int r = e / L.out, col = e % L.out;
        int owner = col / cols, c = col % cols;
        const float* src = slice + r * cols + c;
        act[r * ldn + col] = p.cn > 1 ? ldCluster(src, owner) : *src;
      }
      __syncthreads();
    }
  }
  // keep this CTA's shared memory alive until every peer finished its DSMEM reads
  if (p.cn > 1 && a.layers > 1) clusterSync();
}

}  // namespace

// Builds the plan; returns the dynamic shared-memory size (0 if infeasible).
static size_t planFc(const FcChainArgs& a, int R, int cn, FcPlan& p) {
  p = FcPlan{};
  p.cn = cn;
  p.R = R;
  int off = 0;
  for (int l = 0; l < a.layers; ++l) {
    p.cols[l] = (a.L[l].out + cn - 1) / cn;
    p.wld[l] = padRow(a.L[l].kred);
    p.offW[l] = off;
    off += p.cols[l] * p.wld[l];
  }
  int aldMax = 0;
  p.ald[0] = padRow(a.L[0].kred);
  for (int l = 1; l < a.layers; ++l) p.ald[l] = padRow(a.L[l].kred);
  for (int l = 0; l < a.layers; ++l) aldMax = p.ald[l] > aldMax ? p.ald[l] : aldMax;
  p.offAct = off;
  off += R * aldMax;
  int sliceMax = 0;
  for (int l = 0; l < a.layers; ++l) sliceMax = R * p.cols[l] > sliceMax ? R * p.cols[l] : sliceMax;
  p.offSlice0 = off;
  off += sliceMax;
  p.offSlice1 = off;
  off += sliceMax;
  off = (off + 3) & ~3;  // 16-byte alignment for the mbarriers
  p.offBar = off;
  p.kc = a.L[0].kred;
  p.nchunk0 = 1;
  off += 2 * (R + p.cols[0] + a.layers);  // uint64 barriers: act rows, weight rows, layers
  bool bulk = (a.ldi % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.I) & 15) == 0);
  for (int l = 0; l < a.layers; ++l)
    bulk = bulk && (a.L[l].kred % 4 == 0) && (a.L[l].ldw % 4 == 0) &&
           ((reinterpret_cast<uintptr_t>(a.L[l].W) & 15) == 0);
  p.bulk = bulk ? 1 : 0;
  return (size_t)off * sizeof(float);
}

size_t fcChainSmem(const FcChainArgs& a, int rows, int cn) {
  FcPlan p;
  return planFc(a, rows, cn, p);
}

int fcChainThreads(const FcChainArgs& a, int rows, int cn) {
  int need = 0;
  for (int l = 0; l < a.layers; ++l) {
    int cols = (a.L[l].out + cn - 1) / cn;
    need = cols * rows > need ? cols * rows : need;
  }
  // block size that runs every layer in one pass (any multiple of 32 works;
  // smaller blocks take several passes)
  int t = ((need + 31) / 32) * 32;
  return t > 1024 ? 1024 : t;
}

cudaError_t launchFcChain(const FcChainArgs& a, int rows, int cn, int threads, cudaStream_t s) {
  if (a.batch <= 0) return cudaSuccess;
  FcPlan p;
  size_t smem = planFc(a, rows, cn, p);
  if (smem > 227 * 1024 || cn < 1 || cn > 16 || rows < 1) return cudaErrorInvalidConfiguration;
  if (threads < 32 || threads > 1024 || threads % 32) return cudaErrorInvalidConfiguration;
  cudaFuncSetAttribute(fc_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cn > 8) cudaFuncSetAttribute(fc_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cn, (a.batch + rows - 1) / rows, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cn;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fc_cluster_kernel, a, p);
}

}  // namespace k
}  // namespace tcb
