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
// start warp 0 issues EVERY bulk async copy the CTA will need
// (cp.async.bulk, global → shared, completing on mbarriers): the R input
// rows (padded rows, one copy each) and each layer's weight slice (one
// contiguous copy per layer). Each layer's output value is pushed straight
// into the next layer's input buffer of every CTA of the cluster (mapa +
// st.shared::cluster, double-buffered by layer parity), then one cluster
// barrier (release/acquire) per layer makes the pushes visible: the
// activations never touch HBM except as the layer's own return tensor, and
// no CTA ever waits on a remote load.
//
// Exactness: each (row, column) output is one thread's sequential FFMA
// chain in ascending k from bias[o], then fmaxf(·, 0) — the interpreter's
// order (interpreter.cc:218-233; builtin fmaxf → std::fmax, :22-24).
#include <algorithm>
#include <cstdio>

#include "kernels.cuh"

namespace tcb {
namespace k {

namespace {


struct FcPlan {
  int cn, R;
  int cols[kMaxLayers];     // output columns per CTA
  int ald[kMaxLayers + 1];  // padded row stride of layer l's input activations (floats)
  int wld[kMaxLayers];      // weight-slice row stride: kred rounded up to 4 (dense when kred%4==0)
  int offW[kMaxLayers];     // weight slices [cols][wld] (floats)
  int offAct[kMaxLayers];   // [0]: input rows; [l>0]: layer l-1's output = layer l's input
  int offBar;
  int denseIn;              // input rows land unpadded with one copy (ald[0] == kred, conflict-free)
  int bulk;                 // 1: cp.async.bulk path, 2: 16-byte cp.async path, 0: cooperative loads
  int nch, kc4;             // cp.async path: layer 0 in nch chunks of kc4 float4s of the reduction
  int pair;                 // 1: layer 0 runs two columns (c, c + cols/2) per thread, interleaved
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
    if (spin > (1u << 22)) __trap();  // never hang: the host reports the launch failure
  }
}
__device__ __forceinline__ void bulkCopy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smemAddr(dst)),
      "l"(src), "r"(bytes), "r"(smemAddr(bar))
      : "memory");
}
__device__ __forceinline__ void cpAsync16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smemAddr(dst)), "l"(src) : "memory");
}
template <int N>
__device__ __forceinline__ void cpAsyncWait() {
  if constexpr (N >= 0) asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ unsigned clusterRank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
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

// remote store that completes `bytes` on the destination CTA's mbarrier
// (st.async): the consumer waits on its own barrier, no cluster barrier
__device__ __forceinline__ void stAsyncCluster(const float* local, const uint64_t* localBar, unsigned rank, float v) {
  unsigned ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smemAddr(local)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smemAddr(localBar)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(ra),
               "r"(__float_as_uint(v)), "r"(rb)
               : "memory");
}


// acc = chain over k in [0, n) of x[k] * w[k]; operands addressed as 32-bit
// shared-window byte addresses. Double-buffered 16-wide chunks: the eight
// vector loads of chunk c+1 are issued before the 16 dependent FFMAs of
// chunk c, so shared-load latency hides behind a full chunk of the chain.
// Reads up to 32 floats past n (the plan leaves that slack after every
// operand buffer).
__device__ __noinline__ float chainSegment(unsigned xa, unsigned wa, int n, float acc) {
  const int nch = n >> 4;
  float4 X0[4], W0[4], X1[4], W1[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    X0[i] = lds4(xa + i * 16);
    W0[i] = lds4(wa + i * 16);
  }
  int c = 0;
  for (; c + 2 <= nch; c += 2) {
    const unsigned o = c * 64;
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

// Two chains of one input row against two weight columns, interleaved: per
// 4 steps one input vector load feeds 8 FFMAs (2 loads per 4 in
// chainSegment). The chains are LDS-writeback bound at one output per lane
// (~6.2 cycles per step with 4 warps per SM); 8-step chunks (16-step
// chunks as in chainSegment measured slower: 6.3 vs 5.9 cycles per step); half the lanes with two
// outputs each move a quarter fewer bytes through the register file per
// output. Same slack rules as chainSegment.
__device__ __noinline__ float2 chainSegment2(unsigned xa, unsigned wa, unsigned wb, int n, float accA, float accB) {
  const int nch = n >> 3;
  float4 X0[2], A0[2], B0[2], X1[2], A1[2], B1[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    X0[i] = lds4(xa + i * 16);
    A0[i] = lds4(wa + i * 16);
    B0[i] = lds4(wb + i * 16);
  }
  int c = 0;
  for (; c + 2 <= nch; c += 2) {
    const unsigned o = c * 32;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      X1[i] = lds4(xa + o + 32 + i * 16);
      A1[i] = lds4(wa + o + 32 + i * 16);
      B1[i] = lds4(wb + o + 32 + i * 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      accA = fma4(X0[i], A0[i], accA);
      accB = fma4(X0[i], B0[i], accB);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      X0[i] = lds4(xa + o + 64 + i * 16);
      A0[i] = lds4(wa + o + 64 + i * 16);
      B0[i] = lds4(wb + o + 64 + i * 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      accA = fma4(X1[i], A1[i], accA);
      accB = fma4(X1[i], B1[i], accB);
    }
  }
  if (c < nch) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      accA = fma4(X0[i], A0[i], accA);
      accB = fma4(X0[i], B0[i], accB);
    }
    ++c;
  }
  int kk = c * 8;
  for (; kk + 4 <= n; kk += 4) {
    const float4 x = lds4(xa + kk * 4);
    accA = fma4(x, lds4(wa + kk * 4), accA);
    accB = fma4(x, lds4(wb + kk * 4), accB);
  }
  for (; kk < n; ++kk) {
    const float x = lds1(xa + kk * 4);
    accA = __fmaf_rn(x, lds1(wa + kk * 4), accA);
    accB = __fmaf_rn(x, lds1(wb + kk * 4), accB);
  }
  return make_float2(accA, accB);
}

#ifdef TCB_FC_TRACE
// diagnostic build only (profiles/fc_trace.cu): per-CTA phase timestamps
__device__ unsigned long long g_fc_trace[1024][32];
#define FC_STAMP(ev)                                                                       \
  do {                                                                                     \
    if (threadIdx.x == 0) g_fc_trace[blockIdx.y * gridDim.x + blockIdx.x][ev] = clock64(); \
  } while (0)
#define FC_GSTAMP(ev)                                                                  \
  do {                                                                                 \
    unsigned long long t_;                                                             \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
    if (threadIdx.x == 0) g_fc_trace[blockIdx.y * gridDim.x + blockIdx.x][ev] = t_;    \
  } while (0)
#else
#define FC_STAMP(ev) \
  do {               \
  } while (0)
#define FC_GSTAMP(ev) \
  do {                \
  } while (0)
#endif

// __grid_constant__: the layer loop indexes a.L[l] / p.*[l] dynamically;
// without it those reads go through a local-memory copy of the parameters
// NL = a.layers: every layer loop unrolls with static indices, so the
// parameter reads are constant-bank operands the compiler can hoist and
// overlap. (A runtime layer loop made each layer's reads dependent misses in
// the cold constant cache; MLP3 6.8 -> 5.3 µs, profiles/fc_trace.cu.)
// LM = p.bulk, the load mode, as a template parameter too: each instance
// holds only its own load path (the fused kernel is latency-bound and its
// instruction footprint showed up as ~half of all warp-stall samples,
// "no instruction", in ncu: profiles/r02_fc_icache.txt)
template <int NL, int LM>
__global__ void __launch_bounds__(kFcMaxThreads)
    fc_cluster_kernel(const __grid_constant__ FcChainArgs a, const __grid_constant__ FcPlan p) {
  FC_GSTAMP(13);
  FC_STAMP(0);
  extern __shared__ __align__(128) float sm[];
  const int tid = threadIdx.x, T = blockDim.x, R = p.R;
  const int cn = p.cn;
  constexpr int layers = NL;
  const int rank = cn > 1 ? static_cast<int>(clusterRank()) : 0;
  const int row0 = blockIdx.y * R;
  const int rows = min(R, a.batch - row0);
  // bars[l]: layer l's input activations landed; bars[layers + l]: layer l's weight slice landed
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + p.offBar);

  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < 2 * layers; ++b) mbarInit(&bars[b], 1);
    // the pushed activations of every later layer: R rows x all columns
    // (armed before any peer can push: see the cluster arrive below)
    if (cn > 1)
#pragma unroll
      for (int l = 1; l < layers; ++l) mbarExpectTx(&bars[l], (unsigned)(R * a.L[l - 1].out * 4));
    FC_STAMP(1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    FC_STAMP(5);
    if (LM == 1) {
      // bulk loads: thread 0 arms and issues every copy before anything else
      // touches the parameters (each first read of a parameter line is a
      // ~270-cycle constant-cache miss on the way to the first copy)
      const unsigned rowBytes = (unsigned)a.L[0].kred * 4u;
      mbarExpectTx(&bars[0], rowBytes * rows);
      if (p.denseIn) {  // the CTA's input rows are one contiguous block
        bulkCopy(sm + p.offAct[0], a.I + (int64_t)row0 * a.ldi, rowBytes * rows, &bars[0]);
      } else {
        for (int r = 0; r < rows; ++r)
          bulkCopy(sm + p.offAct[0] + r * p.ald[0], a.I + (int64_t)(row0 + r) * a.ldi, rowBytes, &bars[0]);
      }
      FC_STAMP(24);
#pragma unroll
      for (int l = 0; l < layers; ++l) {
        const int c0 = rank * p.cols[l], nc = max(0, min(p.cols[l], a.L[l].out - c0));
        mbarExpectTx(&bars[layers + l], (unsigned)(a.L[l].kred * 4 * nc));
        if (nc == 0) continue;
        const float* src = a.L[l].W + (int64_t)c0 * a.L[l].ldw;
        if (l < 4) FC_STAMP(25 + l);
        if (a.L[l].ldw == a.L[l].kred) {  // the slice is one contiguous block
          bulkCopy(sm + p.offW[l], src, (unsigned)(nc * a.L[l].kred * 4), &bars[layers + l]);
        } else {
          for (int q = 0; q < nc; ++q)
            bulkCopy(sm + p.offW[l] + q * p.wld[l], src + (int64_t)q * a.L[l].ldw, a.L[l].kred * 4,
                     &bars[layers + l]);
        }
      }
      FC_STAMP(12);
    }
  }
  // first-pass bias of every layer, loaded now so its latency hides behind
  // the weight copies (each chain starts from its bias)
  float biasPre[kMaxLayers];
#pragma unroll
  for (int l = 0; l < kMaxLayers; ++l) {
    const int c = tid / R, c0 = rank * (l < layers ? p.cols[l] : 0);
    biasPre[l] = (l < layers && tid < R * p.cols[l] && c0 + c < a.L[l].out) ? __ldg(a.L[l].bias + c0 + c) : 0.0f;
  }
  // layer 0's second column (column pairs, planFc `pair`)
  const float biasPreB = (NL <= 2 && (p.pair & 1) && tid < R * (p.cols[0] / 2) && rank * p.cols[0] + tid / R + p.cols[0] / 2 < a.L[0].out)
                             ? __ldg(a.L[0].bias + rank * p.cols[0] + tid / R + p.cols[0] / 2)
                             : 0.0f;
  __syncwarp();      // lane 0 rejoins its warp (compute-sanitizer synccheck: no divergent barrier)
  __syncthreads();  // inits visible inside the CTA
  FC_STAMP(8);
  // Peers push layer outputs into this CTA's activation buffers and complete
  // them on this CTA's barriers, so every CTA of the cluster must have
  // initialised its barriers before the first push: arrive now, wait right
  // before pushing (the weight loads and layer 0 hide the barrier).
  if (cn > 1) asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
  FC_STAMP(11);

  // ---- every global load of the kernel is issued up front (bulk copies:
  // by thread 0 right after the barrier inits, above; dealing them
  // round-robin to the warps' lane 0 bought nothing once a CTA is one or two
  // warps and the paper chains need three copies)
  if (LM == 1) {
    // (the copies were issued by thread 0 above) input rows past the batch end are zero
    for (int e = tid; e < (R - rows) * p.ald[0]; e += T) sm[p.offAct[0] + rows * p.ald[0] + e] = 0.0f;
    if (rows < R) __syncthreads();
  } else if (LM == 2) {
    // 16-byte cp.async from every thread (a tunable; see planFc)
    // Layer 0 lands in p.nch reduction chunks (its input rows and weight
    // slice, one commit group per chunk), so its chains start on chunk 0
    // while the rest is in flight; every later layer is one more group.
    for (int e = tid; e < (R - rows) * p.ald[0]; e += T) sm[p.offAct[0] + rows * p.ald[0] + e] = 0.0f;
    {
      const int c0 = rank * p.cols[0], nc = max(0, min(p.cols[0], a.L[0].out - c0));
      const float* src = a.L[0].W + (int64_t)c0 * a.L[0].ldw;
      for (int ch = 0; ch < p.nch; ++ch) {
        const int q0 = ch * p.kc4, q1 = min(q0 + p.kc4, a.L[0].kred >> 2), w4 = q1 - q0;
        for (int e = tid; e < (rows + nc) * w4; e += T) {
          const int j = e / w4, q = q0 + e - j * w4;
          if (j < rows)
            cpAsync16(sm + p.offAct[0] + j * p.ald[0] + 4 * q, a.I + (int64_t)(row0 + j) * a.ldi + 4 * q);
          else
            cpAsync16(sm + p.offW[0] + (j - rows) * p.wld[0] + 4 * q, src + (int64_t)(j - rows) * a.L[0].ldw + 4 * q);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
    }
#pragma unroll
    for (int l = 1; l < layers; ++l) {
      const int c0 = rank * p.cols[l], nc = max(0, min(p.cols[l], a.L[l].out - c0)), k4 = a.L[l].kred >> 2;
      const float* src = a.L[l].W + (int64_t)c0 * a.L[l].ldw;
      for (int e = tid; e < nc * k4; e += T) {
        const int j = e / k4, q = e - j * k4;
        cpAsync16(sm + p.offW[l] + j * p.wld[l] + 4 * q, src + (int64_t)j * a.L[l].ldw + 4 * q);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  } else {
    for (int e = tid; e < R * p.ald[0]; e += T) {
      int r = e / p.ald[0], kk = e % p.ald[0];
      sm[p.offAct[0] + e] = (r < rows && kk < a.L[0].kred) ? a.I[(int64_t)(row0 + r) * a.ldi + kk] : 0.0f;
    }
    for (int l = 0; l < layers; ++l) {
      const int c0 = rank * p.cols[l];
      for (int e = tid; e < p.cols[l] * p.wld[l]; e += T) {
        int j = e / p.wld[l], kk = e % p.wld[l];
        sm[p.offW[l] + e] =
            (c0 + j < a.L[l].out && kk < a.L[l].kred) ? a.L[l].W[(int64_t)(c0 + j) * a.L[l].ldw + kk] : 0.0f;
      }
    }
    __syncthreads();
  }
  FC_STAMP(2);

#pragma unroll
  for (int l = 0; l < layers; ++l) {
    const FcLayer L = a.L[l];
    const int cols = p.cols[l], c0 = rank * cols;
    const bool last = l + 1 == layers;
    const int ald = p.ald[l];
    const unsigned actBase = smemAddr(sm + p.offAct[l]), wBase = smemAddr(sm + p.offW[l]);
    if ((l > 0 && cn > 1) || (l == 0 && LM == 1)) mbarWait(&bars[l], 0, l);
    if (LM == 1) mbarWait(&bars[layers + l], 0, layers + l);
    // cp.async mode: commit groups in flight after layer l's (or layer-0
    // chunk ch's) group; waiting for that leaves only later groups pending
    auto asyncWait = [&](int pending) {
      switch (pending) {
        case 0: cpAsyncWait<0>(); break;
        case 1: cpAsyncWait<1>(); break;
        case 2: cpAsyncWait<2>(); break;
        case 3: cpAsyncWait<3>(); break;
        case 4: cpAsyncWait<4>(); break;
        case 5: cpAsyncWait<5>(); break;
        default: cpAsyncWait<6>(); break;
      }
      __syncthreads();  // this thread's copies landed, then everyone's
    };
    if (LM == 2 && l > 0) asyncWait(NL - 1 - l);
    FC_STAMP(3 + 3 * l);
    if (!last && l == 0 && cn > 1) asm volatile("barrier.cluster.wait;" ::: "memory");
    if (l == 0) FC_STAMP(20);
    // (column pairs only in 1- and 2-layer chains: the extra code path cost
    // the 3-layer kernel register spills)
    if (NL <= 2 && l == 0 && (p.pair & 1)) {
      // one pass: thread t runs columns c and c + cols/2 of row r (planFc:
      // R * cols <= 2T, cols even); dead chains run on row 0 / column 0
      const int half = cols >> 1, idx = tid;
      const int r = idx < R * half ? idx % R : 0, c = idx < R * half ? idx / R : 0;
      const bool liveA = idx < R * half && c0 + c < L.out, liveB = idx < R * half && c0 + c + half < L.out;
      const float bA = biasPre[0], bB = biasPreB;  // (layer 0 only)
      const unsigned xa = actBase + (unsigned)(r * ald) * 4u, wa = wBase + (unsigned)(c * p.wld[l]) * 4u,
                     wb = wa + (unsigned)(half * p.wld[l]) * 4u;
      if (l < 3) FC_STAMP(21 + l);
      const float2 acc = chainSegment2(xa, wa, liveB ? wb : wa, L.kred, liveA ? bA : 0.0f, liveB ? bB : 0.0f);
      FC_STAMP(16 + l);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool live = h ? liveB : liveA;
        if (!live) continue;
        const int cc = c + h * half;
        const float v = fmaxf(h ? acc.y : acc.x, 0.0f);
        if (r < rows) L.O[(int64_t)(row0 + r) * L.out + c0 + cc] = v;
        if (!last) {
          float* dst = sm + p.offAct[l + 1] + r * p.ald[l + 1] + c0 + cc;
          if (cn > 1) {
            for (int q = 0; q < cn; ++q) stAsyncCluster(dst, &bars[l + 1], q, v);
          } else {
            *dst = v;
          }
        }
      }
    } else {
      const int nchains = R * cols;
      for (int base = 0; base < nchains; base += T) {
        // one (row, column) chain per thread and pass, row fastest; idle
        // lanes run a dummy chain on row 0 / column 0 (no branch in the chain)
        const int idx = base + tid;
        const bool live = idx < nchains && c0 + idx / R < L.out;
        const int r = live ? idx % R : 0, c = live ? idx / R : 0;
        float bpre = 0.0f;
  #pragma unroll
        for (int q = 0; q < kMaxLayers; ++q)
          if (q == l) bpre = biasPre[q];  // static register indexing
        float acc = !live ? 0.0f : base == 0 ? bpre : __ldg(L.bias + c0 + c);
        const unsigned xa = actBase + (unsigned)(r * ald) * 4u, wa = wBase + (unsigned)(c * p.wld[l]) * 4u;
        if (l == 0 && LM == 2) {
          for (int ch = 0; ch < p.nch; ++ch) {  // the chain follows the chunks in
            if (base == 0) asyncWait(p.nch - 1 - ch + NL - 1);
            const int k0 = ch * 4 * p.kc4, n = min(4 * p.kc4, L.kred - k0);
            acc = chainSegment(xa + 4u * k0, wa + 4u * k0, n, acc);
          }
        } else {
          if (l < 3) FC_STAMP(21 + l);  // chain entry (thread 0's first pass)
          acc = chainSegment(xa, wa, L.kred, acc);
        }
        FC_STAMP(16 + l);  // chain done (thread 0's first pass), before its stores
        if (live) {
          const float v = fmaxf(acc, 0.0f);
          if (r < rows) L.O[(int64_t)(row0 + r) * L.out + c0 + c] = v;
          if (!last) {  // push into the next layer's input buffer of every cluster CTA
            float* dst = sm + p.offAct[l + 1] + r * p.ald[l + 1] + c0 + c;
            if (cn > 1) {
              for (int q = 0; q < cn; ++q) stAsyncCluster(dst, &bars[l + 1], q, v);
            } else {
              *dst = v;  // a lone CTA: plain store, published by the barrier below
            }
          }
        }
      }
    }
    FC_STAMP(4 + 3 * l);
    if (!last && cn == 1) __syncthreads();
  }
  if (cn > 1 && layers == 1) asm volatile("barrier.cluster.wait;" ::: "memory");  // pair the arrive
  if (LM == 1 || cn > 1) {
    // every wait on the barriers is behind us: invalidate them, so the shared
    // memory they occupied is plain memory again for the next kernel on this
    // SM (compute-sanitizer synccheck otherwise tracks the stale objects)
    __syncthreads();
    if (tid == 0)
#pragma unroll
      for (int b = 0; b < 2 * layers; ++b)
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smemAddr(&bars[b])) : "memory");
  }
  FC_STAMP(15);
  FC_GSTAMP(14);
}

}  // namespace

// Builds the plan; returns the dynamic shared-memory size. Every operand
// buffer is followed by >= 32 floats of slack (the chain prefetches ahead).
static size_t planFc(const FcChainArgs& a, int R, int cn, FcPlan& p, int loads = 0, int threads = 0) {
  p = FcPlan{};
  p.cn = cn;
  p.R = R;
  int off = 0;
  for (int l = 0; l < a.layers; ++l) {
    p.cols[l] = (a.L[l].out + cn - 1) / cn;
    p.wld[l] = up4(a.L[l].kred);
    // a block of half the layer's chains runs them two columns per thread in
    // one pass instead of two passes (bulk loads: every kred row 16-B aligned)
    if (l == 0 && a.layers <= 2 && threads > 0 && p.cols[l] % 2 == 0 && R * p.cols[l] > threads && R * p.cols[l] <= 2 * threads &&
        a.L[l].kred % 4 == 0)
      p.pair = 1;
    p.offW[l] = off;
    off += p.cols[l] * p.wld[l] + 32;
  }
  // layer l >= 1 reads kred_l columns of rows that receive all out_{l-1} pushed columns
  for (int l = 0; l <= a.layers; ++l) {
    int w = l < a.layers ? a.L[l].kred : a.L[l - 1].out;
    if (l > 0 && l < a.layers && a.L[l - 1].out > w) w = a.L[l - 1].out;
    p.ald[l] = padRow(w);
  }
  // dense input rows (one bulk copy) when the unpadded row stride already
  // puts the up-to-8 rows of an LDS.128 wavefront in distinct 16-byte bank groups
  {
    const int k0 = a.L[0].kred, nr = R < 8 ? R : 8;
    bool ok = a.ldi == k0 && k0 % 4 == 0;
    unsigned seen = 0;
    for (int r = 0; r < nr && ok; ++r) {
      const unsigned g = 1u << (((r * k0) / 4) % 8);
      ok = !(seen & g);
      seen |= g;
    }
    p.denseIn = ok ? 1 : 0;
    if (ok) p.ald[0] = k0;
  }
  for (int l = 0; l < a.layers; ++l) {  // one buffer per layer boundary: never reused, so no
    p.offAct[l] = off;                   // "buffer free" handshake between cluster CTAs
    off += R * p.ald[l] + 32;
  }
  off = (off + 3) & ~3;  // 16-byte alignment for the mbarriers
  p.offBar = off;
  off += 2 * (2 * a.layers);  // uint64 barriers: [l]: activations of layer l, [layers + l]: weights of layer l
  bool bulk = (a.ldi % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.I) & 15) == 0);
  for (int l = 0; l < a.layers; ++l)
    bulk = bulk && (a.L[l].kred % 4 == 0) && (a.L[l].ldw % 4 == 0) &&
           ((reinterpret_cast<uintptr_t>(a.L[l].W) & 15) == 0);
  // automatic loads: the bulk-copy engine. 16-byte cp.async from every
  // thread (loads 2/3) measured slower at every paper shape — MLP3 5.95 vs
  // 5.49 us, 2FCRelu 16.9 vs 7.9, MLP1 15.5 vs 6.5: an SM keeps too few
  // cp.async sectors in flight for ~90 KB per CTA (profiles/r02_fc_notes.txt)
  p.bulk = !bulk ? 0 : (loads == 2 || loads == 3) ? 2 : 1;
  if (p.bulk == 2) p.pair = 0;  // layer 0 follows the cp.async chunks (single-column chains)
  const bool oneChunk = loads == 3;
  {
    // layer-0 chunks: ~256-step pieces, at most 4, multiples of 16 steps
    // (chainSegment's granularity; the chunk boundaries keep the k order)
    const int k4 = a.L[0].kred >> 2;
    p.nch = std::max(1, std::min(4, a.L[0].kred / 256));
    p.kc4 = ((k4 + p.nch - 1) / p.nch + 3) & ~3;
    p.nch = (k4 + p.kc4 - 1) / p.kc4;
    if (a.layers + p.nch - 1 > 7 || oneChunk) p.nch = 1, p.kc4 = k4;  // (wait_group immediates up to 6)
  }
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
  return t > kFcMaxThreads ? kFcMaxThreads : (t < 32 ? 32 : t);
}

template <int LM>
static void (*fcKernelLm(int layers))(FcChainArgs, FcPlan) {
  switch (layers) {
    case 1: return fc_cluster_kernel<1, LM>;
    case 2: return fc_cluster_kernel<2, LM>;
    case 3: return fc_cluster_kernel<3, LM>;
    case 4: return fc_cluster_kernel<4, LM>;
    default: return nullptr;
  }
}
static void (*fcKernel(int layers, int lm))(FcChainArgs, FcPlan) {
  return lm == 1 ? fcKernelLm<1>(layers) : lm == 2 ? fcKernelLm<2>(layers) : fcKernelLm<0>(layers);
}

cudaError_t launchFcChain(const FcChainArgs& a, int rows, int cn, int threads, cudaStream_t s, int loads) {
  if (a.batch <= 0) return cudaSuccess;
  if (loads == 4) return launchFcTma(a, rows, cn, threads, s);
  FcPlan p;
  size_t smem = planFc(a, rows, cn, p, loads, threads);
  if (smem > 227 * 1024 || cn < 1 || cn > 16 || rows < 1) return cudaErrorInvalidConfiguration;
  if (threads < 32 || threads > kFcMaxThreads || threads % 32) return cudaErrorInvalidConfiguration;
  void (*kern)(FcChainArgs, FcPlan) = fcKernel(a.layers, p.bulk);
  if (!kern) return cudaErrorInvalidValue;
  {
    cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kern), (int)smem, cn > 8);
    if (e != cudaSuccess) return e;
  }
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
  return cudaLaunchKernelEx(&cfg, kern, a, p);
}

}  // namespace k
}  // namespace tcb
