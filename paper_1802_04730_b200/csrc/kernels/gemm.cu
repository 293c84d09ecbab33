// gemm.cu — exact fp32 NT-GEMM for the contraction family
//   TMM   C(m,n) +=! A(m,kk) * B(n,kk)          proj/kernels/tmm.tc:2-4
//   TBMM  Z(b,n,k) +=! X(b,n,m) * Y(b,k,m)       proj/kernels/tbmm.tc:2-4
//   C3    C3(b,wy) += I3(b,wxx) * W(wy,wxx)      PAPER.md:3035 (in/out)
//   FC    O(b,n) = B(n); O += I(b,m)*W(n,m); O = fmaxf(O,0)   mlp1.tc:2-6
//
// Register-tiled SIMT GEMM on the FP32 FFMA pipe. Each thread owns an
// RM×RN micro-tile and runs every output's k-chain sequentially in
// ascending k from the init value, with one fused multiply-add per step —
// the reference interpreter's per-step rounding order (interpreter.cc:
// 218-233). Operand tiles (TM×TK, TN×TK) are staged row-major in shared
// memory by 16-byte cp.async (zero-filled at the edges) through a 4- or
// 8-stage ring (S-1 tiles in flight: the K loop is load-latency bound),
// with a +4-float row pad that keeps the per-thread float4 k-reads
// conflict-free. Tensor cores are deliberately not used here: their
// internal accumulation order cannot reproduce the reference chain, and
// at the paper shapes these contractions are launch- or HBM-bound.
#include <algorithm>

#include "kernels.cuh"

namespace tcb {
namespace k {

namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ float4 ldsV4(unsigned addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

__device__ __forceinline__ float initValue(const GemmArgs& a, const float* C, int m, int n) {
  if (a.init == kInitInout) return C[(int64_t)m * a.ldc + n];
  if (a.init == kInitBias) return a.bias[n];
  return 0.0f;
}

template <int TM, int TN, int RM, int RN, int TK, int S>
__global__ void __launch_bounds__((TM / RM) * (TN / RN))
    gemm_nt_tiled(const GemmArgs a, const int vec) {
  constexpr int TX = TN / RN, TY = TM / RM, NT = TX * TY;
  constexpr int LD = TK + 4;  // padded row stride, keeps 16B alignment
  extern __shared__ __align__(16) float smem[];
  float (*As)[TM][LD] = reinterpret_cast<float (*)[TM][LD]>(smem);            // [S][TM][LD]
  float (*Bs)[TN][LD] = reinterpret_cast<float (*)[TN][LD]>(smem + S * TM * LD);  // [S][TN][LD]

  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const int n0 = blockIdx.x * TN, m0 = blockIdx.y * TM, b = blockIdx.z;
  const float* A = a.A + (int64_t)b * a.sA;
  const float* B = a.B + (int64_t)b * a.sB;
  float* C = a.C + (int64_t)b * a.sC;

  float acc[RM][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      int m = m0 + ty + i * TY, n = n0 + tx + j * TX;
      acc[i][j] = (m < a.M && n < a.N) ? initValue(a, C, m, n) : 0.0f;
    }

  auto loadTile = [&](int stage, int k0) {
    if (vec) {
      constexpr int C4 = TK / 4;
      for (int l = tid; l < TM * C4; l += NT) {
        int r = l / C4, c = (l % C4) * 4;
        int m = m0 + r, kk = k0 + c;
        bool ok = m < a.M && kk < a.K;
        const float* src = ok ? A + (int64_t)m * a.lda + kk : A;
        cp_async16(&As[stage][r][c], src, ok ? 16 : 0);
      }
      for (int l = tid; l < TN * C4; l += NT) {
        int r = l / C4, c = (l % C4) * 4;
        int n = n0 + r, kk = k0 + c;
        bool ok = n < a.N && kk < a.K;
        const float* src = ok ? B + (int64_t)n * a.ldb + kk : B;
        cp_async16(&Bs[stage][r][c], src, ok ? 16 : 0);
      }
    } else {
      for (int l = tid; l < TM * TK; l += NT) {
        int r = l / TK, c = l % TK;
        int m = m0 + r, kk = k0 + c;
        As[stage][r][c] = (m < a.M && kk < a.K) ? A[(int64_t)m * a.lda + kk] : 0.0f;
      }
      for (int l = tid; l < TN * TK; l += NT) {
        int r = l / TK, c = l % TK;
        int n = n0 + r, kk = k0 + c;
        Bs[stage][r][c] = (n < a.N && kk < a.K) ? B[(int64_t)n * a.ldb + kk] : 0.0f;
      }
    }
  };

  // S-stage cp.async ring: S-1 tiles in flight while one is consumed
  const int ntiles = (a.K + TK - 1) / TK;
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < ntiles) loadTile(s, s * TK);
    cp_async_commit();
  }
  for (int t = 0; t < ntiles; ++t) {
    cp_async_wait<S - 2>();
    __syncthreads();  // tile t landed for everyone; stage (t-1)%S is free
    {
      const int nt = t + S - 1;
      if (nt < ntiles) loadTile(nt % S, nt * TK);
      cp_async_commit();
    }
    const int st = t % S;
    const float* Ast = &As[st][ty][0];
    const float* Bst = &Bs[st][tx][0];
    // volatile shared loads: the compiler keeps them where they are written
    // (it otherwise sinks them next to their FFMAs, exposing the latency)
    const unsigned aS = static_cast<unsigned>(__cvta_generic_to_shared(Ast));
    const unsigned bS = static_cast<unsigned>(__cvta_generic_to_shared(Bst));
    auto loadGroup = [&](int kk, float4* av, float4* bv) {
#pragma unroll
      for (int i = 0; i < RM; ++i) av[i] = ldsV4(aS + (i * TY * LD + kk) * 4);
#pragma unroll
      for (int j = 0; j < RN; ++j) bv[j] = ldsV4(bS + (j * TX * LD + kk) * 4);
    };
    auto fmaGroup = [&](const float4* av, const float4* bv) {  // one 4-k step of every chain
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < RN; ++j) acc[i][j] = __fmaf_rn(av[i].x, bv[j].x, acc[i][j]);
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < RN; ++j) acc[i][j] = __fmaf_rn(av[i].y, bv[j].y, acc[i][j]);
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < RN; ++j) acc[i][j] = __fmaf_rn(av[i].z, bv[j].z, acc[i][j]);
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < RN; ++j) acc[i][j] = __fmaf_rn(av[i].w, bv[j].w, acc[i][j]);
    };
    auto group = [&](int kk) {  // one 4-k step of every chain of the micro-tile
      float4 av[RM], bv[RN];
      loadGroup(kk, av, bv);
      fmaGroup(av, bv);
    };
    const int klim = min(TK, a.K - t * TK);
    if (klim == TK) {
      // full tile: register ring of 3 groups — group g+2's shared loads are
      // issued before group g's FFMAs, so their latency hides behind two
      // groups of FFMAs
      float4 ra[3][RM], rb[3][RN];
      loadGroup(0, ra[0], rb[0]);
      if (TK > 4) loadGroup(4, ra[1], rb[1]);
#pragma unroll
      for (int g = 0; g < TK / 4; ++g) {
        if (g + 2 < TK / 4) loadGroup((g + 2) * 4, ra[(g + 2) % 3], rb[(g + 2) % 3]);
        fmaGroup(ra[g % 3], rb[g % 3]);
      }
    } else {
      const int k4 = klim & ~3;
      int kk = 0;
      for (; kk < k4; kk += 4) group(kk);
      for (; kk < klim; ++kk) {
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) acc[i][j] = __fmaf_rn(Ast[i * TY * LD + kk], Bst[j * TX * LD + kk], acc[i][j]);
      }
    }
  }

#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      int m = m0 + ty + i * TY, n = n0 + tx + j * TX;
      if (m < a.M && n < a.N) {
        float v = acc[i][j];
        if (a.relu) v = fmaxf(v, 0.0f);
        C[(int64_t)m * a.ldc + n] = v;
      }
    }
}

// One output per thread, operands streamed through L1 (no staging). Used
// for tiny problems where staging costs more than it saves.
__global__ void gemm_nt_direct(const GemmArgs a, const int vec) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)a.batch * a.M * a.N;
  if (idx >= total) return;
  int n = (int)(idx % a.N);
  int64_t r = idx / a.N;
  int m = (int)(r % a.M);
  int b = (int)(r / a.M);
  const float* Ar = a.A + (int64_t)b * a.sA + (int64_t)m * a.lda;
  const float* Br = a.B + (int64_t)b * a.sB + (int64_t)n * a.ldb;
  float* C = a.C + (int64_t)b * a.sC;
  float acc = initValue(a, C, m, n);
  int kk = 0;
  if (vec) {
    for (; kk + 4 <= a.K; kk += 4) {
      float4 x = __ldg(reinterpret_cast<const float4*>(Ar + kk));
      float4 y = __ldg(reinterpret_cast<const float4*>(Br + kk));
      acc = __fmaf_rn(x.x, y.x, acc);
      acc = __fmaf_rn(x.y, y.y, acc);
      acc = __fmaf_rn(x.z, y.z, acc);
      acc = __fmaf_rn(x.w, y.w, acc);
    }
  }
  for (; kk < a.K; ++kk) acc = __fmaf_rn(__ldg(Ar + kk), __ldg(Br + kk), acc);
  if (a.relu) acc = fmaxf(acc, 0.0f);
  C[(int64_t)m * a.ldc + n] = acc;
}

// Persistent batched GEMM for many small independent problems (TBMM:
// 500 batches of 26x72 · 72x26). Each CTA walks batches b = blockIdx.x +
// j*gridDim.x; a whole batch (A[b]: M rows, B[b]: N rows, K floats each)
// is one stage of an S-deep shared-memory ring, filled by per-row
// cp.async.bulk copies issued up front by warp 0 and completing on the
// stage's mbarrier — all of a CTA's first S batches are in flight before
// any compute starts. Rows are padded to ldS ≡ 4 (mod 32) floats. Every
// output is one thread's sequential FFMA chain in ascending k (RM x RN
// independent chains per thread), as in gemm_nt_tiled.
__device__ __forceinline__ unsigned smemU32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulkG2S(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smemU32(dst)),
      "l"(src), "r"(bytes), "r"(smemU32(bar))
      : "memory");
}
// Ends an mbarrier's life once every wait on it is behind us, so its shared
// memory is plain memory again for the next kernel on the SM
// (compute-sanitizer synccheck tracks stale barrier objects across kernels).
__device__ __forceinline__ void barInval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smemU32(bar)) : "memory");
}
__device__ __forceinline__ void barWait(uint64_t* bar, unsigned parity) {
  const unsigned addr = smemU32(bar);
  for (unsigned spin = 0;; ++spin) {
    unsigned done;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
    if (spin > (1u << 24)) __trap();  // never hang: the host reports the launch failure
  }
}

template <int RM, int RN>
__global__ void __launch_bounds__(512) gemm_nt_batched(const GemmArgs a, const int ldS, const int S) {
  extern __shared__ __align__(16) float smem[];
  const int stageF = (a.M + a.N) * ldS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * stageF);
  const int tid = threadIdx.x, T = blockDim.x;
  const int nb = (a.batch - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;  // batches of this CTA
  const unsigned rowBytes = (unsigned)a.K * 4u;
  // dense operands (row stride == K, landing unpadded): one copy per operand
  const bool dense = ldS == a.K && a.lda == a.K && a.ldb == a.K;

  auto issue = [&](int j, int s) {  // warp 0: stage s <- batch blockIdx.x + j*gridDim.x
    const int b = blockIdx.x + j * gridDim.x;
    const float* A = a.A + (int64_t)b * a.sA;
    const float* B = a.B + (int64_t)b * a.sB;
    float* dst = smem + s * stageF;
    if (dense) {
      if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smemU32(&bars[s])),
                     "r"(rowBytes * (unsigned)(a.M + a.N))
                     : "memory");
        bulkG2S(dst, A, rowBytes * a.M, &bars[s]);
        bulkG2S(dst + a.M * ldS, B, rowBytes * a.N, &bars[s]);
      }
      return;
    }
    if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smemU32(&bars[s])),
                               "r"(rowBytes * (unsigned)(a.M + a.N))
                               : "memory");
    __syncwarp();
    for (int r = tid; r < a.M + a.N; r += 32) {
      const float* src = r < a.M ? A + (int64_t)r * a.lda : B + (int64_t)(r - a.M) * a.ldb;
      bulkG2S(dst + r * ldS, src, rowBytes, &bars[s]);
    }
  };
  if (tid == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smemU32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();  // barrier inits visible; copies are issued below while the other warps start waiting
  if (tid < 32)
    for (int j = 0; j < min(S, nb); ++j) issue(j, j);

  const int tm = (a.M + RM - 1) / RM, tn = (a.N + RN - 1) / RN, ntask = tm * tn;
  for (int j = 0; j < nb; ++j) {
    const int s = j % S;
    const int b = blockIdx.x + j * gridDim.x;
    barWait(&bars[s], (j / S) & 1);
    const float* As = smem + s * stageF;
    const float* Bs = As + a.M * ldS;
    float* C = a.C + (int64_t)b * a.sC;
    for (int t = tid; t < ntask; t += T) {
      const int ti = t % tm, tj = t / tm;  // consecutive lanes walk A rows (B rows broadcast)
      int mr[RM], nr[RN];
#pragma unroll
      for (int i = 0; i < RM; ++i) mr[i] = min(ti * RM + i, a.M - 1);  // clamped reads, masked stores
#pragma unroll
      for (int q = 0; q < RN; ++q) nr[q] = min(tj * RN + q, a.N - 1);
      float acc[RM][RN];
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int q = 0; q < RN; ++q) acc[i][q] = initValue(a, C, mr[i], nr[q]);
      int kk = 0;
      for (; kk + 4 <= a.K; kk += 4) {
        float4 av[RM], bv[RN];
#pragma unroll
        for (int i = 0; i < RM; ++i) av[i] = *reinterpret_cast<const float4*>(As + mr[i] * ldS + kk);
#pragma unroll
        for (int q = 0; q < RN; ++q) bv[q] = *reinterpret_cast<const float4*>(Bs + nr[q] * ldS + kk);
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int q = 0; q < RN; ++q) acc[i][q] = __fmaf_rn(av[i].x, bv[q].x, acc[i][q]);
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int q = 0; q < RN; ++q) acc[i][q] = __fmaf_rn(av[i].y, bv[q].y, acc[i][q]);
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int q = 0; q < RN; ++q) acc[i][q] = __fmaf_rn(av[i].z, bv[q].z, acc[i][q]);
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int q = 0; q < RN; ++q) acc[i][q] = __fmaf_rn(av[i].w, bv[q].w, acc[i][q]);
      }
      for (; kk < a.K; ++kk)
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int q = 0; q < RN; ++q) acc[i][q] = __fmaf_rn(As[mr[i] * ldS + kk], Bs[nr[q] * ldS + kk], acc[i][q]);
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int q = 0; q < RN; ++q) {
          const int m = ti * RM + i, n = tj * RN + q;
          if (m < a.M && n < a.N) {
            float v = acc[i][q];
            if (a.relu) v = fmaxf(v, 0.0f);
            C[(int64_t)m * a.ldc + n] = v;
          }
        }
    }
    __syncthreads();  // stage s fully consumed
    if (tid < 32 && j + S < nb) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before async refill
      issue(j + S, s);
    }
  }
  __syncthreads();  // every wait on the ring is behind us
  if (tid == 0)
    for (int s = 0; s < S; ++s) barInval(&bars[s]);
}

// "Slab" GEMM for many small batches (TBMM: 500 x (26x72 · 72x26)). One CTA
// owns one batch (or a row/column tile of it); the whole tile's operands
// are in flight from the first cycle, by 16-byte cp.async from every thread,
// in NCH reduction chunks of CQ float4s, one commit group per chunk, so the
// chains of chunk c run while chunks > c are still arriving. Lane j of a
// warp owns output column n = n0 + j: it moves its B row's chunk from shared
// memory into registers (rows padded to an odd number of 16-byte units, so
// eight lanes' float4 reads hit eight bank groups). Warp g owns CH output
// rows and streams their A rows from shared memory, where every lane reads
// the same address (a broadcast: one wavefront per 4 reduction steps for the
// whole warp), so each A value fetched feeds 32 FFMAs. A batch is ~15 KB:
// every CTA of the paper shape is resident in one wave.
// Each output is one thread's sequential FFMA chain in ascending k from its
// init value, as in gemm_nt_tiled.
constexpr int kSlabCq = 6;  // float4s per reduction chunk (24 k steps)

#ifdef TCB_SLAB_TRACE
// diagnostic build only (profiles/slab_trace.cu): per-CTA globaltimer stamps
__device__ unsigned long long g_slab_trace[4096][10];
#define SLAB_STAMP(ev)                                                      \
  do {                                                                      \
    unsigned long long t_;                                                  \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
    if (threadIdx.x == 0 && blockIdx.x < 4096) g_slab_trace[blockIdx.x][ev] = t_; \
  } while (0)
#else
#define SLAB_STAMP(ev) \
  do {                 \
  } while (0)
#endif

template <int CH>
__global__ void __launch_bounds__(256) gemm_nt_slab(const GemmArgs a, const int ng) {
  extern __shared__ __align__(16) float smem[];
  constexpr int CQ = kSlabCq;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = warp % ng, lb = warp / ng;
  const int MT = ng * CH, NT = blockDim.x / ng;  // tile rows / columns
  const int m0 = blockIdx.y * MT, n0 = blockIdx.z * NT, b = blockIdx.x;
  const int n = n0 + lb * 32 + lane;
  const int K4 = a.K >> 2;
  const int ldA = K4, ldB = K4 | 1;  // row strides in float4s
  const float* A = a.A + (int64_t)b * a.sA;
  const float* B = a.B + (int64_t)b * a.sB;
  float* C = a.C + (int64_t)b * a.sC;
  const int rowsA = min(MT, a.M - m0), rowsB = min(NT, a.N - n0);
  float4* As = reinterpret_cast<float4*>(smem);  // [MT][ldA]
  float4* Bs = As + MT * ldA;                    // [NT][ldB]
  SLAB_STAMP(0);

  // every chunk's copies issued up front, one commit group per chunk
  const int nch = (K4 + CQ - 1) / CQ;
  for (int c = 0; c < nch; ++c) {
    const int q0 = c * CQ, cq = min(CQ, K4 - q0);
    for (int e = tid; e < (rowsA + rowsB) * cq; e += blockDim.x) {
      const int r = e / cq, q = q0 + e - r * cq;
      if (r < rowsA)
        cp_async16(As + r * ldA + q, A + (int64_t)(m0 + r) * a.lda + 4 * q, 16);
      else
        cp_async16(Bs + (r - rowsA) * ldB + q, B + (int64_t)(n0 + r - rowsA) * a.ldb + 4 * q, 16);
    }
    cp_async_commit();
  }
  SLAB_STAMP(1);
  float acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int m = m0 + g * CH + c;
    acc[c] = (m < a.M && n < a.N) ? initValue(a, C, m, n) : 0.0f;
  }
  const unsigned aS = static_cast<unsigned>(__cvta_generic_to_shared(As));
  const unsigned bS = static_cast<unsigned>(__cvta_generic_to_shared(Bs + min(lb * 32 + lane, rowsB - 1) * ldB));
  unsigned rowAddr[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) rowAddr[c] = aS + (unsigned)(min(g * CH + c, rowsA - 1) * ldA) * 16u;

  for (int c = 0; c < nch; ++c) {
    switch (nch - 1 - c) {  // this thread's copies of chunks <= c have landed
      case 0: cp_async_wait<0>(); break;
      case 1: cp_async_wait<1>(); break;
      case 2: cp_async_wait<2>(); break;
      case 3: cp_async_wait<3>(); break;
      case 4: cp_async_wait<4>(); break;
      default: cp_async_wait<5>(); break;
    }
    __syncthreads();  // ... and everyone's
    SLAB_STAMP(2 + min(c, 5));
    const int q0 = c * CQ, cq = min(CQ, K4 - q0);
    float4 br[CQ];
#pragma unroll
    for (int q = 0; q < CQ; ++q)
      if (q < cq) br[q] = ldsV4(bS + (q0 + q) * 16);
    float4 av[2][CH];
#pragma unroll
    for (int r = 0; r < CH; ++r) av[0][r] = ldsV4(rowAddr[r] + q0 * 16);
#pragma unroll
    for (int q = 0; q < CQ; ++q) {
      if (q < cq) {  // warp-uniform
        if (q + 1 < cq) {  // next group's A values before this group's FFMAs
#pragma unroll
          for (int r = 0; r < CH; ++r) av[(q + 1) & 1][r] = ldsV4(rowAddr[r] + (q0 + q + 1) * 16);
        }
        const float4* v = av[q & 1];
#pragma unroll
        for (int r = 0; r < CH; ++r) acc[r] = __fmaf_rn(v[r].x, br[q].x, acc[r]);
#pragma unroll
        for (int r = 0; r < CH; ++r) acc[r] = __fmaf_rn(v[r].y, br[q].y, acc[r]);
#pragma unroll
        for (int r = 0; r < CH; ++r) acc[r] = __fmaf_rn(v[r].z, br[q].z, acc[r]);
#pragma unroll
        for (int r = 0; r < CH; ++r) acc[r] = __fmaf_rn(v[r].w, br[q].w, acc[r]);
      }
    }
  }
  SLAB_STAMP(8);
  if (n < a.N) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int m = m0 + g * CH + c;
      if (m < a.M) {
        float v = acc[c];
        if (a.relu) v = fmaxf(v, 0.0f);
        C[(int64_t)m * a.ldc + n] = v;
      }
    }
  }
  SLAB_STAMP(9);
}

// Register-tiled slab: the same one-CTA-per-batch, chunk-pipelined loads as
// gemm_nt_slab, but each lane owns an RM x RN block of outputs (rows
// rg + 4i, columns cg + 8j; lane = rg * 8 + cg), so a warp tile is
// 4*RM x 8*RN (28 x 32 for 7x4: one warp covers a whole 26x26 TBMM batch).
// Shared-memory reads are what bound the broadcast slab (ncu: a broadcast
// LDS.128 costs 2 LSU wavefronts, so 7 A rows per 28 FFMAs saturated the
// LSU pipe and slowed the cp.async fills sharing it); here each 4-step group
// reads RM A float4s (4 distinct rows per instruction) and RN B float4s (8
// distinct rows) for 4*RM*RN FFMAs. Row strides are odd in 16-byte units, so
// consecutive rows fall in distinct bank groups. Each output is one lane's
// sequential FFMA chain in ascending k from its init value.
template <int RM, int RN, bool BULK>
__global__ void __launch_bounds__(256) gemm_nt_slab_rt(const GemmArgs a, const int wm) {
  extern __shared__ __align__(16) float smem[];
  constexpr int CQ = kSlabCq;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rg = lane >> 3, cg = lane & 7;
  const int wr = warp % wm, wc = warp / wm;
  const int MT = wm * 4 * RM, NT = (blockDim.x >> 5) / wm * 8 * RN;
  const int m0 = blockIdx.y * MT, n0 = blockIdx.z * NT, b = blockIdx.x;
  const int K4 = a.K >> 2;
  const int ld = BULK ? K4 : (K4 | 1);  // row stride in float4s (odd unless bulk-filled)
  const float* A = a.A + (int64_t)b * a.sA;
  const float* B = a.B + (int64_t)b * a.sB;
  float* C = a.C + (int64_t)b * a.sC;
  const int rowsA = min(MT, a.M - m0), rowsB = min(NT, a.N - n0);
  float4* As = reinterpret_cast<float4*>(smem);  // [MT][ld]
  float4* Bs = As + MT * ld;                     // [NT][ld]
  SLAB_STAMP(0);

  const int nch = (K4 + CQ - 1) / CQ;
  uint64_t* bars = reinterpret_cast<uint64_t*>(Bs + NT * ld);  // BULK: the fill's mbarrier
  if (BULK) {
    // dense operand tiles (rows of exactly K floats): one bulk copy per
    // operand tile, both on one mbarrier. (Per row-chunk bulk copies were
    // measured at ~6 us to issue 156 of them: a bulk copy costs its issuing
    // thread ~200 cycles.)
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smemU32(&bars[0])));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smemU32(&bars[0])),
                   "r"((unsigned)((rowsA + rowsB) * K4 * 16))
                   : "memory");
      bulkG2S(As, A + (int64_t)m0 * a.lda, (unsigned)(rowsA * K4 * 16), &bars[0]);
      bulkG2S(Bs, B + (int64_t)n0 * a.ldb, (unsigned)(rowsB * K4 * 16), &bars[0]);
    }
    __syncthreads();  // barrier initialised before anyone waits on it
  } else {
    for (int c = 0; c < nch; ++c) {
      const int q0 = c * CQ, cq = min(CQ, K4 - q0);
      for (int e = tid; e < (rowsA + rowsB) * cq; e += blockDim.x) {
        const int r = e / cq, q = q0 + e - r * cq;
        if (r < rowsA)
          cp_async16(As + r * ld + q, A + (int64_t)(m0 + r) * a.lda + 4 * q, 16);
        else
          cp_async16(Bs + (r - rowsA) * ld + q, B + (int64_t)(n0 + r - rowsA) * a.ldb + 4 * q, 16);
      }
      cp_async_commit();
    }
  }
  SLAB_STAMP(1);
  // this lane's rows / columns inside the CTA tile (clamped for reads)
  const int rbase = wr * 4 * RM + rg, cbase = wc * 8 * RN + cg;
  float acc[RM][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int m = m0 + rbase + 4 * i, n = n0 + cbase + 8 * j;
      acc[i][j] = (m < a.M && n < a.N) ? initValue(a, C, m, n) : 0.0f;
    }
  const unsigned aS = static_cast<unsigned>(__cvta_generic_to_shared(As));
  const unsigned bS = static_cast<unsigned>(__cvta_generic_to_shared(Bs));
  unsigned ra[RM], rb[RN];
#pragma unroll
  for (int i = 0; i < RM; ++i) ra[i] = aS + (unsigned)(min(rbase + 4 * i, rowsA - 1) * ld) * 16u;
#pragma unroll
  for (int j = 0; j < RN; ++j) rb[j] = bS + (unsigned)(min(cbase + 8 * j, rowsB - 1) * ld) * 16u;

  for (int c = 0; c < nch; ++c) {
    if (BULK) {
      if (c == 0) barWait(&bars[0], 0);
    } else {
      switch (nch - 1 - c) {
        case 0: cp_async_wait<0>(); break;
        case 1: cp_async_wait<1>(); break;
        case 2: cp_async_wait<2>(); break;
        case 3: cp_async_wait<3>(); break;
        case 4: cp_async_wait<4>(); break;
        default: cp_async_wait<5>(); break;
      }
      __syncthreads();
    }
    SLAB_STAMP(2 + min(c, 5));
    const int q0 = c * CQ, cq = min(CQ, K4 - q0);
    float4 av[2][RM], bv[2][RN];
#pragma unroll
    for (int i = 0; i < RM; ++i) av[0][i] = ldsV4(ra[i] + q0 * 16);
#pragma unroll
    for (int j = 0; j < RN; ++j) bv[0][j] = ldsV4(rb[j] + q0 * 16);
#pragma unroll
    for (int q = 0; q < CQ; ++q) {
      if (q < cq) {  // block-uniform
        if (q + 1 < cq) {
#pragma unroll
          for (int i = 0; i < RM; ++i) av[(q + 1) & 1][i] = ldsV4(ra[i] + (q0 + q + 1) * 16);
#pragma unroll
          for (int j = 0; j < RN; ++j) bv[(q + 1) & 1][j] = ldsV4(rb[j] + (q0 + q + 1) * 16);
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
    }
  }
  if (BULK) {  // the fill's barrier: every wait is behind us
    __syncthreads();
    if (tid == 0) barInval(&bars[0]);
  }
  SLAB_STAMP(8);
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    const int m = m0 + rbase + 4 * i;
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int n = n0 + cbase + 8 * j;
      if (m < a.M && n < a.N) {
        float v = acc[i][j];
        if (a.relu) v = fmaxf(v, 0.0f);
        C[(int64_t)m * a.ldc + n] = v;
      }
    }
  }
  SLAB_STAMP(9);
}

// Warp-per-batch GEMM: for batches whose whole output fits one warp tile
// (M <= 4*RM, N <= 8*RN: TBMM's 26x26 with 7x4). A CTA of W warps owns W
// consecutive batches, one per warp, so the warps of one SM spread over its
// four schedulers (a 1-warp CTA per batch left them on few schedulers:
// profiles/r02_tbmm_trace.txt). Lane 0 of each warp lands its batch's two
// dense operand blocks with two bulk copies on the warp's own mbarrier (or the
// warp's lanes use 16-byte cp.async when the rows are not dense) and the
// warp starts the moment its batch is in. Lane = rg * 8 + cg owns rows
// rg + 4i and columns cg + 8j; each 4-step group reads RM + RN float4s from
// shared memory for 4*RM*RN FFMAs (ncu: the LSU pipe, not the FMA pipe,
// bounded the broadcast slab). Each output is one lane's sequential FFMA
// chain in ascending k from its init value.
template <int RM, int RN>
__global__ void __launch_bounds__(256) gemm_nt_warpbatch(const GemmArgs a, const int dense) {
  extern __shared__ __align__(16) float smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int b = blockIdx.x * W + warp;
  const int K4 = a.K >> 2;
  const int ld = dense ? K4 : (K4 | 1);
  const int slot = (a.M + a.N) * ld;  // float4s per warp
  float4* As = reinterpret_cast<float4*>(smem) + warp * slot;
  float4* Bs = As + a.M * ld;
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<float4*>(smem) + W * slot) + warp;
  SLAB_STAMP(0);
  if (b >= a.batch) return;  // (no CTA-wide barrier below)
  const float* A = a.A + (int64_t)b * a.sA;
  const float* B = a.B + (int64_t)b * a.sB;
  float* C = a.C + (int64_t)b * a.sC;
  if (dense) {
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smemU32(bar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smemU32(bar)),
                   "r"((unsigned)((a.M + a.N) * K4 * 16))
                   : "memory");
      bulkG2S(As, A, (unsigned)(a.M * K4 * 16), bar);
      bulkG2S(Bs, B, (unsigned)(a.N * K4 * 16), bar);
    }
  } else {
    for (int e = lane; e < (a.M + a.N) * K4; e += 32) {
      const int r = e / K4, q = e - r * K4;
      if (r < a.M)
        cp_async16(As + r * ld + q, A + (int64_t)r * a.lda + 4 * q, 16);
      else
        cp_async16(Bs + (r - a.M) * ld + q, B + (int64_t)(r - a.M) * a.ldb + 4 * q, 16);
    }
    cp_async_commit();
  }
  SLAB_STAMP(1);
  const int rg = lane >> 3, cg = lane & 7;
  float acc[RM][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int m = rg + 4 * i, n = cg + 8 * j;
      acc[i][j] = (m < a.M && n < a.N) ? initValue(a, C, m, n) : 0.0f;
    }
  unsigned ra[RM], rb[RN];
#pragma unroll
  for (int i = 0; i < RM; ++i) ra[i] = smemU32(As + min(rg + 4 * i, a.M - 1) * ld);
#pragma unroll
  for (int j = 0; j < RN; ++j) rb[j] = smemU32(Bs + min(cg + 8 * j, a.N - 1) * ld);
  if (dense) {
    __syncwarp();  // lane 0's barrier init before the others poll it
    barWait(bar, 0);
    __syncwarp();
    if (lane == 0) barInval(bar);
  } else {
    cp_async_wait<0>();
    __syncwarp();
  }
  SLAB_STAMP(2);
  float4 av[2][RM], bv[2][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i) av[0][i] = ldsV4(ra[i]);
#pragma unroll
  for (int j = 0; j < RN; ++j) bv[0][j] = ldsV4(rb[j]);
  int q = 0;
  for (; q + 2 <= K4; q += 2) {  // two groups per trip: static register buffers
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (q + h + 1 < K4) {
#pragma unroll
        for (int i = 0; i < RM; ++i) av[h ^ 1][i] = ldsV4(ra[i] + (q + h + 1) * 16);
#pragma unroll
        for (int j = 0; j < RN; ++j) bv[h ^ 1][j] = ldsV4(rb[j] + (q + h + 1) * 16);
      }
      const float4* x = av[h];
      const float4* y = bv[h];
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
  }
  if (q < K4) {  // odd group count: the last group sits in buffer 0
    const float4* x = av[0];
    const float4* y = bv[0];
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
  SLAB_STAMP(8);
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    const int m = rg + 4 * i;
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int n = cg + 8 * j;
      if (m < a.M && n < a.N) {
        float v = acc[i][j];
        if (a.relu) v = fmaxf(v, 0.0f);
        C[(int64_t)m * a.ldc + n] = v;
      }
    }
  }
  SLAB_STAMP(9);
}

int batchedLd(int K) {
  int l = (K + 3) & ~3;
  while (l % 32 != 4) l += 4;
  return l;
}

const GemmVariant kGemmVariants[] = {
    {0, 0, 0, 1, 1, 0, "direct"},
    {1, 16, 16, 1, 1, 32, "t16x16_r1x1_k32"},
    {2, 16, 32, 1, 2, 32, "t16x32_r1x2_k32"},
    {3, 32, 16, 2, 1, 32, "t32x16_r2x1_k32"},
    {4, 32, 32, 2, 2, 32, "t32x32_r2x2_k32"},
    {5, 32, 64, 2, 4, 32, "t32x64_r2x4_k32"},
    {6, 64, 32, 4, 2, 32, "t64x32_r4x2_k32"},
    {7, 64, 64, 4, 4, 32, "t64x64_r4x4_k32"},
    {8, 32, 32, 4, 4, 32, "t32x32_r4x4_k32"},
    {9, 16, 32, 2, 2, 32, "t16x32_r2x2_k32"},
    {10, 32, 32, 2, 2, 64, "t32x32_r2x2_k64"},
    {11, 64, 64, 4, 4, 16, "t64x64_r4x4_k16"},
    {12, 16, 64, 2, 4, 32, "t16x64_r2x4_k32"},
    {13, 32, 32, 2, 4, 32, "t32x32_r2x4_k32"},
    {14, 16, 16, 2, 2, 32, "t16x16_r2x2_k32"},
    {15, 32, 64, 4, 4, 32, "t32x64_r4x4_k32"},
    {16, 32, 32, 2, 2, 32, "t32x32_r2x2_k32_s8", 8},
    {17, 16, 32, 2, 2, 32, "t16x32_r2x2_k32_s8", 8},
    {18, 16, 16, 1, 1, 64, "t16x16_r1x1_k64"},
    // persistent batched (tk = 0 marks "whole reduction per stage")
    {19, 1, 1, 2, 2, 0, "batched_r2x2", 0},
    {20, 1, 1, 1, 1, 0, "batched_r1x1", 0},
    {21, 1, 1, 2, 1, 0, "batched_r2x1", 0},
    {22, 1, 1, 1, 2, 0, "batched_r1x2", 0},
    // deeper k stages for long reductions (more bytes in flight per CTA)
    {23, 32, 32, 2, 2, 64, "t32x32_r2x2_k64_s8", 8},
    {24, 32, 32, 2, 2, 128, "t32x32_r2x2_k128", 4},
    {25, 32, 64, 2, 4, 64, "t32x64_r2x4_k64", 4},
    {26, 16, 64, 2, 4, 64, "t16x64_r2x4_k64", 4},
    {27, 16, 32, 2, 2, 64, "t16x32_r2x2_k64_s8", 8},
    {28, 32, 16, 2, 2, 64, "t32x16_r2x2_k64", 4},
    // slab: one CTA per batch, B rows in registers, A rows broadcast from
    // shared memory (tk = -1; rm = output rows per warp)
    {29, 0, 0, 4, 1, -1, "slab_c4", 0},
    {30, 0, 0, 7, 1, -1, "slab_c7", 0},
    {31, 0, 0, 13, 1, -1, "slab_c13", 0},
    // register-tiled slab (tk = -2): rm x rn outputs per lane
    {32, 0, 0, 7, 4, -2, "slab_rt7x4", 0},
    {33, 0, 0, 4, 4, -2, "slab_rt4x4", 0},
    {34, 0, 0, 4, 2, -2, "slab_rt4x2", 0},
    // ... filled by bulk copies (tk = -3)
    {35, 0, 0, 7, 4, -3, "slab_rt7x4_bulk", 0},
    {36, 0, 0, 4, 4, -3, "slab_rt4x4_bulk", 0},
    {37, 0, 0, 4, 2, -3, "slab_rt4x2_bulk", 0},
    // one warp per batch (tk = -4): the whole batch is one rm x rn warp tile
    {38, 0, 0, 7, 4, -4, "warpbatch_7x4", 0},
    {39, 0, 0, 4, 4, -4, "warpbatch_4x4", 0},
    // TMA-fed tiles (tk = -5, gemm_tma.cu): two tensor copies per 32-deep stage
    {40, 32, 32, 4, 4, -5, "tma_t32x32_r4x4", 8},
    {41, 32, 32, 4, 2, -5, "tma_t32x32_r4x2", 8},
    {42, 32, 64, 4, 4, -5, "tma_t32x64_r4x4", 6},
    {43, 16, 32, 2, 4, -5, "tma_t16x32_r2x4", 8},
    {44, 32, 16, 4, 2, -5, "tma_t32x16_r4x2", 8},
    {45, 64, 32, 4, 4, -5, "tma_t64x32_r4x4", 6},
    {46, 32, 32, 2, 2, -5, "tma_t32x32_r2x2", 8},
    // ... with the A tile multicast over a cluster of `stages` CTAs along N (tk = -6)
    {47, 32, 32, 2, 2, -6, "tma_t32x32_r2x2_mc4", 4},
    {48, 32, 32, 4, 2, -6, "tma_t32x32_r4x2_mc4", 4},
    {49, 32, 16, 2, 2, -6, "tma_t32x16_r2x2_mc4", 4},
    {50, 32, 32, 2, 2, -6, "tma_t32x32_r2x2_mc2", 2},
    // more broadcast-slab row counts per warp (tk = -1)
    {51, 0, 0, 5, 1, -1, "slab_c5", 0},
    {52, 0, 0, 6, 1, -1, "slab_c6", 0},
    {53, 0, 0, 9, 1, -1, "slab_c9", 0},
};

template <int RM, int RN>
cudaError_t launchBatched(const GemmArgs& a, int grid, cudaStream_t s) {
  // dense per-batch operands land with one copy each, unpadded; otherwise
  // one copy per row into rows padded to ldS = 4 (mod 32)
  const bool dense = a.lda == a.K && a.ldb == a.K;
  const int ldS = dense ? a.K : batchedLd(a.K);
  const size_t stageB = (size_t)(a.M + a.N) * ldS * 4;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (grid <= 0) grid = std::min(a.batch, 2 * sms);
  grid = std::min(grid, a.batch);
  const int perCta = (a.batch + grid - 1) / grid;
  int S = std::min(4, perCta);
  while (S > 1 && S * stageB + 64 > 100 * 1024) --S;
  const size_t smem = S * stageB + 8 * S;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  const int ntask = ((a.M + RM - 1) / RM) * ((a.N + RN - 1) / RN);
  const int threads = std::max(32, std::min(512, (ntask + 31) / 32 * 32));
  auto kfn = gemm_nt_batched<RM, RN>;
  {
    cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kfn), (int)smem);
    if (e != cudaSuccess) return e;
  }
  kfn<<<grid, threads, smem, s>>>(a, ldS, S);
  return cudaGetLastError();
}


// slab kernel dispatch: KR4 = register float4s per B row (K <= 4*KR4)
template <int CH>
cudaError_t launchSlabCh(const GemmArgs& a, cudaStream_t s) {
  // warps per lane block: enough row groups to cover M (<= 8), then as many
  // 32-column lane blocks as fit in 256 threads
  int ng = std::min(8, (a.M + CH - 1) / CH);
  int nbMax = std::max(1, 8 / ng);
  int nb = std::min(nbMax, (a.N + 31) / 32);
  dim3 grid(a.batch, (a.M + ng * CH - 1) / (ng * CH), (a.N + 32 * nb - 1) / (32 * nb));
  const int threads = ng * nb * 32;
  const int K4 = a.K / 4;
  const size_t smem = ((size_t)ng * CH * K4 + (size_t)32 * nb * (K4 | 1)) * 16;
  auto kfn = gemm_nt_slab<CH>;
  {
    cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kfn), (int)smem);
    if (e != cudaSuccess) return e;
  }
  kfn<<<grid, threads, smem, s>>>(a, ng);
  return cudaGetLastError();
}

template <int RM, int RN, bool BULK>
cudaError_t launchSlabRt(const GemmArgs& a, cudaStream_t s) {
  // warps along M to cover the rows (<= 8), then along N within 8 warps
  const int wmt = 4 * RM, wnt = 8 * RN;
  int wm = std::min(8, (a.M + wmt - 1) / wmt);
  int wn = std::min(std::max(1, 8 / wm), (a.N + wnt - 1) / wnt);
  dim3 grid(a.batch, (a.M + wm * wmt - 1) / (wm * wmt), (a.N + wn * wnt - 1) / (wn * wnt));
  if (BULK && (a.lda != a.K || a.ldb != a.K)) return launchSlabRt<RM, RN, false>(a, s);
  const int ld = BULK ? a.K / 4 : (a.K / 4) | 1;
  const size_t smem = (size_t)(wm * wmt + wn * wnt) * ld * 16 + 8 * 8;
  auto kfn = gemm_nt_slab_rt<RM, RN, BULK>;
  {
    cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kfn), (int)smem);
    if (e != cudaSuccess) return e;
  }
  kfn<<<grid, wm * wn * 32, smem, s>>>(a, wm);
  return cudaGetLastError();
}

template <int RM, int RN>
cudaError_t launchWarpBatch(const GemmArgs& a, int warps, cudaStream_t s) {
  if (a.M > 4 * RM || a.N > 8 * RN) return cudaErrorInvalidValue;
  const int dense = a.lda == a.K && a.ldb == a.K;
  const int K4 = a.K / 4, ld = dense ? K4 : (K4 | 1);
  if (warps <= 0) warps = 4;
  warps = std::max(1, std::min(8, warps));
  const size_t smem = (size_t)warps * (a.M + a.N) * ld * 16 + 8 * warps;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  auto kfn = gemm_nt_warpbatch<RM, RN>;
  {
    cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kfn), (int)smem);
    if (e != cudaSuccess) return e;
  }
  kfn<<<(a.batch + warps - 1) / warps, warps * 32, smem, s>>>(a, dense);
  return cudaGetLastError();
}

template <int TM, int TN, int RM, int RN, int TK, int S = 4>
cudaError_t launchTiled(const GemmArgs& a, int vec, cudaStream_t s) {
  dim3 grid((a.N + TN - 1) / TN, (a.M + TM - 1) / TM, a.batch);
  const size_t smem = (size_t)S * (TM + TN) * (TK + 4) * sizeof(float);
  auto kfn = gemm_nt_tiled<TM, TN, RM, RN, TK, S>;
  // set on every launch: the attribute is per device context, and a cached
  // per-process flag would leave other devices at the 48 KB default
  {
    cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kfn), (int)smem);
    if (e != cudaSuccess) return e;
  }
  kfn<<<grid, (TM / RM) * (TN / RN), smem, s>>>(a, vec);
  return cudaGetLastError();
}

}  // namespace

int gemmVariantCount() { return sizeof(kGemmVariants) / sizeof(kGemmVariants[0]); }

bool slabOk(const GemmArgs& a) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return a.K > 0 && a.K % 4 == 0 && a.K <= 4 * 6 * kSlabCq && a.lda % 4 == 0 && a.ldb % 4 == 0 && a.sA % 4 == 0 &&
         a.sB % 4 == 0 && al16(a.A) && al16(a.B) && a.batch <= 65535 * 1024;
}

bool batchedOk(const GemmArgs& a) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (a.K % 4 || a.lda % 4 || a.ldb % 4 || a.sA % 4 || a.sB % 4 || !al16(a.A) || !al16(a.B)) return false;
  return (size_t)(a.M + a.N) * batchedLd(a.K) * 4 + 64 <= 100 * 1024;
}
const GemmVariant& gemmVariant(int i) { return kGemmVariants[i]; }

cudaError_t launchGemm(const GemmArgs& a, int variant, int threads, cudaStream_t s) {
  if (a.batch <= 0 || a.M <= 0 || a.N <= 0) return cudaSuccess;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  int vec = (a.K % 4 == 0) && (a.lda % 4 == 0) && (a.ldb % 4 == 0) && (a.sA % 4 == 0) && (a.sB % 4 == 0) &&
            al16(a.A) && al16(a.B);
  switch (variant) {
    case 0: {
      int64_t total = (int64_t)a.batch * a.M * a.N;
      int t = threads > 0 ? threads : 128;
      gemm_nt_direct<<<(unsigned)((total + t - 1) / t), t, 0, s>>>(a, vec);
      return cudaGetLastError();
    }
    case 1: return launchTiled<16, 16, 1, 1, 32>(a, vec, s);
    case 2: return launchTiled<16, 32, 1, 2, 32>(a, vec, s);
    case 3: return launchTiled<32, 16, 2, 1, 32>(a, vec, s);
    case 4: return launchTiled<32, 32, 2, 2, 32>(a, vec, s);
    case 5: return launchTiled<32, 64, 2, 4, 32>(a, vec, s);
    case 6: return launchTiled<64, 32, 4, 2, 32>(a, vec, s);
    case 7: return launchTiled<64, 64, 4, 4, 32>(a, vec, s);
    case 8: return launchTiled<32, 32, 4, 4, 32>(a, vec, s);
    case 9: return launchTiled<16, 32, 2, 2, 32>(a, vec, s);
    case 10: return launchTiled<32, 32, 2, 2, 64>(a, vec, s);
    case 11: return launchTiled<64, 64, 4, 4, 16>(a, vec, s);
    case 12: return launchTiled<16, 64, 2, 4, 32>(a, vec, s);
    case 13: return launchTiled<32, 32, 2, 4, 32>(a, vec, s);
    case 14: return launchTiled<16, 16, 2, 2, 32>(a, vec, s);
    case 15: return launchTiled<32, 64, 4, 4, 32>(a, vec, s);
    case 16: return launchTiled<32, 32, 2, 2, 32, 8>(a, vec, s);
    case 17: return launchTiled<16, 32, 2, 2, 32, 8>(a, vec, s);
    case 18: return launchTiled<16, 16, 1, 1, 64>(a, vec, s);
    case 23: return launchTiled<32, 32, 2, 2, 64, 8>(a, vec, s);
    case 24: return launchTiled<32, 32, 2, 2, 128, 4>(a, vec, s);
    case 25: return launchTiled<32, 64, 2, 4, 64, 4>(a, vec, s);
    case 26: return launchTiled<16, 64, 2, 4, 64, 4>(a, vec, s);
    case 27: return launchTiled<16, 32, 2, 2, 64, 8>(a, vec, s);
    case 28: return launchTiled<32, 16, 2, 2, 64, 4>(a, vec, s);
    case 29:
    case 30:
    case 31: {
      if (!slabOk(a)) return cudaErrorInvalidValue;
      if (variant == 29) return launchSlabCh<4>(a, s);
      if (variant == 30) return launchSlabCh<7>(a, s);
      return launchSlabCh<13>(a, s);
    }
    case 32:
    case 33:
    case 34: {
      if (!slabOk(a)) return cudaErrorInvalidValue;
      if (variant == 32) return launchSlabRt<7, 4, false>(a, s);
      if (variant == 33) return launchSlabRt<4, 4, false>(a, s);
      return launchSlabRt<4, 2, false>(a, s);
    }
    case 35:
    case 36:
    case 37: {
      if (!slabOk(a)) return cudaErrorInvalidValue;
      if (variant == 35) return launchSlabRt<7, 4, true>(a, s);
      if (variant == 36) return launchSlabRt<4, 4, true>(a, s);
      return launchSlabRt<4, 2, true>(a, s);
    }
    case 38:
    case 39: {
      // warp per batch; `threads` carries the warps per CTA (0 = 4)
      if (!slabOk(a)) return cudaErrorInvalidValue;
      if (variant == 38) return launchWarpBatch<7, 4>(a, threads, s);
      return launchWarpBatch<4, 4>(a, threads, s);
    }
    case 40:
    case 41:
    case 42:
    case 43:
    case 44:
    case 45:
    case 46:
    case 47:
    case 48:
    case 49:
    case 50: return launchGemmTma(a, variant - 40, s);
    case 51:
    case 52:
    case 53:
      if (!slabOk(a)) return cudaErrorInvalidValue;
      return variant == 51 ? launchSlabCh<5>(a, s) : variant == 52 ? launchSlabCh<6>(a, s) : launchSlabCh<9>(a, s);
    case 19:
    case 20:
    case 21:
    case 22: {
      if (!batchedOk(a)) return cudaErrorInvalidValue;
      const int g = threads;  // the batched variants take their grid size here (0 = auto)
      if (variant == 19) return launchBatched<2, 2>(a, g, s);
      if (variant == 20) return launchBatched<1, 1>(a, g, s);
      if (variant == 21) return launchBatched<2, 1>(a, g, s);
      return launchBatched<1, 2>(a, g, s);
    }
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace k
}  // namespace tcb
