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
    auto group = [&](int kk) {  // one 4-k step of every chain of the micro-tile
      float4 av[RM], bv[RN];
#pragma unroll
      for (int i = 0; i < RM; ++i) av[i] = *reinterpret_cast<const float4*>(Ast + i * TY * LD + kk);
#pragma unroll
      for (int j = 0; j < RN; ++j) bv[j] = *reinterpret_cast<const float4*>(Bst + j * TX * LD + kk);
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
    const int klim = min(TK, a.K - t * TK);
    if (klim == TK) {
      // full tile: fully unrolled so the scheduler hoists the next group's
      // shared loads above the current group's FFMAs
#pragma unroll
      for (int kk = 0; kk < TK; kk += 4) group(kk);
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
};

template <int TM, int TN, int RM, int RN, int TK, int S = 4>
cudaError_t launchTiled(const GemmArgs& a, int vec, cudaStream_t s) {
  dim3 grid((a.N + TN - 1) / TN, (a.M + TM - 1) / TM, a.batch);
  const size_t smem = (size_t)S * (TM + TN) * (TK + 4) * sizeof(float);
  auto kfn = gemm_nt_tiled<TM, TN, RM, RN, TK, S>;
  static bool attr = false;  // per instantiation
  if (!attr) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  kfn<<<grid, (TM / RM) * (TN / RN), smem, s>>>(a, vec);
  return cudaGetLastError();
}

}  // namespace

int gemmVariantCount() { return sizeof(kGemmVariants) / sizeof(kGemmVariants[0]); }
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
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace k
}  // namespace tcb
