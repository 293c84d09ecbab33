// tc_kru.cu — the 3-factor Kronecker layer on tcgen05
// tensor cores (TF32 / 3xTF32), fused like the FFMA kernel (kru.cu):
//   XW2(m,n0,n1,d2) +=! X(m,n0,n1,r2)   * W2(d2,r2)     step 1
//   XW1(m,n0,d1,d2) +=! XW2(m,n0,r1,d2) * W1(d1,r1)     step 2
//   Y(m,d0,d1,d2)   +=! XW1(m,r0,d1,d2) * W0(d0,r0)     step 3
// A CTA owns (m, a 16-wide chunk of d2). Each step is one UMMA GEMM with a
// K = 16 reduction (two K steps of 8):
//   step 1: rows (n0,n1) x cols d2, A = X[m]      (K-major as stored)
//   step 2: rows (n0,d2) x cols d1, A = XW2 chunk (K = n1)
//   step 3: rows (d1,d2) x cols d0, A = XW1 chunk (K = n0)
// The A operand of steps 2 and 3 is the previous step's result, which the
// epilogue writes straight from TMEM into shared memory in the next step's
// K-major layout ([k/4][row][4 floats]: K-major, no swizzle, 8-row x 16-byte
// core matrices, SBO = 128 B, LBO = one k-plane) while it stores the step's
// return to global memory: every return is written once and the
// intermediates never leave the chip (the FFMA kernel's data flow). The
// weights are the B operands ([k/4][row][4], rows = the output columns).
// 3xTF32 stacks each B as [hi | lo] (N doubled) and issues a_hi*[B] and
// a_lo*[B] per K step; the epilogue adds the column halves.
// Requires N0 = N1 = N2 = 16, D0 = D1 = DN in {16, 32} (compile-time: the
// epilogues' rows stay in registers) and D2 % 16 == 0 (tcKru3Supported). Not FFMA-exact: tensor-core math.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"
#include "sm100.cuh"

namespace tcb {
namespace k {

namespace {

using namespace sm100;

constexpr int kR = 16;   // N0 = N1 = N2: the reduction extent of every step
// d2 chunk per CTA: a template parameter DC (8 or 16); 8 halves the shared
// memory of the step-2/3 operands so more CTAs share an SM
constexpr int kThreadsKru = 128;

// [k/4][rows][4] operand: element (row, k)
__device__ __forceinline__ int kmIdx(int row, int k, int rows) { return ((k >> 2) * rows + row) * 4 + (k & 3); }

template <bool X3>
struct KruCfg {
  // floats of each operand region (hi, then lo for the A operands in 3xTF32)
  __host__ __device__ static int nb(int n) { return X3 ? 2 * n : n; }
  __host__ __device__ static int smemFloats(int D0, int D1, int DC) {
    const int aMul = X3 ? 2 : 1;
    return aMul * (256 * kR) +                         // A1 = X[m] (256 rows = (n0,n1))
           nb(DC) * kR + nb(D1) * kR + nb(D0) * kR +   // B1, B2, B3
           aMul * (kR * DC * kR) +                     // A2 (rows (n0,d2))
           aMul * (D1 * DC * kR);                      // A3 (rows (d1,d2))
  }
};

template <bool X3, int DN, int DC>
__global__ void __launch_bounds__(kThreadsKru) tc_kru3_kernel(const KruArgs a) {
  using Cfg = KruCfg<X3>;
  extern __shared__ uint8_t smraw[];
  float* sm = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  constexpr int D0 = DN, D1 = DN;
  const int D2 = a.D2;
  const int m = blockIdx.y, d2_0 = blockIdx.x * DC;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int nb1 = X3 ? 2 * DC : DC, nb2 = X3 ? 2 * D1 : D1, nb3 = X3 ? 2 * D0 : D0;
  constexpr int rows2 = kR * DC, rows3 = D1 * DC;
  const int aMul = X3 ? 2 : 1;
  float* A1 = sm;                              // hi [, lo at + 256*kR]
  float* B1 = A1 + aMul * 256 * kR;            // [kR/4][nb1][4]
  float* B2 = B1 + nb1 * kR;                   // [kR/4][nb2][4]
  float* B3 = B2 + nb2 * kR;                   // [kR/4][nb3][4]
  float* A2 = B3 + nb3 * kR;                   // hi [, lo]
  float* A3 = A2 + aMul * rows2 * kR;          // hi [, lo]
  uint64_t* bar = reinterpret_cast<uint64_t*>(A3 + aMul * rows3 * kR);
  uint32_t* tmemSlot = reinterpret_cast<uint32_t*>(bar + 1);

  // ---- operands: 16-byte cp.async chunks (a row's 4-float k quad -> its k-plane)
  auto cp16 = [](float* dst, const float* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem(dst)), "l"(src) : "memory");
  };
  const float* Xm = a.X + (int64_t)m * 256 * kR;
  for (int e = tid; e < 256 * 4; e += kThreadsKru) cp16(A1 + (e & 3) * 256 * 4 + (e >> 2) * 4, Xm + e * 4);
  for (int e = tid; e < DC * 4; e += kThreadsKru)
    cp16(B1 + (e & 3) * nb1 * 4 + (e >> 2) * 4, a.W2 + (int64_t)(d2_0 + (e >> 2)) * kR + (e & 3) * 4);
  for (int e = tid; e < D1 * 4; e += kThreadsKru) cp16(B2 + (e & 3) * nb2 * 4 + (e >> 2) * 4, a.W1 + e * 4);
  for (int e = tid; e < D0 * 4; e += kThreadsKru) cp16(B3 + (e & 3) * nb3 * 4 + (e >> 2) * 4, a.W0 + e * 4);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if constexpr (X3) {  // split: A1 lo plane; B rows [n, 2n) = lo of rows [0, n)
    for (int e = tid; e < 256 * kR; e += kThreadsKru) {
      const float x = A1[e], h = rzTf32(x);
      A1[e] = h;
      A1[256 * kR + e] = toTf32(x - h);
    }
    auto splitB = [&](float* B, int n) {
      for (int e = tid; e < n * kR; e += kThreadsKru) {
        const int row = e / kR, k = e - row * kR;
        const float x = B[kmIdx(row, k, 2 * n)], h = rzTf32(x);
        B[kmIdx(row, k, 2 * n)] = h;
        B[kmIdx(n + row, k, 2 * n)] = toTf32(x - h);
      }
    };
    splitB(B1, DC);
    splitB(B2, D1);
    splitB(B3, D0);
  }
  fenceProxyAsyncSmem();
  if (tid == 0) {
    mbarInit(bar, 1);
    fenceBarrierInit();
  }
  // TMEM: step 1 (2 x nb1) then step 2 (2 x nb2) columns, step 3 reuses both
  // (4 x nb3): 128 columns for TF32, so four CTAs' worth fit an SM
  constexpr int kCols = X3 ? 256 : 128;
  if (warp == 0) tmemAlloc<kCols>(tmemSlot);
  tcFenceBefore();
  __syncthreads();
  tcFenceAfter();
  const uint32_t tmem = *tmemSlot;

  // one step: rows/128 row blocks x 2 K steps into TMEM columns col0 + rb*n
  auto mmaStep = [&](const float* A, int rows, const float* B, int n, uint32_t col0, uint32_t parity) {
    if (warp == 0) {
      tcFenceAfter();
      const uint32_t idesc = idescTf32(128, n);
      for (int rb = 0; rb < rows / 128; ++rb)
        for (int ks = 0; ks < 2; ++ks) {
          const uint32_t aoff = (2 * ks * rows + rb * 128) * 16, boff = 2 * ks * n * 16;
          const uint64_t ah = descKInterleave(smem(A) + aoff, rows * 16, 128), bd = descKInterleave(smem(B) + boff, n * 16, 128);
          if (electSync()) {
            mmaTf32(tmem + col0 + rb * n, ah, bd, idesc, ks > 0);
            if constexpr (X3) {
              const uint64_t al = descKInterleave(smem(A + rows * kR) + aoff, rows * 16, 128);
              mmaTf32(tmem + col0 + rb * n, al, bd, idesc, 1);
            }
          }
          __syncwarp();
        }
      if (electSync()) mmaCommit(bar);
      __syncwarp();
    }
    mbarWait(bar, parity, 0);
    tcFenceAfter();
  };
  // TMEM row block rb of this thread's lane quarter: n (+n lo) columns -> v[0, n)
  auto readRow = [&](uint32_t col, auto nConst, float* v) {
    constexpr int n = decltype(nConst)::value;
    const uint32_t t = tmem + (static_cast<uint32_t>(warp * 32) << 16) + col;
#pragma unroll
    for (int c = 0; c < (X3 ? 2 * n : n); c += 16) tmemLoad16(t + c, v + c);
    tmemLoadWait();
    if constexpr (X3) {
#pragma unroll
      for (int j = 0; j < n; ++j) v[j] += v[n + j];  // (hi*hi + lo*hi) + (hi*lo + lo*lo)
    }
  };
  auto putA = [&](float* A, int rows, int row, int k, float x) {  // next step's A (hi [, lo])
    if constexpr (X3) {
      const float h = rzTf32(x);
      A[kmIdx(row, k, rows)] = h;
      A[rows * kR + kmIdx(row, k, rows)] = toTf32(x - h);
    } else {
      A[kmIdx(row, k, rows)] = x;
    }
  };

  // ---- step 1: XW2 rows (n0,n1), cols d2 (chunk)
  mmaStep(A1, 256, B1, nb1, 0, 0);
  for (int rb = 0; rb < 2; ++rb) {
    float v[DC < 16 ? 32 : 2 * DC];  // (x16 TMEM loads: at least 16 columns)
    readRow(rb * nb1, std::integral_constant<int, DC>{}, v);
    const int row = rb * 128 + warp * 32 + lane, n0 = row >> 4, n1 = row & 15;
    float* g = a.XW2 + (((int64_t)m * kR + n0) * kR + n1) * D2 + d2_0;
#pragma unroll
    for (int j = 0; j < DC; j += 4) *reinterpret_cast<float4*>(g + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
#pragma unroll
    for (int j = 0; j < DC; ++j) putA(A2, rows2, n0 * DC + j, n1, v[j]);  // A2 row (n0,d2), k = n1
  }
  tcFenceBefore();
  fenceProxyAsyncSmem();
  __syncthreads();

  // ---- step 2: XW1 rows (n0,d2), cols d1
  const uint32_t c2 = 2 * nb1;  // after step 1's columns
  mmaStep(A2, rows2, B2, nb2, c2, 1);
  for (int rb = 0; rb < rows2 / 128; ++rb) {
    float v[2 * D1];
    readRow(c2 + rb * nb2, std::integral_constant<int, D1>{}, v);
    const int row = rb * 128 + warp * 32 + lane, n0 = row / DC, d2 = row % DC;
    float* g = a.XW1 + ((int64_t)m * kR + n0) * D1 * D2 + d2_0 + d2;
#pragma unroll
    for (int d1 = 0; d1 < D1; ++d1) {
      g[(int64_t)d1 * D2] = v[d1];
      putA(A3, rows3, d1 * DC + d2, n0, v[d1]);  // A3 row (d1,d2), k = n0
    }
  }
  tcFenceBefore();
  fenceProxyAsyncSmem();
  __syncthreads();

  // ---- step 3: Y rows (d1,d2), cols d0 (TMEM columns of steps 1-2 are free again)
  mmaStep(A3, rows3, B3, nb3, 0, 0);
  for (int rb = 0; rb < rows3 / 128; ++rb) {
    float v[2 * D0];
    readRow(rb * nb3, std::integral_constant<int, D0>{}, v);
    const int row = rb * 128 + warp * 32 + lane, d1 = row / DC, d2 = row % DC;
    float* g = a.Y + ((int64_t)m * D0 * D1 + d1) * D2 + d2_0 + d2;
#pragma unroll
    for (int d0 = 0; d0 < D0; ++d0) g[(int64_t)d0 * D1 * D2] = v[d0];
  }
  tcFenceBefore();
  __syncthreads();
  if (warp == 0) {
    tcFenceAfter();
    tmemFree<kCols>(tmem);
  }
}

template <bool X3, int DN, int DC>
cudaError_t launchT(const KruArgs& a, cudaStream_t s) {
  const size_t smemBytes = (size_t)KruCfg<X3>::smemFloats(DN, DN, DC) * 4 + 1024 + 64;
  if (smemBytes > 227 * 1024) return cudaErrorInvalidValue;
  auto kern = tc_kru3_kernel<X3, DN, DC>;
  cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kern), (int)smemBytes);
  if (e != cudaSuccess) return e;
  kern<<<dim3(a.D2 / DC, a.M), kThreadsKru, smemBytes, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

bool tcKru3Supported(const KruArgs& a, const char** why) {
  auto no = [&](const char* w) {
    if (why) *why = w;
    return false;
  };
  if (a.N0 != kR || a.N1 != kR || a.N2 != kR) return no("tensor-core 3-KRU needs N0 = N1 = N2 = 16");
  if (a.D2 % 16) return no("tensor-core 3-KRU needs D2 to be a multiple of 16");
  if (a.D0 != a.D1 || (a.D0 != 16 && a.D0 != 32)) return no("tensor-core 3-KRU needs D0 = D1 = 16 or 32");
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al16(a.X) || !al16(a.W0) || !al16(a.W1) || !al16(a.W2) || !al16(a.XW2))
    return no("tensor-core 3-KRU needs 16-byte aligned tensors");
  if ((size_t)KruCfg<true>::smemFloats(a.D0, a.D1, 16) * 4 + 1088 > 227 * 1024)
    return no("tensor-core 3-KRU operands exceed shared memory");
  return true;
}

cudaError_t launchTcKru3(const KruArgs& a, int math, cudaStream_t s) {
  if (a.M <= 0) return cudaSuccess;
  if (!tcKru3Supported(a, nullptr)) return cudaErrorInvalidValue;
  const bool x3 = math == kMath3xTf32;
  // d2 chunk: 16 for TF32 (21.7 vs 29.2 us at the paper shape), 8 for 3xTF32
  // (38.6 vs 42.1 us: its hi/lo operands need the smaller footprint to share
  // an SM); TCB_KRU_DC overrides (tests run both)
  const char* ev = std::getenv("TCB_KRU_DC");
  const bool dc8 = ev ? std::atoi(ev) == 8 : x3;
  if (a.D0 == 16)  // (step-3 rows D1 * DC must fill 128-row blocks: DC = 8 needs D1 >= 16)
    return x3 ? (dc8 ? launchT<true, 16, 8>(a, s) : launchT<true, 16, 16>(a, s))
              : (dc8 ? launchT<false, 16, 8>(a, s) : launchT<false, 16, 16>(a, s));
  return x3 ? (dc8 ? launchT<true, 32, 8>(a, s) : launchT<true, 32, 16>(a, s))
            : (dc8 ? launchT<false, 32, 8>(a, s) : launchT<false, 32, 16>(a, s));
}

}  // namespace k
}  // namespace tcb
