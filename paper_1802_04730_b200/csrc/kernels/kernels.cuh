// kernels.cuh — launch interfaces of the hand-written sm_100a kernels.
//
// Every kernel here is "FFMA-exact": each output element is produced by a
// single thread that runs the reference's reduction chain in canonical
// order — init value, then acc = fma(a_k, b_k, acc) for k ascending — so
// the result matches the reference interpreter
// (interpreter.cc:218-233: double combine + float narrowing per step) up to
// double-rounding ties of the fused step (≈2^-29 per step; none observed
// on the golden vectors). No kernel reassociates a reduction.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace tcb {
namespace k {

// Sets a kernel's dynamic shared-memory limit (and, when asked, the
// non-portable cluster size permission) on the current device, once per
// (kernel, device, size): function attributes belong to a device context, and
// a cudaFuncSetAttribute on every launch costs host time on the paper's
// synchronised-call protocol. Thread-safe (attr.cu).
cudaError_t ensureFuncAttrs(const void* fn, int smemBytes, bool nonPortableCluster = false);

// ------------------------------------------------------------- GEMM-NT
// C[b][m][n] = epi(init + sum_k A[b][m][k] * B[b][n][k]),  k ascending.
enum InitMode : int { kInitZero = 0, kInitInout = 1, kInitBias = 2 };

struct GemmArgs {
  const float* A;
  const float* B;
  float* C;
  const float* bias;  // kInitBias: bias[n]
  int batch, M, N, K;
  int64_t lda, ldb, ldc;     // row strides (elements)
  int64_t sA, sB, sC;        // batch strides (elements); 0 ⇒ broadcast
  int init;                  // InitMode
  int relu;                  // epilogue fmaxf(acc, 0)
};

// variant ids: see gemm.cu kGemmVariants
struct GemmVariant {
  int id;
  int tm, tn, rm, rn, tk;  // tm==0 ⇒ "direct" (no smem staging, 1 output / thread)
  const char* name;
  int stages = 4;          // cp.async ring depth
};
int gemmVariantCount();
const GemmVariant& gemmVariant(int i);
// threads: the direct variant's block size (≥32, multiple of 32, ≤1024);
// for the persistent batched variants (tk == 0) the grid size (0 = auto)
cudaError_t launchGemm(const GemmArgs& a, int variant, int threads, cudaStream_t s);
// whether the persistent batched variants can take this problem (16-byte
// rows/strides/pointers, one batch's operands fit a shared-memory stage)
bool batchedOk(const GemmArgs& a);
// whether the slab variants (tk == -1) can take this problem: K % 4 == 0,
// K <= 144 (at most six 24-step reduction chunks), 16-byte rows/strides/pointers
bool slabOk(const GemmArgs& a);
// TMA-fed tiles (gemm_tma.cu): 16-byte aligned operands and strides
bool gemmTmaOk(const GemmArgs& a);
cudaError_t launchGemmTma(const GemmArgs& a, int which, cudaStream_t s);

// ------------------------------------------------- GEMM-NT, tensor cores
// tcgen05 .kind::tf32 variant of the same contraction (tc_gemm.cu). Not
// FFMA-exact: selected only when the caller asks for tensor-core math.
enum MathMode : int { kMathFfma = 0, kMathTf32 = 1, kMath3xTf32 = 3 };
struct TcPlan {
  int bn = 128;     // output columns per CTA (UMMA N, multiple of 16 in [16, 256])
  int splits = 1;   // K splits = cluster size along z (power of two <= 16)
  int packP = 0;    // > 1: block-diagonal packing of packP small batches per 128-row tile
};
bool tcGemmSupported(const GemmArgs& a, const char** why);
TcPlan tcGemmPlan(int batch, int M, int N, int K, int sms);
cudaError_t launchTcGemm(const GemmArgs& a, int math, const TcPlan& plan, cudaStream_t s);

// ------------------------------------------------------------ FC chain
// Fused FC+bias+ReLU layers (MLP1 / 2FCRelu / MLP3): a cluster of `cn` CTAs
// per `rows` batch rows; output features split across the cluster,
// activations exchanged over DSMEM between layers.
constexpr int kMaxLayers = 4;
constexpr int kFcMaxThreads = 256;  // fused chain block size bound (register budget, fc_chain.cu)
struct FcLayer {
  const float* W;     // [out][ldw]
  const float* bias;  // [out]
  float* O;           // [batch][out] (global output of this layer)
  int out, kred;      // output features, reduction length
  int64_t ldw;
};
struct FcChainArgs {
  const float* I;  // [batch][ldi] first-layer input
  int64_t ldi;
  int batch;
  int layers;
  FcLayer L[kMaxLayers];
};
// loads: 0 = automatic (bulk copies), 1 = bulk copies, 2 = 16-byte cp.async
// with layer 0 in reduction chunks, 3 = cp.async in one chunk, 4 = layer 0 by
// TMA tensor copies in reduction chunks (fc_tma.cu)
cudaError_t launchFcChain(const FcChainArgs& a, int rows, int cn, int threads, cudaStream_t s, int loads = 0);
size_t fcChainSmem(const FcChainArgs& a, int rows, int cn);
int fcChainThreads(const FcChainArgs& a, int rows, int cn);  // single-pass block size
// register-resident chains (fc_regs.cu): every layer kred <= 128, one CTA per
// `rows` (1, 2, 4) batch rows, one warp group per layer, weights in registers
bool fcRegsSupported(const FcChainArgs& a, int rows, const char** why);
// one-kernel tcgen05 FC chain (tc_fc_fused.cu): every layer in one CTA per
// 128 rows, activations TMEM -> shared memory -> next layer's A operand
bool tcFcFusedSupported(const FcChainArgs& a, int math, const char** why);
cudaError_t launchTcFcFused(const FcChainArgs& a, int math, cudaStream_t s);
// two FC layers in one tcgen05 launch (tc_gemm.cu): layer 1 split-K over a
// cluster, layer 2 in rank 0 from the reduced rows (2FCRelu at K = 1128)
bool tcFc2Supported(const FcChainArgs& a, int math, const char** why);
cudaError_t launchTcFc2(const FcChainArgs& a, int math, int sms, cudaStream_t s);
cudaError_t launchFcRegs(const FcChainArgs& a, int rows, cudaStream_t s);
// the cluster kernel with layer 0 streamed in by TMA tensor copies in 256-step
// reduction chunks (fc_tma.cu): layer 0's chains start on the first chunk
bool fcTmaSupported(const FcChainArgs& a, int rows, int cn, const char** why);
cudaError_t launchFcTma(const FcChainArgs& a, int rows, int cn, int threads, cudaStream_t s);

// ------------------------------------------------------------------ KRU
struct KruArgs {
  const float *W0, *W1, *W2, *X;
  float *Y, *XW1, *XW2;
  int M, N0, N1, N2, D0, D1, D2;
};
cudaError_t launchKru3(const KruArgs& a, int dchunk, int threads, cudaStream_t s);
size_t kru3Smem(const KruArgs& a, int dchunk);
// tensor-core 3-KRU (tc_kru.cu): N0 = N1 = N2 = 16, D0 = D1 in {16, 32}, D2 % 16 == 0
bool tcKru3Supported(const KruArgs& a, const char** why);
cudaError_t launchTcKru3(const KruArgs& a, int math, cudaStream_t s);

// ---------------------------------------------------------------- gconv
struct GconvArgs {
  const float* I;   // [N][G][C][H][W]
  const float* W1;  // [G][F][C][KH][KW]
  const float* B;   // [Mb]
  float* O;         // [N][G][F][Ho][Wo]
  int N, G, C, H, W, F, KH, KW, Mb;
};
struct GconvVariant {
  int id, rf, rw, kw;
  const char* name;
};
int gconvVariantCount();
const GconvVariant& gconvVariant(int i);
cudaError_t launchGconv(const GconvArgs& a, int variant, int th, cudaStream_t s);
// tcgen05 implicit-GEMM gconv (tc_gconv.cu), tensor-core math only
bool tcGconvSupported(const GconvArgs& a, const char** why);
cudaError_t launchTcGconv(const GconvArgs& a, int math, cudaStream_t s);
// the default: NHWC staging copy + TMA-fed tcgen05 (tc_gconv_tma.cu)
cudaError_t launchTcGconvTma(const GconvArgs& a, int math, cudaStream_t s);
// shifted-halo implicit GEMM (tc_gconv_shift.cu): one halo tile per 128
// virtual pixels, every tap a shifted K-major descriptor into it
bool tcGconvShiftSupported(const GconvArgs& a, int math, const char** why);
cudaError_t launchTcGconvShift(const GconvArgs& a, int math, cudaStream_t s);
size_t gconvSmem(const GconvArgs& a, int th, int rw);
int gconvThreads(const GconvArgs& a, int variant, int th);

// ------------------------------------------------------------------ LUT
// O[i][j] = sum_k LUT[I[i][k]][j] (k ascending); out-of-range indices set
// *err (IndexOutOfRange) and leave that row's value unspecified.
struct LutArgs {
  const float* LUT;
  const int32_t* I;
  float* O;
  int64_t E;
  int D, B, L;
  int* err;
};
cudaError_t launchLut(const LutArgs* tables, int ntables, int threads, cudaStream_t s);

// --------------------------------------------------------------- concat
constexpr int kMaxConcat = 8;
struct ConcatArgs {
  const float* src[kMaxConcat];
  int off[kMaxConcat + 1];  // column offsets: src s covers [off[s], off[s+1])
  int n;
  int64_t rows, width;
  float* dst;
};
cudaError_t launchConcat(const ConcatArgs& a, cudaStream_t s);

// ------------------------------------------------------ host transfers
// Up to kMaxSeg copies (4-byte multiples) in one launch; host sides are
// mapped pinned pointers. Segments whose pointers and size are 16-byte
// aligned move as int4.
constexpr int kMaxSeg = 16;
struct SegCopyArgs {
  const void* src[kMaxSeg];
  void* dst[kMaxSeg];
  int64_t start[kMaxSeg + 1];  // prefix of per-segment units (16 B or 4 B)
  bool vec16[kMaxSeg];
  int n;
};
void segCopyAdd(SegCopyArgs& a, void* dst, const void* src, int64_t bytes);
cudaError_t launchSegCopy(const SegCopyArgs& a, int sms, cudaStream_t s);

// ---------------------------------------------------------------- probes
// fp32 FFMA throughput of the whole device (TFLOP/s, 2 flops per FMA)
cudaError_t probeFfma(int sms, double* tflops, float* ms);
// device µs per launch of back-to-back empty kernels in a CUDA graph
cudaError_t probeLaunch(int ctas, int threads, int cluster, double* us);

}  // namespace k
}  // namespace tcb
