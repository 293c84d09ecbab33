// ops.h — from a specialized TC definition to hand-written kernels.
//
// The reference turns every definition into a generated loop nest
// (pipeline::compile, pipeline.cc:69-101) and runs it on its CPU emulator
// (backend::emulate, emulator.cc:448-559). tc-b200 instead recognises the
// definition — by its positional canonical form (cache::canonicalize, the
// same text the cache keys on) — as one of the registered paper operators
// (tc/ops.tc), binds the caller's tensors to the operands of that
// operator's kernel family, and maps the reference's MappingOptions genes
// onto that family's kernel parameters. A definition with no registered
// form fails with ErrorKind::NoKernel (never a CPU fallback).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "kernels/kernels.cuh"
#include "options.h"
#include "sem.h"

namespace tcb {
namespace ops {

enum class Family { Gemm, FcChain, Kru3, Gconv, Lut };
const char* familyName(Family f);

// A tensor of the run call: inputs[idx] (parameters, declaration order) or
// outputs[idx] (returns, declaration order).
struct Ref {
  bool out = false;
  int idx = -1;
  bool valid() const { return idx >= 0; }
};

struct GemmDesc {
  Ref A, B, C, bias;
  int batch = 1, M = 0, N = 0, K = 0;
  int64_t lda = 0, ldb = 0, ldc = 0, sA = 0, sB = 0, sC = 0;
  int init = k::kInitZero, relu = 0;
};
struct FcLayerDesc {
  Ref W, bias, O;
  int out = 0, kred = 0;
  int64_t ldw = 0;
};
struct FcDesc {
  Ref I;
  int64_t ldi = 0;
  int batch = 0;
  std::vector<FcLayerDesc> layers;
};
struct KruDesc {
  Ref W0, W1, W2, X, Y, XW1, XW2;
  int M = 0, N0 = 0, N1 = 0, N2 = 0, D0 = 0, D1 = 0, D2 = 0;
};
struct GconvDesc {
  Ref I, W1, B, O;
  int N = 0, G = 0, C = 0, H = 0, W = 0, F = 0, KH = 0, KW = 0, Mb = 0;
};
struct LutTable {
  Ref LUT, I, O;
  int64_t E = 0;
  int D = 0, B = 0, L = 0;
};

struct Problem {
  std::string form;  // registered def name in tc/ops.tc
  Family family = Family::Gemm;
  GemmDesc gemm;
  FcDesc fc;
  KruDesc kru;
  GconvDesc gconv;
  std::vector<LutTable> lut;
  double flops = 0;  // algorithmic FLOPs per call (2 per multiply-add)
  double bytes = 0;  // algorithmic HBM bytes per call (inputs once, outputs once, in/out read once)
};

struct Mapping {
  // arithmetic: k::kMathFfma (the exact FFMA kernels, default) or a
  // tensor-core mode (k::kMathTf32 / k::kMath3xTf32, tc_gemm.cu)
  int math = k::kMathFfma;
  k::TcPlan tc;  // tensor-core tile plan (math != FFMA); per-layer plans are derived at launch
  bool tcAuto = true;
  bool tcFused = false;  // FC chains in tensor-core math: the one-kernel chain (tc_fc_fused.cu)
  bool tcFc2 = false;    // ... or the fused two-layer split-K kernel (tc_gemm.cu, launchTcFc2)
  // Gemm (and unfused FC layers)
  int gemmVariant = 4, gemmThreads = 0;
  // FcChain
  bool fused = true;
  int fcKind = 0;  // fused: 0 = cluster kernel (fc_chain.cu), 1 = register chains (fc_regs.cu)
  int fcLoads = 0;  // cluster kernel loads: 0 automatic, 1 bulk copies, 2 cp.async (chunked), 3 cp.async,
                    // 4 layer 0 by TMA tensor copies in reduction chunks (fc_tma.cu)
  int rows = 1, cn = 1, threads = 128;
  // Kru3
  int dchunk = 16;
  // Gconv
  int gconvVariant = 0, th = 4;
  std::string describe() const;
  Family family = Family::Gemm;
};

// Registered forms: canonical text → def name, from the embedded tc/ops.tc.
const std::string& opsSource();
std::vector<std::string> registeredForms();
std::string formOf(const std::string& canonicalTc);  // "" if unregistered

Problem match(const sem::Specialized& s, const std::string& canonicalTc);  // Error(NoKernel)
// math: k::MathMode. Tensor-core modes exist for the GEMM-NT family
// (TMM, TBMM, C3), the FC chains (per-layer GEMMs), gconv (implicit GEMM)
// and 3-KRU (three chained GEMMs); the LUT family raises MappingInvalid.
Mapping decode(const Problem& p, const MappingOptions& o, int math = k::kMathFfma);  // Error(MappingInvalid)
MappingOptions defaultOptions(const Problem& p, int math = k::kMathFfma);
const char* mathName(int math);
int mathFromName(const std::string& s);  // Error(MappingInvalid)

// Gene pools for the tuner (TuningSpace per family; see tuner.cc).
struct GenePools {
  std::vector<int64_t> tile0, tile1, tile2, tx, ty, tz;
  std::vector<int64_t> bz{1};  // block_shape[2]: tensor-core K splits (1 for the FFMA families)
  std::vector<Fusion> fusion;
  std::vector<int> useShared;  // {0,1} or {1}
};
GenePools genePools(const Problem& p, int math = k::kMathFfma);
// the tuner's acceptance bound for a tensor-core candidate against the
// default tensor-core plan of the same problem (accumulation order only),
// max |got - ref| / max(|ref|, 1); see ops.cc
double tcTolerance(const Problem& p, int math);

// Batch sharding: every registered form has one
// independent outer dimension (TBMM/C3/TMM/FC rows, 3-KRU M, gconv N, LUT B)
// with no reduction across it. shardExtent() is its length; shardOf()
// rewrites a problem and its tensor pointers so the launch covers only
// [lo, hi) of that dimension, reading and writing the full tensors in place.
int64_t shardExtent(const Problem& p);
void shardRange(int64_t n, int rank, int world, int64_t* lo, int64_t* hi);  // balanced contiguous split
Problem shardOf(const Problem& p, int64_t lo, int64_t hi, std::vector<void*>& in, std::vector<void*>& out);

// Launches the whole definition on `stream`. in/out are device pointers in
// declaration order. errFlag: device int for data-dependent index checks.
void launch(const Problem& p, const Mapping& m, void* const* in, void* const* out, int* errFlag,
            cudaStream_t stream);

}  // namespace ops
}  // namespace tcb
