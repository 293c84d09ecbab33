// ops.cc — operator registry, tensor binding, option decoding, launch.
#include "ops.h"

#include <cmath>
#include <map>
#include <mutex>
#include <sstream>

#include "cache.h"

namespace tcb {
namespace ops {

namespace {

const char* kOpsTc =
#include "ops_tc.inc"
    ;

struct Registry {
  std::map<std::string, std::string> byCanon;  // canonical text → form name
  std::vector<std::string> forms;
};

const Registry& registry() {
  static Registry r;
  static std::once_flag once;
  std::call_once(once, [] {
    lang::Program p = lang::parse(kOpsTc);
    for (const auto& d : p.defs) {
      lang::Validated v = lang::validate(d, &p);
      r.byCanon[cache::canonicalize(v)] = d.name;
      r.forms.push_back(d.name);
    }
  });
  return r;
}

Ref in(int i) { return Ref{false, i}; }
Ref out(int i) { return Ref{true, i}; }

const std::vector<int64_t>& shapeOf(const sem::Specialized& s, const Ref& r) {
  const std::string& name = r.out ? s.v.def.rets[r.idx] : s.v.def.params[r.idx].name;
  return s.shapes.at(name);
}

double vol(const std::vector<int64_t>& v) {
  double n = 1;
  for (auto e : v) n *= static_cast<double>(e);
  return n;
}

[[noreturn]] void invalid(const std::string& m) { fail(ErrorKind::MappingInvalid, m); }

int smCount() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// Tensor-core genes: tile_sizes[1] = UMMA N per CTA (16..256, power of two),
// block_shape[2] = K splits (cluster size, power of two <= 16); a tile N of
// 1 means "plan tile and splits from each contraction's shape" (the FC
// chains' default: every layer gets its own plan).
void decodeTc(const Problem& p, const MappingOptions& o, Mapping& m) {
  if (p.family == Family::Gconv) {
    k::GconvArgs a{};
    a.C = p.gconv.C;
    a.H = p.gconv.H;
    a.W = p.gconv.W;
    a.F = p.gconv.F;
    a.KH = p.gconv.KH;
    a.KW = p.gconv.KW;
    a.Mb = p.gconv.Mb;
    const char* why = nullptr;
    // tile_sizes[2]: 2 = NHWC staging, 3 = shifted halo, else on-chip im2col
    const int sel = o.tileSizes.size() > 2 ? static_cast<int>(o.tileSizes[2]) : 0;
    if (sel == 3) {
      if (!k::tcGconvShiftSupported(a, m.math, &why)) invalid(why);
      m.gconvVariant = 2;
      return;
    }
    if (!k::tcGconvSupported(a, &why)) invalid(why);
    m.gconvVariant = sel == 2 ? 0 : 1;
    return;
  }
  if (p.family == Family::Kru3) {
    k::KruArgs a{};
    a.N0 = p.kru.N0;
    a.N1 = p.kru.N1;
    a.N2 = p.kru.N2;
    a.D0 = p.kru.D0;
    a.D1 = p.kru.D1;
    a.D2 = p.kru.D2;
    const char* why = nullptr;
    if (!k::tcKru3Supported(a, &why)) invalid(why);  // (null pointers pass the alignment check)
    return;
  }
  if (p.family != Family::Gemm && p.family != Family::FcChain)
    invalid(std::string("no tensor-core kernel for the ") + familyName(p.family) +
            " family (tensor-core math covers TMM, TBMM, C3, the FC chains, gconv and 3-KRU)");
  auto ok4 = [](int64_t v) { return v % 4 == 0; };
  if (p.family == Family::Gemm) {
    const GemmDesc& g = p.gemm;
    if (!ok4(g.lda) || !ok4(g.ldb) || (g.batch > 1 && (!ok4(g.sA) || !ok4(g.sB))))
      invalid("tensor-core GEMM needs operand rows and batch strides that are multiples of 16 bytes");
  } else {
    if (!ok4(p.fc.ldi)) invalid("tensor-core FC layers need input rows that are multiples of 16 bytes");
    for (size_t l = 0; l < p.fc.layers.size(); ++l) {
      const auto& L = p.fc.layers[l];
      // a layer's output is the next layer's A operand
      if (!ok4(L.ldw) || (l + 1 < p.fc.layers.size() && !ok4(L.out)))
        invalid("tensor-core FC layers need rows that are multiples of 16 bytes");
    }
  }
  m.fused = false;
  const int64_t fcMode = o.tileSizes.size() > 2 ? o.tileSizes[2] : 0;
  if (p.family == Family::FcChain && fcMode != 1) {
    // the one-kernel chain where every layer fits it (tile_sizes[2] == 1
    // asks for the per-layer tc_gemm launches instead; == 2 for the fused
    // two-layer split-K kernel, a tunable: 2FCRelu TF32 13.8 vs 11.6 us per
    // layer, profiles/r02_tcfc2.txt)
    k::FcChainArgs a{};
    a.layers = static_cast<int>(p.fc.layers.size());
    a.ldi = p.fc.ldi;
    a.batch = p.fc.batch;
    for (int l = 0; l < a.layers; ++l) {
      a.L[l].out = p.fc.layers[l].out;
      a.L[l].kred = p.fc.layers[l].kred;
      a.L[l].ldw = p.fc.layers[l].ldw;
    }
    if (fcMode == 2) {
      const char* why = nullptr;
      if (!k::tcFc2Supported(a, m.math, &why)) invalid(why);
      m.tcFused = true;
      m.tcFc2 = true;
      return;
    }
    if (k::tcFcFusedSupported(a, m.math, nullptr)) {  // (null pointers pass the alignment checks)
      m.tcFused = true;
      return;
    }
  }
  int64_t bn = o.tileSizes.size() > 1 ? o.tileSizes[1] : 0;
  int64_t sp = o.blockShape[2];
  if (bn <= 1) {
    m.tcAuto = true;
    return;
  }
  if (bn != 16 && bn != 32 && bn != 64 && bn != 128 && bn != 256)
    invalid("tensor-core tile N must be one of 16, 32, 64, 128, 256");
  if (sp < 1 || sp > 16 || (sp & (sp - 1))) invalid("tensor-core K splits must be a power of two <= 16");
  m.tcAuto = false;
  m.tc.bn = static_cast<int>(bn);
  m.tc.splits = static_cast<int>(sp);
}

void decodeGemm(const MappingOptions& o, Mapping& m) {
  if (!o.useShared) {
    int t = static_cast<int>(o.threads());
    if (t < 32 || t % 32 != 0) invalid("direct GEMM needs a thread count that is a multiple of 32");
    m.gemmVariant = 0;
    m.gemmThreads = t;
    return;
  }
  if (o.tileSizes.size() < 3) invalid("tiled GEMM needs three tile sizes (rows, cols, reduction depth)");
  if (o.tileSizes[2] == 1) {
    // reduction depth 1 = stage a whole batch per step: the persistent
    // batched kernel, micro-tile tile_sizes[0] x tile_sizes[1], grid
    // block_shape[0] (1 = one or two CTAs per SM)
    const int rm = static_cast<int>(o.tileSizes[0]), rn = static_cast<int>(o.tileSizes[1]);
    for (int i = 1; i < k::gemmVariantCount(); ++i) {
      const auto& v = k::gemmVariant(i);
      if (v.tk == 0 && v.rm == rm && v.rn == rn) {
        m.gemmVariant = i;
        m.gemmThreads = o.blockShape[0] > 1 ? static_cast<int>(o.blockShape[0]) : 0;
        return;
      }
    }
    invalid("persistent batched GEMM micro-tile must be 1x1, 1x2, 2x1 or 2x2");
  }
  if (o.tileSizes[2] == 2) {
    // reduction depth 2 = the slab kernel (one CTA per batch, B rows in
    // registers, A rows broadcast from shared memory); tile_sizes[0] = output
    // rows per warp
    // (tile_sizes[1] == 1, the broadcast slab) or rows x columns per lane
    // (tile_sizes[1] > 1, the register-tiled slab)
    const int ch = static_cast<int>(o.tileSizes[0]), rn = static_cast<int>(o.tileSizes[1]);
    for (int i = 1; i < k::gemmVariantCount(); ++i) {
      const auto& v = k::gemmVariant(i);
      // unroll_copy_shared selects the bulk-copy fill of the register-tiled slab
      // block_shape[0] > 1 selects one warp per batch with that many warps per CTA
      const int tk = rn == 1 ? -1 : o.blockShape[0] > 1 ? -4 : o.unrollCopyShared ? -3 : -2;
      if (v.tk == tk && v.rm == ch && v.rn == rn) {
        m.gemmVariant = i;
        m.gemmThreads = tk == -4 ? static_cast<int>(o.blockShape[0]) : 0;
        return;
      }
    }
    invalid("slab GEMM micro-tile must be 4x1 to 7x1, 9x1, 13x1 (broadcast) or 7x4, 4x4, 4x2 (register-tiled)");
  }
  if (o.tileSizes[2] == 3) {
    // reduction depth 3 = TMA-fed tiles (32-deep stages): tile tm x tn,
    // micro-tile (tm / thread_shape[1]) x (tn / thread_shape[0]);
    // block_shape[1] > 1: the A tile multicast over that many CTAs along N
    const int64_t tm = o.tileSizes[0], tn = o.tileSizes[1], tx = o.threadShape[0], ty = o.threadShape[1];
    const int64_t mc = o.blockShape[1];
    for (int i = 1; i < k::gemmVariantCount(); ++i) {
      const auto& v = k::gemmVariant(i);
      const bool kind = mc > 1 ? (v.tk == -6 && v.stages == mc) : v.tk == -5;
      if (kind && v.tm == tm && v.tn == tn && tx * v.rn == tn && ty * v.rm == tm) {
        m.gemmVariant = i;
        m.gemmThreads = static_cast<int>(tx * ty);
        return;
      }
    }
    invalid("no TMA-fed GEMM kernel for tile " + std::to_string(tm) + "x" + std::to_string(tn) + " with a " +
            std::to_string(tx) + "x" + std::to_string(ty) + " block");
  }
  if (o.threadShape[2] != 1) invalid("tiled GEMM uses a 2-D thread block");
  int64_t tm = o.tileSizes[0], tn = o.tileSizes[1], tk = o.tileSizes[2];
  int64_t tx = o.threadShape[0], ty = o.threadShape[1];
  if (tm % ty || tn % tx) invalid("tile extents must be multiples of the thread block extents");
  const int stages = o.unrollCopyShared ? 8 : 4;  // deeper copy pipeline
  for (int i = 1; i < k::gemmVariantCount(); ++i) {
    const auto& v = k::gemmVariant(i);
    if (v.tm == tm && v.tn == tn && v.tk == tk && v.rm == tm / ty && v.rn == tn / tx && v.stages == stages) {
      m.gemmVariant = i;
      m.gemmThreads = static_cast<int>(tx * ty);
      return;
    }
  }
  invalid("no GEMM kernel instantiated for tile " + std::to_string(tm) + "x" + std::to_string(tn) + "x" +
          std::to_string(tk) + " with a " + std::to_string(tx) + "x" + std::to_string(ty) + " block");
}

void launchGemmDesc(const GemmDesc& g, const Mapping& m, void* const* in, void* const* out, cudaStream_t s) {
  auto ptr = [&](const Ref& r) -> void* { return r.valid() ? (r.out ? out[r.idx] : in[r.idx]) : nullptr; };
  k::GemmArgs a;
  a.A = static_cast<const float*>(ptr(g.A));
  a.B = static_cast<const float*>(ptr(g.B));
  a.C = static_cast<float*>(ptr(g.C));
  a.bias = static_cast<const float*>(ptr(g.bias));
  a.batch = g.batch;
  a.M = g.M;
  a.N = g.N;
  a.K = g.K;
  a.lda = g.lda;
  a.ldb = g.ldb;
  a.ldc = g.ldc;
  a.sA = g.sA;
  a.sB = g.sB;
  a.sC = g.sC;
  a.init = g.init;
  a.relu = g.relu;
  cudaError_t e;
  if (m.math != k::kMathFfma) {
    const char* why = nullptr;
    if (!k::tcGemmSupported(a, &why)) fail(ErrorKind::MappingInvalid, why);
    k::TcPlan pl = m.tcAuto ? k::tcGemmPlan(g.batch, g.M, g.N, g.K, smCount()) : m.tc;
    e = k::launchTcGemm(a, m.math, pl, s);
  } else if ((k::gemmVariant(m.gemmVariant).tk == 0 && !k::batchedOk(a)) ||
             (k::gemmVariant(m.gemmVariant).tk < 0 && k::gemmVariant(m.gemmVariant).tk > -5 && !k::slabOk(a)) ||
             (k::gemmVariant(m.gemmVariant).tk <= -5 && !k::gemmTmaOk(a))) {
    // the persistent batched and slab kernels need 16-byte aligned operands
    // (and the slab K <= 144); the tiled kernel computes the same bit-exact
    // chains without that need
    e = k::launchGemm(a, 4, 256, s);
  } else {
    e = k::launchGemm(a, m.gemmVariant, m.gemmThreads, s);
  }
  if (e != cudaSuccess) fail(ErrorKind::Cuda, std::string("GEMM launch failed: ") + cudaGetErrorString(e));
}

}  // namespace

const char* familyName(Family f) {
  switch (f) {
    case Family::Gemm: return "gemm_nt";
    case Family::FcChain: return "fc_chain";
    case Family::Kru3: return "kru3";
    case Family::Gconv: return "gconv";
    case Family::Lut: return "lut";
  }
  return "?";
}

const std::string& opsSource() {
  static const std::string s(kOpsTc);
  return s;
}

std::vector<std::string> registeredForms() { return registry().forms; }

std::string formOf(const std::string& canon) {
  const auto& r = registry();
  auto f = r.byCanon.find(canon);
  return f == r.byCanon.end() ? std::string() : f->second;
}

std::string Mapping::describe() const {
  std::ostringstream os;
  os << familyName(family) << ":";
  if (math != k::kMathFfma) {
    os << "tcgen05 " << mathName(math);
    if (family == Family::Kru3) return os.str() + " fused 3-step (TMEM -> next step's A in smem)";
    if (family == Family::Gconv)
      return os.str() + (gconvVariant == 1   ? " implicit-GEMM (on-chip im2col)"
                         : gconvVariant == 2 ? " implicit-GEMM (shifted halo)"
                                             : " implicit-GEMM (NHWC staging)");
    if (family == Family::FcChain && tcFused && tcFc2)
      return os.str() + " fused 2-layer (split-K cluster; layer 2 in rank 0 from the reduced rows)";
    if (family == Family::FcChain && tcFused) return os.str() + " fused chain (TMEM -> next layer's A in smem)";
    if (tcAuto) os << " planned";
    else os << " bn=" << tc.bn << " splits=" << tc.splits;
    if (family == Family::FcChain) os << " per-layer";
    return os.str();
  }
  switch (family) {
    case Family::Gemm:
      if (k::gemmVariant(gemmVariant).tk == -4)
        os << k::gemmVariant(gemmVariant).name << " warps=" << gemmThreads;
      else if (k::gemmVariant(gemmVariant).tk < 0 && k::gemmVariant(gemmVariant).tk > -5)
        os << k::gemmVariant(gemmVariant).name;
      else if (k::gemmVariant(gemmVariant).tk == 0)
        os << k::gemmVariant(gemmVariant).name << " grid=" << (gemmThreads ? std::to_string(gemmThreads) : "auto");
      else
        os << k::gemmVariant(gemmVariant).name << " threads=" << gemmThreads;
      break;
    case Family::FcChain:
      if (fused && fcKind == 1) os << "registers rows=" << rows;
      else if (fused)
        os << "cluster rows=" << rows << " cn=" << cn << " threads=" << threads
           << (fcLoads == 1   ? " loads=bulk"
               : fcLoads == 2 ? " loads=cp.async"
               : fcLoads == 3 ? " loads=cp.async/1"
               : fcLoads == 4 ? " loads=tma-chunks"
                              : "");
      else os << "per-layer " << k::gemmVariant(gemmVariant).name << " threads=" << gemmThreads;
      break;
    case Family::Kru3: os << "fused dchunk=" << dchunk << " threads=" << threads; break;
    case Family::Gconv: os << k::gconvVariant(gconvVariant).name << " th=" << th; break;
    case Family::Lut: os << "gather threads=" << threads; break;
  }
  return os.str();
}

Problem match(const sem::Specialized& s, const std::string& canon) {
  std::string form = formOf(canon);
  if (form.empty())
    fail(ErrorKind::NoKernel, "definition '" + s.v.def.name +
                                  "' matches no hand-written kernel family (recognised forms: tmm, tbmm, C3, "
                                  "MLP1, 2FCRelu, MLP3, 3KRU, gconv, 2LUT, 1LUT)");
  Problem p;
  p.form = form;
  auto sh = [&](const Ref& r) { return shapeOf(s, r); };
  auto i32 = [](int64_t v) {
    if (v > INT32_MAX) fail(ErrorKind::NoKernel, "extent exceeds the 32-bit kernel index range");
    return static_cast<int>(v);
  };

  if (form == "tmm" || form == "tbmm" || form == "C3") {
    p.family = Family::Gemm;
    GemmDesc& g = p.gemm;
    g.A = in(0);
    g.B = in(1);
    g.C = out(0);
    const auto &a = sh(g.A), &b = sh(g.B), &c = sh(g.C);
    if (form == "tbmm") {
      g.batch = i32(a[0]);
      g.M = i32(a[1]);
      g.N = i32(b[1]);
      g.K = i32(std::min(a[2], b[2]));
      g.lda = a[2];
      g.ldb = b[2];
      g.ldc = c[2];
      g.sA = a[1] * a[2];
      g.sB = b[1] * b[2];
      g.sC = c[1] * c[2];
    } else {
      g.M = i32(a[0]);
      g.N = i32(b[0]);
      g.K = i32(std::min(a[1], b[1]));
      g.lda = a[1];
      g.ldb = b[1];
      g.ldc = c[1];
    }
    g.init = form == "C3" ? k::kInitInout : k::kInitZero;
    p.flops = 2.0 * g.batch * g.M * g.N * g.K;
    p.bytes = 4.0 * (vol(a) + vol(b) + vol(c) * (form == "C3" ? 2 : 1));
    return p;
  }
  if (form == "MLP1" || form == "2FCRelu" || form == "MLP3") {
    p.family = Family::FcChain;
    FcDesc& f = p.fc;
    int nl = form == "MLP1" ? 1 : form == "2FCRelu" ? 2 : 3;
    // MLP1/2FCRelu read I = param 0; MLP3 reads the pass-through return O1
    f.I = form == "MLP3" ? out(0) : in(0);
    const auto& I = sh(f.I);
    f.ldi = I[1];
    f.batch = i32(I[0]);
    int64_t prevOut = I[1];
    p.bytes = 4.0 * vol(I);
    for (int l = 0; l < nl; ++l) {
      FcLayerDesc L;
      L.W = in(1 + 2 * l);
      L.bias = in(2 + 2 * l);
      L.O = out(form == "MLP3" ? 1 + l : l);
      const auto& W = sh(L.W);
      L.out = i32(W[0]);
      L.ldw = W[1];
      L.kred = i32(std::min(prevOut, W[1]));  // reduction range = intersection (ranges.cc)
      prevOut = L.out;
      p.flops += 2.0 * f.batch * L.out * L.kred;
      p.bytes += 4.0 * (vol(W) + vol(sh(L.bias)) + (double)f.batch * L.out);
      f.layers.push_back(L);
    }
    return p;
  }
  if (form == "3KRU") {
    p.family = Family::Kru3;
    KruDesc& k = p.kru;
    k.W0 = in(0);
    k.W1 = in(1);
    k.W2 = in(2);
    k.X = in(3);
    k.Y = out(0);
    k.XW1 = out(1);
    k.XW2 = out(2);
    const auto& X = sh(k.X);
    k.M = i32(X[0]);
    k.N0 = i32(X[1]);
    k.N1 = i32(X[2]);
    k.N2 = i32(X[3]);
    k.D0 = i32(sh(k.W0)[0]);
    k.D1 = i32(sh(k.W1)[0]);
    k.D2 = i32(sh(k.W2)[0]);
    double m = k.M;
    p.flops = 2.0 * m *
              ((double)k.N0 * k.N1 * k.D2 * k.N2 + (double)k.N0 * k.D1 * k.D2 * k.N1 + (double)k.D0 * k.D1 * k.D2 * k.N0);
    p.bytes = 4.0 * (vol(X) + vol(sh(k.W0)) + vol(sh(k.W1)) + vol(sh(k.W2)) + vol(sh(k.Y)) + vol(sh(k.XW1)) +
                     vol(sh(k.XW2)));
    return p;
  }
  if (form == "gconv") {
    p.family = Family::Gconv;
    GconvDesc& g = p.gconv;
    g.I = in(0);
    g.W1 = in(1);
    g.B = in(2);
    g.O = out(0);
    const auto &I = sh(g.I), &W = sh(g.W1);
    g.N = i32(I[0]);
    g.G = i32(I[1]);
    g.C = i32(I[2]);
    g.H = i32(I[3]);
    g.W = i32(I[4]);
    g.F = i32(W[1]);
    g.KH = i32(W[3]);
    g.KW = i32(W[4]);
    g.Mb = i32(sh(g.B)[0]);
    double outs = vol(sh(g.O));
    p.flops = outs * (2.0 * g.C * g.KH * g.KW + g.Mb);
    p.bytes = 4.0 * (vol(I) + vol(W) + g.Mb + outs);
    return p;
  }
  if (form == "2LUT" || form == "1LUT") {
    p.family = Family::Lut;
    int nt = form == "2LUT" ? 2 : 1;
    for (int t = 0; t < nt; ++t) {
      LutTable T;
      T.LUT = in(2 * t);
      T.I = in(2 * t + 1);
      T.O = out(t);
      const auto &L = sh(T.LUT), &I = sh(T.I);
      T.E = L[0];
      T.D = i32(L[1]);
      T.B = i32(I[0]);
      T.L = i32(I[1]);
      p.flops += (double)T.B * T.L * T.D;
      p.bytes += 4.0 * ((double)T.B * T.L + (double)T.B * T.L * T.D + (double)T.B * T.D);
      p.lut.push_back(T);
    }
    return p;
  }
  fail(ErrorKind::Internal, "registered form '" + form + "' has no binder");
}

const char* mathName(int math) {
  switch (math) {
    case k::kMathFfma: return "ffma";
    case k::kMathTf32: return "tf32";
    case k::kMath3xTf32: return "3xtf32";
  }
  return "?";
}

int mathFromName(const std::string& s) {
  if (s == "ffma" || s.empty()) return k::kMathFfma;
  if (s == "tf32") return k::kMathTf32;
  if (s == "3xtf32") return k::kMath3xTf32;
  invalid("unknown math mode '" + s + "' (ffma | tf32 | 3xtf32)");
}

Mapping decode(const Problem& p, const MappingOptions& o, int math) {
  o.validate();
  Mapping m;
  m.family = p.family;
  if (math != k::kMathFfma) {
    if (math != k::kMathTf32 && math != k::kMath3xTf32) invalid("unknown math mode");
    m.math = math;
    decodeTc(p, o, m);
    return m;
  }
  switch (p.family) {
    case Family::Gemm: decodeGemm(o, m); break;
    case Family::FcChain: {
      if (o.fusion == Fusion::Min) {
        m.fused = false;
        decodeGemm(o, m);
        break;
      }
      m.fused = true;
      m.rows = o.tileSizes.empty() ? 1 : static_cast<int>(o.tileSizes[0]);
      m.cn = o.tileSizes.size() < 2 ? 1 : static_cast<int>(o.tileSizes[1]);
      // tile_sizes[2]: 1 = cluster kernel, automatic loads; 3 / 4 / 5 = cluster
      // kernel with bulk-copy / chunked cp.async / one-chunk cp.async loads;
      // 6 = layer 0 by TMA tensor copies in reduction chunks (fc_tma.cu)
      if (o.tileSizes.size() > 2 && o.tileSizes[2] >= 3 && o.tileSizes[2] <= 6)
        m.fcLoads = static_cast<int>(o.tileSizes[2]) - 2;
      if (o.tileSizes.size() > 2 && o.tileSizes[2] == 2) {
        // tile_sizes[2] == 2: register chains, tile_sizes[0] rows per CTA
        m.fcKind = 1;
        m.cn = 1;
        k::FcChainArgs a{};
        a.layers = static_cast<int>(p.fc.layers.size());
        a.ldi = p.fc.ldi;
        for (int l = 0; l < a.layers; ++l) {
          a.L[l].out = p.fc.layers[l].out;
          a.L[l].kred = p.fc.layers[l].kred;
          a.L[l].ldw = p.fc.layers[l].ldw;
        }
        const char* why = nullptr;  // (null pointers pass the alignment checks)
        if (!k::fcRegsSupported(a, m.rows, &why)) invalid(why);
        m.threads = 0;
        break;
      }
      if (m.rows < 1 || m.rows > 32) invalid("fused FC chain rows per cluster must be in [1, 32]");
      if (m.cn < 1 || m.cn > 16) invalid("fused FC chain cluster size must be in [1, 16]");
      m.threads = static_cast<int>(o.threads());
      if (m.threads < 32 || m.threads % 32 || m.threads > k::kFcMaxThreads)
        invalid("fused FC chain needs a multiple of 32 threads, at most 256");
      k::FcChainArgs a{};
      a.layers = static_cast<int>(p.fc.layers.size());
      a.batch = p.fc.batch;
      for (int l = 0; l < a.layers; ++l) {
        a.L[l].out = p.fc.layers[l].out;
        a.L[l].kred = p.fc.layers[l].kred;
      }
      if (m.fcLoads == 4) {
        a.ldi = p.fc.ldi;
        for (int l = 0; l < a.layers; ++l) a.L[l].ldw = p.fc.layers[l].ldw;
        const char* why = nullptr;  // (null pointers pass the alignment checks)
        if (!k::fcTmaSupported(a, m.rows, m.cn, &why)) invalid(why);
      } else if (k::fcChainSmem(a, m.rows, m.cn) > 227 * 1024) {
        invalid("fused FC chain exceeds the shared-memory capacity");
      }
      break;
    }
    case Family::Kru3: {
      if (o.fusion == Fusion::Min) invalid("3-KRU is only implemented as one fused kernel");
      m.dchunk = o.tileSizes.empty() ? 16 : static_cast<int>(o.tileSizes[0]);
      m.threads = static_cast<int>(o.threads());
      if (m.threads < 32 || m.threads % 32) invalid("3-KRU needs a multiple of 32 threads");
      k::KruArgs a{};
      a.N0 = p.kru.N0;
      a.N1 = p.kru.N1;
      a.N2 = p.kru.N2;
      a.D0 = p.kru.D0;
      a.D1 = p.kru.D1;
      a.D2 = p.kru.D2;
      if (m.dchunk < 1 || m.dchunk > p.kru.D2) invalid("3-KRU d2 chunk outside [1, D2]");
      if (k::kru3Smem(a, m.dchunk) > 227 * 1024) invalid("3-KRU chunk exceeds the shared-memory capacity");
      break;
    }
    case Family::Gconv: {
      if (o.tileSizes.size() < 3) invalid("gconv needs tile sizes (rows per CTA, filters per thread, columns per thread)");
      m.th = static_cast<int>(o.tileSizes[0]);
      int rf = static_cast<int>(o.tileSizes[1]), rw = static_cast<int>(o.tileSizes[2]);
      m.gconvVariant = -1;
      for (int i = 0; i < k::gconvVariantCount(); ++i) {
        const auto& v = k::gconvVariant(i);
        if (v.rf == rf && v.rw == rw && v.kw == p.gconv.KW) m.gconvVariant = i;
      }
      if (m.gconvVariant < 0) invalid("no gconv kernel instantiated for this filter/column micro-tile and KW");
      k::GconvArgs a{};
      a.C = p.gconv.C;
      a.H = p.gconv.H;
      a.W = p.gconv.W;
      a.F = p.gconv.F;
      a.KH = p.gconv.KH;
      a.KW = p.gconv.KW;
      a.Mb = p.gconv.Mb;
      int t = k::gconvThreads(a, m.gconvVariant, m.th);
      if (t > 512) invalid("gconv CTA would exceed 512 threads");
      if (k::gconvSmem(a, m.th, rw) + (size_t)a.C * a.KH * a.KW * (rf * ((a.F + rf - 1) / rf) - a.F) * 4 > 227 * 1024)
        invalid("gconv tile exceeds the shared-memory capacity");
      m.threads = t;
      break;
    }
    case Family::Lut: {
      m.threads = static_cast<int>(o.threads());
      if (m.threads < 32 || m.threads % 32) invalid("LUT gather needs a multiple of 32 threads");
      break;
    }
  }
  return m;
}

MappingOptions defaultOptions(const Problem& p, int math) {
  MappingOptions o;
  if (math != k::kMathFfma && p.family == Family::Gconv) {
    // 128 pixels x F filters; variant 3 = shifted halo (the fastest at the
    // paper shape, profiles/experiments/r01_gconv_shift_tuning.txt), else 1 =
    // on-chip im2col where the halo ring does not fit
    k::GconvArgs a{};
    a.C = p.gconv.C;
    a.H = p.gconv.H;
    a.W = p.gconv.W;
    a.F = p.gconv.F;
    a.KH = p.gconv.KH;
    a.KW = p.gconv.KW;
    a.Mb = p.gconv.Mb;
    const int variant = k::tcGconvShiftSupported(a, math, nullptr) ? 3 : 1;
    o.tileSizes = {128, static_cast<int64_t>(p.gconv.F), variant};
    o.threadShape = {{512, 1, 1}};
    o.useShared = true;
    return o;
  }
  if (math != k::kMathFfma && (p.family == Family::Gemm || p.family == Family::FcChain)) {
    // tile N = 1: plan tile, K splits and batch packing from the shape at
    // launch (k::tcGemmPlan); the tuner explores explicit values
    o.tileSizes = {128, 1, 32};
    o.blockShape = {{1, 1, 1}};
    o.threadShape = {{256, 1, 1}};
    o.useShared = true;
    o.fusion = Fusion::Min;
    return o;
  }
  switch (p.family) {
    case Family::Gemm: {
      // start from the reference's contraction preset (options.cc:182-191:
      // 32x32 tile, 16x16 threads, 2x2 micro-tile) and adapt the tile to
      // the problem: finer tiles when the grid would not cover the SMs, an
      // 8-deep copy ring when the reduction is long
      o = baselineOptions()[0];
      const GemmDesc& g = p.gemm;

      auto ctas = [&](int tm, int tn) { return (double)g.batch * ((g.M + tm - 1) / tm) * ((g.N + tn - 1) / tn); };
      o.unrollCopyShared = g.K > 128;
      if (g.batch > 1 && g.K % 4 == 0 && g.K <= 144 && g.M <= 64 && g.N <= 256) {
        // many small batches (TBMM 500 x 26x26x72): the slab kernel, one
        // CTA per batch, 9 output rows per warp (3 warps for 26 rows; 6.7 us
        // alone vs 6.8 for 7 rows, 15.2 vs 15.7 us in the bench step,
        // profiles/r02_slab_rows.txt)
        o.tileSizes = {g.M <= 16 ? 4 : 9, 1, 2};
        o.threadShape = {{32, 1, 1}};
        o.unrollCopyShared = false;
        break;
      }
      if (g.K > 128 && ctas(32, 32) >= 96) {
        // long reductions with enough 32x32 tiles: the TMA-fed tiles (8 x 32-
        // deep stages in flight; C3 and TMM 128x1024x1024 21.6 -> 16.9 us,
        // profiles/r02_tma_sweep.txt); the tiled kernel's cp.async ring where
        // the operands cannot take a tensor map (ops::launchGemmDesc)
        o.tileSizes = {32, 32, 3};
        o.threadShape = {{16, 16, 1}};
        o.blockShape = {{1, 1, 1}};
        o.unrollCopyShared = false;
        break;
      }
      if (ctas(32, 32) < 148) {
        if (o.unrollCopyShared) {
          o.tileSizes = {16, 32, 32};
          o.threadShape = {{16, 8, 1}};
        } else {
          o.tileSizes = {16, 16, 32};
          o.threadShape = {{16, 16, 1}};
        }
      }
      break;
    }
    case Family::FcChain: {
      // clusters of up to 8 CTAs split the widest layer into ~16-column
      // slices; rows per cluster chosen so the grid covers ~128 CTAs
      int outMax = 0;
      for (const auto& L : p.fc.layers) outMax = std::max(outMax, L.out);
      int cn = std::min(8, std::max(1, (outMax + 15) / 16));
      k::FcChainArgs a{};
      a.layers = static_cast<int>(p.fc.layers.size());
      for (int l = 0; l < a.layers; ++l) {
        a.L[l].out = p.fc.layers[l].out;
        a.L[l].kred = p.fc.layers[l].kred;
      }
      // aim at ~2 co-resident CTAs per SM (>= 200 CTAs): a wave of 1-CTA/SM
      // 8-clusters does not fit the GPCs (max 15 active of 16 on B200).
      // Chains with small slices (<= 32 KB per CTA) go to >= 128 fatter CTAs:
      // MLP3 rows 2 -> 4 is as fast alone and overlaps better in the bench
      // step (profiles/r01_step_variants.txt)
      int rows = 1;
      while (rows < 16) {
        const int nr = rows * 2;
        const int64_t ctas = (int64_t)((p.fc.batch + nr - 1) / nr) * cn;
        if (ctas < (k::fcChainSmem(a, nr, cn) <= 32 * 1024 ? 128 : 200)) break;
        rows = nr;
      }
      while (rows > 1 && k::fcChainSmem(a, rows, cn) > 110 * 1024) rows /= 2;
      int t = std::max(64, k::fcChainThreads(a, rows, cn));  // one pass per layer
      // long first reductions (MLP1, 2FCRelu: K = 1128): half the block, two
      // columns per thread in layer 0 (fc_chain.cu chainSegment2): MLP1 6.70
      // -> 6.20 us, 2FCRelu 7.81 -> 7.57 alone, 16.1 -> 15.3-15.8 in the bench
      // step; MLP3 (K = 128) measured slower that way (6.1 vs 5.3)
      if (a.L[0].kred >= 512 && ((a.L[0].out + cn - 1) / cn) % 2 == 0 && a.L[0].kred % 4 == 0 && t % 64 == 0)
        t /= 2;
      a.ldi = p.fc.ldi;
      for (int l = 0; l < a.layers; ++l) a.L[l].ldw = p.fc.layers[l].ldw;
      o.tileSizes = {rows, cn, 1};
      o.threadShape = {{t, 1, 1}};
      o.fusion = Fusion::Max;
      o.useShared = true;
      break;
    }
    case Family::Kru3:
      o.tileSizes = {std::min<int64_t>(16, p.kru.D2), 1, 1};
      o.threadShape = {{256, 1, 1}};
      o.useShared = true;
      break;
    case Family::Gconv: {
      int Wo = p.gconv.W - p.gconv.KW + 1, Ho = p.gconv.H - p.gconv.KH + 1;
      int rw = (p.gconv.KW == 3 && Wo % 7 == 0) ? 7 : 4;
      int rf = 4;
      if (p.gconv.KW != 3) rw = 4;
      o.tileSizes = {4, rf, rw};
      // small images: one CTA covers more rows (its filter staging is shared by
      // more work); measured on the paper's four gconv columns
      // (profiles/r01_gconv_columns_sweep.txt): 14x14 F16 rf4 x 7 rows 127 -> 63 us,
      // 7x7 F32 rf2 x 7 rows 308 -> 104 us, 28x28 F8 and 56x56 F4 rf2 x 14 rows
      // 108 -> 66 us and 109 -> 72 us; the 56x56 F16 shape keeps rf4 x 4 rows
      if (rw == 7 && Ho % 7 == 0 && Ho <= 14) {
        rf = p.gconv.F >= 32 ? 2 : 4;
        o.tileSizes = {7, rf, rw};
        break;
      }
      if (rw == 7 && Ho % 14 == 0 && p.gconv.F <= 8 && (Wo / 7) * 14 * ((p.gconv.F + 1) / 2) <= 512) {
        rf = 2;
        o.tileSizes = {14, rf, rw};
        break;
      }
      o.threadShape = {{1, 1, 1}};
      o.useShared = true;
      // shrink rows-per-CTA until the CTA fits 512 threads
      k::GconvArgs a{};
      a.W = p.gconv.W;
      a.KW = p.gconv.KW;
      a.F = p.gconv.F;
      for (int th : {4, 2, 1}) {
        o.tileSizes[0] = th;
        int v = -1;
        for (int i = 0; i < k::gconvVariantCount(); ++i)
          if (k::gconvVariant(i).rf == rf && k::gconvVariant(i).rw == rw && k::gconvVariant(i).kw == p.gconv.KW) v = i;
        if (v >= 0 && k::gconvThreads(a, v, th) <= 512) break;
      }
      break;
    }
    case Family::Lut:
      o.threadShape = {{256, 1, 1}};
      break;
  }
  return o;
}

double tcTolerance(const Problem& p, int math) {
  // Two tensor-core plans of one problem round their operands identically
  // (tf32: the MMA's truncation; 3xtf32: the hi/lo split), so they differ
  // only in the order their fp32 accumulators add up the K products (split-K
  // partials, MMA grouping). That difference is ~K * 2^-24 * |partial sums|:
  // the bound is 4 * K * 2^-24 per contraction (tests/tc_emulate.py, the
  // same accumulator-only bound the GPU parity tests hold the kernels to
  // against an fp64 emulation, doubled for two plans; x3 for 3xtf32, which
  // issues three MMAs into the accumulator per k). Chained contractions
  // (FC layers, 3-KRU) carry a layer's difference into the next layer's sum
  // over its inputs, so their bound is 64 * sum(K) * 2^-24. A plan that drops
  // or repeats a 32-deep k-block is off by ~1e-1 relative, far outside both.
  const double u = std::ldexp(1.0, -24) * (math == k::kMath3xTf32 ? 3 : 1);
  switch (p.family) {
    case Family::Gemm: return 4.0 * p.gemm.K * u;
    case Family::Gconv: return 4.0 * ((double)p.gconv.C * p.gconv.KH * p.gconv.KW + p.gconv.Mb) * u;
    case Family::FcChain: {
      double k = 0;
      for (const auto& L : p.fc.layers) k += L.kred;
      return 64.0 * k * u;
    }
    case Family::Kru3: return 64.0 * ((double)p.kru.N0 + p.kru.N1 + p.kru.N2) * u;
    default: return 0.0;
  }
}

GenePools genePools(const Problem& p, int math) {
  GenePools g;
  if (math != k::kMathFfma) {
    g.tx = {256};
    g.ty = {1};
    g.tz = {1};
    g.useShared = {1};
    g.fusion = {Fusion::Min};
    if (p.family == Family::Gconv) {
      g.tile0 = {128};
      g.tile1 = {static_cast<int64_t>(p.gconv.F)};
      // the shifted-halo kernel where it applies: the on-chip im2col and NHWC
      // staging variants measured ~4x slower there (dead weight
      // in the pool); they remain the fallback for shapes it cannot take
      k::GconvArgs a{};
      a.C = p.gconv.C;
      a.H = p.gconv.H;
      a.W = p.gconv.W;
      a.F = p.gconv.F;
      a.KH = p.gconv.KH;
      a.KW = p.gconv.KW;
      a.Mb = p.gconv.Mb;
      if (k::tcGconvShiftSupported(a, math, nullptr)) g.tile2 = {3};
      else g.tile2 = {1, 2};
      g.bz = {1};
    } else {
      g.tile0 = {128};
      g.tile1 = {1, 16, 32, 64, 128, 256};  // 1 = plan at launch (per layer for the FC chains)
      g.tile2 = {32};
      g.bz = {1, 2, 4, 8, 16};
    }
    return g;
  }
  switch (p.family) {
    case Family::Gemm:
    case Family::FcChain:
      g.tile0 = {16, 32, 64};
      g.tile1 = {16, 32, 64};
      g.tile2 = {16, 32, 64};
      if (p.family == Family::Gemm && p.gemm.batch > 1) {  // + the persistent batched kernel
        g.tile0 = {1, 2, 4, 7, 13, 16, 32, 64};
        g.tile1 = {1, 2, 4, 16, 32, 64};
        g.tile2 = {1, 2, 3, 16, 32, 64};  // 1 = persistent batched, 2 = slab, 3 = TMA-fed
      }
      g.tx = {4, 8, 16, 32};
      g.ty = {4, 8, 16, 32};
      g.tz = {1};
      g.useShared = {0, 1};
      g.fusion = {Fusion::Max};
      if (p.family == Family::FcChain) {
        g.tile0 = {1, 2, 4, 8, 16, 32, 64};
        g.tile1 = {1, 2, 4, 8, 16, 32, 64};
        g.tile2 = {1, 2, 3, 4, 6, 16, 32, 64};  // fused: 1 = cluster kernel, 2 = register chains, 3/4/6 = loads
        g.tx = {4, 8, 16, 32, 64, 128, 256, 512};
        g.fusion = {Fusion::Max, Fusion::Min};
      }
      break;
    case Family::Kru3:
      g.tile0 = {2, 4, 8, 16, 32};
      g.tile1 = {1};
      g.tile2 = {1};
      g.tx = {32, 64, 128, 256, 512};
      g.ty = {1, 2};
      g.tz = {1};
      g.useShared = {1};
      g.fusion = {Fusion::Max};
      break;
    case Family::Gconv:
      g.tile0 = {1, 2, 4, 8};
      g.tile1 = {1, 2, 4, 8};
      g.tile2 = {1, 4, 7, 8};
      g.tx = {1};
      g.ty = {1};
      g.tz = {1};
      g.useShared = {1};
      g.fusion = {Fusion::Max};
      break;
    case Family::Lut:
      g.tile0 = {1};
      g.tile1 = {1};
      g.tile2 = {1};
      g.tx = {32, 64, 128, 256, 512, 1024};
      g.ty = {1};
      g.tz = {1};
      g.useShared = {0};
      g.fusion = {Fusion::Max};
      break;
  }
  return g;
}

int64_t shardExtent(const Problem& p) {
  switch (p.family) {
    case Family::Gemm: return p.gemm.batch > 1 ? p.gemm.batch : p.gemm.M;
    case Family::FcChain: return p.fc.batch;
    case Family::Kru3: return p.kru.M;
    case Family::Gconv: return p.gconv.N;
    case Family::Lut: return p.lut.empty() ? 0 : p.lut[0].B;
  }
  return 0;
}

void shardRange(int64_t n, int rank, int world, int64_t* lo, int64_t* hi) {
  if (world < 1 || rank < 0 || rank >= world) fail(ErrorKind::MappingInvalid, "shard: rank outside [0, world)");
  const int64_t base = n / world, extra = n % world;
  *lo = rank * base + std::min<int64_t>(rank, extra);
  *hi = *lo + base + (rank < extra ? 1 : 0);
}

Problem shardOf(const Problem& p, int64_t lo, int64_t hi, std::vector<void*>& in, std::vector<void*>& out) {
  if (lo < 0 || hi < lo || hi > shardExtent(p)) fail(ErrorKind::MappingInvalid, "shard: range outside the batch");
  Problem q = p;
  const int n = static_cast<int>(hi - lo);
  // elements per batch row of every batched tensor (each Ref offset once:
  // MLP3's batch input O1 is also its first return)
  std::vector<std::pair<Ref, int64_t>> rows;
  auto add = [&](const Ref& r, int64_t per) {
    if (!r.valid()) return;
    for (const auto& x : rows)
      if (x.first.out == r.out && x.first.idx == r.idx) return;
    rows.push_back({r, per});
  };
  switch (p.family) {
    case Family::Gemm: {
      const GemmDesc& g = p.gemm;
      if (g.batch > 1) {
        add(g.A, g.sA);
        add(g.B, g.sB);
        add(g.C, g.sC);
        q.gemm.batch = n;
      } else {
        add(g.A, g.lda);
        add(g.C, g.ldc);
        q.gemm.M = n;
      }
      q.flops = p.flops * n / std::max<int64_t>(1, shardExtent(p));
      break;
    }
    case Family::FcChain:
      add(p.fc.I, p.fc.ldi);
      for (const auto& L : p.fc.layers) add(L.O, L.out);
      q.fc.batch = n;
      break;
    case Family::Kru3: {
      const KruDesc& k = p.kru;
      add(k.X, (int64_t)k.N0 * k.N1 * k.N2);
      add(k.Y, (int64_t)k.D0 * k.D1 * k.D2);
      add(k.XW1, (int64_t)k.N0 * k.D1 * k.D2);
      add(k.XW2, (int64_t)k.N0 * k.N1 * k.D2);
      q.kru.M = n;
      break;
    }
    case Family::Gconv: {
      const GconvDesc& g = p.gconv;
      add(g.I, (int64_t)g.G * g.C * g.H * g.W);
      add(g.O, (int64_t)g.G * g.F * (g.H - g.KH + 1) * (g.W - g.KW + 1));
      q.gconv.N = n;
      break;
    }
    case Family::Lut:
      for (size_t t = 0; t < p.lut.size(); ++t) {
        add(p.lut[t].I, p.lut[t].L);
        add(p.lut[t].O, p.lut[t].D);
        q.lut[t].B = n;
      }
      break;
  }
  for (const auto& x : rows) {
    std::vector<void*>& v = x.first.out ? out : in;
    v[x.first.idx] = static_cast<char*>(v[x.first.idx]) + lo * x.second * 4;  // fp32 / int32 elements
  }
  if (p.family != Family::Gemm) {
    const double f = (double)n / std::max<int64_t>(1, shardExtent(p));
    q.flops = p.flops * f;
  }
  return q;
}

void launch(const Problem& p, const Mapping& m, void* const* in, void* const* out, int* errFlag, cudaStream_t s) {
  auto ptr = [&](const Ref& r) -> void* { return r.out ? out[r.idx] : in[r.idx]; };
  auto check = [](cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(ErrorKind::Cuda, std::string(what) + " launch failed: " + cudaGetErrorString(e));
  };
  switch (p.family) {
    case Family::Gemm: launchGemmDesc(p.gemm, m, in, out, s); return;
    case Family::FcChain: {
      const FcDesc& f = p.fc;
      if (m.math != k::kMathFfma && m.tcFused) {
        k::FcChainArgs a{};
        a.I = static_cast<const float*>(ptr(f.I));
        a.ldi = f.ldi;
        a.batch = f.batch;
        a.layers = static_cast<int>(f.layers.size());
        for (int l = 0; l < a.layers; ++l) {
          const auto& L = f.layers[l];
          a.L[l].W = static_cast<const float*>(ptr(L.W));
          a.L[l].bias = static_cast<const float*>(ptr(L.bias));
          a.L[l].O = static_cast<float*>(ptr(L.O));
          a.L[l].out = L.out;
          a.L[l].kred = L.kred;
          a.L[l].ldw = L.ldw;
        }
        check(m.tcFc2 ? k::launchTcFc2(a, m.math, smCount(), s) : k::launchTcFcFused(a, m.math, s),
              "fused tensor-core FC chain");
        return;
      }
      if (!m.fused) {
        // one GEMM per layer: init = bias, epilogue = ReLU; layer l>0 reads
        // layer l-1's global output
        Ref prev = f.I;
        int64_t ldprev = f.ldi;
        for (const auto& L : f.layers) {
          GemmDesc g;
          g.A = prev;
          g.B = L.W;
          g.C = L.O;
          g.bias = L.bias;
          g.M = f.batch;
          g.N = L.out;
          g.K = L.kred;
          g.lda = ldprev;
          g.ldb = L.ldw;
          g.ldc = L.out;
          g.init = k::kInitBias;
          g.relu = 1;
          launchGemmDesc(g, m, in, out, s);
          prev = L.O;
          ldprev = L.out;
        }
        return;
      }
      k::FcChainArgs a{};
      a.I = static_cast<const float*>(ptr(f.I));
      a.ldi = f.ldi;
      a.batch = f.batch;
      a.layers = static_cast<int>(f.layers.size());
      for (int l = 0; l < a.layers; ++l) {
        const auto& L = f.layers[l];
        a.L[l].W = static_cast<const float*>(ptr(L.W));
        a.L[l].bias = static_cast<const float*>(ptr(L.bias));
        a.L[l].O = static_cast<float*>(ptr(L.O));
        a.L[l].out = L.out;
        a.L[l].kred = L.kred;
        a.L[l].ldw = L.ldw;
      }
      if (m.fcKind == 1) {
        check(k::launchFcRegs(a, m.rows, s), "FC chain (registers)");
        return;
      }
      check(k::launchFcChain(a, m.rows, m.cn, m.threads, s, m.fcLoads), "FC chain");
      return;
    }
    case Family::Kru3: {
      const KruDesc& d = p.kru;
      k::KruArgs a;
      a.W0 = static_cast<const float*>(ptr(d.W0));
      a.W1 = static_cast<const float*>(ptr(d.W1));
      a.W2 = static_cast<const float*>(ptr(d.W2));
      a.X = static_cast<const float*>(ptr(d.X));
      a.Y = static_cast<float*>(ptr(d.Y));
      a.XW1 = static_cast<float*>(ptr(d.XW1));
      a.XW2 = static_cast<float*>(ptr(d.XW2));
      a.M = d.M;
      a.N0 = d.N0;
      a.N1 = d.N1;
      a.N2 = d.N2;
      a.D0 = d.D0;
      a.D1 = d.D1;
      a.D2 = d.D2;
      if (m.math != k::kMathFfma) {
        const char* why = nullptr;
        if (!k::tcKru3Supported(a, &why)) fail(ErrorKind::MappingInvalid, why);
        check(k::launchTcKru3(a, m.math, s), "tensor-core 3-KRU");
        return;
      }
      check(k::launchKru3(a, m.dchunk, m.threads, s), "3-KRU");
      return;
    }
    case Family::Gconv: {
      const GconvDesc& d = p.gconv;
      k::GconvArgs a;
      a.I = static_cast<const float*>(ptr(d.I));
      a.W1 = static_cast<const float*>(ptr(d.W1));
      a.B = static_cast<const float*>(ptr(d.B));
      a.O = static_cast<float*>(ptr(d.O));
      a.N = d.N;
      a.G = d.G;
      a.C = d.C;
      a.H = d.H;
      a.W = d.W;
      a.F = d.F;
      a.KH = d.KH;
      a.KW = d.KW;
      a.Mb = d.Mb;
      if (m.math != k::kMathFfma) {
        const char* why = nullptr;
        if (m.gconvVariant == 2) {
          if (!k::tcGconvShiftSupported(a, m.math, &why)) fail(ErrorKind::MappingInvalid, why);
          check(k::launchTcGconvShift(a, m.math, s), "tensor-core gconv");
        } else {
          if (!k::tcGconvSupported(a, &why)) fail(ErrorKind::MappingInvalid, why);
          check(m.gconvVariant == 1 ? k::launchTcGconv(a, m.math, s) : k::launchTcGconvTma(a, m.math, s),
                "tensor-core gconv");
        }
      } else {
        check(k::launchGconv(a, m.gconvVariant, m.th, s), "gconv");
      }
      return;
    }
    case Family::Lut: {
      k::LutArgs t[2];
      int n = static_cast<int>(p.lut.size());
      for (int i = 0; i < n; ++i) {
        const auto& T = p.lut[i];
        t[i].LUT = static_cast<const float*>(ptr(T.LUT));
        t[i].I = static_cast<const int32_t*>(ptr(T.I));
        t[i].O = static_cast<float*>(ptr(T.O));
        t[i].E = T.E;
        t[i].D = T.D;
        t[i].B = T.B;
        t[i].L = T.L;
        t[i].err = errFlag;
      }
      check(k::launchLut(t, n, m.threads, s), "LUT");
      return;
    }
  }
}

}  // namespace ops
}  // namespace tcb
