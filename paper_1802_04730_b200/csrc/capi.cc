// capi.cc — the ExecutionEngine behind the C ABI (include/tcb.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <memory>
#include <random>
#include <mutex>
#include <sstream>

#include "../../include/tcb.h"
#include "cache.h"
#include "json.h"
#include "ops.h"
#include "session.h"
#include "tensor_file.h"
#include "tuner.h"

using namespace tcb;

namespace {

thread_local std::string g_lastError;

int report(const Error& e) {
  g_lastError = std::string(errorKindName(e.kind())) + ": " + e.what();
  if (e.pos().line) g_lastError += " (at " + std::to_string(e.pos().line) + ":" + std::to_string(e.pos().col) + ")";
  return static_cast<int>(e.kind()) + 1;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    return report(e);
  } catch (const std::exception& e) {
    return report(Error(ErrorKind::Internal, e.what()));
  }
}

void cudaOk(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(ErrorKind::Cuda, std::string(what) + ": " + cudaGetErrorString(e));
}

void copyOut(const std::string& s, char* buf, int len) {
  if (!buf || len <= 0) return;
  if (static_cast<int>(s.size()) >= len) fail(ErrorKind::Io, "output buffer too small (" + std::to_string(s.size() + 1) + " bytes needed)");
  std::memcpy(buf, s.c_str(), s.size() + 1);
}

cache::Cache& globalCache() {
  static cache::Cache c;
  return c;
}

std::vector<int64_t> shapeOf(const tcb_tensor& t) {
  if (t.rank < 0 || t.rank > TCB_MAX_RANK) fail(ErrorKind::ShapeMismatch, "tensor rank outside 0..8");
  return std::vector<int64_t>(t.shape, t.shape + t.rank);
}

struct DefEntry {
  std::shared_ptr<lang::Program> program;
  lang::Validated v;
};

struct Compiled {
  std::string name;
  sem::Specialized spec;
  std::string canon;
  cache::Key key;
  ops::Problem prob;
  MappingOptions opts;
  ops::Mapping map;
  std::string source;
  int math = 0;
  int* dErr = nullptr;
  cudaStream_t lastStream = nullptr;
  // staging for TCB_HOST tensors
  // host runs alternate between two staging sets, so an async host run can
  // land its inputs while the previous one (on another stream) still runs
  // its kernel or returns its outputs
  static constexpr int kStagingSets = 2;
  std::vector<void*> dInSet[kStagingSets], dOutSet[kStagingSets];
  std::vector<size_t> inBytes, outBytes;
  int stagingNext = 0;
  std::vector<bool> outInout;
  // the compiled tensor signature, flattened once (tcb_run's per-call check
  // compares against it without map lookups or allocations)
  struct Sig {
    int rank = 0, dtype = TCB_F32;
    bool scalar = false;
    int64_t dims[TCB_MAX_RANK] = {};
    const std::string* name = nullptr;
  };
  std::vector<Sig> inSig, outSig;
  std::once_flag sigOnce;
  // recorded after a host run's last read of the staging buffers (its D2H);
  // the next host run, on any stream, waits for it before overwriting them
  cudaEvent_t stagingFree[kStagingSets] = {};
  bool stagingPending[kStagingSets] = {};
  std::mutex runMu;
  ~Compiled() {
    for (int k = 0; k < kStagingSets; ++k) {
      if (stagingFree[k]) cudaEventDestroy(stagingFree[k]);
      for (void* p : dInSet[k]) cudaFree(p);
      for (void* p : dOutSet[k]) cudaFree(p);
    }
    if (dErr) cudaFree(dErr);
  }
};

}  // namespace

struct tcb_engine {
  std::mutex mu;
  std::map<std::string, DefEntry> defs;
  std::vector<std::unique_ptr<Compiled>> handles;

  const DefEntry& def(const std::string& name) {
    auto f = defs.find(name);
    if (f == defs.end()) fail(ErrorKind::Name, "no def named '" + name + "' has been defined");
    return f->second;
  }

  // shapes of the caller's tensors: every parameter, plus returns given rank>0
  std::map<std::string, std::vector<int64_t>> provided(const DefEntry& d, const tcb_tensor* in, int nin,
                                                       const tcb_tensor* out, int nout) {
    const auto& params = d.v.def.params;
    if (nin != static_cast<int>(params.size()))
      fail(ErrorKind::ShapeMismatch, "def '" + d.v.def.name + "' takes " + std::to_string(params.size()) +
                                         " parameters, got " + std::to_string(nin));
    std::map<std::string, std::vector<int64_t>> m;
    for (int i = 0; i < nin; ++i) {
      const auto& p = params[i];
      if (p.scalar()) continue;
      int want = p.elem == lang::Elem::Int ? TCB_I32 : TCB_F32;
      if (in[i].data && in[i].dtype != want)  // shape-only descriptors carry no dtype
        fail(ErrorKind::ShapeMismatch, "parameter '" + p.name + "' must be " + (want == TCB_I32 ? "int32" : "float32"));
      m[p.name] = shapeOf(in[i]);
    }
    if (out) {
      if (nout != static_cast<int>(d.v.def.rets.size()))
        fail(ErrorKind::ShapeMismatch, "def '" + d.v.def.name + "' has " + std::to_string(d.v.def.rets.size()) +
                                           " returns, got " + std::to_string(nout));
      for (int i = 0; i < nout; ++i)
        if (out[i].rank > 0) m[d.v.def.rets[i]] = shapeOf(out[i]);
    }
    return m;
  }

  sem::Specialized specialize(const std::string& name, const tcb_tensor* in, int nin, const tcb_tensor* out,
                              int nout) {
    const DefEntry& d = def(name);
    return sem::specialize(d.v, provided(d, in, nin, out, nout));
  }

  std::map<std::string, std::vector<int64_t>> paramShapes(const sem::Specialized& s) {
    std::map<std::string, std::vector<int64_t>> m;
    for (const auto& p : s.v.def.params)
      if (!p.scalar()) m[p.name] = s.shapes.at(p.name);
    return m;
  }

  Compiled& handle(uint64_t h) {
    if (h == 0 || h > handles.size() || !handles[h - 1])
      fail(ErrorKind::Name, "unknown (or released) kernel handle " + std::to_string(h));
    return *handles[h - 1];
  }
};

extern "C" {

const char* tcb_version(void) { return "tc-b200 0.1 (sm_100a, FFMA-exact kernels)"; }

const char* tcb_last_error(void) { return g_lastError.c_str(); }

int tcb_device_info(int dev, char* buf, int len) {
  return guarded([&] {
    cudaDeviceProp p;
    cudaOk(cudaGetDeviceProperties(&p, dev), "cudaGetDeviceProperties");
    std::ostringstream os;
    os << p.name << " sm_" << p.major << p.minor << " sms=" << p.multiProcessorCount
       << " smem_optin=" << p.sharedMemPerBlockOptin << " l2=" << p.l2CacheSize << " hbm=" << p.totalGlobalMem;
    copyOut(os.str(), buf, len);
  });
}

int tcb_measure_peaks(int dev, char* buf, int len) {
  return guarded([&] {
    cudaOk(cudaSetDevice(dev), "cudaSetDevice");
    cudaDeviceProp p;
    cudaOk(cudaGetDeviceProperties(&p, dev), "cudaGetDeviceProperties");
    double ffma = 0;
    float ms = 0;
    cudaOk(k::probeFfma(p.multiProcessorCount, &ffma, &ms), "ffma probe");
    double l1 = 0, l148 = 0, lcl = 0;
    cudaOk(k::probeLaunch(1, 32, 1, &l1), "launch probe");
    cudaOk(k::probeLaunch(2 * p.multiProcessorCount, 256, 1, &l148), "launch probe");
    cudaOk(k::probeLaunch(256, 64, 8, &lcl), "launch probe");
    std::ostringstream os;
    os << "{\"ffma_tflops\": " << ffma << ", \"ffma_probe_ms\": " << ms
       << ", \"launch_floor_us\": {\"1x32\": " << l1 << ", \"" << 2 * p.multiProcessorCount
       << "x256\": " << l148 << ", \"256x64_cluster8\": " << lcl << "}"
       << ", \"sms\": " << p.multiProcessorCount << "}";
    copyOut(os.str(), buf, len);
  });
}

int tcb_engine_create(tcb_engine** out) {
  return guarded([&] { *out = new tcb_engine(); });
}

void tcb_engine_destroy(tcb_engine* e) { delete e; }

const char* tcb_builtin_ops(void) { return ops::opsSource().c_str(); }

int tcb_define(tcb_engine* e, const char* src) {
  return guarded([&] {
    auto prog = std::make_shared<lang::Program>(lang::parse(src));
    std::map<std::string, DefEntry> fresh;
    for (const auto& d : prog->defs) {
      DefEntry de;
      de.program = prog;
      de.v = lang::validate(d, prog.get());
      fresh[d.name] = std::move(de);
    }
    std::lock_guard<std::mutex> g(e->mu);
    for (auto& kv : fresh) e->defs[kv.first] = std::move(kv.second);
  });
}

int tcb_def_signature(tcb_engine* e, const char* name, int* np, int* nr, char* names, int len) {
  return guarded([&] {
    std::lock_guard<std::mutex> g(e->mu);
    const DefEntry& d = e->def(name);
    *np = static_cast<int>(d.v.def.params.size());
    *nr = static_cast<int>(d.v.def.rets.size());
    std::string s;
    for (size_t i = 0; i < d.v.def.params.size(); ++i) s += (i ? "," : "") + d.v.def.params[i].name;
    s += ";";
    for (size_t i = 0; i < d.v.def.rets.size(); ++i) s += (i ? "," : "") + d.v.def.rets[i];
    copyOut(s, names, len);
  });
}

int tcb_infer_outputs(tcb_engine* e, const char* name, const tcb_tensor* in, int nin, tcb_tensor* out, int nout) {
  return guarded([&] {
    std::lock_guard<std::mutex> g(e->mu);
    sem::Specialized s = e->specialize(name, in, nin, out, nout);
    for (int i = 0; i < nout; ++i) {
      const auto& shp = s.shapes.at(s.v.def.rets[i]);
      out[i].rank = static_cast<int32_t>(shp.size());
      for (size_t d = 0; d < shp.size(); ++d) out[i].shape[d] = shp[d];
      out[i].dtype = TCB_F32;
    }
  });
}

int tcb_compile_ex(tcb_engine* e, const char* name, const tcb_tensor* in, int nin, const tcb_tensor* out, int nout,
                   const char* options_json, int math, uint64_t* handle) {
  return guarded([&] {
    if (math != TCB_MATH_FFMA && math != TCB_MATH_TF32 && math != TCB_MATH_3XTF32)
      fail(ErrorKind::MappingInvalid, "unknown math mode " + std::to_string(math));
    std::lock_guard<std::mutex> g(e->mu);
    auto c = std::make_unique<Compiled>();
    c->name = name;
    c->math = math;
    c->spec = e->specialize(name, in, nin, out, nout);
    c->canon = cache::canonicalize(c->spec.v);
    c->prob = ops::match(c->spec, c->canon);
    const std::string suffix = math ? std::string(" math=") + ops::mathName(math) : std::string();
    if (options_json) {
      c->opts = MappingOptions::fromJson(options_json);
      c->source = "explicit";
    } else {
      c->key = cache::makeKey(c->spec.v, e->paramShapes(c->spec), MappingOptions{}, suffix);
      if (auto hit = globalCache().lookup(c->key)) {
        c->opts = hit->options;
        c->source = "cache";
      } else {
        c->opts = ops::defaultOptions(c->prob, math);
        c->source = "default";
      }
    }
    c->key = cache::makeKey(c->spec.v, e->paramShapes(c->spec), c->opts, suffix);
    c->map = ops::decode(c->prob, c->opts, math);
    e->handles.push_back(std::move(c));
    *handle = e->handles.size();
  });
}

int tcb_compile(tcb_engine* e, const char* name, const tcb_tensor* in, int nin, const tcb_tensor* out, int nout,
                const char* options_json, uint64_t* handle) {
  return tcb_compile_ex(e, name, in, nin, out, nout, options_json, TCB_MATH_FFMA, handle);
}

int tcb_describe(tcb_engine* e, uint64_t h, char* buf, int len) {
  return guarded([&] {
    std::lock_guard<std::mutex> g(e->mu);
    Compiled& c = e->handle(h);
    Json j = Json::object();
    j["def"] = Json(c.name);
    j["form"] = Json(c.prob.form);
    j["family"] = Json(ops::familyName(c.prob.family));
    j["kernel"] = Json(c.map.describe());
    j["options"] = Json::parse(c.opts.toJson());
    j["options_source"] = Json(c.source);
    j["math"] = Json(ops::mathName(c.math));
    j["flops"] = Json(static_cast<int64_t>(c.prob.flops));
    j["bytes"] = Json(static_cast<int64_t>(c.prob.bytes));
    j["canonical_tc"] = Json(c.canon);
    j["lookup_key"] = Json(c.key.lookupKey());
    j["options_digest"] = Json(c.opts.digest());
    Json inout = Json::array();
    for (const auto& r : sem::inoutReturns(c.spec.v)) inout.push(Json(r));
    j["inout_returns"] = inout;
    copyOut(j.dump(), buf, len);
  });
}

namespace {

// largest host tensor moved by the segment-copy kernel instead of a DMA
// (TCB_ZEROCOPY_MAX bytes; 0 disables it)
int64_t zeroCopyMax() {
  static const int64_t v = [] {
    const char* e = std::getenv("TCB_ZEROCOPY_MAX");
    return e ? std::atoll(e) : static_cast<int64_t>(1) << 20;
  }();
  return v;
}

// the device address of a pinned (page-locked, UVA-mapped) host buffer, or
// null for pageable memory
const void* mappedHost(const void* p) {
  if (zeroCopyMax() <= 0) return nullptr;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

int deviceSms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

}  // namespace

namespace {

// device staging buffers of a handle run on host tensors
void ensureStaging(Compiled& c, int set) {
  const auto& params = c.spec.v.def.params;
  const auto& rets = c.spec.v.def.rets;
  const int nin = static_cast<int>(params.size()), nout = static_cast<int>(rets.size());
  if (c.inBytes.empty()) {
    auto inout = sem::inoutReturns(c.spec.v);
    for (int i = 0; i < nin; ++i) {
      size_t b = 4;
      if (!params[i].scalar())
        for (auto x : c.spec.shapes.at(params[i].name)) b *= static_cast<size_t>(x);
      c.inBytes.push_back(b);
    }
    for (int i = 0; i < nout; ++i) {
      size_t b = 4;
      for (auto x : c.spec.shapes.at(rets[i])) b *= static_cast<size_t>(x);
      c.outBytes.push_back(b);
      c.outInout.push_back(std::find(inout.begin(), inout.end(), rets[i]) != inout.end());
    }
  }
  if (c.dInSet[set].empty()) {
    for (int i = 0; i < nin; ++i) {
      void* p = nullptr;
      cudaOk(cudaMalloc(&p, c.inBytes[i]), "cudaMalloc");
      c.dInSet[set].push_back(p);
    }
    for (int i = 0; i < nout; ++i) {
      void* p = nullptr;
      cudaOk(cudaMalloc(&p, c.outBytes[i]), "cudaMalloc");
      c.dOutSet[set].push_back(p);
    }
  }
}

}  // namespace

// flattens the compiled tensor signature of a handle (once)
static void buildSigOnce(Compiled& c) {
  std::vector<Compiled::Sig> in, out;
  for (const auto& p : c.spec.v.def.params) {
    Compiled::Sig s;
    s.name = &p.name;
    s.scalar = p.scalar();
    if (!s.scalar) {
      const auto& sh = c.spec.shapes.at(p.name);
      s.rank = static_cast<int>(sh.size());
      std::copy(sh.begin(), sh.end(), s.dims);
      s.dtype = p.elem == lang::Elem::Int ? TCB_I32 : TCB_F32;
    }
    in.push_back(s);
  }
  for (const auto& r : c.spec.v.def.rets) {
    Compiled::Sig s;
    s.name = &r;
    const auto& sh = c.spec.shapes.at(r);
    s.rank = static_cast<int>(sh.size());
    std::copy(sh.begin(), sh.end(), s.dims);
    out.push_back(s);
  }
  c.outSig = std::move(out);
  c.inSig = std::move(in);
}
static void buildSig(Compiled& c) { std::call_once(c.sigOnce, [&] { buildSigOnce(c); }); }

int tcb_run(tcb_engine* e, uint64_t h, const tcb_tensor* in, int nin, const tcb_tensor* out, int nout, void* stream,
            int flags, int64_t* duration_ns) {
  return guarded([&] {
    Compiled* cp;
    {
      std::lock_guard<std::mutex> g(e->mu);
      cp = &e->handle(h);
    }
    Compiled& c = *cp;
    const auto& params = c.spec.v.def.params;
    const auto& rets = c.spec.v.def.rets;
    if (nin != static_cast<int>(params.size()) || nout != static_cast<int>(rets.size()))
      fail(ErrorKind::ShapeMismatch, "run: wrong number of inputs or outputs for '" + c.name + "'");
    bool host = false, dev = false;
    buildSig(c);
    auto checkT = [&](const tcb_tensor& t, const Compiled::Sig& g) {
      bool ok = t.rank == g.rank;
      for (int d = 0; ok && d < g.rank; ++d) ok = t.shape[d] == g.dims[d];
      if (!ok) fail(ErrorKind::ShapeMismatch, "run: tensor '" + *g.name + "' does not have the compiled shape");
      if (t.dtype != g.dtype) fail(ErrorKind::ShapeMismatch, "run: tensor '" + *g.name + "' has the wrong dtype");
      if (!t.data) fail(ErrorKind::Io, "run: tensor '" + *g.name + "' has no data");
      (t.location == TCB_HOST ? host : dev) = true;
    };
    for (int i = 0; i < nin; ++i)
      if (!c.inSig[i].scalar) checkT(in[i], c.inSig[i]);
    for (int i = 0; i < nout; ++i) checkT(out[i], c.outSig[i]);
    if (host && dev) fail(ErrorKind::Io, "run: mixing host and device tensors in one call is not supported");
    cudaStream_t s = static_cast<cudaStream_t>(stream);

    std::lock_guard<std::mutex> rg(c.runMu);
    if (!c.dErr) {
      cudaOk(cudaMalloc(&c.dErr, sizeof(int)), "cudaMalloc");
      cudaOk(cudaMemset(c.dErr, 0, sizeof(int)), "cudaMemset");
    }
    c.lastStream = s;
    // per-call pointer lists without heap allocations for the usual arity
    void* dinBuf[16];
    void* doutBuf[16];
    const void* mapBuf[16];
    std::vector<void*> dinV, doutV;
    std::vector<const void*> mapV;
    void** din = dinBuf;
    void** dout = doutBuf;
    const void** outMapped = mapBuf;
    if (nin > 16) dinV.resize(nin), din = dinV.data();
    if (nout > 16) doutV.resize(nout), mapV.resize(nout), dout = doutV.data(), outMapped = mapV.data();
    for (int i = 0; i < nout; ++i) outMapped[i] = nullptr;
    bool profile = (flags & TCB_RUN_PROFILE) != 0;
    // host tensors: mapped pinned buffers up to zeroCopyMax() move in one
    // segment-copy launch per direction; the rest (pageable or large) by DMA
    k::SegCopyArgs up{}, down{};
    const int set = host ? c.stagingNext : 0;
    if (host) {
      c.stagingNext = (c.stagingNext + 1) % Compiled::kStagingSets;
      ensureStaging(c, set);
      if (!c.stagingFree[set])
        cudaOk(cudaEventCreateWithFlags(&c.stagingFree[set], cudaEventDisableTiming), "event");
      // an earlier async host run (possibly on another stream) may still be
      // reading this staging set
      if (c.stagingPending[set]) cudaOk(cudaStreamWaitEvent(s, c.stagingFree[set], 0), "stream wait");
      auto stage = [&](k::SegCopyArgs& a, void* dst, const void* src, const void* mapped, size_t bytes,
                       cudaMemcpyKind kind) {
        if (mapped && a.n < k::kMaxSeg && static_cast<int64_t>(bytes) <= zeroCopyMax() && bytes % 4 == 0) {
          if (kind == cudaMemcpyHostToDevice)
            k::segCopyAdd(a, dst, mapped, static_cast<int64_t>(bytes));
          else
            k::segCopyAdd(a, const_cast<void*>(mapped), src, static_cast<int64_t>(bytes));
        } else {
          cudaOk(cudaMemcpyAsync(dst, src, bytes, kind, s), kind == cudaMemcpyHostToDevice ? "H2D" : "D2H");
        }
      };
      for (int i = 0; i < nin; ++i) {
        din[i] = c.dInSet[set][i];
        if (!params[i].scalar())
          stage(up, din[i], in[i].data, mappedHost(in[i].data), c.inBytes[i], cudaMemcpyHostToDevice);
      }
      for (int i = 0; i < nout; ++i) {
        dout[i] = c.dOutSet[set][i];
        outMapped[i] = mappedHost(out[i].data);
        if (c.outInout[i]) stage(up, dout[i], out[i].data, outMapped[i], c.outBytes[i], cudaMemcpyHostToDevice);
      }
      cudaOk(k::launchSegCopy(up, deviceSms(), s), "host copy");
    } else {
      for (int i = 0; i < nin; ++i) din[i] = in[i].data;
      for (int i = 0; i < nout; ++i) dout[i] = out[i].data;
    }
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (profile) {
      cudaOk(cudaEventCreate(&ev0), "event");
      cudaOk(cudaEventCreate(&ev1), "event");
      cudaOk(cudaEventRecord(ev0, s), "record");
    }
    ops::launch(c.prob, c.map, din, dout, c.dErr, s);
    if (profile) cudaOk(cudaEventRecord(ev1, s), "record");
    if (host) {
      for (int i = 0; i < nout; ++i) {
        if (outMapped[i] && down.n < k::kMaxSeg && static_cast<int64_t>(c.outBytes[i]) <= zeroCopyMax())
          k::segCopyAdd(down, const_cast<void*>(outMapped[i]), dout[i], static_cast<int64_t>(c.outBytes[i]));
        else
          cudaOk(cudaMemcpyAsync(out[i].data, dout[i], c.outBytes[i], cudaMemcpyDeviceToHost, s), "D2H");
      }
      cudaOk(k::launchSegCopy(down, deviceSms(), s), "host copy");
      cudaOk(cudaEventRecord(c.stagingFree[set], s), "record");
      c.stagingPending[set] = (flags & TCB_RUN_ASYNC) != 0;
      if (!(flags & TCB_RUN_ASYNC)) cudaOk(cudaStreamSynchronize(s), "sync");
    }
    if (profile) {
      cudaOk(cudaEventSynchronize(ev1), "sync");
      float ms = 0;
      cudaOk(cudaEventElapsedTime(&ms, ev0, ev1), "elapsed");
      if (duration_ns) *duration_ns = static_cast<int64_t>(ms * 1e6);
      cudaEventDestroy(ev0);
      cudaEventDestroy(ev1);
    }
    if (c.prob.family == ops::Family::Lut && !(flags & (TCB_RUN_NOCHECK | TCB_RUN_ASYNC))) {
      int flag = 0;
      cudaOk(cudaMemcpyAsync(&flag, c.dErr, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
      cudaOk(cudaStreamSynchronize(s), "sync");
      if (flag) {
        cudaOk(cudaMemset(c.dErr, 0, sizeof(int)), "cudaMemset");
        fail(ErrorKind::IndexOutOfRange, "a data-dependent subscript escaped its tensor's extent");
      }
    }
  });
}

int tcb_shard_range(tcb_engine* e, uint64_t h, int rank, int world, int64_t* lo, int64_t* hi, int64_t* extent) {
  return guarded([&] {
    Compiled* cp;
    {
      std::lock_guard<std::mutex> g(e->mu);
      cp = &e->handle(h);
    }
    const int64_t n = ops::shardExtent(cp->prob);
    int64_t a = 0, b = 0;
    ops::shardRange(n, rank, world, &a, &b);
    if (lo) *lo = a;
    if (hi) *hi = b;
    if (extent) *extent = n;
  });
}

int tcb_run_shard(tcb_engine* e, uint64_t h, const tcb_tensor* in, int nin, const tcb_tensor* out, int nout,
                  int rank, int world, void* stream, int flags) {
  return guarded([&] {
    Compiled* cp;
    {
      std::lock_guard<std::mutex> g(e->mu);
      cp = &e->handle(h);
    }
    Compiled& c = *cp;
    const auto& params = c.spec.v.def.params;
    const auto& rets = c.spec.v.def.rets;
    if (nin != static_cast<int>(params.size()) || nout != static_cast<int>(rets.size()))
      fail(ErrorKind::ShapeMismatch, "run_shard: wrong number of inputs or outputs for '" + c.name + "'");
    auto checkT = [&](const tcb_tensor& t, const std::string& nm, bool isInt) {
      if (shapeOf(t) != c.spec.shapes.at(nm))
        fail(ErrorKind::ShapeMismatch, "run_shard: tensor '" + nm + "' does not have the compiled (full) shape");
      if (t.dtype != (isInt ? TCB_I32 : TCB_F32)) fail(ErrorKind::ShapeMismatch, "run_shard: tensor '" + nm + "' has the wrong dtype");
      if (!t.data) fail(ErrorKind::Io, "run_shard: tensor '" + nm + "' has no data");
      if (t.location == TCB_HOST) fail(ErrorKind::Io, "run_shard: shards run on device tensors (one process per GPU)");
    };
    std::vector<void*> din(nin), dout(nout);
    for (int i = 0; i < nin; ++i) {
      if (!params[i].scalar()) checkT(in[i], params[i].name, params[i].elem == lang::Elem::Int);
      din[i] = in[i].data;
    }
    for (int i = 0; i < nout; ++i) {
      checkT(out[i], rets[i], false);
      dout[i] = out[i].data;
    }
    int64_t lo = 0, hi = 0;
    ops::shardRange(ops::shardExtent(c.prob), rank, world, &lo, &hi);
    if (hi == lo) return;
    ops::Problem q = ops::shardOf(c.prob, lo, hi, din, dout);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> rg(c.runMu);
    if (!c.dErr) {
      cudaOk(cudaMalloc(&c.dErr, sizeof(int)), "cudaMalloc");
      cudaOk(cudaMemset(c.dErr, 0, sizeof(int)), "cudaMemset");
    }
    c.lastStream = s;
    ops::launch(q, c.map, din.data(), dout.data(), c.dErr, s);
    if (c.prob.family == ops::Family::Lut && !(flags & (TCB_RUN_NOCHECK | TCB_RUN_ASYNC))) {
      int flag = 0;
      cudaOk(cudaMemcpyAsync(&flag, c.dErr, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
      cudaOk(cudaStreamSynchronize(s), "sync");
      if (flag) {
        cudaOk(cudaMemset(c.dErr, 0, sizeof(int)), "cudaMemset");
        fail(ErrorKind::IndexOutOfRange, "a data-dependent subscript escaped its tensor's extent");
      }
    }
  });
}

int tcb_release(tcb_engine* e, uint64_t h) {
  return guarded([&] {
    std::unique_ptr<Compiled> dead;
    {
      std::lock_guard<std::mutex> g(e->mu);
      e->handle(h);  // validates
      dead = std::move(e->handles[h - 1]);
    }
    // its device staging / error flag are freed once its last run is done
    if (dead->lastStream) cudaStreamSynchronize(dead->lastStream);
    std::lock_guard<std::mutex> rg(dead->runMu);
  });
}

int tcb_check(tcb_engine* e, uint64_t h) {
  return guarded([&] {
    Compiled* cp;
    {
      std::lock_guard<std::mutex> g(e->mu);
      cp = &e->handle(h);
    }
    if (!cp->dErr) return;
    cudaOk(cudaStreamSynchronize(cp->lastStream), "sync");
    int flag = 0;
    cudaOk(cudaMemcpy(&flag, cp->dErr, sizeof(int), cudaMemcpyDeviceToHost), "D2H");
    if (flag) {
      cudaOk(cudaMemset(cp->dErr, 0, sizeof(int)), "cudaMemset");
      fail(ErrorKind::IndexOutOfRange, "a data-dependent subscript escaped its tensor's extent");
    }
  });
}

int tcb_tune(tcb_engine* e, const char* name, const tcb_tensor* in, int nin, const tcb_tensor* out, int nout,
             const char* topts, char* best, int len) {
  return guarded([&] {
    std::lock_guard<std::mutex> g(e->mu);
    sem::Specialized s = e->specialize(name, in, nin, out, nout);
    std::string canon = cache::canonicalize(s.v);
    ops::Problem p = ops::match(s, canon);
    TuneOptions o;
    if (topts && *topts) {
      Json j;
      try {
        j = Json::parse(topts);
      } catch (const std::exception& ex) {
        fail(ErrorKind::CorruptStore, std::string("malformed tune options: ") + ex.what());
      }
      if (j.has("population")) o.population = static_cast<size_t>(j.at("population").asInt());
      if (j.has("generations")) o.generations = static_cast<size_t>(j.at("generations").asInt());
      if (j.has("mutation_rate")) {
        const Json& m = j.at("mutation_rate");
        o.mutationRate = m.type() == Json::T::Float ? std::stod(m.dump()) : static_cast<double>(m.asInt());
      }
      if (j.has("seed")) o.seed = j.at("seed").asUInt();
      if (j.has("timing_iters")) o.timingIters = static_cast<int>(j.at("timing_iters").asInt());
      if (j.has("cold_l2")) o.coldL2 = j.at("cold_l2").asBool();
      if (j.has("session_log")) o.sessionLog = j.at("session_log").asStr();
      if (j.has("use_baselines")) o.useBaselines = j.at("use_baselines").asBool();
      if (j.has("math")) o.math = ops::mathFromName(j.at("math").asStr());
      if (j.has("devices")) {
        const Json& d = j.at("devices");
        if (d.type() == Json::T::Str && d.asStr() == "all") {
          int n = 0;
          cudaOk(cudaGetDeviceCount(&n), "device count");
          for (int i = 0; i < n; ++i) o.devices.push_back(i);
        } else {
          for (const auto& x : d.items()) o.devices.push_back(static_cast<int>(x.asInt()));
        }
      }
    }
    const std::string suffix = o.math ? std::string(" math=") + ops::mathName(o.math) : std::string();
    cache::Key key = cache::makeKey(s.v, e->paramShapes(s), MappingOptions{}, suffix);
    TuneResult r = tune(s, p, key, o, &globalCache());
    Json res = Json::parse(r.best.toJson());
    copyOut(res.dump(), best, len);
  });
}

int tcb_cache_load(const char* path) {
  return guarded([&] { globalCache().load(path); });
}
int tcb_cache_save(const char* path) {
  return guarded([&] { globalCache().save(path); });
}
int tcb_cache_size(void) { return static_cast<int>(globalCache().size()); }
int tcb_cache_purge(void) {
  return guarded([&] { globalCache().purge(); });
}
int tcb_cache_set_history(const char* path) {
  return guarded([&] { globalCache().setHistoryPath(path ? path : ""); });
}
int tcb_cache_serialize(char* buf, int len) {
  return guarded([&] { copyOut(globalCache().serialize(), buf, len); });
}
int tcb_cache_deserialize(const char* text) {
  return guarded([&] { globalCache().deserialize(text); });
}

int tcb_cache_lookup(tcb_engine* e, const char* name, const tcb_tensor* in, int nin, const tcb_tensor* out, int nout,
                     int* hit, char* opts, int len) {
  return guarded([&] {
    std::lock_guard<std::mutex> g(e->mu);
    sem::Specialized s = e->specialize(name, in, nin, out, nout);
    cache::Key key = cache::makeKey(s.v, e->paramShapes(s), MappingOptions{});
    auto f = globalCache().lookup(key);
    *hit = f ? 1 : 0;
    if (f) copyOut(f->options.toJson(), opts, len);
  });
}

int tcb_cache_inject(tcb_engine* e, const char* name, const tcb_tensor* in, int nin, const tcb_tensor* out, int nout,
                     const char* options_json, int64_t cost) {
  return guarded([&] {
    std::lock_guard<std::mutex> g(e->mu);
    sem::Specialized s = e->specialize(name, in, nin, out, nout);
    MappingOptions o = MappingOptions::fromJson(options_json);
    cache::Entry en;
    en.key = cache::makeKey(s.v, e->paramShapes(s), o);
    en.options = o;
    en.cost = cost;
    en.createdAt = static_cast<int64_t>(std::time(nullptr));
    en.origin = cache::Origin::Injected;
    globalCache().update(en, "inject");
  });
}

int tcb_canonical(tcb_engine* e, const char* name, const tcb_tensor* in, int nin, const tcb_tensor* out, int nout,
                  char* canon, int clen, char* key, int klen) {
  return guarded([&] {
    std::lock_guard<std::mutex> g(e->mu);
    sem::Specialized s = e->specialize(name, in, nin, out, nout);
    cache::Key k = cache::makeKey(s.v, e->paramShapes(s), MappingOptions{});
    copyOut(k.canonicalTc, canon, clen);
    copyOut(k.lookupKey(), key, klen);
  });
}

int tcb_session_inputs(tcb_engine* e, const char* name, const tcb_tensor* in, int nin, const tcb_tensor* out,
                       int nout, uint64_t seed) {
  return guarded([&] {
    std::lock_guard<std::mutex> g(e->mu);
    sem::Specialized s = e->specialize(name, in, nin, out, nout);
    auto t = sessionInputs(s, seed);
    for (int i = 0; i < nin; ++i) {
      const auto& p = s.v.def.params[i];
      if (p.scalar()) continue;
      HostTensor& h = t.at(p.name);
      if (!in[i].data || in[i].location != TCB_HOST) fail(ErrorKind::Io, "session inputs need host buffers");
      std::memcpy(in[i].data, h.data(), static_cast<size_t>(h.volume()) * 4);
    }
  });
}

int tcb_fill_uniform(void* host, int64_t n, int32_t dtype, uint64_t seed, double lo, double hi) {
  return guarded([&] {
    std::mt19937_64 g(seed);
    if (dtype == TCB_F32) {
      float* f = static_cast<float*>(host);
      for (int64_t k = 0; k < n; ++k) f[k] = static_cast<float>(uniformReal(g, lo, hi));
    } else {
      int32_t* p = static_cast<int32_t*>(host);
      int64_t ilo = static_cast<int64_t>(std::ceil(lo)), ihi = static_cast<int64_t>(std::ceil(hi)) - 1;
      if (ihi < ilo) fail(ErrorKind::Internal, "empty integer fill range");
      for (int64_t k = 0; k < n; ++k) p[k] = static_cast<int32_t>(uniformInt(g, ilo, ihi));
    }
  });
}

int tcb_options_validate(const char* j) {
  return guarded([&] { MappingOptions::fromJson(j).validate(); });
}
int tcb_options_normalize(const char* j, char* out, int len) {
  return guarded([&] { copyOut(MappingOptions::fromJson(j).toJson(), out, len); });
}
int tcb_options_digest(const char* j, char* out, int len) {
  return guarded([&] { copyOut(MappingOptions::fromJson(j).digest(), out, len); });
}
int tcb_options_baseline(int i, char* out, int len) {
  return guarded([&] {
    auto v = baselineOptions();
    if (i < 0 || i >= static_cast<int>(v.size())) fail(ErrorKind::Name, "no baseline preset " + std::to_string(i));
    copyOut(v[i].toJson(), out, len);
  });
}
int tcb_options_default(tcb_engine* e, const char* name, const tcb_tensor* in, int nin, const tcb_tensor* out,
                        int nout, char* buf, int len) {
  return guarded([&] {
    std::lock_guard<std::mutex> g(e->mu);
    sem::Specialized s = e->specialize(name, in, nin, out, nout);
    ops::Problem p = ops::match(s, cache::canonicalize(s.v));
    copyOut(ops::defaultOptions(p).toJson(), buf, len);
  });
}

int tcb_tensor_file_write(const char* path, const tcb_tensor* t) {
  return guarded([&] {
    if (!t || !t->data) fail(ErrorKind::Io, "tensor has no host data");
    if (t->location != TCB_HOST) fail(ErrorKind::Io, "tensor files are written from host tensors");
    TensorFile h;
    h.isInt = t->dtype == TCB_I32;
    h.shape = shapeOf(*t);
    int64_t n = 1;
    for (auto e : h.shape) n *= e;
    h.bits.assign(static_cast<const uint32_t*>(t->data), static_cast<const uint32_t*>(t->data) + n);
    writeTensorFile(path, h);
  });
}

int tcb_tensor_file_read(const char* path, tcb_tensor* t) {
  return guarded([&] {
    TensorFile h = readTensorFile(path);
    size_t bytes = std::max<size_t>(4, h.bits.size() * 4);
    void* p = std::malloc(bytes);
    if (!p) fail(ErrorKind::Io, "out of host memory reading '" + std::string(path) + "'");
    std::memcpy(p, h.bits.data(), h.bits.size() * 4);
    t->data = p;
    t->dtype = h.isInt ? TCB_I32 : TCB_F32;
    t->rank = static_cast<int32_t>(h.shape.size());
    for (size_t d = 0; d < h.shape.size(); ++d) t->shape[d] = h.shape[d];
    t->location = TCB_HOST;
    t->reserved = 0;
  });
}

void tcb_tensor_file_free(void* data) { std::free(data); }

int tcb_concat_cols(const float* const* srcs, const int64_t* widths, int n, int64_t rows, float* dst,
                    void* stream) {
  return guarded([&] {
    if (n < 1 || n > k::kMaxConcat) fail(ErrorKind::ShapeMismatch, "concat takes 1..8 sources");
    k::ConcatArgs a{};
    a.n = n;
    a.rows = rows;
    a.dst = dst;
    a.off[0] = 0;
    for (int i = 0; i < n; ++i) {
      if (!srcs[i] || widths[i] < 1) fail(ErrorKind::ShapeMismatch, "concat source without data or columns");
      a.src[i] = srcs[i];
      a.off[i + 1] = a.off[i] + static_cast<int>(widths[i]);
    }
    a.width = a.off[n];
    cudaOk(k::launchConcat(a, static_cast<cudaStream_t>(stream)), "concat launch");
  });
}

int tcb_def_params(tcb_engine* e, const char* name, char* buf, int len) {
  return guarded([&] {
    std::lock_guard<std::mutex> g(e->mu);
    const DefEntry& d = e->def(name);
    Json j = Json::object();
    Json ps = Json::array();
    for (const auto& p : d.v.def.params) {
      Json q = Json::object();
      q["name"] = Json(p.name);
      q["elem"] = Json(p.elem == lang::Elem::Int ? "int" : "float");
      Json dims = Json::array();
      for (const auto& x : p.dims) dims.push(Json(x));
      q["dims"] = dims;
      ps.push(q);
    }
    j["params"] = ps;
    Json rs = Json::array();
    for (const auto& r : d.v.def.rets) rs.push(Json(r));
    j["returns"] = rs;
    Json io = Json::array();
    for (const auto& r : sem::inoutReturns(d.v)) io.push(Json(r));
    j["inout_returns"] = io;
    copyOut(j.dump(), buf, len);
  });
}

int tcb_cache_entries(char* buf, int len) {
  return guarded([&] {
    Json a = Json::array();
    for (const auto& en : globalCache().entries()) {
      Json j = Json::object();
      j["canonical_tc"] = Json(en.key.canonicalTc);
      Json sh = Json::array();
      for (const auto& s : en.key.inputShapes) sh.push(Json(s));
      j["input_shapes"] = sh;
      j["target"] = Json(en.key.target);
      j["options_digest"] = Json(en.key.optionsDigest);
      j["options"] = Json::parse(en.options.toJson());
      j["kernel"] = Json(en.kernelText);
      j["cost_ns"] = Json(en.cost);
      j["created_at"] = Json(en.createdAt);
      j["origin"] = Json(cache::originName(en.origin));
      a.push(j);
    }
    copyOut(a.dump(), buf, len);
  });
}

int tcb_host_alloc(void** p, int64_t bytes) {
  return guarded([&] { cudaOk(cudaMallocHost(p, static_cast<size_t>(bytes)), "cudaMallocHost"); });
}
int tcb_host_free(void* p) {
  return guarded([&] { cudaOk(cudaFreeHost(p), "cudaFreeHost"); });
}
int tcb_device_alloc(void** p, int64_t bytes) {
  return guarded([&] { cudaOk(cudaMalloc(p, static_cast<size_t>(bytes)), "cudaMalloc"); });
}
int tcb_device_free(void* p) {
  return guarded([&] { cudaOk(cudaFree(p), "cudaFree"); });
}
int tcb_copy(void* dst, const void* src, int64_t bytes) {
  return guarded([&] { cudaOk(cudaMemcpy(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault), "cudaMemcpy"); });
}
int tcb_stream_sync(void* stream) {
  return guarded([&] { cudaOk(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "sync"); });
}

}  // extern "C"

namespace tcb {
namespace cache {

std::string targetDescriptor() {
  static std::string d = [] {
    int sms = 148, dev = 0;
    size_t smem = 232448;
    cudaDeviceProp p;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaGetDeviceProperties(&p, dev) == cudaSuccess) {
      sms = p.multiProcessorCount;
      smem = p.sharedMemPerBlockOptin;
    } else {
      cudaGetLastError();
    }
    return "tc-b200/1 sm_100a sms=" + std::to_string(sms) + " smem=" + std::to_string(smem);
  }();
  return d;
}

}  // namespace cache
}  // namespace tcb
