// tcb — command-line driver over the tc-b200 C ABI (include/tcb.h), the
// B200 counterpart of the reference's CLI module:
//
//   tcb check   FILE [--def NAME]
//   tcb compile FILE --def NAME --sizes N=128,M=32 [options] [--cache PATH]
//   tcb run     FILE --def NAME --sizes ... [--inputs A=a.tctn,...] [--seed S]
//               [--outputs C=c.tctn,...] [--compare C=golden.tctn,... [--tol T]]
//               [options] [--cache PATH] [--profile]
//   tcb tune    FILE --def NAME --sizes ... [--pop P] [--gens G] [--seed S]
//               [--log PATH] --cache PATH
//   tcb latency FILE --def NAME --sizes ... [--iters N] [--warmup W] [options]
//               the paper's protocol: N synchronised
//               calls of tcb_run on device tensors (session inputs), host
//               wall time per call (launch + kernel + sync); prints one JSON
//               line with p0/p50/p90/p99 in us and the device time
//   tcb cache   list|inspect|inject|purge --cache PATH
//               [inspect: --index I] [inject: FILE --def NAME --sizes ... --options JSON --cost NS]
//
// options: --options JSON | --tile a,b,c --threads x,y,z --blocks x,y,z ;
//          --math ffma|tf32|3xtf32 (tensor-core variants).
// Sizes bind the size symbols of the def's parameter declarations; a
// read-only return's shape (MLP3's O1) is bound as O1__0=..,O1__1=..
// (the reference's synthesized symbols, ranges.cc:458-466).
// Every verb is a thin composition of C-ABI calls. Exit codes follow the
// spec's contract: 0 success, 1 user/input error, 2 internal.
// `run` has no CPU path: the reference interpreter is not part of tc-b200
// (use --compare against tensors the reference wrote).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../../../include/tcb.h"
#include "../json.h"

namespace {

using tcb::Json;

struct Exit {
  int code;
  std::string msg;
};

[[noreturn]] void die(int code, const std::string& m) { throw Exit{code, m}; }

// error code → exit code: Internal and Cuda are internal (2), the rest user (1)
void ck(int rc, const char* what) {
  if (rc == 0) return;
  std::string m = std::string(what) + ": " + tcb_last_error();
  die(rc == TCB_ERR_INTERNAL || rc == TCB_ERR_CUDA ? 2 : 1, m);
}

std::vector<std::string> split(const std::string& s, char c) {
  std::vector<std::string> out;
  if (s.empty()) return out;
  std::stringstream ss(s);
  std::string x;
  while (std::getline(ss, x, c)) out.push_back(x);
  return out;
}

std::map<std::string, std::string> kv(const std::string& s) {
  std::map<std::string, std::string> m;
  for (const auto& p : split(s, ',')) {
    auto e = p.find('=');
    if (e == std::string::npos) die(1, "expected NAME=VALUE, got '" + p + "'");
    m[p.substr(0, e)] = p.substr(e + 1);
  }
  return m;
}

struct Args {
  std::string verb, sub, file;
  std::map<std::string, std::string> flags;
  bool has(const std::string& k) const { return flags.count(k) != 0; }
  std::string get(const std::string& k, const std::string& d = "") const {
    auto f = flags.find(k);
    return f == flags.end() ? d : f->second;
  }
  std::string need(const std::string& k) const {
    if (!has(k)) die(1, "missing --" + k);
    return get(k);
  }
};

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 2) die(1, "usage: tcb check|compile|run|tune|cache ... (see tcb_main.cc)");
  a.verb = argv[1];
  int i = 2;
  if (a.verb == "cache") {
    if (argc < 3) die(1, "usage: tcb cache list|inspect|inject|purge --cache PATH");
    a.sub = argv[2];
    i = 3;
  }
  for (; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) == 0) {
      std::string k = s.substr(2);
      if (k == "profile") {
        a.flags[k] = "1";
        continue;
      }
      if (i + 1 >= argc) die(1, "flag --" + k + " needs a value");
      a.flags[k] = argv[++i];
    } else if (a.file.empty()) {
      a.file = s;
    } else {
      die(1, "unexpected argument '" + s + "'");
    }
  }
  return a;
}

std::string readFile(const std::string& path) {
  std::ifstream is(path);
  if (!is) die(1, "Io: cannot open '" + path + "'");
  std::stringstream ss;
  ss << is.rdbuf();
  return ss.str();
}

struct Engine {
  tcb_engine* e = nullptr;
  Engine() { ck(tcb_engine_create(&e), "engine"); }
  ~Engine() { tcb_engine_destroy(e); }
};

std::string defParams(tcb_engine* e, const std::string& def) {
  std::vector<char> b(1 << 16);
  ck(tcb_def_params(e, def.c_str(), b.data(), static_cast<int>(b.size())), "def");
  return b.data();
}

// shape-only descriptors for the def's parameters and returns from --sizes
struct Shapes {
  std::vector<std::string> pnames, rnames, inout;
  std::vector<bool> pint;
  std::vector<tcb_tensor> in, out;
};

Shapes bindSizes(tcb_engine* e, const std::string& def, const std::string& sizes) {
  Json j = Json::parse(defParams(e, def));
  auto sz = kv(sizes);
  Shapes s;
  for (const auto& p : j.at("params").items()) {
    tcb_tensor t{};
    t.dtype = p.at("elem").asStr() == "int" ? TCB_I32 : TCB_F32;
    t.location = TCB_HOST;
    const auto& dims = p.at("dims").items();
    t.rank = static_cast<int32_t>(dims.size());
    if (t.rank > TCB_MAX_RANK) die(1, "parameter rank above 8");
    for (size_t d = 0; d < dims.size(); ++d) {
      const std::string& x = dims[d].asStr();
      char* end = nullptr;
      long long lit = std::strtoll(x.c_str(), &end, 10);
      if (end && *end == '\0' && !x.empty()) {
        t.shape[d] = lit;
      } else {
        auto f = sz.find(x);
        if (f == sz.end()) die(1, "MissingBinding: size symbol '" + x + "' of parameter '" + p.at("name").asStr() +
                                      "' is not bound by --sizes");
        t.shape[d] = std::atoll(f->second.c_str());
        if (t.shape[d] < 1) die(1, "MissingBinding: size symbol '" + x + "' must be >= 1");
      }
    }
    s.pnames.push_back(p.at("name").asStr());
    s.pint.push_back(t.dtype == TCB_I32);
    s.in.push_back(t);
  }
  for (const auto& r : j.at("returns").items()) {
    tcb_tensor t{};
    t.dtype = TCB_F32;
    t.location = TCB_HOST;
    const std::string rn = r.asStr();
    for (int d = 0; d < TCB_MAX_RANK; ++d) {  // read-only return shapes: O1__0, O1__1, ...
      auto f = sz.find(rn + "__" + std::to_string(d));
      if (f == sz.end()) break;
      t.shape[d] = std::atoll(f->second.c_str());
      t.rank = d + 1;
    }
    s.rnames.push_back(rn);
    s.out.push_back(t);
  }
  for (const auto& r : j.at("inout_returns").items()) s.inout.push_back(r.asStr());
  ck(tcb_infer_outputs(e, def.c_str(), s.in.data(), static_cast<int>(s.in.size()), s.out.data(),
                       static_cast<int>(s.out.size())),
     "shape inference");
  return s;
}

std::string optionsJson(const Args& a, tcb_engine* e, const std::string& def, const Shapes& s) {
  if (a.has("options")) return a.get("options");
  if (!a.has("tile") && !a.has("threads") && !a.has("blocks")) return "";
  std::vector<char> b(1 << 14);
  ck(tcb_options_default(e, def.c_str(), s.in.data(), static_cast<int>(s.in.size()), s.out.data(),
                         static_cast<int>(s.out.size()), b.data(), static_cast<int>(b.size())),
     "options");
  Json o = Json::parse(b.data());
  auto ints = [](const std::string& v) {
    Json arr = Json::array();
    for (const auto& x : split(v, ',')) arr.push(Json(static_cast<int64_t>(std::atoll(x.c_str()))));
    return arr;
  };
  if (a.has("tile")) o["tile_sizes"] = ints(a.get("tile"));
  if (a.has("threads")) o["thread_shape"] = ints(a.get("threads"));
  if (a.has("blocks")) o["block_shape"] = ints(a.get("blocks"));
  return o.dump();
}

int mathOf(const Args& a) {
  std::string m = a.get("math", "ffma");
  if (m == "ffma") return TCB_MATH_FFMA;
  if (m == "tf32") return TCB_MATH_TF32;
  if (m == "3xtf32") return TCB_MATH_3XTF32;
  die(1, "--math must be ffma, tf32 or 3xtf32");
}

void loadCache(const Args& a) {
  if (!a.has("cache")) return;
  std::ifstream probe(a.get("cache"));
  if (probe) ck(tcb_cache_load(a.get("cache").c_str()), "cache load");
  if (a.has("history")) ck(tcb_cache_set_history(a.get("history").c_str()), "history");
}

uint64_t compile(const Args& a, tcb_engine* e, const std::string& def, const Shapes& s, Json* desc) {
  std::string opt = optionsJson(a, e, def, s);
  uint64_t h = 0;
  ck(tcb_compile_ex(e, def.c_str(), s.in.data(), static_cast<int>(s.in.size()), s.out.data(),
                    static_cast<int>(s.out.size()), opt.empty() ? nullptr : opt.c_str(), mathOf(a), &h),
     "compile");
  std::vector<char> b(1 << 16);
  ck(tcb_describe(e, h, b.data(), static_cast<int>(b.size())), "describe");
  *desc = Json::parse(b.data());
  return h;
}

int64_t volume(const tcb_tensor& t) {
  int64_t n = 1;
  for (int d = 0; d < t.rank; ++d) n *= t.shape[d];
  return n;
}

// ----------------------------------------------------------------- verbs
int cmdCheck(const Args& a) {
  Engine E;
  std::string src = readFile(a.file);
  ck(tcb_define(E.e, src.c_str()), "check");
  if (a.has("def")) {
    int np = 0, nr = 0;
    std::vector<char> b(1 << 14);
    ck(tcb_def_signature(E.e, a.get("def").c_str(), &np, &nr, b.data(), static_cast<int>(b.size())), "def");
    std::printf("ok: %s(%s)\n", a.get("def").c_str(), b.data());
  } else {
    std::printf("ok: %s\n", a.file.c_str());
  }
  return 0;
}

int cmdCompile(const Args& a) {
  Engine E;
  loadCache(a);
  std::string src = readFile(a.file), def = a.need("def");
  ck(tcb_define(E.e, src.c_str()), "define");
  Shapes s = bindSizes(E.e, def, a.need("sizes"));
  Json d;
  compile(a, E.e, def, s, &d);
  if (d.at("options_source").asStr() == "cache")
    std::fprintf(stderr, "cache hit: %s reproduced from the cache without retuning\n", def.c_str());
  std::printf("%s\n", d.dump().c_str());
  return 0;
}

int cmdRun(const Args& a) {
  Engine E;
  loadCache(a);
  std::string src = readFile(a.file), def = a.need("def");
  ck(tcb_define(E.e, src.c_str()), "define");
  Shapes s = bindSizes(E.e, def, a.need("sizes"));
  // host buffers: session inputs (the tuner's makeSessionInputs, seeded),
  // overridden by --inputs files; returns zero unless given (in/out)
  std::vector<std::vector<uint32_t>> pin(s.in.size()), pout(s.out.size());
  for (size_t i = 0; i < s.in.size(); ++i) {
    pin[i].assign(static_cast<size_t>(volume(s.in[i])), 0u);
    s.in[i].data = pin[i].data();
  }
  for (size_t i = 0; i < s.out.size(); ++i) {
    pout[i].assign(static_cast<size_t>(volume(s.out[i])), 0u);
    s.out[i].data = pout[i].data();
  }
  const uint64_t seed = std::strtoull(a.get("seed", "0").c_str(), nullptr, 10);
  ck(tcb_session_inputs(E.e, def.c_str(), s.in.data(), static_cast<int>(s.in.size()), s.out.data(),
                        static_cast<int>(s.out.size()), seed),
     "session inputs");
  auto load = [&](const std::string& name, const std::string& path, tcb_tensor& dst, std::vector<uint32_t>& buf) {
    tcb_tensor t{};
    ck(tcb_tensor_file_read(path.c_str(), &t), "read");
    bool same = t.rank == dst.rank && t.dtype == dst.dtype;
    for (int d = 0; same && d < t.rank; ++d) same = t.shape[d] == dst.shape[d];
    if (!same) {
      tcb_tensor_file_free(t.data);
      die(1, "ShapeMismatch: '" + path + "' does not have the declared shape/kind of '" + name + "'");
    }
    std::memcpy(buf.data(), t.data, buf.size() * 4);
    tcb_tensor_file_free(t.data);
  };
  for (const auto& f : kv(a.get("inputs"))) {
    bool found = false;
    for (size_t i = 0; i < s.pnames.size() && !found; ++i)
      if (s.pnames[i] == f.first) load(f.first, f.second, s.in[i], pin[i]), found = true;
    for (size_t i = 0; i < s.rnames.size() && !found; ++i)
      if (s.rnames[i] == f.first) load(f.first, f.second, s.out[i], pout[i]), found = true;
    if (!found) die(1, "Name: '" + f.first + "' is neither a parameter nor a return of " + def);
  }
  Json d;
  uint64_t h = compile(a, E.e, def, s, &d);
  int64_t ns = 0;
  ck(tcb_run(E.e, h, s.in.data(), static_cast<int>(s.in.size()), s.out.data(), static_cast<int>(s.out.size()),
             nullptr, a.has("profile") ? TCB_RUN_PROFILE : 0, &ns),
     "run");
  std::printf("ran %s on %s", def.c_str(), d.at("kernel").asStr().c_str());
  if (a.has("profile")) std::printf(" (%.3f us device)", ns * 1e-3);
  std::printf("\n");
  for (const auto& f : kv(a.get("outputs"))) {
    bool found = false;
    for (size_t i = 0; i < s.rnames.size(); ++i)
      if (s.rnames[i] == f.first) {
        ck(tcb_tensor_file_write(f.second.c_str(), &s.out[i]), "write");
        found = true;
      }
    if (!found) die(1, "Name: '" + f.first + "' is not a return of " + def);
  }
  int rc = 0;
  const double tol = std::atof(a.get("tol", "1e-5").c_str());
  for (const auto& f : kv(a.get("compare"))) {
    size_t i = 0;
    while (i < s.rnames.size() && s.rnames[i] != f.first) ++i;
    if (i == s.rnames.size()) die(1, "Name: '" + f.first + "' is not a return of " + def);
    tcb_tensor g{};
    ck(tcb_tensor_file_read(f.second.c_str(), &g), "read");
    bool same = g.rank == s.out[i].rank && g.dtype == TCB_F32;
    for (int k = 0; same && k < g.rank; ++k) same = g.shape[k] == s.out[i].shape[k];
    double worst = same ? 0.0 : INFINITY;  // maxRelError, tensor_data.cc:221-234
    int64_t diff = 0, n = volume(s.out[i]);
    const float* got = reinterpret_cast<const float*>(pout[i].data());
    const float* ref = static_cast<const float*>(g.data);
    for (int64_t k = 0; same && k < n; ++k) {
      double r = ref[k], v = got[k];
      worst = std::fmax(worst, std::fabs(v - r) / std::fmax(std::fabs(r), 1.0));
      diff += std::memcmp(&got[k], &ref[k], 4) != 0;
    }
    tcb_tensor_file_free(g.data);
    std::printf("compare %s: maxRelError %.3g, %lld of %lld elements differ bitwise%s\n", f.first.c_str(), worst,
                static_cast<long long>(diff), static_cast<long long>(n), worst <= tol ? "" : "  (above tolerance)");
    if (!(worst <= tol)) rc = 1;
  }
  return rc;
}

int cmdTune(const Args& a) {
  Engine E;
  loadCache(a);
  std::string src = readFile(a.file), def = a.need("def"), cachePath = a.need("cache");
  ck(tcb_define(E.e, src.c_str()), "define");
  Shapes s = bindSizes(E.e, def, a.need("sizes"));
  Json t = Json::object();
  t["population"] = Json(static_cast<int64_t>(std::atoll(a.get("pop", "100").c_str())));
  t["generations"] = Json(static_cast<int64_t>(std::atoll(a.get("gens", "25").c_str())));
  t["seed"] = Json(static_cast<int64_t>(std::atoll(a.get("seed", "0").c_str())));
  if (a.has("log")) t["session_log"] = Json(a.get("log"));
  std::vector<char> b(1 << 14);
  ck(tcb_tune(E.e, def.c_str(), s.in.data(), static_cast<int>(s.in.size()), s.out.data(),
              static_cast<int>(s.out.size()), t.dump().c_str(), b.data(), static_cast<int>(b.size())),
     "tune");
  ck(tcb_cache_save(cachePath.c_str()), "cache save");
  std::printf("%s\n", b.data());
  return 0;
}

int cmdCache(const Args& a) {
  const std::string path = a.need("cache");
  loadCache(a);
  if (a.sub == "purge") {
    ck(tcb_cache_purge(), "purge");
    ck(tcb_cache_save(path.c_str()), "cache save");
    std::printf("purged %s\n", path.c_str());
    return 0;
  }
  if (a.sub == "inject") {
    Engine E;
    std::string src = readFile(a.file), def = a.need("def");
    ck(tcb_define(E.e, src.c_str()), "define");
    Shapes s = bindSizes(E.e, def, a.need("sizes"));
    ck(tcb_cache_inject(E.e, def.c_str(), s.in.data(), static_cast<int>(s.in.size()), s.out.data(),
                        static_cast<int>(s.out.size()), a.need("options").c_str(),
                        std::atoll(a.get("cost", "0").c_str())),
       "inject");
    ck(tcb_cache_save(path.c_str()), "cache save");
    std::printf("injected into %s (%d entries)\n", path.c_str(), tcb_cache_size());
    return 0;
  }
  std::vector<char> b(1 << 24);
  ck(tcb_cache_entries(b.data(), static_cast<int>(b.size())), "entries");
  Json es = Json::parse(b.data());
  if (a.sub == "list") {
    int i = 0;
    for (const auto& en : es.items()) {
      std::string canon = en.at("canonical_tc").asStr();
      std::string head = canon.substr(0, canon.find('\n'));
      std::string shapes = en.at("input_shapes").dump();
      std::printf("%3d  %-8s cost=%-10lld shapes=%-28s %s | %s\n", i++, en.at("origin").asStr().c_str(),
                  static_cast<long long>(en.at("cost_ns").asInt()), shapes.c_str(), head.c_str(),
                  en.at("target").asStr().c_str());
    }
    return 0;
  }
  if (a.sub == "inspect") {
    const int idx = std::atoi(a.need("index").c_str());
    if (idx < 0 || idx >= static_cast<int>(es.items().size())) die(1, "Io: no cache entry " + std::to_string(idx));
    std::printf("%s\n", es.items()[static_cast<size_t>(idx)].dump().c_str());
    return 0;
  }
  die(1, "unknown cache verb '" + a.sub + "' (list | inspect | inject | purge)");
}

}  // namespace

int cmdLatency(const Args& a) {
  Engine E;
  loadCache(a);
  std::string src = readFile(a.file), def = a.need("def");
  ck(tcb_define(E.e, src.c_str()), "define");
  Shapes s = bindSizes(E.e, def, a.need("sizes"));
  std::vector<std::vector<uint32_t>> hin(s.in.size()), hout(s.out.size());
  for (size_t i = 0; i < s.in.size(); ++i) {
    hin[i].assign(static_cast<size_t>(volume(s.in[i])), 0u);
    s.in[i].data = hin[i].data();
  }
  for (size_t i = 0; i < s.out.size(); ++i) {
    hout[i].assign(static_cast<size_t>(volume(s.out[i])), 0u);
    s.out[i].data = hout[i].data();
  }
  ck(tcb_session_inputs(E.e, def.c_str(), s.in.data(), static_cast<int>(s.in.size()), s.out.data(),
                        static_cast<int>(s.out.size()), 0),
     "session inputs");
  // device copies of every tensor: the call under test reads device tensors,
  // as the reference's caller passes DLTensors resident on the GPU
  std::vector<tcb_tensor> din = s.in, dout = s.out;
  std::vector<void*> bufs;
  auto toDev = [&](tcb_tensor& t) {
    void* p = nullptr;
    const int64_t bytes = volume(t) * 4;
    ck(tcb_device_alloc(&p, bytes), "device alloc");
    ck(tcb_copy(p, t.data, bytes), "copy");
    t.data = p;
    t.location = TCB_DEVICE;
    bufs.push_back(p);
  };
  for (auto& t : din) toDev(t);
  for (auto& t : dout) toDev(t);
  Json d;
  uint64_t h = compile(a, E.e, def, s, &d);
  const int iters = std::atoi(a.get("iters", "1000").c_str()), warm = std::atoi(a.get("warmup", "100").c_str());
  auto call = [&] {
    ck(tcb_run(E.e, h, din.data(), static_cast<int>(din.size()), dout.data(), static_cast<int>(dout.size()), nullptr,
               TCB_RUN_NOCHECK, nullptr),
       "run");
    ck(tcb_stream_sync(nullptr), "sync");
  };
  for (int i = 0; i < warm; ++i) call();
  std::vector<double> us(iters);
  for (int i = 0; i < iters; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    call();
    us[i] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  }
  std::sort(us.begin(), us.end());
  // host cost of one tcb_run alone: enqueue-only calls back to back
  ck(tcb_stream_sync(nullptr), "sync");
  const int nh = std::min(iters, 200);
  auto h0 = std::chrono::steady_clock::now();
  for (int i = 0; i < nh; ++i)
    ck(tcb_run(E.e, h, din.data(), static_cast<int>(din.size()), dout.data(), static_cast<int>(dout.size()), nullptr,
               TCB_RUN_NOCHECK, nullptr),
       "run");
  const double hostUs = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count() / nh;
  ck(tcb_stream_sync(nullptr), "sync");
  int64_t ns = 0;
  ck(tcb_run(E.e, h, din.data(), static_cast<int>(din.size()), dout.data(), static_cast<int>(dout.size()), nullptr,
             TCB_RUN_PROFILE, &ns),
     "run");
  auto pct = [&](double q) { return us[std::min<size_t>(us.size() - 1, static_cast<size_t>(q * us.size()))]; };
  std::printf("{\"def\": \"%s\", \"kernel\": \"%s\", \"iters\": %d, \"us_p0\": %.2f, \"us_p50\": %.2f, "
              "\"us_p90\": %.2f, \"us_p99\": %.2f, \"device_us\": %.3f, \"host_enqueue_us\": %.2f}\n",
              def.c_str(), d.at("kernel").asStr().c_str(), iters, us[0], pct(0.5), pct(0.9), pct(0.99), ns * 1e-3,
              hostUs);
  for (void* p : bufs) tcb_device_free(p);
  return 0;
}

int main(int argc, char** argv) {
  try {
    Args a = parse(argc, argv);
    if (a.verb != "cache" && a.file.empty()) die(1, "missing the .tc file argument");
    if (a.verb == "check") return cmdCheck(a);
    if (a.verb == "compile") return cmdCompile(a);
    if (a.verb == "run") return cmdRun(a);
    if (a.verb == "tune") return cmdTune(a);
    if (a.verb == "cache") return cmdCache(a);
    if (a.verb == "latency") return cmdLatency(a);
    die(1, "unknown verb '" + a.verb + "' (check | compile | run | tune | cache | latency)");
  } catch (const Exit& e) {
    std::fprintf(stderr, "tcb: %s\n", e.msg.c_str());
    return e.code;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "tcb: %s\n", e.what());
    return 2;
  }
}
