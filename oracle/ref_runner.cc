/*
 * ref_runner.cc — TEST INFRASTRUCTURE ONLY. A C-callable shim around the
 * UNMODIFIED reference library (/root/reference/proj/src, compiled by
 * oracle/Makefile into oracle/_ref/libtcref.so). Nothing here re-implements
 * reference behaviour: every entry point calls the reference's own
 * functions, in the order its pipeline uses them:
 *   tcref_run      → lang::parse / pipeline::check / pipeline::specialize /
 *                    backend::interpretReference   (pipeline.cc:36-67,
 *                    interpreter.cc:301-349)
 *   tcref_key      → cache::makeKey(...).lookupKey() + canonical text
 *                    (cache.cc:233-281)
 *   tcref_session  → tuner::makeSessionInputs (genetic.cc:255-291)
 *   tcref_options  → tuner::baselineOptions()[i].toJson()/digest()
 *                    (options.cc:82-208)
 * Error convention: 0 = ok, else (int)ErrorKind + 1, message in `err`.
 */
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "tc/backend/interpreter.h"
#include "tc/cache/cache.h"
#include "tc/lang/parser.h"
#include "tc/pipeline.h"
#include "tc/tuner/genetic.h"
#include "tc/tuner/options.h"

using namespace tc;

namespace {

void setErr(char* err, int errlen, const std::string& msg) {
  if (err && errlen > 0) {
    std::strncpy(err, msg.c_str(), errlen - 1);
    err[errlen - 1] = 0;
  }
}

// Bind size symbols from the shapes of the provided tensors: declared dims
// of parameters, and the synthesized `T__d` symbols of read-only returns
// (ranges.cc:458-466).
std::map<std::string, int64_t> bindSizes(
    const pipeline::Checked& checked,
    const std::map<std::string, std::vector<int64_t>>& shapes) {
  std::map<std::string, int64_t> sizes;
  for (const auto& p : checked.vdef.def.params) {
    auto it = shapes.find(p.name);
    if (it == shapes.end() || p.isScalar()) continue;
    for (size_t d = 0; d < p.dims.size() && d < it->second.size(); ++d) sizes[p.dims[d]] = it->second[d];
  }
  for (const auto& r : checked.vdef.def.returns) {
    auto it = shapes.find(r);
    if (it == shapes.end()) continue;
    for (size_t d = 0; d < it->second.size(); ++d) {
      std::string sym = r + "__" + std::to_string(d);
      if (checked.ranges.sizeSymbols.count(sym)) sizes[sym] = it->second[d];
    }
  }
  return sizes;
}

struct Prepared {
  lang::Program program;
  pipeline::Checked checked;
  std::shared_ptr<sem::SpecializedDef> def;
};

Prepared prepare(const char* src, const char* entry, int n_in, const char** names,
                 const int* ranks, const int64_t* shapes_flat) {
  Prepared p;
  p.program = lang::parse(src);
  const lang::TcDef& d = pipeline::selectDef(p.program, entry ? entry : "");
  p.checked = pipeline::check(d, &p.program);
  std::map<std::string, std::vector<int64_t>> shapes;
  const int64_t* s = shapes_flat;
  for (int i = 0; i < n_in; ++i) {
    shapes[names[i]] = std::vector<int64_t>(s, s + ranks[i]);
    s += ranks[i];
  }
  p.def = std::make_shared<sem::SpecializedDef>(pipeline::specialize(p.checked, bindSizes(p.checked, shapes)));
  return p;
}

} // namespace

extern "C" {

/* Runs the reference interpreter. Inputs: n_in named tensors (params, plus
 * optionally seeded returns), kinds 0=float 1=int, row-major data. Outputs:
 * each requested tensor of the final storage is copied into out_data[i]
 * (capacity out_caps[i] elements); its shape goes to out_shapes (rank ≤ 8
 * per tensor, 8 slots each) and out_ranks. */
int tcref_run(const char* src, const char* entry, int n_in, const char** names,
              const int* kinds, const int* ranks, const int64_t* shapes_flat,
              const void** data, int n_out, const char** out_names, void** out_data,
              const int64_t* out_caps, int64_t* out_shapes, int* out_ranks, char* err,
              int errlen) {
  try {
    Prepared p = prepare(src, entry, n_in, names, ranks, shapes_flat);
    backend::TensorMap inputs;
    const int64_t* s = shapes_flat;
    for (int i = 0; i < n_in; ++i) {
      std::vector<int64_t> shape(s, s + ranks[i]);
      s += ranks[i];
      backend::TensorData t = backend::TensorData::zeros(
          kinds[i] ? lang::ElemKind::Int : lang::ElemKind::Float, shape);
      int64_t n = t.volume();
      if (kinds[i]) std::memcpy(t.i.data(), data[i], n * 4);
      else std::memcpy(t.f.data(), data[i], n * 4);
      inputs.emplace(names[i], std::move(t));
    }
    backend::TensorMap out = backend::interpretReference(*p.def, inputs, {});
    for (int o = 0; o < n_out; ++o) {
      auto it = out.find(out_names[o]);
      if (it == out.end()) {
        setErr(err, errlen, std::string("no tensor ") + out_names[o]);
        return (int)ErrorKind::Io + 1;
      }
      const auto& t = it->second;
      int64_t n = t.volume();
      if (n > out_caps[o]) {
        setErr(err, errlen, "output buffer too small");
        return (int)ErrorKind::Io + 1;
      }
      if (t.elemKind == lang::ElemKind::Float) std::memcpy(out_data[o], t.f.data(), n * 4);
      else std::memcpy(out_data[o], t.i.data(), n * 4);
      out_ranks[o] = (int)t.shape.size();
      for (size_t d = 0; d < t.shape.size() && d < 8; ++d) out_shapes[o * 8 + d] = t.shape[d];
    }
    return 0;
  } catch (const Error& e) {
    setErr(err, errlen, e.what());
    return (int)e.kind() + 1;
  } catch (const std::exception& e) {
    setErr(err, errlen, e.what());
    return (int)ErrorKind::Internal + 1;
  }
}

/* Canonical TC text (cache::canonicalize) and the lookup key
 * (CacheKey::lookupKey) for the given input-parameter shapes. */
int tcref_key(const char* src, const char* entry, int n_in, const char** names,
              const int* ranks, const int64_t* shapes_flat, char* canon, int canon_len,
              char* key, int key_len, char* err, int errlen) {
  try {
    Prepared p = prepare(src, entry, n_in, names, ranks, shapes_flat);
    std::map<std::string, std::vector<int64_t>> shapes;
    for (const auto& kv : p.def->shapes) shapes[kv.first] = kv.second;
    cache::CacheKey k = cache::makeKey(p.def->vdef, shapes, tuner::MappingOptions{});
    setErr(canon, canon_len, k.canonicalTc);
    setErr(key, key_len, k.lookupKey());
    return 0;
  } catch (const Error& e) {
    setErr(err, errlen, e.what());
    return (int)e.kind() + 1;
  }
}

/* tuner::makeSessionInputs(def, seed): inputs in std::map (sorted-name)
 * order; copies the named tensors out. */
int tcref_session(const char* src, const char* entry, int n_in, const char** names,
                  const int* ranks, const int64_t* shapes_flat, uint64_t seed, int n_out,
                  const char** out_names, void** out_data, const int64_t* out_caps,
                  char* err, int errlen) {
  try {
    Prepared p = prepare(src, entry, n_in, names, ranks, shapes_flat);
    tuner::SessionInputs si = tuner::makeSessionInputs(*p.def, seed);
    for (int o = 0; o < n_out; ++o) {
      auto it = si.tensors.find(out_names[o]);
      if (it == si.tensors.end()) return (int)ErrorKind::Io + 1;
      const auto& t = it->second;
      if (t.volume() > out_caps[o]) return (int)ErrorKind::Io + 1;
      if (t.elemKind == lang::ElemKind::Float) std::memcpy(out_data[o], t.f.data(), t.volume() * 4);
      else std::memcpy(out_data[o], t.i.data(), t.volume() * 4);
    }
    return 0;
  } catch (const Error& e) {
    setErr(err, errlen, e.what());
    return (int)e.kind() + 1;
  }
}

/* baselineOptions()[i] as JSON + digest; returns -1 past the end. */
int tcref_options(int i, char* json, int json_len, char* digest, int digest_len) {
  auto v = tuner::baselineOptions();
  if (i < 0 || i >= (int)v.size()) return -1;
  setErr(json, json_len, v[i].toJson());
  setErr(digest, digest_len, v[i].digest());
  return 0;
}

/* MappingOptions::fromJson(text).toJson() — round trip / validation probe. */
int tcref_options_roundtrip(const char* text, char* out, int out_len, char* err, int errlen) {
  try {
    tuner::MappingOptions o = tuner::MappingOptions::fromJson(text);
    setErr(out, out_len, o.toJson());
    return 0;
  } catch (const Error& e) {
    setErr(err, errlen, e.what());
    return (int)e.kind() + 1;
  }
}

/* cache round trip: builds a store with one entry and serializes it. */
int tcref_cache_serialize_one(const char* src, const char* entry, int n_in,
                              const char** names, const int* ranks,
                              const int64_t* shapes_flat, const char* options_json,
                              int64_t cost, int64_t created_at, char* out, int out_len,
                              char* err, int errlen) {
  try {
    Prepared p = prepare(src, entry, n_in, names, ranks, shapes_flat);
    std::map<std::string, std::vector<int64_t>> shapes;
    for (const auto& kv : p.def->shapes) shapes[kv.first] = kv.second;
    tuner::MappingOptions o = tuner::MappingOptions::fromJson(options_json);
    cache::CacheEntry e;
    e.key = cache::makeKey(p.def->vdef, shapes, o);
    e.options = o;
    e.kernelText = "";
    e.cost = cost;
    e.createdAt = created_at;
    e.origin = cache::EntryOrigin::Tuned;
    cache::Cache c;
    c.update(e);
    setErr(out, out_len, c.serialize());
    return 0;
  } catch (const Error& e) {
    setErr(err, errlen, e.what());
    return (int)e.kind() + 1;
  }
}

// TCTN1 through the reference's own writer / reader
// (proj/src/support/tensor_data.cc:122-189), for the byte-compatibility test.
int tcref_write_tensor(const char* path, int kind, int rank, const int64_t* shape, const void* data, char* err,
                       int errlen) {
  try {
    std::vector<int64_t> sh(shape, shape + rank);
    backend::TensorData t = backend::TensorData::zeros(kind ? lang::ElemKind::Int : lang::ElemKind::Float, sh);
    int64_t n = t.volume();
    if (kind) std::memcpy(t.i.data(), data, n * 4);
    else std::memcpy(t.f.data(), data, n * 4);
    backend::writeTensorFile(path, t);
    return 0;
  } catch (const Error& e) {
    setErr(err, errlen, e.what());
    return (int)e.kind() + 1;
  }
}

// reads a TCTN1 file; returns the volume (or -(ErrorKind+1)); fills kind/rank/shape/data up to cap values
int64_t tcref_read_tensor(const char* path, int* kind, int* rank, int64_t* shape, void* data, int64_t cap, char* err,
                          int errlen) {
  try {
    backend::TensorData t = backend::readTensorFile(path);
    *kind = t.elemKind == lang::ElemKind::Int ? 1 : 0;
    *rank = (int)t.shape.size();
    for (size_t d = 0; d < t.shape.size(); ++d) shape[d] = t.shape[d];
    int64_t n = t.volume();
    if (n <= cap) std::memcpy(data, *kind ? (const void*)t.i.data() : (const void*)t.f.data(), n * 4);
    return n;
  } catch (const Error& e) {
    setErr(err, errlen, e.what());
    return -((int64_t)e.kind() + 1);
  }
}

} // extern "C"
