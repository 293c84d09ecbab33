// cache.h — the shape-keyed compilation cache (proj/include/tc/cache/cache.h,
// proj/src/cache/cache.cc), kept format-compatible:
//   * positional canonicalization of the TC (def → f, tensors → T0.., size
//     symbols → S0.., iterators → i0.. per statement), printed with the
//     reference printer's layout (cache.cc:48-152,233-235);
//   * key = (canonical TC, per-parameter input shapes, target descriptor,
//     options digest); lookups ignore the digest (cache.cc:243-255);
//   * min-update with incumbent-wins ties, append-only history (JSONL when
//     a history path is set), one mutex (cache.cc:308-338);
//   * store = "TCCACHE 1 <bytes>\n<json>\nFNV1A64 <hex>\n" (cache.cc:365-439).
// The only semantic change is the target descriptor: a B200 string, so
// entries tuned by the reference's emulator never hit here and vice versa.
#pragma once

#include <map>
#include <mutex>
#include <optional>
#include <string>
#include <vector>

#include "lang.h"
#include "options.h"

namespace tcb {
namespace cache {

std::string canonicalize(const lang::Validated& v);
std::string targetDescriptor();

struct Key {
  std::string canonicalTc;
  std::vector<std::vector<int64_t>> inputShapes;  // per parameter; scalars → {}
  std::string target;
  std::string optionsDigest;
  std::string lookupKey() const;
};

// targetSuffix distinguishes tensor-core math modes (" math=tf32"): their
// kernels and results differ from the exact default, so they never share
// cache entries with it.
Key makeKey(const lang::Validated& v, const std::map<std::string, std::vector<int64_t>>& shapes,
            const MappingOptions& o, const std::string& targetSuffix = "");

enum class Origin { Tuned, Injected, Baseline };
const char* originName(Origin o);

struct Entry {
  Key key;
  MappingOptions options;
  std::string kernelText;  // here: the kernel variant name + launch geometry
  int64_t cost = 0;        // device nanoseconds per call (reference: emulated cost)
  int64_t createdAt = 0;
  Origin origin = Origin::Tuned;
};

class Cache {
 public:
  std::optional<Entry> lookup(const Key& k) const;
  bool update(const Entry& e, const std::string& session = "");
  std::vector<Entry> entries() const;
  size_t historySize() const;
  size_t size() const;
  void purge();
  std::string serialize() const;
  void deserialize(const std::string& text);  // Error(CorruptStore)
  void save(const std::string& path) const;   // Error(Io)
  void load(const std::string& path);         // Error(Io / CorruptStore)
  void setHistoryPath(const std::string& p);

 private:
  mutable std::mutex mu_;
  std::map<std::string, Entry> entries_;
  size_t history_ = 0;
  std::string historyPath_;
};

}  // namespace cache
}  // namespace tcb
