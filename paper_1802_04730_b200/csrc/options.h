// options.h — MappingOptions, the reference's tunable knob vector
// (proj/include/tc/tuner/options.h:29-63), kept field-for-field with the
// same JSON spelling, validation rules and FNV digest so option files and
// cache entries are interchangeable with the reference.
//
// How tc-b200 reads the genes (per kernel family; see ops.cc):
//   tile_sizes[0..2]  CTA tile along the output rows / output columns /
//                     reduction staging depth (GEMM-like families), or
//                     rows-per-CTA / output-chunk / — (chain families)
//   thread_shape      CTA block extents x,y,z (threads per block = product)
//   block_shape       grid extents; 1s mean "derive from the problem"
//   fusion_strategy   max = one fused kernel for multi-statement defs,
//                     min = one kernel per layer/statement group
//   use_shared        stage operands in shared memory (vs. L1/L2 direct)
//   use_private       register-tile the outputs (micro-tile from tile/threads)
//   unroll_factor     inner reduction unroll
//   unroll_copy_shared, shared_memory_budget, rng_seed: carried verbatim
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

namespace tcb {

enum class Fusion { Max = 0, Min = 1, Preserve3 = 2 };
const char* fusionName(Fusion f);
Fusion fusionFromName(const std::string& s);  // Error(CorruptStore)

struct MappingOptions {
  std::vector<int64_t> tileSizes;
  std::array<int64_t, 3> blockShape{{1, 1, 1}};   // grid extents
  std::array<int64_t, 3> threadShape{{1, 1, 1}};  // block extents
  Fusion fusion = Fusion::Max;
  bool useShared = false;
  bool usePrivate = false;
  bool unrollCopyShared = false;
  int64_t unrollFactor = 1;
  int64_t sharedMemoryBudget = 48 * 1024;
  uint64_t rngSeed = 0;

  void validate() const;  // Error(MappingInvalid), options.cc:57-80
  std::string toJson() const;
  static MappingOptions fromJson(const std::string& text);  // Error(CorruptStore)
  std::string digest() const;                                // %016llx of fnv1a64(toJson())
  int64_t threads() const { return threadShape[0] * threadShape[1] * threadShape[2]; }
  bool operator==(const MappingOptions& o) const { return toJson() == o.toJson(); }
  bool operator!=(const MappingOptions& o) const { return !(*this == o); }
};

// The reference's three presets (options.cc:178-208), verbatim.
std::vector<MappingOptions> baselineOptions();

}  // namespace tcb
