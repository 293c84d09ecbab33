// tuner.h — the genetic autotuner (proj/include/tc/tuner/genetic.h,
// proj/src/tuner/genetic.cc) re-targeted at real B200 execution.
//
// Kept from the reference: the 14-gene genome over MappingOptions, the
// seeding order (cached best, extra starts, baselines, uniform random
// top-up), fitness-proportional roulette, three-parent uniform crossover,
// per-gene mutation, elitism, restart on a degenerate generation, a min-
// update of the cache for every evaluated candidate, one JSONL session-log
// line per generation. Changed: admissible gene values come from the
// kernel family's instantiated variants (ops::genePools) instead of the
// problem's ceil-divisors, and a candidate's cost is its measured device
// time (median of CUDA-event timings, ns) instead of the emulator's
// statement count. A candidate fails (fitness 0) when its options do not
// decode to a kernel, its launch fails, or its outputs differ bit-wise
// from the reference candidate's — the B200 stand-in for the emulator's
// race detector (genetic.cc:112-117).
#pragma once

#include <string>
#include <vector>

#include "cache.h"
#include "ops.h"

namespace tcb {

struct TuneOptions {
  size_t population = 100;
  size_t generations = 25;
  double mutationRate = 0.05;
  uint64_t seed = 0;
  int timingIters = 10;
  bool coldL2 = true;  // rewrite a 2x-L2 buffer before each timed launch
  std::string sessionLog;
  bool useBaselines = true;
  std::vector<MappingOptions> extraStarting;
  // k::MathMode. Tensor-core modes tune the tcgen05 tile/split genes; a
  // candidate then passes when it agrees with the mode's default plan within
  // ops::tcTolerance (different K splits sum in different orders), instead
  // of the FFMA modes' bit equality.
  int math = 0;
  // Devices that score candidates in parallel, one host thread per entry
  // (the reference scores candidates on a worker pool, genetic.cc:317-345;
  // the paper tuned on 8 GPUs). Empty = the current
  // device. A device may be listed twice (two workers sharing one GPU: the
  // code path, not a timing setup).
  std::vector<int> devices;
};

struct TuneResult {
  MappingOptions best;
  int64_t bestCost = 0;
  size_t evaluated = 0, failed = 0;
  std::vector<size_t> perWorker;  // candidates scored by each device worker
};

TuneResult tune(const sem::Specialized& s, const ops::Problem& p, const cache::Key& key, const TuneOptions& o,
                cache::Cache* c);

}  // namespace tcb
