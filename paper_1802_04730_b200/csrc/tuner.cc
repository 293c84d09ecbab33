// tuner.cc — see tuner.h.
#include "tuner.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <ctime>
#include <fstream>
#include <atomic>
#include <memory>
#include <optional>
#include <random>
#include <thread>

#include "session.h"

namespace tcb {

namespace {

constexpr size_t kGenes = 14;

double uniform01(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
size_t pickIndex(std::mt19937_64& g, size_t n) { return static_cast<size_t>(g() % n); }

struct Space {
  ops::GenePools pools;
  std::vector<int64_t> unrollPool{1, 2, 4};
  int64_t sharedBudget = 48 * 1024;

  int64_t pick(const std::vector<int64_t>& v, std::mt19937_64& g) const { return v[pickIndex(g, v.size())]; }

  void normalize(MappingOptions& o) const {
    o.tileSizes.resize(3, 1);
    o.sharedMemoryBudget = sharedBudget;
    o.rngSeed = 0;
  }
  int64_t get(const MappingOptions& o, size_t gene) const {
    if (gene < 3) return o.tileSizes[gene];
    if (gene < 6) return o.blockShape[gene - 3];
    if (gene < 9) return o.threadShape[gene - 6];
    switch (gene) {
      case 9: return static_cast<int64_t>(o.fusion);
      case 10: return o.useShared;
      case 11: return o.usePrivate;
      case 12: return o.unrollCopyShared;
      default: return o.unrollFactor;
    }
  }
  void set(MappingOptions& o, size_t gene, int64_t v) const {
    if (gene < 3) o.tileSizes[gene] = v;
    else if (gene < 6) o.blockShape[gene - 3] = v;
    else if (gene < 9) o.threadShape[gene - 6] = v;
    else if (gene == 9) o.fusion = static_cast<Fusion>(v);
    else if (gene == 10) o.useShared = v != 0;
    else if (gene == 11) o.usePrivate = v != 0;
    else if (gene == 12) o.unrollCopyShared = v != 0;
    else o.unrollFactor = v;
  }
  int64_t randomGene(size_t gene, std::mt19937_64& g) const {
    switch (gene) {
      case 0: return pick(pools.tile0, g);
      case 1: return pick(pools.tile1, g);
      case 2: return pick(pools.tile2, g);
      case 3:
      case 4: return 1;  // grid extents are derived from the problem
      case 5: return pick(pools.bz, g);  // tensor-core K splits (1 otherwise)
      case 6: return pick(pools.tx, g);
      case 7: return pick(pools.ty, g);
      case 8: return pick(pools.tz, g);
      case 9: return static_cast<int64_t>(pools.fusion[pickIndex(g, pools.fusion.size())]);
      case 10: return pools.useShared[pickIndex(g, pools.useShared.size())];
      case 11:
      case 12: return static_cast<int64_t>(g() & 1);
      default: return pick(unrollPool, g);
    }
  }
  MappingOptions random(std::mt19937_64& g) const {
    MappingOptions o;
    normalize(o);
    for (size_t i = 0; i < kGenes; ++i) set(o, i, randomGene(i, g));
    return o;
  }
  MappingOptions crossover(const MappingOptions& a, const MappingOptions& b, const MappingOptions& c,
                           std::mt19937_64& g) const {
    const MappingOptions* par[3] = {&a, &b, &c};
    MappingOptions child;
    normalize(child);
    for (size_t i = 0; i < kGenes; ++i) set(child, i, get(*par[pickIndex(g, 3)], i));
    return child;
  }
  void mutate(MappingOptions& o, double rate, std::mt19937_64& g) const {
    for (size_t i = 0; i < kGenes; ++i)
      if (uniform01(g) < rate) set(o, i, randomGene(i, g));
  }
};

struct Candidate {
  MappingOptions genome;
  bool ok = false;
  int64_t cost = 0;
  double fitness = 0;
  std::string text, failure;
};

void cudaOk(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(ErrorKind::Cuda, std::string(what) + ": " + cudaGetErrorString(e));
}

// Device-resident session: parameters from makeSessionInputs, returns
// (in/out ones seeded from a second stream, seed ^ 0x5eed) and their
// pristine copies.
struct DeviceSession {
  std::vector<void*> in, out, outInit;
  std::vector<size_t> outBytes;
  int* err = nullptr;
  cudaStream_t stream = nullptr;

  DeviceSession(const sem::Specialized& s, uint64_t seed) {
    auto host = sessionInputs(s, seed);
    cudaOk(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
    for (const auto& p : s.v.def.params) {
      if (p.scalar()) {
        in.push_back(nullptr);
        continue;
      }
      HostTensor& h = host.at(p.name);
      size_t bytes = static_cast<size_t>(h.volume()) * 4;
      void* d = nullptr;
      cudaOk(cudaMalloc(&d, std::max<size_t>(bytes, 16)), "cudaMalloc");
      cudaOk(cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice), "H2D");
      in.push_back(d);
    }
    std::mt19937_64 g(seed ^ 0x5EEDULL);
    for (const auto& r : s.v.def.rets) {
      int64_t n = 1;
      for (auto e : s.shapes.at(r)) n *= e;
      std::vector<float> init(static_cast<size_t>(n));
      for (auto& v : init) v = static_cast<float>(uniformReal(g, -1.0, 1.0));
      size_t bytes = static_cast<size_t>(n) * 4;
      void *d = nullptr, *d0 = nullptr;
      cudaOk(cudaMalloc(&d, std::max<size_t>(bytes, 16)), "cudaMalloc");
      cudaOk(cudaMalloc(&d0, std::max<size_t>(bytes, 16)), "cudaMalloc");
      cudaOk(cudaMemcpy(d0, init.data(), bytes, cudaMemcpyHostToDevice), "H2D");
      out.push_back(d);
      outInit.push_back(d0);
      outBytes.push_back(bytes);
    }
    cudaOk(cudaMalloc(&err, sizeof(int)), "cudaMalloc");
  }
  // cold-L2 timing: a scratch buffer of twice the L2 is rewritten before each
  // timed launch, so candidates are costed on cold operands as the bench and a
  // serving step see them (warm timing favoured plans that re-read from L2)
  void* flushBuf = nullptr;
  size_t flushBytes = 0;
  void flushL2() {
    if (!flushBuf) {
      int dev = 0, l2 = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
      flushBytes = static_cast<size_t>(std::max(l2, 1 << 20)) * 2;
      if (cudaMalloc(&flushBuf, flushBytes) != cudaSuccess) {
        cudaGetLastError();
        flushBuf = nullptr;
        flushBytes = 0;
        return;
      }
    }
    static unsigned char v = 0;
    cudaOk(cudaMemsetAsync(flushBuf, ++v, flushBytes, stream), "flush");
  }
  ~DeviceSession() {
    if (flushBuf) cudaFree(flushBuf);
    for (void* p : in) cudaFree(p);
    for (void* p : out) cudaFree(p);
    for (void* p : outInit) cudaFree(p);
    cudaFree(err);
    cudaStreamDestroy(stream);
  }
  void reset() {
    for (size_t i = 0; i < out.size(); ++i)
      cudaOk(cudaMemcpyAsync(out[i], outInit[i], outBytes[i], cudaMemcpyDeviceToDevice, stream), "reset");
    cudaOk(cudaMemsetAsync(err, 0, sizeof(int), stream), "memset");
  }
  std::vector<std::vector<char>> snapshot() {
    cudaOk(cudaStreamSynchronize(stream), "sync");
    std::vector<std::vector<char>> v;
    for (size_t i = 0; i < out.size(); ++i) {
      v.emplace_back(outBytes[i]);
      cudaOk(cudaMemcpy(v.back().data(), out[i], outBytes[i], cudaMemcpyDeviceToHost), "D2H");
    }
    return v;
  }
};

// max |a - b| / max(|b|, 1) over fp32 buffers (tensor_data.cc:221-234)
double maxRel(const std::vector<std::vector<char>>& a, const std::vector<std::vector<char>>& b) {
  double worst = 0;
  for (size_t t = 0; t < a.size() && t < b.size(); ++t) {
    const size_t n = std::min(a[t].size(), b[t].size()) / 4;
    const float* x = reinterpret_cast<const float*>(a[t].data());
    const float* y = reinterpret_cast<const float*>(b[t].data());
    for (size_t i = 0; i < n; ++i) {
      const double d = std::fabs((double)x[i] - (double)y[i]) / std::max(1.0, std::fabs((double)y[i]));
      if (!(d <= worst)) worst = d;  // NaN propagates as a failure
    }
  }
  return worst;
}

void score(Candidate& c, const ops::Problem& p, DeviceSession& ds, int iters,
           std::optional<std::vector<std::vector<char>>>& refOut, int math = 0, bool coldL2 = true) {
  try {
    ops::Mapping m = ops::decode(p, c.genome, math);
    c.text = m.describe();
    // correctness run from pristine outputs
    ds.reset();
    ops::launch(p, m, ds.in.data(), ds.out.data(), ds.err, ds.stream);
    auto got = ds.snapshot();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(ErrorKind::Cuda, cudaGetErrorString(e));
    if (!refOut) {
      refOut = got;
    } else if (math == 0 ? got != *refOut : !(maxRel(got, *refOut) <= ops::tcTolerance(p, math))) {
      c.ok = false;
      c.fitness = 0;
      c.failure = math == 0 ? "output mismatch against the reference candidate"
                            : "outside the tensor-core tolerance of the reference candidate";
      return;
    }
    cudaEvent_t a, b;
    cudaOk(cudaEventCreate(&a), "event");
    cudaOk(cudaEventCreate(&b), "event");
    std::vector<float> ms;
    for (int i = 0; i < 2 + iters; ++i) {
      if (coldL2) ds.flushL2();
      cudaOk(cudaEventRecord(a, ds.stream), "record");
      ops::launch(p, m, ds.in.data(), ds.out.data(), ds.err, ds.stream);
      cudaOk(cudaEventRecord(b, ds.stream), "record");
      cudaOk(cudaEventSynchronize(b), "sync");
      float t = 0;
      cudaOk(cudaEventElapsedTime(&t, a, b), "elapsed");
      if (i >= 2) ms.push_back(t);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    std::sort(ms.begin(), ms.end());
    c.cost = std::max<int64_t>(1, static_cast<int64_t>(ms[ms.size() / 2] * 1e6));
    c.fitness = 1.0 / static_cast<double>(c.cost);
    c.ok = true;
  } catch (const Error& e) {
    c.ok = false;
    c.fitness = 0;
    c.failure = std::string(errorKindName(e.kind())) + ": " + e.what();
    cudaGetLastError();  // clear a sticky launch-config error
  }
}

size_t roulette(const std::vector<Candidate>& pop, double total, std::mt19937_64& g) {
  double point = uniform01(g) * total, acc = 0;
  for (size_t i = 0; i < pop.size(); ++i) {
    acc += pop[i].fitness;
    if (point < acc) return i;
  }
  return pop.size() - 1;
}

}  // namespace

TuneResult tune(const sem::Specialized& s, const ops::Problem& p, const cache::Key& key, const TuneOptions& o,
                cache::Cache* c) {
  TCB_CHECK(o.population >= 1, "population must hold at least one genome");
  Space space;
  space.pools = ops::genePools(p, o.math);

  std::vector<MappingOptions> starting;
  if (c) {
    if (auto hit = c->lookup(key)) starting.push_back(hit->options);
  }
  for (const auto& x : o.extraStarting) starting.push_back(x);
  starting.push_back(ops::defaultOptions(p, o.math));
  if (o.useBaselines && o.math == 0)  // the reference presets describe FFMA mappings
    for (const auto& b : baselineOptions()) starting.push_back(b);

  std::mt19937_64 g(o.seed);
  auto seedPop = [&](const std::vector<MappingOptions>& start) {
    std::vector<Candidate> pop;
    for (const auto& st : start) {
      if (pop.size() == o.population) break;
      Candidate cd;
      cd.genome = st;
      space.normalize(cd.genome);
      pop.push_back(cd);
    }
    while (pop.size() < o.population) {
      Candidate cd;
      cd.genome = space.random(g);
      pop.push_back(cd);
    }
    return pop;
  };
  std::vector<Candidate> pop = seedPop(starting);

  // one scoring worker per listed device: its own session (the same seeded
  // inputs) and its own reference output from the family default mapping
  std::vector<int> devs = o.devices;
  int cur = 0;
  cudaOk(cudaGetDevice(&cur), "device");
  if (devs.empty()) devs.push_back(cur);
  struct Worker {
    int dev;
    std::unique_ptr<DeviceSession> ds;
    std::optional<std::vector<std::vector<char>>> refOut;
  };
  std::vector<Worker> workers(devs.size());
  for (size_t w = 0; w < devs.size(); ++w) {
    workers[w].dev = devs[w];
    cudaOk(cudaSetDevice(devs[w]), "device");
    workers[w].ds = std::make_unique<DeviceSession>(s, o.seed ^ fnv1a64("session-inputs"));
    Candidate ref;
    ref.genome = ops::defaultOptions(p, o.math);
    score(ref, p, *workers[w].ds, 1, workers[w].refOut, o.math);
    if (!ref.ok) fail(ErrorKind::NoViableCandidate, "the default mapping failed: " + ref.failure);
  }
  cudaOk(cudaSetDevice(cur), "device");
  TuneResult res;
  res.perWorker.assign(workers.size(), 0);
  // scores every candidate of a generation: workers take the next unscored
  // index; each writes only its own candidates (the reference's per-slot
  // writes, genetic.h:99-104); cache updates follow in candidate order
  auto scoreAll = [&](std::vector<Candidate>& cands) {
    if (workers.size() == 1) {
      for (auto& cd : cands) score(cd, p, *workers[0].ds, o.timingIters, workers[0].refOut, o.math, o.coldL2);
      res.perWorker[0] += cands.size();
      return;
    }
    std::atomic<size_t> next{0};
    std::vector<std::thread> th;
    std::vector<std::string> errs(workers.size());
    for (size_t w = 0; w < workers.size(); ++w)
      th.emplace_back([&, w] {
        try {
          cudaOk(cudaSetDevice(workers[w].dev), "device");
          for (size_t i; (i = next.fetch_add(1)) < cands.size();) {
            score(cands[i], p, *workers[w].ds, o.timingIters, workers[w].refOut, o.math, o.coldL2);
            ++res.perWorker[w];
          }
        } catch (const std::exception& e) {
          errs[w] = e.what();
        }
      });
    for (auto& t : th) t.join();
    cudaSetDevice(cur);
    for (const auto& e : errs)
      if (!e.empty()) fail(ErrorKind::Cuda, "tuner worker: " + e);
  };

  const std::string session = "tune-" + hex16(fnv1a64(key.canonicalTc + std::to_string(o.seed)));
  std::ofstream log;
  if (!o.sessionLog.empty()) log.open(o.sessionLog, std::ios::app);

  std::optional<Candidate> best;
  for (size_t gen = 0;; ++gen) {
    scoreAll(pop);
    for (auto& cd : pop) {
      ++res.evaluated;
      if (!cd.ok) {
        ++res.failed;
        continue;
      }
      if (!best || cd.cost < best->cost) best = cd;
      if (c) {
        cache::Entry e;
        e.key = key;
        e.key.optionsDigest = cd.genome.digest();
        e.options = cd.genome;
        e.kernelText = cd.text;
        e.cost = cd.cost;
        e.createdAt = static_cast<int64_t>(std::time(nullptr));
        e.origin = cache::Origin::Tuned;
        c->update(e, session);
      }
    }
    if (log) {
      std::string pw;
      for (size_t w = 0; w < res.perWorker.size(); ++w) pw += (w ? "," : "") + std::to_string(res.perWorker[w]);
      log << "{\"generation\":" << gen << ",\"best_cost\":" << (best ? std::to_string(best->cost) : "null")
          << ",\"genome\":" << (best ? best->genome.toJson() : "null") << ",\"scored_per_device_worker\":[" << pw
          << "]}\n";
    }
    if (gen == o.generations) break;
    double total = 0;
    size_t eliteIdx = 0;
    for (size_t i = 0; i < pop.size(); ++i) {
      total += pop[i].fitness;
      if (pop[i].fitness > pop[eliteIdx].fitness) eliteIdx = i;
    }
    if (total <= 0) {  // DegeneratePopulation → restart from random genomes
      pop = seedPop({});
      continue;
    }
    std::vector<Candidate> next;
    Candidate elite;
    elite.genome = pop[eliteIdx].genome;
    next.push_back(elite);
    while (next.size() < pop.size()) {
      const Candidate& a = pop[roulette(pop, total, g)];
      const Candidate& b = pop[roulette(pop, total, g)];
      const Candidate& d = pop[roulette(pop, total, g)];
      Candidate child;
      child.genome = space.crossover(a.genome, b.genome, d.genome, g);
      space.mutate(child.genome, o.mutationRate, g);
      next.push_back(child);
    }
    pop = std::move(next);
  }
  if (!best) fail(ErrorKind::NoViableCandidate, "no genome of any generation compiled and ran");
  res.best = best->genome;
  res.bestCost = best->cost;
  return res;
}

}  // namespace tcb
