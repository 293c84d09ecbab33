// session.h — deterministic tuning-session inputs, bit-compatible with the
// reference's tuner::makeSessionInputs (genetic.cc:255-291) and
// backend::fillUniform (tensor_data.cc:191-209): one std::mt19937_64 stream
// seeded with `seed`, input tensors filled in sorted-name order, floats
// from uniform_real_distribution<double>(-1, 1) narrowed to float, int
// tensors from uniform_int_distribution<int64_t> over [0, min input extent).
#pragma once

#include <cstdint>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "sem.h"

namespace tcb {

struct HostTensor {
  bool isInt = false;
  std::vector<int64_t> shape;
  std::vector<float> f;
  std::vector<int32_t> i;
  int64_t volume() const {
    int64_t n = 1;
    for (auto e : shape) n *= e;
    return n;
  }
  void* data() { return isInt ? static_cast<void*>(i.data()) : static_cast<void*>(f.data()); }
};

// libstdc++'s uniform_real_distribution<double>(lo, hi) on mt19937_64
double uniformReal(std::mt19937_64& g, double lo, double hi);
// libstdc++'s uniform_int_distribution<int64_t>(lo, hi), inclusive
int64_t uniformInt(std::mt19937_64& g, int64_t lo, int64_t hi);

// inputs by tensor name (parameters only, like the reference)
std::map<std::string, HostTensor> sessionInputs(const sem::Specialized& s, uint64_t seed);

}  // namespace tcb
