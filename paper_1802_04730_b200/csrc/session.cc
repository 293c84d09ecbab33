#include "session.h"

#include <cmath>
#include <limits>

namespace tcb {

double uniformReal(std::mt19937_64& g, double lo, double hi) {
  // generate_canonical<double, 53> draws one 64-bit word and divides by 2^64
  double u = static_cast<double>(g()) / 18446744073709551616.0;
  if (u >= 1.0) u = std::nextafter(1.0, 0.0);
  return u * (hi - lo) + lo;
}

int64_t uniformInt(std::mt19937_64& g, int64_t lo, int64_t hi) {
  // Lemire's nearly-divisionless downscaling (libstdc++ _S_nd, 128-bit)
  uint64_t range = static_cast<uint64_t>(hi - lo) + 1;
  unsigned __int128 prod = static_cast<unsigned __int128>(g()) * range;
  uint64_t low = static_cast<uint64_t>(prod);
  if (low < range) {
    uint64_t threshold = (0 - range) % range;
    while (low < threshold) {
      prod = static_cast<unsigned __int128>(g()) * range;
      low = static_cast<uint64_t>(prod);
    }
  }
  return static_cast<int64_t>(static_cast<uint64_t>(prod >> 64)) + lo;
}

std::map<std::string, HostTensor> sessionInputs(const sem::Specialized& s, uint64_t seed) {
  std::mt19937_64 g(seed);
  int64_t minExtent = std::numeric_limits<int64_t>::max();
  for (const auto& [name, t] : s.v.tensors) {
    if (t.role != lang::Role::Input) continue;
    for (int64_t e : s.shapes.at(name)) minExtent = std::min(minExtent, e);
  }
  if (minExtent == std::numeric_limits<int64_t>::max() || minExtent < 1) minExtent = 1;
  std::map<std::string, HostTensor> out;
  for (const auto& [name, t] : s.v.tensors) {  // std::map: sorted by name
    if (t.role != lang::Role::Input) continue;
    HostTensor h;
    h.isInt = t.elem == lang::Elem::Int;
    h.shape = s.shapes.at(name);
    int64_t n = h.volume();
    if (h.isInt) {
      h.i.resize(n);
      for (int64_t k = 0; k < n; ++k) h.i[k] = static_cast<int32_t>(uniformInt(g, 0, minExtent - 1));
    } else {
      h.f.resize(n);
      for (int64_t k = 0; k < n; ++k) h.f[k] = static_cast<float>(uniformReal(g, -1.0, 1.0));
    }
    out.emplace(name, std::move(h));
  }
  return out;
}

}  // namespace tcb
