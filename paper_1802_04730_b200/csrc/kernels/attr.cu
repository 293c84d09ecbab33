// attr.cu — per-device cache of kernel function attributes (kernels.cuh).
#include <mutex>
#include <vector>

#include "kernels.cuh"

namespace tcb {
namespace k {

namespace {
struct AttrEntry {
  const void* fn;
  int dev, smem;
  bool npc;
};
std::mutex g_attrMu;
std::vector<AttrEntry> g_attrs;
}  // namespace

cudaError_t ensureFuncAttrs(const void* fn, int smemBytes, bool nonPortableCluster) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(g_attrMu);
  for (const auto& a : g_attrs)
    if (a.fn == fn && a.dev == dev && a.smem >= smemBytes && (a.npc || !nonPortableCluster)) return cudaSuccess;
  if (smemBytes > 48 * 1024) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smemBytes);
    if (e != cudaSuccess) return e;
  }
  if (nonPortableCluster) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  for (auto& a : g_attrs)
    if (a.fn == fn && a.dev == dev) {
      a.smem = smemBytes > a.smem ? smemBytes : a.smem;
      a.npc = a.npc || nonPortableCluster;
      return cudaSuccess;
    }
  g_attrs.push_back({fn, dev, smemBytes, nonPortableCluster});
  return cudaSuccess;
}

}  // namespace k
}  // namespace tcb
