// sm100.cuh — thin inline-PTX wrappers for the sm_100a async machinery the
// tensor-core kernels use: mbarriers, TMA tensor loads, thread-block
// cluster/DSMEM, and tcgen05 (TMEM alloc, MMA, commit, TMEM loads).
// Descriptor bit layouts follow the PTX ISA "tcgen05 matrix descriptors"
// (shared-memory descriptor: start>>4 [0,14), LBO>>4 [16,30), SBO>>4
// [32,46), version=1 [46,48), base offset [49,52), layout [61,64)) and
// the instruction descriptor for .kind::tf32 (c_format [4,6), a/b format
// [7,10)/[10,13), a/b major [15]/[16], N>>3 [17,23), M>>4 [24,29)).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <mutex>

namespace tcb {
namespace k {
namespace sm100 {

// host: the driver's cuTensorMapEncodeTiled, fetched once through the runtime
// (no -lcuda link); null if the driver does not provide it
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline EncodeFn encodeFn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// host: 3-D map {K, rows, batch} of a row-major fp32 operand, box {boxK,
// boxRows, 1}, 128-byte swizzle, cached by (pointer, geometry, device):
// graph capture and repeated host calls re-use the encoded map
// (cuTensorMapEncodeTiled costs host time on every synchronised call
// otherwise). Shared by the TMA-fed FFMA GEMM and the tcgen05 GEMM.
inline bool cachedMapF32Sw128(CUtensorMap* m, const float* base, int K, int rows, int batch, int64_t ld,
                              int64_t sBatch, int boxK, int boxRows) {
  struct Key {
    const void* p;
    int64_t K, rows, batch, ld, sb;
    int boxK, boxRows, dev;
    bool operator==(const Key& o) const {
      return p == o.p && K == o.K && rows == o.rows && batch == o.batch && ld == o.ld && sb == o.sb &&
             boxK == o.boxK && boxRows == o.boxRows && dev == o.dev;
    }
  };
  static std::mutex mu;
  static Key keys[128];
  static CUtensorMap maps[128];
  static int n = 0, next = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const Key key{base, K, rows, batch, ld, sBatch, boxK, boxRows, dev};
  {
    std::lock_guard<std::mutex> g(mu);
    for (int i = 0; i < n; ++i)
      if (keys[i] == key) {
        *m = maps[i];
        return true;
      }
  }
  EncodeFn enc = encodeFn();
  if (!enc) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(batch)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 4,
                           static_cast<cuuint64_t>(batch > 1 ? sBatch : ld * rows) * 4};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(boxK), static_cast<cuuint32_t>(boxRows), 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  std::lock_guard<std::mutex> g(mu);
  keys[next] = key;  // a ring of the 128 most recent geometries
  maps[next] = *m;
  next = (next + 1) % 128;
  if (n < 128) ++n;
  return true;
}

__device__ __forceinline__ uint32_t smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbarInit(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem(bar)), "r"(count));
}
// Ends an mbarrier's life once no wait or arrival on it is pending, so its
// shared memory is plain memory again for the next kernel on the SM
// (compute-sanitizer synccheck tracks stale barrier objects across kernels).
__device__ __forceinline__ void mbarInval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem(bar)) : "memory");
}
__device__ __forceinline__ void fenceBarrierInit() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbarExpectTx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbarArrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem(bar)) : "memory");
}
// Spins on the barrier phase; traps (reported by the host as a CUDA error)
// instead of hanging when the phase never completes.
__device__ __forceinline__ void mbarWait(uint64_t* bar, uint32_t parity, int tag) {
  const uint32_t addr = smem(bar);
  for (uint32_t spin = 0;; ++spin) {
    uint32_t done;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
#ifdef TCB_MBAR_TEST_WAIT
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
#else
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
#endif
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
#ifdef TCB_DEBUG_BARRIERS
    if (spin > (1u << 20)) {  // diagnostic builds: record the stuck barrier and give up
      printf("tc-b200 debug: mbarrier tag %d parity %u stuck (block %d thread %d)\n", tag, parity, blockIdx.x,
             threadIdx.x);
      return;
    }
#else
    if (spin > (1u << 24)) __trap();  // never hang: the host reports the launch failure
#endif
  }
}

// ------------------------------------------------------------------ TMA
__device__ __forceinline__ void tmaPrefetch(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
__device__ __forceinline__ void tmaLoad3d(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem(bar))
      : "memory");
}
// shared -> global tensor store of one box (bulk group; the issuing thread
// waits with tmaStoreWaitRead before the source is overwritten)
__device__ __forceinline__ void tmaStore3d(const void* tmap, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem(src))
               : "memory");
}
__device__ __forceinline__ void tmaStoreCommit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tmaStoreWaitRead() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tmaStoreWaitAll() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes → visible to the async proxy (tcgen05.mma operands)
__device__ __forceinline__ void fenceProxyAsyncSmem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// -------------------------------------------------------------- cluster
__device__ __forceinline__ uint32_t clusterRank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void clusterSync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ float ldsCluster(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ float4 ldsCluster4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

// -------------------------------------------------------------- tcgen05
template <int kCols>
__device__ __forceinline__ void tmemAlloc(uint32_t* slot) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem(slot)), "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int kCols>
__device__ __forceinline__ void tmemFree(uint32_t base) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(kCols) : "memory");
}
__device__ __forceinline__ void tcFenceBefore() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tcFenceAfter() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major operand tile written by TMA with SWIZZLE_128B: rows of 128 B,
// 8-row atoms 1024 B apart. LBO is unused for swizzled K-major layouts.
__device__ __forceinline__ uint64_t descSw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>(1) << 16;            // LBO (ignored)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;    // SBO: next 8-row atom
  d |= static_cast<uint64_t>(1) << 46;            // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;            // SWIZZLE_128B
  return d;
}
// K-major operand without swizzle (CuTe INTERLEAVE): 8-row x 16-byte core
// matrices; LBO = byte distance to the next core matrix along K, SBO = to the
// next 8-row group
__device__ __forceinline__ uint64_t descKInterleave(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>(lbo >> 4) << 16;
  d |= static_cast<uint64_t>(sbo >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version; layout type 0 = SWIZZLE_NONE
  return d;
}
// .kind::tf32, fp32 accumulate, both operands K-major
__host__ __device__ constexpr uint32_t idescTf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void mmaTf32(uint32_t tmemD, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmemD),
      "l"(a), "l"(b), "r"(idesc), "r"(accum)
      : "memory");
}
// the same MMA with A read from TMEM (lane = row, one 32-bit column per k)
__device__ __forceinline__ void mmaTf32Tmem(uint32_t tmemD, uint32_t tmemA, uint64_t b, uint32_t idesc,
                                            uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmemD),
      "r"(tmemA), "l"(b), "r"(idesc), "r"(accum)
      : "memory");
}
// one lane of the (converged) warp: issue tcgen05.mma from a warp-uniform
// branch (elect.sync) instead of `lane == 0`, so the operands stay in uniform
// registers and each MMA issues without a per-lane waterfall (~40 vs ~100
// cycles per MMA at small N, profiles/umma_rate.cu)
__device__ __forceinline__ bool electSync() {
  uint32_t pred;
  asm volatile("{ .reg .pred p; elect.sync _|p, 0xffffffff; selp.u32 %0, 1, 0, p; }" : "=r"(pred));
  return pred != 0;
}
// arrives on `bar` when every previously issued tcgen05.mma of this thread completes
__device__ __forceinline__ void mmaCommit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem(bar))
               : "memory");
}
// multicast tensor copy: the box lands at the same offset in every CTA of
// ctaMask and completes its bytes on each one's barrier at the same offset
__device__ __forceinline__ void tmaLoad3dMc(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar,
                                            uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%0], "
      "[%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem(bar)), "h"(mask)
      : "memory");
}
// 32 lanes x 32 columns of fp32: thread i of the warp gets lane (base lane + i), columns c..c+31
__device__ __forceinline__ void tmemLoad32(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmemLoad16(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmemLoadWait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// thread i of the warp writes lane (base lane + i), columns c..c+31
__device__ __forceinline__ void tmemStore32(uint32_t taddr, const float* v) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmemStoreWait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// the tf32 value a tcgen05 .kind::tf32 MMA takes from an fp32 operand: the top
// 19 bits (round toward zero). The 3xTF32 split of every kernel is
// hi = rzTf32(x) (what the MMA would read from x itself), lo = toTf32(x - hi)
// (x - hi is exact in fp32), so a kernel may feed raw x as hi.
__device__ __forceinline__ float rzTf32(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
// fp32 → tf32 (round to nearest, ties away), result in a 32-bit container with the low 13 bits zero
__device__ __forceinline__ float toTf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

}  // namespace sm100
}  // namespace k
}  // namespace tcb
