// lut.cu — embedding lookup-table reductions (1LUT / 2LUT,
// proj/kernels/2lut.tc:2-6):   O(i,j) +=! LUT(I(i,k), j)
// Default (D % 4 == 0, 16-byte aligned): lut_smem_kernel, one CTA per
// (row, table) staging all gathered rows in shared memory before the ordered
// sum. Fallback (lut_kernel): a warp-group of D/4 (or D) threads owns one
// batch row i; each thread owns four consecutive columns j and walks k
// ascending, gathering 16-byte slices of the indexed table rows. Both add in
// k order (__fadd_rn — the reference's double add narrowed to float is the
// correctly rounded float add up to a double-rounding tie). Indices are validated on the device: an
// index outside [0, E) raises the kernel's error flag, the reference's
// IndexOutOfRange (interpreter.cc:284-292), and is never clamped. Both
// tables of 2LUT run in one launch (blockIdx.y selects the table).
#include "kernels.cuh"

namespace tcb {
namespace k {

namespace {

struct LutPack {
  LutArgs t[2];
};

__global__ void lut_kernel(const LutArgs a0, const LutArgs a1, const int vec) {
  const LutArgs& a = blockIdx.y == 0 ? a0 : a1;
  const int lanesPerRow = vec ? a.D / 4 : a.D;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = gid / lanesPerRow;
  const int lane = (int)(gid % lanesPerRow);
  if (row >= a.B) return;
  const int32_t* idx = a.I + row * a.L;
  if (vec) {
    // two-stage loading: a chunk of kChunk indices is
    // read and validated first, then all kChunk table rows are gathered with
    // independent loads, then added in k order — the gathers of a chunk are
    // in flight together instead of one dependent miss per k
    constexpr int kChunk = 16;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    bool bad = false;
    for (int k0 = 0; k0 < a.L; k0 += kChunk) {
      int64_t e[kChunk];
#pragma unroll
      for (int j = 0; j < kChunk; ++j) e[j] = k0 + j < a.L ? (int64_t)__ldg(idx + k0 + j) : 0;
      float4 v[kChunk];
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        const bool ok = e[j] >= 0 && e[j] < a.E;
        bad |= (k0 + j < a.L) && !ok;
        v[j] = (k0 + j < a.L && ok) ? __ldg(reinterpret_cast<const float4*>(a.LUT + e[j] * a.D) + lane)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        if (k0 + j < a.L) {
          acc.x = __fadd_rn(acc.x, v[j].x);
          acc.y = __fadd_rn(acc.y, v[j].y);
          acc.z = __fadd_rn(acc.z, v[j].z);
          acc.w = __fadd_rn(acc.w, v[j].w);
        }
      }
    }
    if (bad) atomicOr(a.err, 1);  // IndexOutOfRange; the row's value is unspecified
    reinterpret_cast<float4*>(a.O + row * a.D)[lane] = acc;
  } else {
    float acc = 0.f;
    for (int k = 0; k < a.L; ++k) {
      int64_t e = __ldg(idx + k);
      if (e < 0 || e >= a.E) {
        atomicOr(a.err, 1);
        break;
      }
      acc = __fadd_rn(acc, __ldg(a.LUT + e * a.D + lane));
    }
    a.O[row * a.D + lane] = acc;
  }
}

// Two-stage loading in shared memory, one CTA per
// (batch row, table): stage 1 reads the row's L indices and validates them;
// stage 2 has every thread of the CTA issue its share of the L x D/4
// 16-byte gathers at once (all of the row's table rows in flight together)
// into shared memory; stage 3 sums them in k order, each thread owning the
// float4 columns tid, tid + T, ... (__fadd_rn, the interpreter's order), so
// any block size covers any D. Chunks of kRows rows keep the staging buffer
// bounded for any L.
constexpr int kRows = 64;
constexpr int kMaxColsPerThread = 8;  // float4 columns per thread: D <= 32 * T
__global__ void lut_smem_kernel(const LutArgs a0, const LutArgs a1) {
  const LutArgs& a = blockIdx.y == 0 ? a0 : a1;
  const int64_t row = blockIdx.x;
  if (row >= a.B) return;
  extern __shared__ float4 stage[];  // [kRows][D/4]
  __shared__ int64_t sIdx[kRows];
  __shared__ int sBad;
  const int cols = a.D / 4, T = blockDim.x, tid = threadIdx.x;
  const int32_t* idx = a.I + row * a.L;
  if (tid == 0) sBad = 0;
  float4 acc[kMaxColsPerThread];
#pragma unroll
  for (int j = 0; j < kMaxColsPerThread; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k0 = 0; k0 < a.L; k0 += kRows) {
    const int nk = min(kRows, a.L - k0);
    __syncthreads();  // previous chunk consumed
    for (int k = tid; k < nk; k += T) {
      const int64_t e = __ldg(idx + k0 + k);
      const bool ok = e >= 0 && e < a.E;
      if (!ok) sBad = 1;
      sIdx[k] = ok ? e : 0;  // never clamped into the result: the row is flagged
    }
    __syncthreads();
    for (int q = tid; q < nk * cols; q += T) {
      const int k = q / cols, c = q % cols;
      stage[q] = __ldg(reinterpret_cast<const float4*>(a.LUT + sIdx[k] * a.D) + c);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kMaxColsPerThread; ++j) {
      const int c = tid + j * T;
      if (c < cols) {
        for (int k = 0; k < nk; ++k) {
          const float4 v = stage[k * cols + c];
          acc[j].x = __fadd_rn(acc[j].x, v.x);
          acc[j].y = __fadd_rn(acc[j].y, v.y);
          acc[j].z = __fadd_rn(acc[j].z, v.z);
          acc[j].w = __fadd_rn(acc[j].w, v.w);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kMaxColsPerThread; ++j) {
    const int c = tid + j * T;
    if (c < cols) reinterpret_cast<float4*>(a.O + row * a.D)[c] = acc[j];
  }
  if (tid == 0 && sBad) atomicOr(a.err, 1);  // IndexOutOfRange; the row's value is unspecified
}

}  // namespace

cudaError_t launchLut(const LutArgs* tables, int ntables, int threads, cudaStream_t s) {
  if (ntables < 1 || ntables > 2) return cudaErrorInvalidValue;
  LutPack p;
  p.t[0] = tables[0];
  p.t[1] = ntables > 1 ? tables[1] : tables[0];
  int vec = 1;
  int64_t maxLanes = 0;
  for (int i = 0; i < ntables; ++i) {
    const LutArgs& a = tables[i];
    vec &= (a.D % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.LUT) & 15) == 0) &&
           ((reinterpret_cast<uintptr_t>(a.O) & 15) == 0);
  }
  for (int i = 0; i < ntables; ++i) {
    int64_t lanes = (int64_t)tables[i].B * (vec ? tables[i].D / 4 : tables[i].D);
    maxLanes = lanes > maxLanes ? lanes : maxLanes;
  }
  if (maxLanes == 0) return cudaSuccess;
  int maxD = 0;
  int64_t maxB = 0;
  for (int i = 0; i < ntables; ++i) {
    maxD = tables[i].D > maxD ? tables[i].D : maxD;
    maxB = tables[i].B > maxB ? tables[i].B : maxB;
  }
  const size_t smem = (size_t)kRows * maxD * 4;
  int t = threads > 0 ? threads : 256;
  if (vec && smem <= 160 * 1024 && maxD / 4 <= kMaxColsPerThread * t) {
    // two-stage shared-memory gather: `threads` per (row, table) CTA. The
    // attribute is per device context: set on every launch (a per-process
    // flag would leave a second device at the 48 KB default)
    if (smem > 48 * 1024) {
      cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(lut_smem_kernel), 160 * 1024);
      if (e != cudaSuccess) return e;
    }
    lut_smem_kernel<<<dim3((unsigned)maxB, ntables), t, smem, s>>>(p.t[0], p.t[1]);
    return cudaGetLastError();
  }
  dim3 grid((unsigned)((maxLanes + t - 1) / t), ntables);
  lut_kernel<<<grid, t, 0, s>>>(p.t[0], p.t[1], vec);
  return cudaGetLastError();
}

}  // namespace k
}  // namespace tcb
