// fc_regs.cu — FC chains whose layers are all short reductions (MLP3:
// 128 -> 64 -> 32 -> 2, proj/kernels/mlp3.tc:4-16; kred <= 128 per layer),
// one CTA per R batch rows, no cluster, no shared-memory weight staging.
//
// The cluster kernel (fc_chain.cu) spends most of an MLP3 call before its
// first FFMA: bulk-copy issue (~0.1-0.2 us per copy on the SM's TMA unit),
// DSMEM pushes and cluster barriers between layers (fc_trace: the first
// layer's data lands ~5400 cycles after entry; the whole chain is ~1100
// cycles of FFMA latency). Here every warp is assigned to one layer and one
// lane to one output column of it. At entry the CTA issues plain coalesced
// 16-byte loads of every layer's weights and its R input rows into shared
// memory (all in flight within the first few hundred cycles); each lane
// then moves its weight row into registers (<= 32 float4s). Layer by layer
// (one CTA barrier between layers) the layer's lanes run their R chains
// from registers (weights) and shared-memory broadcasts (activations),
// write the layer's return and leave it in shared memory for the next.
//
// Exactness: each (row, column) output is one lane's sequential FFMA chain
// in ascending k from bias[o], then fmaxf(., 0) — the interpreter's order
// (interpreter.cc:218-233; builtin fmaxf -> std::fmax, :22-24).
#include "kernels.cuh"

namespace tcb {
namespace k {

namespace {

constexpr int kRegsKq = 32;  // float4s per weight row (kred <= 128)

struct FcRegsPlan {
  int vecW[kMaxLayers];         // weight rows load as float4 (ldw % 4 == 0, 16-byte aligned)
  int wOff[kMaxLayers];         // weights in shared memory (floats)
  int wld4[kMaxLayers];         // their row stride (float4s, odd)
  int vecI;                     // input rows load as float4
  int warpOff[kMaxLayers + 1];  // first warp of each layer
  int ald[kMaxLayers + 1];      // activation row strides (floats, multiple of 4)
  int actOff[kMaxLayers + 1];   // activation buffers in shared memory (floats)
};

__device__ __forceinline__ float4 ldsA(unsigned addr) {
  float4 v;
  asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

#ifdef TCB_FCR_TRACE
// diagnostic build only (profiles/fc_regs_trace.cu): per-CTA globaltimer stamps
__device__ unsigned long long g_fcr_trace[1024][8];
#define FCR_STAMP(ev)                                                          \
  do {                                                                         \
    unsigned long long t_;                                                     \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                    \
    if (threadIdx.x == 0 && blockIdx.x < 1024) g_fcr_trace[blockIdx.x][ev] = t_; \
  } while (0)
#else
#define FCR_STAMP(ev) \
  do {                \
  } while (0)
#endif

template <int NL, int R>
__global__ void __launch_bounds__(256) fc_regs_kernel(const __grid_constant__ FcChainArgs a,
                                                       const __grid_constant__ FcRegsPlan p) {
  extern __shared__ __align__(16) float act[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row0 = blockIdx.x * R;
  const int rows = min(R, a.batch - row0);
  FCR_STAMP(0);
  int layer = -1;
#pragma unroll
  for (int l = 0; l < NL; ++l)
    if (warp >= p.warpOff[l] && warp < p.warpOff[l + 1]) layer = l;

  // ---- every global load up front, coalesced: all layers' weights into
  // shared memory (rows padded to an odd number of float4s, so the lanes'
  // row reads below hit distinct bank groups) and the CTA's input rows, by
  // 16-byte cp.async where the rows allow it (asynchronous: a load-then-store
  // loop serialised every thread on one L2 round trip per 16 bytes, ~6 us
  // for MLP3's 40 KB, profiles/fc_regs_trace.cu). Each lane owns one output
  // column of one layer. (Each lane loading its own weight row straight from
  // global memory put 32 scattered sectors in every warp load instead.)
  auto stage = [&](float4* dst, const float* src, int kr, bool vec) {
    // one zero-padded float4 of a row: 4 k values starting at src
    if (vec) {
      const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
    } else {
      float4 v;
      v.x = 0 < kr ? __ldg(src) : 0.0f;
      v.y = 1 < kr ? __ldg(src + 1) : 0.0f;
      v.z = 2 < kr ? __ldg(src + 2) : 0.0f;
      v.w = 3 < kr ? __ldg(src + 3) : 0.0f;
      *dst = v;
    }
  };
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const int kr = a.L[l].kred, k4 = (kr + 3) >> 2, n = a.L[l].out;
    float4* dst = reinterpret_cast<float4*>(act + p.wOff[l]);
    for (int e = tid; e < n * k4; e += blockDim.x) {
      const int r = e / k4, q = e - r * k4;
      stage(dst + r * p.wld4[l] + q, a.L[l].W + (int64_t)r * a.L[l].ldw + 4 * q, kr - 4 * q,
            p.vecW[l] && 4 * q + 4 <= kr);
    }
  }
  {
    const int kr = a.L[0].kred, k0 = (kr + 3) >> 2;
    float4* a0 = reinterpret_cast<float4*>(act + p.actOff[0]);
    for (int e = tid; e < R * k0; e += blockDim.x) {
      const int r = e / k0, q = e - r * k0;
      if (r < rows)
        stage(a0 + r * (p.ald[0] >> 2) + q, a.I + (int64_t)(row0 + r) * a.ldi + 4 * q, kr - 4 * q,
              p.vecI && 4 * q + 4 <= kr);
      else
        a0[r * (p.ald[0] >> 2) + q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  float bias = 0.0f;
  int col = 0, K4 = 0, KT = 0;  // full float4 groups, tail steps (kred % 4)
  bool live = false;
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    if (layer == l) {
      col = (warp - p.warpOff[l]) * 32 + lane;
      live = col < a.L[l].out;
      K4 = a.L[l].kred >> 2;
      KT = a.L[l].kred & 3;
      bias = live ? __ldg(a.L[l].bias + col) : 0.0f;
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  FCR_STAMP(1);

#pragma unroll
  for (int l = 0; l < NL; ++l) {
    if (layer == l) {
      const float* in = act + p.actOff[l];
      float acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = bias;
      // weights: this lane's row in shared memory (odd float4 stride: the
      // lanes' reads hit distinct bank groups); activations: broadcasts.
      // A compact loop: fully unrolled per-layer chains overflowed the
      // instruction cache (~38 cycles per step)
      const unsigned wr = static_cast<unsigned>(__cvta_generic_to_shared(act + p.wOff[l])) +
                          (unsigned)(min(col, a.L[l].out - 1) * p.wld4[l]) * 16u;
      const unsigned xr = static_cast<unsigned>(__cvta_generic_to_shared(in));
      const unsigned xs = (unsigned)p.ald[l] * 4u;
#pragma unroll 2
      for (int q = 0; q < K4; ++q) {
        const float4 wv = ldsA(wr + q * 16);
        float4 x[R];
#pragma unroll
        for (int r = 0; r < R; ++r) x[r] = ldsA(xr + r * xs + q * 16);
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = __fmaf_rn(x[r].x, wv.x, acc[r]);
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = __fmaf_rn(x[r].y, wv.y, acc[r]);
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = __fmaf_rn(x[r].z, wv.z, acc[r]);
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = __fmaf_rn(x[r].w, wv.w, acc[r]);
      }
      if (KT) {  // the kred % 4 tail steps, still in order
        const float4 wv = ldsA(wr + K4 * 16);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float4 x = ldsA(xr + r * xs + K4 * 16);
          acc[r] = __fmaf_rn(x.x, wv.x, acc[r]);
          if (KT > 1) acc[r] = __fmaf_rn(x.y, wv.y, acc[r]);
          if (KT > 2) acc[r] = __fmaf_rn(x.z, wv.z, acc[r]);
        }
      }
      if (live) {
        float* nxt = act + p.actOff[l + 1];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float v = fmaxf(acc[r], 0.0f);
          nxt[r * p.ald[l + 1] + col] = v;
          if (r < rows) a.L[l].O[(int64_t)(row0 + r) * a.L[l].out + col] = v;
        }
      }
    }
    if (l + 1 < NL) __syncthreads();  // layer l's activations complete
#ifdef TCB_FCR_TRACE
    if (l + 1 == NL) __syncthreads();
#endif
    FCR_STAMP(2 + l);
  }
}

template <int NL>
void* pickRegs(int R) {
  switch (R) {
    case 1: return reinterpret_cast<void*>(fc_regs_kernel<NL, 1>);
    case 2: return reinterpret_cast<void*>(fc_regs_kernel<NL, 2>);
    case 4: return reinterpret_cast<void*>(fc_regs_kernel<NL, 4>);
    default: return nullptr;
  }
}

}  // namespace

size_t fcRegsSmem(const FcChainArgs& a, int rows) {
  size_t f = 0;
  for (int l = 0; l <= a.layers; ++l) {
    const int w = l == 0 ? a.L[0].kred : a.L[l - 1].out;
    f += (size_t)rows * ((w + 3) & ~3);
  }
  for (int l = 0; l < a.layers; ++l) f += (size_t)a.L[l].out * ((((a.L[l].kred + 3) / 4) | 1) * 4);
  return f * 4;
}

bool fcRegsSupported(const FcChainArgs& a, int rows, const char** why) {
  auto no = [&](const char* m) {
    if (why) *why = m;
    return false;
  };
  if (rows != 1 && rows != 2 && rows != 4) return no("register FC chain rows per CTA must be 1, 2 or 4");
  if (a.layers < 1 || a.layers > 3) return no("register FC chain takes 1 to 3 layers");
  int warps = 0;
  for (int l = 0; l < a.layers; ++l) {
    // kred_l of the kRegsKq register float4s, the last one possibly partial
    if (a.L[l].kred > 4 * kRegsKq) return no("register FC chain needs every reduction <= 128 steps");
    warps += (a.L[l].out + 31) / 32;
  }
  if (warps > 8) return no("register FC chain: more than 256 output columns in all layers");
  if (fcRegsSmem(a, rows) > 200 * 1024) return no("register FC chain: weights exceed shared memory");
  return true;
}


cudaError_t launchFcRegs(const FcChainArgs& a, int rows, cudaStream_t s) {
  if (a.batch <= 0) return cudaSuccess;
  if (!fcRegsSupported(a, rows, nullptr)) return cudaErrorInvalidValue;
  FcRegsPlan p{};
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  for (int l = 0; l < a.layers; ++l) p.vecW[l] = a.L[l].ldw % 4 == 0 && al16(a.L[l].W);
  p.vecI = a.ldi % 4 == 0 && al16(a.I);
  int warps = 0, off = 0;
  for (int l = 0; l < a.layers; ++l) {
    p.warpOff[l] = warps;
    warps += (a.L[l].out + 31) / 32;
  }
  p.warpOff[a.layers] = warps;
  for (int l = 0; l <= a.layers; ++l) {
    const int w = l == 0 ? a.L[0].kred : a.L[l - 1].out;
    p.ald[l] = (w + 3) & ~3;  // zero-padded to whole float4s (the tail group reads them, never uses them)
    p.actOff[l] = off;
    off += rows * p.ald[l];
  }
  for (int l = 0; l < a.layers; ++l) {
    p.wOff[l] = off;
    p.wld4[l] = ((a.L[l].kred + 3) / 4) | 1;
    off += a.L[l].out * p.wld4[l] * 4;
  }
  const size_t smem = (size_t)off * 4;
  void* kern = a.layers == 1 ? pickRegs<1>(rows) : a.layers == 2 ? pickRegs<2>(rows) : pickRegs<3>(rows);
  if (!kern) return cudaErrorInvalidValue;
  {
    cudaError_t e = ensureFuncAttrs(reinterpret_cast<const void*>(kern), (int)smem);
    if (e != cudaSuccess) return e;
  }
  void* args[] = {const_cast<FcChainArgs*>(&a), &p};
  return cudaLaunchKernel(kern, dim3((a.batch + rows - 1) / rows), dim3(warps * 32), args, smem, s);
}

}  // namespace k
}  // namespace tcb
