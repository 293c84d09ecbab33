// fc_chain.cu — fused chains of FC+bias+ReLU layers in ONE kernel:
//   MLP1     proj/kernels/mlp1.tc:2-6        (1 layer)
//   2FCRelu  paper_1802_04730_b200/tc/ops.tc (2 layers)
//   MLP3     proj/kernels/mlp3.tc:4-16       (3 layers, single kernel as in
//            the paper's claim)
//
// One CTA owns R batch rows. Every layer's input activations live in
// shared memory (the first layer's rows are staged once, each later
// layer reads the previous layer's smem output), so intermediate layers
// never round-trip through HBM; each layer's output is also written to its
// global return tensor. Weights stream through a double-buffered
// shared-memory ring of KC-wide column chunks filled by 16-byte cp.async.
// Thread t owns output features t, t+T (Q ≤ 2 per thread) for all R rows:
// R independent chains per feature, each a sequential FFMA chain in
// ascending k starting from bias[o] — the reference order — followed by
// fmaxf(·, 0) (interpreter.cc:22-24: std::fmax, NaN-ignoring).
#include "kernels.cuh"

namespace tcb {
namespace k {

namespace {

constexpr int KC = 32;       // weight chunk depth (columns)
constexpr int WLD = KC + 4;  // padded smem row stride

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}

__host__ __device__ inline int up4(int x) { return (x + 3) & ~3; }

template <int R, int Q>
__global__ void fc_chain_kernel(const FcChainArgs a, const int wvec, const int outMax) {
  extern __shared__ __align__(16) float sm[];
  const int T = blockDim.x, tid = threadIdx.x;
  const int row0 = blockIdx.x * R;

  // [2][outMax][WLD] weight ring, then the activation buffers: each
  // layer's input [R][ld] is followed by its output (the next layer's input)
  float* wbuf = sm;
  float* in = wbuf + 2 * outMax * WLD;
  int ldi = up4(a.L[0].kred);

  // stage the first layer's input rows (only the kred columns it reads)
  for (int e = tid; e < R * ldi; e += T) {
    int r = e / ldi, c = e % ldi;
    int b = row0 + r;
    in[e] = (b < a.batch && c < a.L[0].kred) ? a.I[(int64_t)b * a.ldi + c] : 0.0f;
  }

#pragma unroll
  for (int l = 0; l < kMaxLayers; ++l) {
    if (l >= a.layers) break;
    const FcLayer L = a.L[l];
    float acc[Q][R];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      int o = tid + q * T;
#pragma unroll
      for (int r = 0; r < R; ++r) acc[q][r] = (o < L.out) ? __ldg(L.bias + o) : 0.0f;
    }
    const int nch = (L.kred + KC - 1) / KC;
    auto loadChunk = [&](int stage, int k0) {
      float* dst = wbuf + stage * outMax * WLD;
      if (wvec) {
        for (int e = tid; e < L.out * (KC / 4); e += T) {
          int o = e / (KC / 4), c = (e % (KC / 4)) * 4;
          bool ok = k0 + c < L.kred;
          const float* src = ok ? L.W + (int64_t)o * L.ldw + k0 + c : L.W;
          cp_async16(dst + o * WLD + c, src, ok ? 16 : 0);
        }
      } else {
        for (int e = tid; e < L.out * KC; e += T) {
          int o = e / KC, c = e % KC;
          dst[o * WLD + c] = (k0 + c < L.kred) ? L.W[(int64_t)o * L.ldw + k0 + c] : 0.0f;
        }
      }
    };
    __syncthreads();  // previous layer's outputs (this layer's inputs) complete; wbuf free
    loadChunk(0, 0);
    asm volatile("cp.async.commit_group;\n" ::);
    for (int c = 0; c < nch; ++c) {
      const int st = c & 1;
      if (c + 1 < nch) {
        loadChunk(st ^ 1, (c + 1) * KC);
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 1;\n" ::);
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::);
      }
      __syncthreads();
      const float* wch = wbuf + st * outMax * WLD;
      const int k0 = c * KC;
      const int klim = min(KC, L.kred - k0);
      const int k4 = klim & ~3;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        int o = tid + q * T;
        if (o < L.out) {
          const float* wr = wch + o * WLD;
          int kk = 0;
          for (; kk < k4; kk += 4) {
            float4 w4 = *reinterpret_cast<const float4*>(wr + kk);
#pragma unroll
            for (int r = 0; r < R; ++r) {
              float4 x4 = *reinterpret_cast<const float4*>(in + r * ldi + k0 + kk);
              float v = acc[q][r];
              v = __fmaf_rn(x4.x, w4.x, v);
              v = __fmaf_rn(x4.y, w4.y, v);
              v = __fmaf_rn(x4.z, w4.z, v);
              v = __fmaf_rn(x4.w, w4.w, v);
              acc[q][r] = v;
            }
          }
          for (; kk < klim; ++kk) {
            float w = wr[kk];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[q][r] = __fmaf_rn(in[r * ldi + k0 + kk], w, acc[q][r]);
          }
        }
      }
      __syncthreads();
    }
    // epilogue: ReLU, keep in smem for the next layer, write the return
    float* nxt = in + R * ldi;
    const int ldn = up4(L.out);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      int o = tid + q * T;
      if (o < L.out) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float v = fmaxf(acc[q][r], 0.0f);
          nxt[r * ldn + o] = v;
          int b = row0 + r;
          if (b < a.batch) L.O[(int64_t)b * L.out + o] = v;
        }
      }
    }
    // zero the pad columns so float4 reads of the next layer stay defined
    for (int e = tid; e < R * (ldn - L.out); e += T) {
      int r = e / (ldn - L.out), c = L.out + e % (ldn - L.out);
      nxt[r * ldn + c] = 0.0f;
    }
    in = nxt;
    ldi = ldn;
  }
}

template <int R>
cudaError_t launchR(const FcChainArgs& a, int threads, int wvec, int outMax, size_t smem, cudaStream_t s) {
  dim3 grid((a.batch + R - 1) / R);
  int q = (outMax + threads - 1) / threads;
  if (q <= 1) {
    auto kfn = fc_chain_kernel<R, 1>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kfn<<<grid, threads, smem, s>>>(a, wvec, outMax);
  } else if (q == 2) {
    auto kfn = fc_chain_kernel<R, 2>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kfn<<<grid, threads, smem, s>>>(a, wvec, outMax);
  } else {
    return cudaErrorInvalidConfiguration;
  }
  return cudaGetLastError();
}

int outMaxOf(const FcChainArgs& a) {
  int m = 0;
  for (int l = 0; l < a.layers; ++l) m = a.L[l].out > m ? a.L[l].out : m;
  return m;
}

}  // namespace

size_t fcChainSmem(const FcChainArgs& a, int rows) {
  size_t floats = (size_t)rows * up4(a.L[0].kred);
  for (int l = 0; l < a.layers; ++l) floats += (size_t)rows * up4(a.L[l].out);
  floats += 2 * (size_t)outMaxOf(a) * WLD;
  return floats * sizeof(float);
}

cudaError_t launchFcChain(const FcChainArgs& a, int rows, int threads, cudaStream_t s) {
  if (a.batch <= 0) return cudaSuccess;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  int wvec = 1;
  for (int l = 0; l < a.layers; ++l)
    wvec &= (a.L[l].ldw % 4 == 0) && al16(a.L[l].W);
  int outMax = outMaxOf(a);
  size_t smem = fcChainSmem(a, rows);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  switch (rows) {
    case 1: return launchR<1>(a, threads, wvec, outMax, smem, s);
    case 2: return launchR<2>(a, threads, wvec, outMax, smem, s);
    case 4: return launchR<4>(a, threads, wvec, outMax, smem, s);
    case 8: return launchR<8>(a, threads, wvec, outMax, smem, s);
    default: return cudaErrorInvalidConfiguration;
  }
}

}  // namespace k
}  // namespace tcb
