// fc_trace.cu — diagnostic harness: builds the FC-chain kernel with phase
// timestamps (TCB_FC_TRACE) and prints per-phase cycle offsets from kernel
// entry (median / max over CTAs) for the paper shapes. Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_FC_TRACE \
//        -I paper_1802_04730_b200/csrc profiles/fc_trace.cu -o profiles/fc_trace && profiles/fc_trace
#include "kernels/fc_chain.cu"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

using namespace tcb::k;

static void run(const char* label, FcChainArgs a, int rows, int cn, int threads) {
  static unsigned long long z[1024][32];
  {
    FcPlan pl;
    size_t smem = planFc(a, rows, cn, pl);
    auto kern = fcKernel(a.layers, pl.bulk);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cn > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cn, (a.batch + rows - 1) / rows, 1);
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cn;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, kern, &cfg);
    printf("[%s] smem %zu B, grid %d clusters, max active clusters %d (%s)\n", label, smem,
           (a.batch + rows - 1) / rows, nc, cudaGetErrorString(e));
  }
  for (int it = 0; it < 3; ++it) launchFcChain(a, rows, cn, threads, 0);
  cudaDeviceSynchronize();
  cudaMemcpyToSymbol(g_fc_trace, z, sizeof(z));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  launchFcChain(a, rows, cn, threads, 0);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  static unsigned long long tr[1024][32];
  cudaMemcpyFromSymbol(tr, g_fc_trace, sizeof(tr));
  int nblk = cn * ((a.batch + rows - 1) / rows);
  printf("%s: %s  %.2f us  (%d CTAs)\n", label, cudaGetErrorString(err), ms * 1e3, nblk);
  const char* names[32] = {"start", "bar_init", "copies_issued", "L0_data", "L0_done", "init_fence", "L1_data",
                           "L1_done", "cta_sync", "L2_data", "L2_done", "cl_arrive", "expects", "-", "-", "end",
                           "L0_chain", "L1_chain", "L2_chain", "L3_chain", "L0_clwait", "L0_enter", "L1_enter", "L2_enter",
                           "in_copies", "w0_start", "w1_start", "w2_start", "w3_start", "-", "-", "-"};
  unsigned long long g0 = ~0ull, g1 = 0;
  for (int b = 0; b < nblk; ++b) {
    if (tr[b][13]) g0 = std::min(g0, tr[b][13]);
    g1 = std::max(g1, tr[b][14]);
  }
  std::vector<long long> st;
  for (int b = 0; b < nblk; ++b) st.push_back((long long)(tr[b][13] - g0));
  std::sort(st.begin(), st.end());
  printf("  globaltimer: first CTA start -> last CTA end %.2f us; CTA start skew median %lld max %lld ns\n",
         (g1 - g0) * 1e-3, st[st.size() / 2], st.back());
  const int order[] = {1, 5, 8, 11, 12, 24, 25, 26, 27, 28, 2, 3, 20, 21, 16, 4, 6, 22, 17, 7, 9, 23, 18, 10, 19, 15};
  for (int ev : order) {
    std::vector<long long> d;
    for (int b = 0; b < nblk; ++b)
      if (tr[b][ev] && tr[b][0]) d.push_back((long long)(tr[b][ev] - tr[b][0]));
    if (d.empty()) continue;
    std::sort(d.begin(), d.end());
    printf("  %-13s median %7lld  max %7lld cycles\n", names[ev], d[d.size() / 2], d.back());
  }
}

int main() {
  auto alloc = [](size_t n) {
    float* p;
    cudaMalloc(&p, n * 4);
    cudaMemset(p, 0, n * 4);
    return p;
  };
  FcChainArgs f{};
  f.I = alloc(128 * 1128);
  f.ldi = 1128;
  f.batch = 128;
  f.layers = 2;
  f.L[0] = {alloc(128 * 1128), alloc(128), alloc(128 * 128), 128, 1128, 1128};
  f.L[1] = {alloc(64 * 128), alloc(64), alloc(128 * 64), 64, 128, 128};
  FcChainArgs one = f;
  one.layers = 1;
  FcChainArgs m{};
  m.I = alloc(128 * 128);
  m.ldi = 128;
  m.batch = 128;
  m.layers = 3;
  m.L[0] = {alloc(64 * 128), alloc(64), alloc(128 * 64), 64, 128, 128};
  m.L[1] = {alloc(32 * 64), alloc(32), alloc(128 * 32), 32, 64, 64};
  m.L[2] = {alloc(2 * 32), alloc(2), alloc(128 * 2), 2, 32, 32};
  // the default plans of the bench step (ops.cc defaultOptions)
  run("2FCRelu rows=4 cn=8", f, 4, 8, 64);
  if (getenv("FC_TRACE_2FC")) {  // other 2FCRelu plans (r02: rows=8 cn=8 t=128 measured 15 us in the sweep)
    run("2FCRelu rows=4 cn=8 t=32 (column pairs)", f, 4, 8, 32);
    run("MLP1 rows=4 cn=8 t=32 (column pairs)", one, 4, 8, 32);
    run("2FCRelu rows=8 cn=8 t=64 (column pairs)", f, 8, 8, 64);
    if (getenv("FC_TRACE_PAIR_ONLY")) return 0;
    run("2FCRelu rows=8 cn=8 t=128", f, 8, 8, 128);
    run("2FCRelu rows=8 cn=16 t=64", f, 8, 16, 64);
    run("2FCRelu rows=2 cn=8 t=32", f, 2, 8, 32);
    run("2FCRelu rows=8 cn=4 t=256", f, 8, 4, 256);
    return 0;
  }
  run("MLP1 rows=4 cn=8", one, 4, 8, 64);
  run("MLP3 rows=2 cn=4", m, 2, 4, 64);
  run("MLP3 rows=4 cn=4", m, 4, 4, 64);
  run("MLP3 rows=1 cn=1", m, 1, 1, 64);
  return 0;
}
