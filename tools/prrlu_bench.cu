// Standalone prrLU microbenchmark with per-phase cycle counts (development tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/prrlu_bench tools/prrlu_bench.cu
#define ACI_PRRLU_TIMING 1
#include "../paper_2604_00037_b200/csrc/prrlu.cu"

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

int main(int argc, char **argv) {
  // {m, n, kmax, static size}: static 1024 exercises the 8-warp instantiation on small live blocks
  int sizes[][4] = {{64, 64, 64, 0}, {128, 128, 128, 0}, {256, 256, 256, 0}, {512, 512, 512, 0}, {1024, 1024, 512, 0},
                    {64, 64, 64, 1024}, {128, 128, 128, 1024}, {256, 256, 256, 1024}, {512, 512, 512, 1024},
                    {64, 64, 64, 256}, {128, 128, 128, 256}, {256, 128, 128, 256}, {128, 256, 128, 256},
                    {200, 250, 200, 256}, {256, 64, 64, 256}, {64, 256, 64, 256}, {128, 64, 64, 256},
                    {96, 96, 96, 256},
                    // the product's dominant shapes at configs[3] chi = 256 (oracle log: m, n, r x bonds)
                    {512, 1024, 512, 1024}, {512, 256, 256, 1024}, {128, 256, 128, 1024}, {128, 64, 64, 1024},
                    {256, 1024, 256, 1024}, {512, 128, 128, 1024},
                    // hand-off pivots that are not multiples of 4 before rounding (prrlu.cu ho_round)
                    {300, 130, 130, 1024}, {450, 250, 250, 1024}, {500, 200, 200, 1024}, {400, 1000, 400, 1024}};
  double *dM, *dU, *deps;
  unsigned long long *dcol;
  int *drows, *dcols, *dr;
  unsigned long long *dkeys;
  unsigned *dctr, *depoch;
  LuDims *ddims;
  unsigned long long *dscale;
  long long *ddbg;
  cudaMalloc(&dM, sizeof(double) * 1024 * 1024);
  cudaMalloc(&dU, sizeof(double) * 1024 * 1024);
  cudaMalloc(&dcol, (size_t)16 * 2 * 148 * 1024 * kColSpread);
  cudaMemset(dcol, 0, (size_t)16 * 2 * 148 * 1024 * kColSpread);
  cudaMalloc(&depoch, 4);
  cudaMemset(depoch, 0, 4);
  cudaMalloc(&deps, 8);
  cudaMalloc(&drows, 4 * 1024);
  cudaMalloc(&dcols, 4 * 1024);
  cudaMalloc(&dr, 4);
  cudaMalloc(&dkeys, 32 * 2 * 148);
  cudaMemset(dkeys, 0, 32 * 2 * 148);
  cudaMalloc(&dctr, 4);
  cudaMalloc(&ddims, sizeof(LuDims));
  cudaMalloc(&dscale, 8);
  cudaMalloc(&ddbg, 64);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  std::vector<double> h(1024 * 1024);
  for (auto &x : h) x = nd(rng);
  cudaMemcpy(dM, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int only = argc > 1 ? atoi(argv[1]) : -1;
  prrlu_init();
  {
    const void *kern = (const void *)prrlu_kernel<kNWT, 2, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c : {8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c * 8);
      cfg.blockDim = dim3(kNWT * 32);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int n = 0;
      cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
      printf("max active %d-CTA clusters of prrlu_kernel: %d\n", c, n);
    }
  }
  for (auto &sz : sizes) {
    int m = sz[0], n = sz[1], kmax = sz[2], stat = sz[3] ? sz[3] : sz[0];
    if (only > 0 && m != only) continue;
    LuDims D{m, n, n, kmax, n};
    cudaMemcpy(ddims, &D, sizeof(D), cudaMemcpyHostToDevice);
    LuArgs a = {};
    a.M = dM; a.dims = ddims; a.tol = 0.0; a.thr_mode = 2; a.scale_bits = dscale;
    a.rows = drows; a.cols = dcols; a.r_out = dr; a.eps_out = deps; a.U = dU;
    a.colpub = dcol; a.colcap = 1024; a.keys = dkeys; a.counter = dctr; a.epoch = depoch; a.dbg = ddbg;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(ddbg, 0, 64);
      cudaEventRecord(e0);
      launch_prrlu(a, stat, stat, 0);
      cudaEventRecord(e1);
      cudaError_t err = cudaEventSynchronize(e1);
      if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      int r;
      long long dbg[8];
      cudaMemcpy(&r, dr, 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(dbg, ddbg, 64, cudaMemcpyDeviceToHost);
      if (rep == 2) {
        // FNV-1a over the ordered pivots: variants must take identical decisions
        std::vector<int> hr(r), hc(r);
        cudaMemcpy(hr.data(), drows, 4 * r, cudaMemcpyDeviceToHost);
        cudaMemcpy(hc.data(), dcols, 4 * r, cudaMemcpyDeviceToHost);
        unsigned long long hsh = 1469598103934665603ull;
        for (int t = 0; t < r; ++t) hsh = (hsh ^ (unsigned)(hr[t] * 4099 + hc[t])) * 1099511628211ull;
        printf("%4dx%4d (static %4d) r=%4d: %8.1f us total, %6.3f us/pivot | cycles/pivot:", m, n, stat, r, ms * 1e3,
               ms * 1e3 / r);
        for (int t = 0; t < 8; ++t) printf(" p%d=%lld", t, dbg[t] / (r > 0 ? r : 1));
        printf(" | piv %016llx\n", hsh);
      }
    }
  }
  return 0;
}
