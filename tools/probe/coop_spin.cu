// Probe: is a COOPERATIVE launch with a cluster dimension refused when its clusters cannot all be
// co-resident (the guarantee a spinning multi-cluster prrLU grid needs)? Each CTA (1 per SM: 200 KB
// of shared memory) arrives on a counter and spins, with a ~0.5 s timeout, until all have arrived.
// Not product code.
#include <cstdio>
__global__ void spin(unsigned *ctr, unsigned *timeouts) {
  extern __shared__ char big[];
  big[threadIdx.x] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(ctr, 1u);
    long long t0 = clock64();
    while (atomicAdd(ctr, 0u) < gridDim.x) {
      if (clock64() - t0 > 1000000000ll) { atomicAdd(timeouts, 1u); break; }
    }
  }
}
int main() {
  unsigned *d;
  cudaMalloc(&d, 8);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(spin, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {8, 16}) {
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(cs); q.blockDim = dim3(256); q.dynamicSmemBytes = smem;
    cudaLaunchAttribute a1[1];
    a1[0].id = cudaLaunchAttributeClusterDimension;
    a1[0].val.clusterDim.x = cs; a1[0].val.clusterDim.y = 1; a1[0].val.clusterDim.z = 1;
    q.attrs = a1; q.numAttrs = 1;
    int nmax = 0;
    cudaOccupancyMaxActiveClusters(&nmax, spin, &q);
    printf("cluster %d: max active clusters %d\n", cs, nmax);
    for (int ncl = nmax - 1; ncl <= nmax + 2; ++ncl) {
      for (int coop = 0; coop < 2; ++coop) {
        if (!coop && ncl > nmax) continue;  // a plain launch beyond co-residency would just time out
        cudaMemset(d, 0, 8);
        cudaLaunchConfig_t cfg = q;
        cfg.gridDim = dim3(cs * ncl);
        cudaLaunchAttribute at[2];
        at[0] = a1[0];
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = coop;
        cfg.attrs = at; cfg.numAttrs = 2;
        cudaError_t e = cudaLaunchKernelEx(&cfg, spin, d, d + 1);
        cudaError_t e2 = cudaDeviceSynchronize();
        unsigned h[2] = {0, 0};
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("  %2d clusters (%3d CTAs) coop=%d: launch=%s sync=%s arrived=%u timeouts=%u\n", ncl, cs * ncl, coop,
               cudaGetErrorString(e), cudaGetErrorString(e2), h[0], h[1]);
        cudaGetLastError();
      }
    }
  }
  return 0;
}
