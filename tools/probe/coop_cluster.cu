// Probe: does the driver accept a COOPERATIVE launch with a thread-block-cluster dimension
// (co-residency guarantee for the multi-cluster prrLU tier)? Not product code.
#include <cstdio>
__global__ void k(int *out) {
  if (threadIdx.x == 0) atomicAdd(out, 1);
}
int main() {
  int *d;
  cudaMalloc(&d, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {8, 16}) {
    for (int grid : {cs * 4, cs * 7, cs * 8, cs * 9}) {
      cudaMemset(d, 0, 4);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(256);
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeCooperative;
      at[1].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      cudaError_t e = cudaLaunchKernelEx(&cfg, k, d);
      cudaError_t e2 = cudaDeviceSynchronize();
      int h = 0;
      cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
      printf("cluster %2d grid %3d cooperative: launch=%s sync=%s ctas_ran=%d\n", cs, grid, cudaGetErrorString(e),
             cudaGetErrorString(e2), h);
      cudaGetLastError();
    }
  }
  return 0;
}
