// Cluster-tier exchange probe: C-CTA cluster (8 or 16), per step: key to own smem, candidate
// column (m doubles) to global, barrier.cluster, every warp reads the C keys via DSMEM, all
// threads read the winner's column from L2. Not part of the product path.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)
__device__ unsigned pseudo(unsigned g, unsigned k) { return (g * 2654435761u + k * 40503u) & 0xffffu; }

__global__ void __launch_bounds__(512) kern(double *cols, int steps, int m, long long *out) {
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), rank = cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  __shared__ unsigned s_key[2][2];
  __shared__ double s_l[1024];
  double sink = 0;
  long long ta = 0, tb = 0, tc = 0, td = 0;
  const int gbase = blockIdx.x - rank;  // first CTA of this cluster
  for (int k = 0; k < steps; ++k) {
    const int par = k & 1;
    long long t0 = clock64();
    if (w == 1) {
      double *dst = cols + ((size_t)par * gridDim.x + blockIdx.x) * m;
      for (int i = lane; i < m; i += 32) __stcg(dst + i, (double)(i + k));
      if (lane == 0) { s_key[par][0] = pseudo(blockIdx.x, k); s_key[par][1] = rank; }
    }
    long long t1 = clock64();
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    long long t2 = clock64();
    unsigned best = 0, bi = 0;
    if (lane < C) {
      unsigned *pk = cl.map_shared_rank(&s_key[par][0], lane);
      best = pk[0]; bi = pk[1];
    }
    for (int o = 16; o; o >>= 1) { unsigned ob = __shfl_xor_sync(~0u, best, o), oi = __shfl_xor_sync(~0u, bi, o); if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; } }
    long long t3 = clock64();
    const double *src = cols + ((size_t)par * gridDim.x + gbase + bi) * m;
    double v0 = 0, v1 = 0;
    if (tid < m) v0 = __ldcg(src + tid);
    if (tid + 512 < m) v1 = __ldcg(src + tid + 512);
    if (tid < m) s_l[tid] = v0;
    if (tid + 512 < m) s_l[tid + 512] = v1;
    __syncthreads();
    long long t4 = clock64();
    sink += s_l[(tid * 7 + k) % m];
    ta += t1 - t0; tb += t2 - t1; tc += t3 - t2; td += t4 - t3;
  }
  if (tid == 0 && blockIdx.x == 0) { out[0] = ta / steps; out[1] = tb / steps; out[2] = tc / steps; out[3] = td / steps; }
  if (sink == -1) out[5] = 1;
}

int main() {
  double *cols; long long *out;
  CK(cudaMalloc(&cols, 8 * 2 * 160 * 1024)); CK(cudaMalloc(&out, 64));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int steps = 4000; float ms; long long h[4];
  for (int C : {4, 8, 16}) for (int ncl : {1, 4}) for (int m : {512, 1024}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C * ncl); cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int ncl_max = 0;
    cudaOccupancyMaxActiveClusters(&ncl_max, (void *)kern, &cfg);
    cudaEventRecord(e0);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, cols, steps, m, out);
    cudaEventRecord(e1);
    if (e != cudaSuccess) { printf("C=%d ncl=%d: %s\n", C, ncl, cudaGetErrorString(e)); cudaGetLastError(); continue; }
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    CK(cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost));
    printf("C=%2d clusters=%d (max active %d) m=%4d: %.3f us/step | cycles: publish %lld, barrier %lld, dsmem keys %lld, column %lld\n",
           C, ncl, ncl_max, m, ms * 1e3 / steps, h[0], h[1], h[2], h[3]);
  }
  return 0;
}
