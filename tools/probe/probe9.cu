// DSMEM pull probe (development tool, not part of the product path): per step every CTA of a
// C-CTA cluster pulls an M-double column from ONE owner CTA's shared memory (owner = step % C)
// with ld.shared::cluster (all threads, 16-byte loads), then the cluster re-synchronises with a
// st.async key exchange (probe7). Reports cycles of the pull phase (thread 0 of CTA 0) and
// us/step, to compare with the ~1000-cycle L2 column read of the grid tier.
#include <cstdio>
#include <cstdint>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned rank) {
  unsigned r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank)); return r;
}
__device__ __forceinline__ void mbar_init(unsigned a, unsigned cnt) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(cnt) : "memory"); }
__device__ __forceinline__ void mbar_expect(unsigned a, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned par) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(a),
      "r"(par) : "memory");
}
__device__ __forceinline__ void st_async_v4(unsigned raddr, uint4 v, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar) : "memory");
}
__device__ __forceinline__ double2 ld_cl_v2(unsigned a) {
  double2 r;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(a) : "memory");
  return r;
}

__global__ void __launch_bounds__(256) kern(int steps, int M, long long *out) {
  unsigned rank; asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  unsigned C; asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(C));
  const int tid = threadIdx.x;
  __shared__ alignas(16) double col[1024];
  __shared__ alignas(16) double dst[1024];
  __shared__ alignas(16) uint4 keys[2][16];
  __shared__ alignas(8) unsigned long long mb[2];
  for (int i = tid; i < 1024; i += blockDim.x) col[i] = rank * 1000 + i;
  if (tid == 0) {
    mbar_init(smem_u32(&mb[0]), 1); mbar_init(smem_u32(&mb[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect(smem_u32(&mb[0]), C * 16); mbar_expect(smem_u32(&mb[1]), C * 16);
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long ta = 0, tb = 0;
  for (int k = 0; k < steps; ++k) {
    const int par = k & 1;
    const unsigned mk = smem_u32(&mb[par]);
    long long t0 = clock64();
    const unsigned owner = k % C;
    const unsigned base = mapa(smem_u32(&col[0]), owner);
    for (int i = 2 * tid; i < M; i += 2 * blockDim.x) {
      double2 v = ld_cl_v2(base + 8 * i);
      dst[i] = v.x; dst[i + 1] = v.y;
    }
    __syncthreads();
    long long t1 = clock64();
    if (tid < (int)C) st_async_v4(mapa(smem_u32(&keys[par][rank]), tid), make_uint4(k, 0, rank, 0), mapa(mk, tid));
    mbar_wait(mk, (k >> 1) & 1);
    if (tid == 0) mbar_expect(mk, C * 16);
    __syncthreads();
    long long t2 = clock64();
    ta += t1 - t0; tb += t2 - t1;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (tid == 0 && blockIdx.x == 0) { out[0] = ta / steps; out[1] = tb / steps; out[2] = (long long)dst[5]; }
}

int main() {
  long long *out;
  CK(cudaMalloc(&out, 64));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int steps = 4000;
  for (int C : {2, 4, 8, 16})
    for (int M : {128, 256, 512, 1024}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C); cfg.blockDim = dim3(256);
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      long long h[3];
      float ms;
      cudaEventRecord(e0);
      cudaError_t e = cudaLaunchKernelEx(&cfg, kern, steps, M, out);
      cudaEventRecord(e1);
      if (e != cudaSuccess) { printf("C=%d: %s\n", C, cudaGetErrorString(e)); cudaGetLastError(); continue; }
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      CK(cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost));
      printf("C=%2d M=%4d: %.3f us/step | cycles: pull %lld, key exchange %lld\n", C, M, ms * 1e3 / steps, h[0], h[1]);
    }
  return 0;
}
