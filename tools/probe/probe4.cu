// Phase timing of the grid-tier exchange (variant A of probe3): per step, CTA 0 records
// (a) column publish + release + poll done, (b) key read + reduce, (c) winner column read.
#include <cstdio>
#include <cstdint>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void red_release_add(unsigned *p, unsigned v) { asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ void red_relaxed_add(unsigned *p, unsigned v) { asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__device__ unsigned pseudo(unsigned g, unsigned k) { return (g * 2654435761u + k * 40503u) & 0xffffu; }

template <int MODE>  // 0: release/acquire; 1: fence + relaxed; 2: no column publish (barrier only)
__global__ void kern(uint4 *keys, double *cols, unsigned *ctr, int steps, int m, long long *out) {
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  __shared__ double s_l[1024];
  double sink = 0;
  long long ta = 0, tb = 0, tc = 0, td = 0;
  for (int k = 0; k < steps; ++k) {
    const int par = k & 1;
    long long t0 = clock64();
    if (w == 0) {
      if (MODE != 2) {
        double *dst = cols + ((size_t)par * G + g) * m;
        for (int i = lane; i < m; i += 32) __stcg(dst + i, (double)(i + k));
      }
      __syncwarp();
      if (lane == 0) {
        __stcg(keys + par * G + g, make_uint4(pseudo(g, k), 0, g, 0));
        if (MODE == 1) { __threadfence(); red_relaxed_add(ctr, 1u); }
        else red_release_add(ctr, 1u);
      }
    }
    long long t1 = clock64();
    if (tid == 0) {
      if (MODE == 1) { while (ld_relaxed_u32(ctr) < (unsigned)(k + 1) * G) {} __threadfence(); }
      else while (ld_acquire_u32(ctr) < (unsigned)(k + 1) * G) {}
    }
    __syncthreads();
    long long t2 = clock64();
    unsigned best = 0, bi = 0;
    for (int t = lane; t < G; t += 32) { uint4 q = __ldcg(keys + par * G + t); if (q.x > best || (q.x == best && q.z < bi)) { best = q.x; bi = q.z; } }
    for (int o = 16; o; o >>= 1) { unsigned ob = __shfl_xor_sync(~0u, best, o), oi = __shfl_xor_sync(~0u, bi, o); if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; } }
    long long t3 = clock64();
    if (MODE != 2) {
      const double *src = cols + ((size_t)par * G + bi) * m;
      for (int i = tid; i < m; i += blockDim.x) s_l[i] = __ldcg(src + i);
    }
    __syncthreads();
    long long t4 = clock64();
    sink += s_l[(tid * 7 + k) % m];
    ta += t1 - t0; tb += t2 - t1; tc += t3 - t2; td += t4 - t3;
  }
  if (tid == 0 && g == 0) { out[0] = ta / steps; out[1] = tb / steps; out[2] = tc / steps; out[3] = td / steps; }
  if (sink == -1) out[5] = 1;
}

int main() {
  uint4 *keys; double *cols; unsigned *ctr; long long *out;
  CK(cudaMalloc(&keys, 16 * 2 * 160)); CK(cudaMalloc(&cols, 8 * 2 * 160 * 1024)); CK(cudaMalloc(&ctr, 4)); CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int steps = 4000; float ms; long long h[4];
  const char *names[] = {"rel/acq", "fence+relaxed", "barrier-only"};
  for (int mode = 0; mode < 3; ++mode)
    for (int G : {16, 64, 128}) {
      int m = 1024;
      CK(cudaMemset(ctr, 0, 4));
      void *args[] = {&keys, &cols, &ctr, &steps, &m, &out};
      const void *f = mode == 0 ? (const void *)kern<0> : mode == 1 ? (const void *)kern<1> : (const void *)kern<2>;
      cudaEventRecord(e0);
      CK(cudaLaunchCooperativeKernel(f, G, 256, args, 0, 0));
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      CK(cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost));
      printf("%-14s G=%3d: %.3f us/step | cycles: publish %lld, wait %lld, keys %lld, column %lld\n", names[mode], G,
             ms * 1e3 / steps, h[0], h[1], h[2], h[3]);
    }
  return 0;
}
