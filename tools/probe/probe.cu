// Microbenchmarks that size the design (not part of the product path):
//  1. DMMA.8x8x4 (mma.sync f64) throughput per SM and chip-wide.
//  2. Per-step latency of the inter-CTA exchanges a full-pivoting prrLU needs:
//     (a) all-to-all flag exchange through L2 over G co-resident CTAs,
//     (b) the same plus reading an 8 KB "winner column" published by one CTA,
//     (c) hardware cluster barrier + DSMEM read for 8/16-CTA clusters,
//     (d) __syncthreads inside one CTA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[4][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[8] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t] = fma(a, b, c[t]);
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t];
  if (s == 12345.0) out[0] = s;
}

struct Slot { unsigned long long flag; double val; int idx; int pad; };

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v; asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

// all-to-all exchange: each CTA writes its slot (+ optionally its 'column'), then polls everyone's flag.
__global__ void a2a_exchange(Slot* slots, double* cols, int steps, int colLen, long long* cycles) {
  int G = gridDim.x;
  __shared__ double sred[32];
  __shared__ int winner;
  long long t0 = clock64();
  for (int k = 1; k <= steps; ++k) {
    int par = k & 1;
    if (colLen > 0) {
      double* my = cols + ((size_t)par * G + blockIdx.x) * colLen;
      for (int i = threadIdx.x; i < colLen; i += blockDim.x) my[i] = k + i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      Slot* s = slots + par * G + blockIdx.x;
      s->val = (double)((blockIdx.x * 7 + k) % G);
      s->idx = blockIdx.x;
      st_release(&s->flag, (unsigned long long)k);
    }
    // warp 0 polls all flags
    if (threadIdx.x < 32) {
      double best = -1; int bi = 0;
      for (int g = threadIdx.x; g < G; g += 32) {
        Slot* s = slots + par * G + g;
        while (ld_acquire(&s->flag) < (unsigned long long)k) {}
        double v = s->val;
        if (v > best) { best = v; bi = g; }
      }
      for (int o = 16; o; o >>= 1) {
        double ob = __shfl_xor_sync(0xffffffff, best, o);
        int oi = __shfl_xor_sync(0xffffffff, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (threadIdx.x == 0) winner = bi;
    }
    __syncthreads();
    if (colLen > 0) {
      const double* w = cols + ((size_t)par * G + winner) * colLen;
      double acc = 0;
      for (int i = threadIdx.x; i < colLen; i += blockDim.x) acc += __ldcg(w + i);
      sred[threadIdx.x & 31] = acc;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = t1 - t0;
}

// cooperative-groups grid.sync per step
__global__ void cg_gridsync(int steps, long long* cycles) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int k = 0; k < steps; ++k) g.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = t1 - t0;
}

// cluster barrier + DSMEM read of a peer's 'column'
__global__ void cluster_exchange(int steps, int colLen, long long* cycles, double* out) {
  extern __shared__ double col[];
  cg::cluster_group cl = cg::this_cluster();
  unsigned int rank = cl.block_rank();
  unsigned int csz = cl.num_blocks();
  double acc = 0;
  long long t0 = clock64();
  for (int k = 0; k < steps; ++k) {
    int par = k & 1;
    for (int i = threadIdx.x; i < colLen; i += blockDim.x) col[par * colLen + i] = k + i + rank;
    cl.sync();
    unsigned int w = (k * 5) % csz;
    double* peer = cl.map_shared_rank(col, w);
    for (int i = threadIdx.x; i < colLen; i += blockDim.x) acc += peer[par * colLen + i];
  }
  cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = t1 - t0;
  if (acc == -1.0) out[0] = acc;
}

__global__ void cta_sync(int steps, long long* cycles, double* out) {
  __shared__ double x[1024];
  double acc = 0;
  long long t0 = clock64();
  for (int k = 0; k < steps; ++k) {
    x[threadIdx.x] = k + threadIdx.x;
    __syncthreads();
    acc += x[(threadIdx.x * 7 + k) & (blockDim.x - 1)];
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
  if (acc == -1.0) out[0] = acc;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d clock %d kHz smemOptin %zu\n", p.name, p.multiProcessorCount, clk_khz, p.sharedMemPerBlockOptin);
  int nsm = p.multiProcessorCount;
  double* dout; CK(cudaMalloc(&dout, 1 << 20));
  long long* dcyc; CK(cudaMalloc(&dcyc, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // 1. DMMA throughput
  for (int warps : {4, 8, 16}) {
    int iters = 20000;
    dmma_loop<<<nsm * 2, warps * 32>>>(dout, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_loop<<<nsm * 2, warps * 32>>>(dout, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 4 * (double)iters * warps * nsm * 2;
    printf("DMMA m8n8k4: %d warps/CTA x %d CTAs: %.2f TFLOP/s\n", warps, nsm * 2, flops / ms / 1e9);
  }
  for (int warps : {8, 16}) {
    int iters = 20000;
    cudaEventRecord(e0);
    dfma_loop<<<nsm * 2, warps * 32>>>(dout, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * warps * 32 * nsm * 2;
    printf("DFMA: %d warps/CTA: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  // 2. exchanges
  Slot* slots; CK(cudaMalloc(&slots, sizeof(Slot) * 2 * 1024));
  double* cols; CK(cudaMalloc(&cols, sizeof(double) * 2 * 1024 * 1024));
  int steps = 2000;
  for (int G : {16, 32, 64, 128, 148}) {
    for (int colLen : {0, 512, 1024}) {
      CK(cudaMemset(slots, 0, sizeof(Slot) * 2 * 1024));
      void* args[] = {&slots, &cols, &steps, &colLen, &dcyc};
      cudaEventRecord(e0);
      CK(cudaLaunchCooperativeKernel((void*)a2a_exchange, G, 512, args, 0, 0));
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      long long cyc; CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
      printf("a2a flags G=%3d col=%4d: %.3f us/step (%.0f cyc/step)\n", G, colLen, ms * 1e3 / steps, (double)cyc / steps);
    }
  }
  for (int G : {64, 148}) {
    void* args[] = {&steps, &dcyc};
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)cg_gridsync, G, 512, args, 0, 0));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("cg grid.sync G=%d: %.3f us/step\n", G, ms * 1e3 / steps);
  }
  CK(cudaFuncSetAttribute(cluster_exchange, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(cluster_exchange, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  for (int csz : {2, 4, 8, 16}) {
    for (int colLen : {512, 1024}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(csz); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 2 * colLen * 8;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaEventRecord(e0);
      cudaError_t e = cudaLaunchKernelEx(&cfg, cluster_exchange, steps, colLen, dcyc, dout);
      cudaEventRecord(e1);
      if (e != cudaSuccess) { printf("cluster %d: %s\n", csz, cudaGetErrorString(e)); cudaGetLastError(); continue; }
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("cluster sync+DSMEM csz=%2d col=%4d: %.3f us/step\n", csz, colLen, ms * 1e3 / steps);
    }
  }
  for (int nt : {256, 512, 1024}) {
    cudaEventRecord(e0);
    cta_sync<<<1, nt>>>(steps * 10, dcyc, dout);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("CTA __syncthreads x2 nt=%d: %.3f us/step\n", nt, ms * 1e3 / (steps * 10));
  }
  // launch latency
  cudaEventRecord(e0);
  for (int i = 0; i < 1000; ++i) cta_sync<<<1, 32>>>(0, dcyc, dout);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  printf("empty launch back-to-back: %.3f us\n", ms);
  return 0;
}
