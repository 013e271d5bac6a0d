// Second exchange probe: cheaper all-to-all flag exchange variants for the
// grid-tier prrLU (one exchange per pivot step). Not part of the product path.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

struct __align__(16) Slot { double val; unsigned int idx; unsigned int tag; };

__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int* p) {
  unsigned int v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// mode 0: flag-only release store, parallel relaxed polling, fence, then read slot data.
// mode 1: relaxed 16B vector store of {val,idx,tag} (no release), relaxed 16B poll (data+tag in one load).
template <int MODE>
__global__ void a2a_v2(Slot* slots, double* cols, int steps, int colLen, long long* cycles) {
  const int G = gridDim.x;
  __shared__ double s_best[8];
  __shared__ int s_bi[8];
  __shared__ int winner;
  long long t0 = clock64();
  double sink = 0;
  for (int k = 1; k <= steps; ++k) {
    const int par = k & 3;
    if (colLen > 0) {
      double* my = cols + ((size_t)(k & 1) * G + blockIdx.x) * colLen;
      for (int i = threadIdx.x; i < colLen; i += blockDim.x) __stcg(my + i, (double)(k + i));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      Slot* s = slots + par * G + blockIdx.x;
      double v = (double)((blockIdx.x * 7 + k) % G);
      if (MODE == 0) {
        s->val = v; s->idx = blockIdx.x;
        st_release_u32(&s->tag, (unsigned)k);
      } else {
        // release fence covers the column stores, then a single 16-byte store
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        unsigned long long w0 = __double_as_longlong(v);
        unsigned long long w1 = ((unsigned long long)k << 32) | blockIdx.x;
        asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" :: "l"(s), "l"(w0), "l"(w1) : "memory");
      }
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nPollWarps = (G + 31) / 32;
    if (w < nPollWarps) {
      int g = w * 32 + lane;
      double best = -1; int bi = 0x7fffffff;
      if (g < G) {
        Slot* s = slots + par * G + g;
        if (MODE == 0) {
          while (ld_relaxed_u32(&s->tag) != (unsigned)k) {}
          fence_acq_rel();
          best = *(volatile double*)&s->val; bi = *(volatile unsigned*)&s->idx;
        } else {
          unsigned long long w0, w1;
          do {
            asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(s) : "memory");
          } while ((unsigned)(w1 >> 32) != (unsigned)k);
          best = __longlong_as_double(w0); bi = (int)(w1 & 0xffffffffu);
        }
      }
      for (int o = 16; o; o >>= 1) {
        double ob = __shfl_xor_sync(0xffffffff, best, o);
        int oi = __shfl_xor_sync(0xffffffff, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) { s_best[w] = best; s_bi[w] = bi; }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double best = s_best[0]; int bi = s_bi[0];
      for (int i = 1; i < nPollWarps; ++i) if (s_best[i] > best || (s_best[i] == best && s_bi[i] < bi)) { best = s_best[i]; bi = s_bi[i]; }
      winner = bi;
    }
    __syncthreads();
    if (colLen > 0) {
      if (MODE == 1) fence_acq_rel();
      const double* wc = cols + ((size_t)(k & 1) * G + winner) * colLen;
      for (int i = threadIdx.x; i < colLen; i += blockDim.x) sink += __ldcg(wc + i);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = t1 - t0;
  if (sink == -1.0) cycles[1] = 1;
}

// counter barrier (arrive atomically, poll generation)
__global__ void atomic_barrier(unsigned int* ctr, int steps, long long* cycles) {
  long long t0 = clock64();
  for (int k = 1; k <= steps; ++k) {
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(ctr) : "memory");
      unsigned target = (unsigned)k * gridDim.x;
      while (ld_relaxed_u32(ctr) < target) {}
      fence_acq_rel();
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = t1 - t0;
}

int main() {
  long long* dcyc; CK(cudaMalloc(&dcyc, 64));
  Slot* slots; CK(cudaMalloc(&slots, sizeof(Slot) * 4 * 1024));
  double* cols; CK(cudaMalloc(&cols, sizeof(double) * 2 * 1024 * 1024));
  unsigned int* ctr; CK(cudaMalloc(&ctr, 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms; int steps = 4000;
  for (int mode = 0; mode < 2; ++mode)
    for (int G : {8, 16, 32, 64, 96, 148})
      for (int colLen : {0, 1024}) {
        CK(cudaMemset(slots, 0, sizeof(Slot) * 4 * 1024));
        void* args[] = {&slots, &cols, &steps, &colLen, &dcyc};
        cudaEventRecord(e0);
        if (mode == 0) CK(cudaLaunchCooperativeKernel((void*)a2a_v2<0>, G, 256, args, 0, 0));
        else CK(cudaLaunchCooperativeKernel((void*)a2a_v2<1>, G, 256, args, 0, 0));
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        printf("a2a v2 mode=%d G=%3d col=%4d: %.3f us/step\n", mode, G, colLen, ms * 1e3 / steps);
      }
  for (int G : {16, 64, 148}) {
    CK(cudaMemset(ctr, 0, 4));
    void* args[] = {&ctr, &steps, &dcyc};
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)atomic_barrier, G, 256, args, 0, 0));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("atomic barrier G=%3d: %.3f us/step\n", G, ms * 1e3 / steps);
  }
  return 0;
}
