// Exchange-primitive probe for the grid-tier prrLU step: G CTAs each contribute a key and an
// m-double candidate column; all must learn the argmax key and read the winner's column.
// Variants:
//   A: per-CTA key slot + red.release counter + poll + key read + column read (current design)
//   B: tagged key slots (key + step in one 16 B store), every CTA polls all G slots (no counter)
//   C: 2-level: cluster of 8 reduces via DSMEM + barrier.cluster; leaders exchange tagged slots;
//      barrier.cluster broadcast; column read from L2
// Not part of the product path.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void red_release_add(unsigned *p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 ld_relaxed_v4(const uint4 *p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_v4(uint4 *p, uint4 v) {
  asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

__device__ unsigned pseudo(unsigned g, unsigned k) { return (g * 2654435761u + k * 40503u) & 0xffffu; }

// ---- A
__global__ void varA(uint4 *keys, double *cols, unsigned *ctr, int steps, int m, long long *out) {
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  __shared__ unsigned s_win;
  __shared__ double s_l[1024];
  double sink = 0;
  long long t0 = clock64();
  for (int k = 0; k < steps; ++k) {
    const int par = k & 1;
    if (w == 0) {
      double *dst = cols + ((size_t)par * G + g) * m;
      for (int i = lane; i < m; i += 32) __stcg(dst + i, (double)(i + k));
      __syncwarp();
      if (lane == 0) {
        __stcg(keys + par * G + g, make_uint4(pseudo(g, k), 0, g, 0));
        red_release_add(ctr, 1u);
        while (ld_acquire_u32(ctr) < (unsigned)(k + 1) * G) {}
      }
    }
    __syncthreads();
    unsigned best = 0, bi = 0;
    for (int t = lane; t < G; t += 32) { uint4 q = __ldcg(keys + par * G + t); if (q.x > best || (q.x == best && q.z < bi)) { best = q.x; bi = q.z; } }
    for (int o = 16; o; o >>= 1) { unsigned ob = __shfl_xor_sync(~0u, best, o), oi = __shfl_xor_sync(~0u, bi, o); if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; } }
    const double *src = cols + ((size_t)par * G + bi) * m;
    for (int i = tid; i < m; i += blockDim.x) s_l[i] = __ldcg(src + i);
    __syncthreads();
    sink += s_l[(tid * 7 + k) % m];
  }
  if (tid == 0 && g == 0) out[0] = clock64() - t0;
  if (sink == -1) out[1] = 1;
}

// ---- B: tagged slots (tag = step+1 in .w), all-to-all polling by warp 0
__global__ void varB(uint4 *keys, double *cols, int steps, int m, long long *out) {
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  __shared__ unsigned s_win;
  __shared__ double s_l[1024];
  double sink = 0;
  long long t0 = clock64();
  for (int k = 0; k < steps; ++k) {
    const int par = k & 1;
    if (w == 0) {
      double *dst = cols + ((size_t)par * G + g) * m;
      for (int i = lane; i < m; i += 32) __stcg(dst + i, (double)(i + k));
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        st_relaxed_v4(keys + par * G + g, make_uint4(pseudo(g, k), 0, g, (unsigned)(k + 1)));
      }
      unsigned best = 0, bi = 0;
      for (int t = lane; t < G; t += 32) {
        uint4 q;
        do { q = ld_relaxed_v4(keys + par * G + t); } while (q.w != (unsigned)(k + 1));
        if (q.x > best || (q.x == best && q.z < bi)) { best = q.x; bi = q.z; }
      }
      for (int o = 16; o; o >>= 1) { unsigned ob = __shfl_xor_sync(~0u, best, o), oi = __shfl_xor_sync(~0u, bi, o); if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; } }
      if (lane == 0) s_win = bi;
      __threadfence();
    }
    __syncthreads();
    const double *src = cols + ((size_t)par * G + s_win) * m;
    for (int i = tid; i < m; i += blockDim.x) s_l[i] = __ldcg(src + i);
    __syncthreads();
    sink += s_l[(tid * 7 + k) % m];
  }
  if (tid == 0 && g == 0) out[0] = clock64() - t0;
  if (sink == -1) out[1] = 1;
}

// ---- C: clusters of CS; leaders (rank 0) exchange tagged slots; DSMEM inside the cluster
template <int CS>
__global__ void __cluster_dims__(CS, 1, 1) varC(uint4 *keys, double *cols, int steps, int m, long long *out) {
  cg::cluster_group cl = cg::this_cluster();
  const int g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int rank = cl.block_rank(), ncl = gridDim.x / CS, cid = g / CS;
  __shared__ unsigned s_key[2][2];   // my candidate (value, idx)
  __shared__ unsigned s_win;
  __shared__ double s_l[1024];
  double sink = 0;
  long long t0 = clock64();
  for (int k = 0; k < steps; ++k) {
    const int par = k & 1;
    if (w == 0) {
      double *dst = cols + ((size_t)par * gridDim.x + g) * m;
      for (int i = lane; i < m; i += 32) __stcg(dst + i, (double)(i + k));
      if (lane == 0) { s_key[par][0] = pseudo(g, k); s_key[par][1] = g; }
      __syncwarp();
      if (lane == 0) __threadfence();
    }
    cl.sync();  // all candidates of the cluster visible (DSMEM) and columns fenced
    if (rank == 0 && w == 0) {
      unsigned best = 0, bi = 0;
      if (lane < CS) {
        unsigned *pk = cl.map_shared_rank(&s_key[par][0], lane);
        best = pk[0]; bi = pk[1];
      }
      for (int o = 16; o; o >>= 1) { unsigned ob = __shfl_xor_sync(~0u, best, o), oi = __shfl_xor_sync(~0u, bi, o); if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; } }
      if (lane == 0) st_relaxed_v4(keys + par * ncl + cid, make_uint4(best, 0, bi, (unsigned)(k + 1)));
      unsigned gb = 0, gi = 0;
      for (int t = lane; t < ncl; t += 32) {
        uint4 q;
        do { q = ld_relaxed_v4(keys + par * ncl + t); } while (q.w != (unsigned)(k + 1));
        if (q.x > gb || (q.x == gb && q.z < gi)) { gb = q.x; gi = q.z; }
      }
      for (int o = 16; o; o >>= 1) { unsigned ob = __shfl_xor_sync(~0u, gb, o), oi = __shfl_xor_sync(~0u, gi, o); if (ob > gb || (ob == gb && oi < gi)) { gb = ob; gi = oi; } }
      if (lane < CS) *cl.map_shared_rank(&s_win, lane) = gi;
    }
    cl.sync();
    const double *src = cols + ((size_t)par * gridDim.x + s_win) * m;
    for (int i = tid; i < m; i += blockDim.x) s_l[i] = __ldcg(src + i);
    __syncthreads();
    sink += s_l[(tid * 7 + k) % m];
  }
  if (tid == 0 && g == 0) out[0] = clock64() - t0;
  if (sink == -1) out[1] = 1;
}

int main() {
  uint4 *keys; double *cols; unsigned *ctr; long long *out;
  CK(cudaMalloc(&keys, 16 * 2 * 160)); CK(cudaMalloc(&cols, 8 * 2 * 160 * 1024)); CK(cudaMalloc(&ctr, 4)); CK(cudaMalloc(&out, 16));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int steps = 4000; float ms;
  for (int m : {512, 1024}) {
    for (int G : {32, 64, 128}) {
      CK(cudaMemset(ctr, 0, 4)); CK(cudaMemset(keys, 0, 16 * 2 * 160));
      void *args[] = {&keys, &cols, &ctr, &steps, &m, &out};
      cudaEventRecord(e0);
      CK(cudaLaunchCooperativeKernel((void *)varA, G, 256, args, 0, 0));
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("A counter     m=%4d G=%3d: %.3f us/step\n", m, G, ms * 1e3 / steps);
      CK(cudaMemset(keys, 0, 16 * 2 * 160));
      void *argsB[] = {&keys, &cols, &steps, &m, &out};
      cudaEventRecord(e0);
      CK(cudaLaunchCooperativeKernel((void *)varB, G, 256, argsB, 0, 0));
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("B tagged a2a  m=%4d G=%3d: %.3f us/step\n", m, G, ms * 1e3 / steps);
      CK(cudaMemset(keys, 0, 16 * 2 * 160));
      cudaEventRecord(e0);
      varC<8><<<G, 256>>>(keys, cols, steps, m, out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("C cluster8    m=%4d G=%3d: %.3f us/step\n", m, G, ms * 1e3 / steps);
      CK(cudaMemset(keys, 0, 16 * 2 * 160));
      cudaEventRecord(e0);
      varC<4><<<G, 256>>>(keys, cols, steps, m, out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("C cluster4    m=%4d G=%3d: %.3f us/step\n", m, G, ms * 1e3 / steps);
    }
  }
  return 0;
}
