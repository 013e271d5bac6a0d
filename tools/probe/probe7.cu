// Cluster push-exchange probe (development tool, not part of the product path).
// C = R x Cc CTAs of one thread-block cluster; per step:
//   (1) every CTA pushes a 16-byte key into every CTA's smem with st.async (complete_tx on the
//       destination's mbarrier), waits on its own mbarrier, reduces the C keys;
//   (2) the "winner" owners push segments: CTA (i, jq) pushes its m/R-double column segment to
//       the Cc CTAs of row block i, CTA (ip, j) its n/Cc-double row segment to the R CTAs of
//       column block j; receivers wait on a second mbarrier.
// MODE 0: segments by st.async.v2.b64 from a warp; MODE 1: cp.async.bulk smem->remote smem;
// MODE 2: keys only (no segments).
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
__device__ __forceinline__ void st_async_v2d(unsigned raddr, double a, double b, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr), "d"(a),
               "d"(b), "r"(rbar) : "memory");
}
__device__ __forceinline__ void bulk_s2c(unsigned rdst, unsigned src, unsigned bytes, unsigned rbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rdst),
               "r"(src), "r"(bytes), "r"(rbar) : "memory");
}
__device__ unsigned pseudo(unsigned g, unsigned k) { return (g * 2654435761u + k * 40503u) & 0xffffu; }

template <int MODE>
__global__ void __launch_bounds__(512) kern(int steps, int m, int n, int R, long long *out) {
  unsigned rank; asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  unsigned C; asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(C));
  const int Cc = C / R;
  const int myi = rank / Cc, myj = rank % Cc;
  const int MR = m / R, NC = n / Cc;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  __shared__ alignas(16) uint4 keys[2][16];
  __shared__ alignas(16) double lseg[2][1024];
  __shared__ alignas(16) double useg[2][1024];
  __shared__ alignas(16) double stage[2][512];
  __shared__ alignas(8) unsigned long long mb[4];
  if (tid == 0) { for (int t = 0; t < 4; ++t) mbar_init(smem_u32(&mb[t]), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  for (int i = tid; i < 512; i += blockDim.x) { stage[0][i] = i; stage[1][i] = -i; }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long ta = 0, tb = 0, tc = 0;
  double sink = 0;
  for (int k = 0; k < steps; ++k) {
    const int par = k & 1;
    const unsigned ph = (k >> 1) & 1;
    const unsigned mk = smem_u32(&mb[par]), ms = smem_u32(&mb[2 + par]);
    long long t0 = clock64();
    if (tid == 0) mbar_expect(mk, C * 16);
    if (tid < (int)C) st_async_v4(mapa(smem_u32(&keys[par][rank]), tid), make_uint4(pseudo(rank, k), 0, rank, 0), mapa(mk, tid));
    mbar_wait(mk, ph);
    unsigned best = 0, bi = 0;
    if (lane < (int)C) { uint4 q = keys[par][lane]; best = q.x; bi = q.z; }
    for (int o = 16; o; o >>= 1) {
      unsigned ob = __shfl_xor_sync(~0u, best, o), oi = __shfl_xor_sync(~0u, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    long long t1 = clock64();
    if (MODE != 2) {
      const int ip = bi / Cc, jq = bi % Cc;  // winner coordinates
      if (tid == 0) mbar_expect(ms, (MR + NC) * 8);
      if (MODE == 0) {
        if (myj == jq && w < Cc) {  // warp w pushes my column segment to CTA (myi, w)
          const unsigned dr = myi * Cc + w;
          const unsigned rb = mapa(ms, dr), base = mapa(smem_u32(&lseg[par][0]), dr);
          for (int i = 2 * lane; i < MR; i += 64) st_async_v2d(base + 8 * i, stage[par][i], stage[par][i + 1], rb);
        }
        if (myi == ip && w >= 8 && w - 8 < R) {  // warp 8+r pushes my row segment to CTA (r, myj)
          const unsigned dr = (w - 8) * Cc + myj;
          const unsigned rb = mapa(ms, dr), base = mapa(smem_u32(&useg[par][0]), dr);
          for (int i = 2 * lane; i < NC; i += 64) st_async_v2d(base + 8 * i, stage[par][i], stage[par][i + 1], rb);
        }
      } else {
        if (myj == jq && tid < Cc) {
          const unsigned dr = myi * Cc + tid;
          bulk_s2c(mapa(smem_u32(&lseg[par][0]), dr), smem_u32(&stage[par][0]), MR * 8, mapa(ms, dr));
        }
        if (myi == ip && tid >= 32 && tid - 32 < R) {
          const unsigned dr = (tid - 32) * Cc + myj;
          bulk_s2c(mapa(smem_u32(&useg[par][0]), dr), smem_u32(&stage[par][0]), NC * 8, mapa(ms, dr));
        }
      }
      mbar_wait(ms, ph);
      sink += lseg[par][tid % MR] + useg[par][tid % NC];
    }
    long long t2 = clock64();
    __syncthreads();
    long long t3 = clock64();
    ta += t1 - t0; tb += t2 - t1; tc += t3 - t2;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (tid == 0 && blockIdx.x == 0) { out[0] = ta / steps; out[1] = tb / steps; out[2] = tc / steps; }
  if (sink == -1) out[5] = 1;
}

int main() {
  long long *out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const void *fs[3] = {(const void *)kern<0>, (const void *)kern<1>, (const void *)kern<2>};
  const char *names[3] = {"st.async seg", "bulk seg", "keys only"};
  for (int i = 0; i < 3; ++i) CK(cudaFuncSetAttribute(fs[i], cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  int steps = 4000;
  struct Cfg { int C, R, m, n; } cfgs[] = {{8, 2, 512, 512}, {8, 2, 1024, 1024}, {16, 4, 512, 512}, {16, 4, 1024, 1024},
                                           {4, 2, 256, 256}, {16, 2, 512, 1024}};
  for (int mode = 0; mode < 3; ++mode)
    for (auto c : cfgs) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c.C); cfg.blockDim = dim3(512);
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c.C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int ncl = 0;
      cudaOccupancyMaxActiveClusters(&ncl, fs[mode], &cfg);
      cudaError_t e;
      long long h[3];
      float ms;
      cudaEventRecord(e0);
      if (mode == 0) e = cudaLaunchKernelEx(&cfg, kern<0>, steps, c.m, c.n, c.R, out);
      else if (mode == 1) e = cudaLaunchKernelEx(&cfg, kern<1>, steps, c.m, c.n, c.R, out);
      else e = cudaLaunchKernelEx(&cfg, kern<2>, steps, c.m, c.n, c.R, out);
      cudaEventRecord(e1);
      if (e != cudaSuccess) { printf("%s C=%d: launch %s\n", names[mode], c.C, cudaGetErrorString(e)); cudaGetLastError(); continue; }
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      CK(cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost));
      printf("%-13s C=%2d (%dx%d, max active %3d) m=%4d n=%4d: %.3f us/step | cycles: keys %lld, segs %lld, bar %lld\n",
             names[mode], c.C, c.R, c.C / c.R, ncl, c.m, c.n, ms * 1e3 / steps, h[0], h[1], h[2]);
    }
  return 0;
}
