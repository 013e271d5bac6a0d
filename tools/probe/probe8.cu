// Cluster exchange probe, part 2 (development tool, not part of the product path).
// Same R x Cc layout and traffic as probe7, other signalling schemes:
//   MODE 0: keys and segments as TAGGED 8-byte words (32-bit payload | 32-bit step tag) written
//           with weak st.shared::cluster.v2.u64; receivers spin on their OWN smem until every
//           word carries this step's tag (no mbarrier, no fence).
//   MODE 1: keys by st.async (mbarrier complete_tx); segments by weak st.shared::cluster.v2.f64,
//           __syncwarp, then one mbarrier.arrive.release.cluster on the remote barrier.
//   MODE 2: tagged keys only.
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
__device__ __forceinline__ void mbar_arrive_remote(unsigned rbar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
}
__device__ __forceinline__ void st_async_v4(unsigned raddr, uint4 v, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar) : "memory");
}
__device__ __forceinline__ void st_cl_v2u64(unsigned raddr, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.cluster.shared::cluster.v2.u64 [%0], {%1, %2};" ::"r"(raddr), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st_cl_v2f64(unsigned raddr, double a, double b) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(raddr), "d"(a), "d"(b) : "memory");
}
__device__ __forceinline__ void ld_vol_v2u64(const unsigned long long *p, unsigned long long &a, unsigned long long &b) {
  asm volatile("ld.relaxed.cluster.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(smem_u32(p)) : "memory");
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
  __shared__ alignas(16) unsigned long long keys[2][16][2];
  __shared__ alignas(16) unsigned long long lseg[2][1024];  // tagged: 2 words per double (MODE 0) / doubles (MODE 1)
  __shared__ alignas(16) unsigned long long useg[2][1024];
  __shared__ alignas(16) uint4 akeys[2][16];
  __shared__ alignas(8) unsigned long long mb[4];
  if (tid == 0) {
    mbar_init(smem_u32(&mb[0]), 1); mbar_init(smem_u32(&mb[1]), 1);
    mbar_init(smem_u32(&mb[2]), 2); mbar_init(smem_u32(&mb[3]), 2);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 2 * 1024; i += blockDim.x) { (&lseg[0][0])[i] = 0; (&useg[0][0])[i] = 0; }
  for (int i = tid; i < 2 * 16 * 2; i += blockDim.x) (&keys[0][0][0])[i] = 0;
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long ta = 0, tb = 0, tc = 0;
  double sink = 0;
  for (int k = 0; k < steps; ++k) {
    const int par = k & 1;
    const unsigned ph = (k >> 1) & 1;
    const unsigned long long tag = (unsigned long long)(k + 1) << 32;
    long long t0 = clock64();
    unsigned best = 0, bi = 0;
    if (MODE == 1) {
      const unsigned mk = smem_u32(&mb[par]);
      if (tid == 0) mbar_expect(mk, C * 16);
      if (tid < (int)C) st_async_v4(mapa(smem_u32(&akeys[par][rank]), tid), make_uint4(pseudo(rank, k), 0, rank, 0), mapa(mk, tid));
      mbar_wait(mk, ph);
      if (lane < (int)C) { uint4 q = akeys[par][lane]; best = q.x; bi = q.z; }
    } else {
      if (tid < (int)C) st_cl_v2u64(mapa(smem_u32(&keys[par][rank][0]), tid), tag | pseudo(rank, k), tag | rank);
      if (lane < (int)C) {
        unsigned long long a, b;
        do { ld_vol_v2u64(&keys[par][lane][0], a, b); } while ((a >> 32) != (unsigned long long)(k + 1) || (b >> 32) != (unsigned long long)(k + 1));
        best = (unsigned)a; bi = (unsigned)b;
      }
    }
    for (int o = 16; o; o >>= 1) {
      unsigned ob = __shfl_xor_sync(~0u, best, o), oi = __shfl_xor_sync(~0u, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    long long t1 = clock64();
    if (MODE != 2) {
      const int ip = bi / Cc, jq = bi % Cc;
      if (MODE == 0) {
        // column segment: MR doubles as MR tagged pairs (lo word, hi word) -> 16 B per double
        if (myj == jq && w < Cc) {
          const unsigned base = mapa(smem_u32(&lseg[par][0]), myi * Cc + w);
          for (int i = lane; i < MR; i += 32) st_cl_v2u64(base + 16 * i, tag | (unsigned)(2 * i + k), tag | (unsigned)(2 * i + 1));
        }
        if (myi == ip && w >= 8 && w - 8 < R) {
          const unsigned base = mapa(smem_u32(&useg[par][0]), (w - 8) * Cc + myj);
          for (int i = lane; i < NC; i += 32) st_cl_v2u64(base + 16 * i, tag | (unsigned)(2 * i + k), tag | (unsigned)(2 * i + 1));
        }
        // receivers: every thread validates its share (MR/2 + NC/2 pairs) in its own smem
        for (int i = tid; i < MR + NC; i += blockDim.x) {
          const unsigned long long *p = i < MR ? &lseg[par][2 * i] : &useg[par][2 * (i - MR)];
          unsigned long long a, b;
          do { ld_vol_v2u64(p, a, b); } while ((a >> 32) != (unsigned long long)(k + 1) || (b >> 32) != (unsigned long long)(k + 1));
          sink += (double)(unsigned)a;
        }
      } else {
        const unsigned msb = smem_u32(&mb[2 + par]);
        if (myj == jq && w < Cc) {
          const unsigned dr = myi * Cc + w;
          const unsigned base = mapa(smem_u32(&lseg[par][0]), dr);
          for (int i = 2 * lane; i < MR; i += 64) st_cl_v2f64(base + 8 * i, (double)i, (double)(i + 1));
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(mapa(msb, dr));
        }
        if (myi == ip && w >= 8 && w - 8 < R) {
          const unsigned dr = (w - 8) * Cc + myj;
          const unsigned base = mapa(smem_u32(&useg[par][0]), dr);
          for (int i = 2 * lane; i < NC; i += 64) st_cl_v2f64(base + 8 * i, (double)i, (double)(i + 1));
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(mapa(msb, dr));
        }
        mbar_wait(msb, ph);
        sink += __longlong_as_double(lseg[par][tid % MR]) + __longlong_as_double(useg[par][tid % NC]);
      }
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
  const char *names[3] = {"tagged", "weak+arrive", "tagged keys"};
  for (int i = 0; i < 3; ++i) CK(cudaFuncSetAttribute(fs[i], cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  int steps = 4000;
  struct Cfg { int C, R, m, n; } cfgs[] = {{4, 2, 256, 256}, {8, 2, 512, 512}, {16, 4, 512, 512}, {16, 4, 1024, 1024},
                                           {16, 2, 512, 1024}, {8, 2, 256, 256}};
  for (int mode = 0; mode < 3; ++mode)
    for (auto c : cfgs) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c.C); cfg.blockDim = dim3(512);
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c.C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
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
      printf("%-12s C=%2d (%dx%d) m=%4d n=%4d: %.3f us/step | cycles: keys %lld, segs %lld, bar %lld\n", names[mode], c.C,
             c.R, c.C / c.R, c.m, c.n, ms * 1e3 / steps, h[0], h[1], h[2]);
    }
  return 0;
}
