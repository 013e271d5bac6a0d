// FP64 tensor-core (DMMA) GEMMs of the 2-site update:
//   a1/a2: A^n = L^n_{l-1} X^n_l, B^n = X^n_{l+1} R^n_{l+2}  (FUSE = false)
//   a3+a4 (Eq. pifromframes, f of P:459-462): Pi = f(A^1 B^1, ..., A^N B^N) (FUSE = true)
// On sm_100a FP64 matrix math exists only as warp-level mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4
// (tcgen05 has no f64 kind); see DESIGN.md §5.
//
// CTA tile 64x64, BK = 16, 8 warps each owning a 32x16 warp tile (4x2 DMMA tiles), 3-stage
// cp.async pipeline; <= 128 registers so 2-3 CTAs (16-24 warps) share an SM (DMMA needs more
// than one warp per SMSP to cover its latency). Problem sizes are read from device descriptors (live ranks); CTAs whose
// tile lies outside the live M x N exit immediately. In FUSE mode the per-input products never
// reach HBM: f, the NaN check and max|Pi| run on the accumulator registers.
#include "aci_common.cuh"

namespace {

constexpr int BM = 64, BN = 64, BK = 16, STAGES = 3, NT = 256;
constexpr int WN = 16, NI = WN / 8;  // warp tile 32 x 16
constexpr int LDA_S = BK + 4;   // 20 doubles: conflict-free A-fragment loads
constexpr int LDB_S = BN + 8;   // 72 doubles: conflict-free B-fragment loads

__device__ __forceinline__ void cp_async8(double *sdst, const double *gsrc, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gsrc), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

struct Smem {
  double A[STAGES][BM][LDA_S];
  double B[STAGES][BK][LDB_S];
};

__device__ __forceinline__ void load_stage(Smem &sm, int st, const double *A, int lda, const double *B, int ldb,
                                           int M, int N, int K, int m0, int n0, int k0) {
  const int t = threadIdx.x;
#pragma unroll
  for (int i = 0; i < (BM * BK) / NT; ++i) {
    int e = t + NT * i;
    int row = e / BK, kc = e % BK;
    bool v = (m0 + row < M) && (k0 + kc < K);
    const double *src = v ? A + (size_t)(m0 + row) * lda + (k0 + kc) : A;
    cp_async8(&sm.A[st][row][kc], src, v);
  }
#pragma unroll
  for (int i = 0; i < (BK * BN) / NT; ++i) {
    int e = t + NT * i;
    int kr = e / BN, col = e % BN;
    bool v = (k0 + kr < K) && (n0 + col < N);
    const double *src = v ? B + (size_t)(k0 + kr) * ldb + (n0 + col) : B;
    cp_async8(&sm.B[st][kr][col], src, v);
  }
}

// acc += A (M x K) * B (K x N) for this CTA's 64x64 tile.
__device__ __forceinline__ void mainloop(Smem &sm, double (&acc)[4][NI][2], const double *A, int lda,
                                         const double *B, int ldb, int M, int N, int K, int m0, int n0) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int wm = (w >> 2) * 32, wn = (w & 3) * WN;
  const int nk = (K + BK - 1) / BK;
  __syncthreads();  // smem reuse across inputs
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(sm, s, A, lda, B, ldb, M, N, K, m0, n0, s * BK);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nxt = kt + STAGES - 1;
      if (nxt < nk) load_stage(sm, nxt % STAGES, A, lda, B, ldb, M, N, K, m0, n0, nxt * BK);
      cp_async_commit();
    }
    const int st = kt % STAGES;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[4], b[NI];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = sm.A[st][wm + mi * 8 + g][kk * 4 + c];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) b[ni] = sm.B[st][kk * 4 + c][wn + ni * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
    }
  }
  cp_async_wait<0>();
}

// EPI: 0 = store A B, 1 = f(A1 B1, ...) (FUSE), 2 = S - A B.
template <int NIN, bool FUSE, int EPI = FUSE ? 1 : 0>
__global__ void __launch_bounds__(NT, 2) gemm_dmma_kernel(const GemmDesc *__restrict__ descs, FOp op,
                                                       unsigned long long *scale_bits, int *nonfinite) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem &sm = *reinterpret_cast<Smem *>(smem_raw);
  const GemmDesc &D = descs[blockIdx.z];
  const int M = D.M, N = D.N;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= M || n0 >= N) return;

  double acc[NIN][4][NI][2];
#pragma unroll
  for (int i = 0; i < NIN; ++i)
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) acc[i][mi][ni][0] = acc[i][mi][ni][1] = 0.0;

#pragma unroll
  for (int i = 0; i < NIN; ++i) mainloop(sm, acc[i], D.A[i], D.lda[i], D.B[i], D.ldb[i], M, N, D.K[i], m0, n0);

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int wm = (w >> 2) * 32, wn = (w & 3) * WN;
  double vmax = 0.0;
  int bad = 0;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int row = m0 + wm + mi * 8 + g, col = n0 + wn + ni * 8 + 2 * c + e;
        if (row < M && col < N) {
          double y;
          if (FUSE) {
            // same operation order as the oracle's apply_f
            y = 0.0;
            for (int t = 0; t < op.T; ++t) {
              double p = op.coef[t];
#pragma unroll
              for (int i = 0; i < NIN; ++i)
                for (int q = 0; q < op.expo[t * op.N + i]; ++q) p *= acc[i][mi][ni][e];
              y += p;
            }
            if (!isfinite(y)) bad = 1;
            vmax = fmax(vmax, fabs(y));
          } else if (EPI == 2) {
            y = D.S[(size_t)row * D.lds + col] - acc[0][mi][ni][e];
          } else {
            y = acc[0][mi][ni][e];
          }
          D.C[(size_t)row * D.ldc + col] = y;
        }
      }
  if (FUSE) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
      bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if (lane == 0) {
      if (vmax > 0.0) atomicMax(scale_bits, (unsigned long long)__double_as_longlong(vmax));
      if (bad) atomicOr(nonfinite, 1);
    }
  }
}

template <int NIN, bool FUSE>
void launch_t(const GemmDesc *d, int ndesc, int max_m, int max_n, const FOp &op, unsigned long long *sb, int *nf,
              cudaStream_t st) {
  const int smem = (int)sizeof(Smem);
  dim3 grid((max_n + BN - 1) / BN, (max_m + BM - 1) / BM, ndesc);
  gemm_dmma_kernel<NIN, FUSE><<<grid, NT, smem, st>>>(d, op, sb, nf);
}

}  // namespace

void gemm_init() {
  // kernel attributes are set once, outside any stream capture
  static bool done = false;
  if (done) return;
  const int smem = (int)sizeof(Smem);
  cudaFuncSetAttribute(gemm_dmma_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gemm_dmma_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gemm_dmma_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gemm_dmma_kernel<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gemm_dmma_kernel<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gemm_dmma_kernel<1, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  done = true;
}

void launch_gemm_sub(const GemmDesc *d, int ndesc, int max_m, int max_n, cudaStream_t st) {
  if (max_m <= 0 || max_n <= 0 || ndesc <= 0) return;
  const int smem = (int)sizeof(Smem);
  dim3 grid((max_n + BN - 1) / BN, (max_m + BM - 1) / BM, ndesc);
  FOp op = {};
  gemm_dmma_kernel<1, false, 2><<<grid, NT, smem, st>>>(d, op, nullptr, nullptr);
}

void launch_gemm(const GemmDesc *d_descs, int ndesc, int max_m, int max_n, int nin, bool fuse, const FOp &op,
                 unsigned long long *scale_bits, int *nonfinite, cudaStream_t st) {
  if (max_m <= 0 || max_n <= 0 || ndesc <= 0) return;
  if (!fuse) {
    launch_t<1, false>(d_descs, ndesc, max_m, max_n, op, scale_bits, nonfinite, st);
    return;
  }
  switch (nin) {
    case 1: launch_t<1, true>(d_descs, ndesc, max_m, max_n, op, scale_bits, nonfinite, st); break;
    case 2: launch_t<2, true>(d_descs, ndesc, max_m, max_n, op, scale_bits, nonfinite, st); break;
    case 3: launch_t<3, true>(d_descs, ndesc, max_m, max_n, op, scale_bits, nonfinite, st); break;
    default: launch_t<4, true>(d_descs, ndesc, max_m, max_n, op, scale_bits, nonfinite, st); break;
  }
}
