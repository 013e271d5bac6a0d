// Stream-K / data-parallel + stream-K variants of the full-size Pi GEMM (development tool, measured
// NOT adopted: tools/gemm_bench_sk.cu, profiles/r02v_gemm_sk.txt). Builds on the
// product's tile kernel header (Cfg, cp.async staging, smem_bytes).
#pragma once
#include "../paper_2604_00037_b200/csrc/gemm_kernel.cuh"

namespace gemmk {

// VEC = 1 main loop over the k-tiles [kb, ke) of this CTA's tile: acc += A[:, kb*BK : ke*BK] B[...]
// (ke > kb; the whole-K tile kernel and the stream-K kernel's segments both run it)
template <class CF>
__device__ __forceinline__ void mainloop_v(typename CF::Smem &sm, double (&acc)[CF::MI][CF::NI][2], const double *A,
                                           int lda, const double *B, int ldb, int M, int N, int K, int m0, int n0,
                                           int kb, int ke) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int wm = (w / CF::WARPS_N) * CF::WM, wn = (w % CF::WARPS_N) * CF::WN;
  const bool vec = !((lda | ldb) & 1) && !((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15);
  __syncthreads();  // shared memory reuse across inputs
#pragma unroll
  for (int s = 0; s < CF::STAGES - 1; ++s) {
    if (kb + s < ke) load_stage_v<CF>(sm, s, A, lda, B, ldb, M, N, K, m0, n0, (kb + s) * CF::BK, vec);
    cp_async_commit();
  }
  for (int kt = 0; kt < ke - kb; ++kt) {
    cp_async_wait<CF::STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + CF::STAGES - 1;
      if (kb + nxt < ke)
        load_stage_v<CF>(sm, nxt % CF::STAGES, A, lda, B, ldb, M, N, K, m0, n0, (kb + nxt) * CF::BK, vec);
      cp_async_commit();
    }
    const int st = kt % CF::STAGES;
#pragma unroll
    for (int ks = 0; ks < CF::BK / 4; ++ks) {
      double a[CF::MI], b[CF::NI];
#pragma unroll
      for (int mi = 0; mi < CF::MI; ++mi) a[mi] = sm.A[st][wm + mi * 8 + g][4 * ks + c];
#pragma unroll
      for (int ni = 0; ni < CF::NI; ++ni) b[ni] = sm.B[st][4 * ks + c][wn + ni * 8 + g];
#pragma unroll
      for (int mi = 0; mi < CF::MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < CF::NI; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
    }
  }
  cp_async_wait<0>();
}

// EPI_F on a finished tile: Pi = f(x_1, ..., x_N) from the accumulators (inputs 0..NBIG-1) and the
// small-K operands in shared memory (inputs NBIG..), stored to D.C; max |Pi| and the NaN flag of the
// real entries accumulate into vmax / bad
template <class CF, int NBIG, int NSMALL, int NB>
__device__ __forceinline__ void epi_f(const GemmDesc &D, const FOp &op, const double (&acc)[NB][CF::MI][CF::NI][2],
                                      const double *sA, const double *sB, int M, int N, int m0, int n0, double &vmax,
                                      bool &bad) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int wm = (w / CF::WARPS_N) * CF::WM, wn = (w % CF::WARPS_N) * CF::WN;
  // small inputs: this thread's MI rows of A_s and 2*NI columns of B_s in registers
  constexpr int NS = NSMALL > 0 ? NSMALL : 1;
  double ra[NS][CF::MI][kSmallK], rb[NS][CF::NI][2][kSmallK];
  int ks[NS];
#pragma unroll
  for (int s_ = 0; s_ < NSMALL; ++s_) {
    ks[s_] = D.K[NBIG + s_];
#pragma unroll
    for (int kk = 0; kk < kSmallK; ++kk) {
#pragma unroll
      for (int mi = 0; mi < CF::MI; ++mi)
        ra[s_][mi][kk] = sA[s_ * CF::BM * kSmallK + (wm + mi * 8 + g) * kSmallK + kk];
#pragma unroll
      for (int ni = 0; ni < CF::NI; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) rb[s_][ni][e][kk] = sB[s_ * kSmallK * CF::BN + kk * CF::BN + wn + ni * 8 + 2 * c + e];
    }
  }
  const bool mono = op.monomial_all_ones != 0;
  const double coef0 = op.coef[0];
#pragma unroll
  for (int mi = 0; mi < CF::MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < CF::NI; ++ni) {
      const int row = m0 + wm + mi * 8 + g, col0 = n0 + wn + ni * 8 + 2 * c;
      double y2[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double x[NBIG + NSMALL];
#pragma unroll
        for (int i = 0; i < NBIG; ++i) x[i] = acc[i][mi][ni][e];
#pragma unroll
        for (int s_ = 0; s_ < NSMALL; ++s_) {
          double v = 0.0;
#pragma unroll
          for (int kk = 0; kk < kSmallK; ++kk)
            if (kk < ks[s_]) v = fma(ra[s_][mi][kk], rb[s_][ni][e][kk], v);
          x[NBIG + s_] = v;
        }
        double y;
        if (mono) {
          // f = coef * prod x_i, multiplied in the oracle's order (apply_f with one term)
          double p = coef0;
#pragma unroll
          for (int i = 0; i < NBIG + NSMALL; ++i) p *= x[i];
          y = p;
        } else {
          y = 0.0;
          for (int t = 0; t < op.T; ++t) {
            double p = op.coef[t];
#pragma unroll
            for (int i = 0; i < NBIG + NSMALL; ++i)
              for (int q = 0; q < op.expo[t * op.N + i]; ++q) p *= x[i];
            y += p;
          }
        }
        // padded lanes hold f(0) (nonzero for a constant term): never part of s or the NaN check
        if (row < M && col0 + e < N) {
          bad |= !isfinite(y);
          vmax = fmax(vmax, fabs(y));
        }
        y2[e] = y;
      }
      if (row < M) {
        double *dst = D.C + (size_t)row * D.ldc + col0;
        if (col0 + 1 < N) {
          dst[0] = y2[0];
          dst[1] = y2[1];
        } else if (col0 < N) {
          dst[0] = y2[0];
        }
      }
    }
}

// warp max of |Pi| into the running s (scale_bits, atomicMax on the bits) and the NaN flag
__device__ __forceinline__ void epi_scale(double vmax, bool bad, unsigned long long *scale_bits, int *nonfinite) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    bad = bad | (__shfl_xor_sync(0xffffffffu, (int)bad, o) != 0);
  }
  if (lane == 0) {
    // s only grows: a warp whose max does not exceed the value it reads skips the atomic (a stale
    // read is never larger than the current value, so no needed update is skipped) — 8 warps x
    // 256 CTAs of atomics on one address cost ~2 us per full-size Pi otherwise
    const unsigned long long vb = (unsigned long long)__double_as_longlong(vmax);
    if (vmax > 0.0 && vb > *(volatile const unsigned long long *)scale_bits) atomicMax(scale_bits, vb);
    if (bad) atomicOr(nonfinite, 1);
  }
}

// Stream-K variant of the EPI_F kernel for one DMMA input (NBIG = 1, any number of small-K inputs)
// on large grids. The full-size Pi of configs[3] chi = 256 (1024 x 1024, 256 64x64 tiles) on 148 SMs
// leaves 108 SMs with two tiles and 40 with one; here the U = tiles x k-tiles units are split evenly
// over a persistent grid of G co-resident CTAs. CTA q (logical id from a ticket counter: every lower
// id has already started) owns the units [qU/G, (q+1)U/G) and walks its tiles from the highest down:
//   * its first segment may stop short of the tile's last k-tile: the partial accumulator goes to
//     its own slot part[q] (thread-major) and flags[q] is raised — it never waits;
//   * tiles it holds whole are finished at once (f, max|Pi|, store: the EPI_F epilogue);
//   * its last segment holds the end of a tile whose beginning lower ids hold: it waits for their
//     flags (they stored those partials first thing), adds them in descending id order (a fixed
//     order: results are deterministic) and clears the flags for the next launch.
// Only the grouping of the k-sum differs from the tile kernel (rounding-level differences in Pi).
template <class CF, int NSMALL>
__global__ void __launch_bounds__(CF::NT, CF::MINB)
    gemm_sk_kernel(const GemmDesc *__restrict__ descs, FOp op, unsigned long long *scale_bits, int *nonfinite,
                   double *__restrict__ part, unsigned *flags, unsigned long long *ticket, int nsk) {
  static_assert(CF::VEC != 0, "stream-K runs the VEC main loop");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto &sm = *reinterpret_cast<typename CF::Smem *>(smem_raw);
  double *sA = reinterpret_cast<double *>(smem_raw + sizeof(typename CF::Smem));
  double *sB = sA + NSMALL * CF::BM * kSmallK;
  __shared__ int s_q;
  constexpr int TE = CF::MI * CF::NI * 2;  // accumulator doubles per thread
  const GemmDesc &D = descs[0];
  const int M = D.M, N = D.N, K = D.K[0];
  const int tn = (N + CF::BN - 1) / CF::BN, tm = (M + CF::BM - 1) / CF::BM;
  const int KT = K > 0 ? (K + CF::BK - 1) / CF::BK : 1;
  // the first gridDim.x - nsk CTAs take one whole tile each (data-parallel); the last nsk CTAs
  // split the remaining tiles' k-tiles evenly (stream-K)
  const int ndp = gridDim.x - nsk, tdp = min(tm * tn, ndp);
  if ((int)blockIdx.x < ndp && (int)blockIdx.x >= tdp) return;
  const int G = nsk;
  int q = -1;
  if ((int)blockIdx.x >= ndp) {
    if (threadIdx.x == 0) s_q = (int)(atomicAdd(ticket, 1ull) % (unsigned long long)G);
    __syncthreads();
    q = s_q;
  }
  const long long U = (long long)(tm * tn - tdp) * KT, base = (long long)tdp * KT;
  auto bound = [&](int i) { return base + U * i / G; };
  const long long s0 = q < 0 ? (long long)blockIdx.x * KT : bound(q), e0 = q < 0 ? s0 + KT : bound(q + 1);
  double vmax = 0.0;
  bool bad = false;
  for (long long t = s0 < e0 ? (e0 - 1) / KT : -1; t >= 0 && t >= s0 / KT; --t) {
    const long long ts = t * KT, te = ts + KT;
    const int kb = (int)((s0 > ts ? s0 : ts) - ts), ke = (int)((e0 < te ? e0 : te) - ts);
    const bool finisher = ke == KT;
    const int m0 = (int)(t / tn) * CF::BM, n0 = (int)(t % tn) * CF::BN;
    __syncthreads();  // the previous tile's epilogue is done with sA / sB
    if (NSMALL > 0 && finisher) {  // small-K operands of this tile (hidden under its main loop)
#pragma unroll
      for (int s_ = 0; s_ < NSMALL; ++s_) {
        const int i = 1 + s_, Ks = D.K[i];
        for (int x = threadIdx.x; x < CF::BM * kSmallK; x += CF::NT) {
          const int row = x / kSmallK, kk = x % kSmallK;
          const bool v = kk < Ks && m0 + row < M;
          cp_async8(&sA[s_ * CF::BM * kSmallK + x], v ? D.A[i] + (size_t)(m0 + row) * D.lda[i] + kk : D.A[i], v);
        }
        for (int x = threadIdx.x; x < kSmallK * CF::BN; x += CF::NT) {
          const int kk = x / CF::BN, col = x % CF::BN;
          const bool v = kk < Ks && n0 + col < N;
          cp_async8(&sB[s_ * kSmallK * CF::BN + x], v ? D.B[i] + (size_t)kk * D.ldb[i] + n0 + col : D.B[i], v);
        }
      }
      cp_async_commit();
    }
    double acc[1][CF::MI][CF::NI][2];
#pragma unroll
    for (int mi = 0; mi < CF::MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < CF::NI; ++ni) acc[0][mi][ni][0] = acc[0][mi][ni][1] = 0.0;
    if (K > 0) mainloop_v<CF>(sm, acc[0], D.A[0], D.lda[0], D.B[0], D.ldb[0], M, N, K, m0, n0, kb, ke);
    if (!finisher) {  // hand the partial sum to the tile's finisher
      double *dst = part + (size_t)q * (CF::BM * CF::BN) + threadIdx.x;
#pragma unroll
      for (int mi = 0; mi < CF::MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < CF::NI; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) __stcg(dst + ((mi * CF::NI + ni) * 2 + e) * CF::NT, acc[0][mi][ni][e]);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(flags + q), "r"(1u) : "memory");
      }
      continue;
    }
    if (kb > 0) {  // the tile's earlier k-tiles: lower ids, nearest first
      for (int p = q - 1; p >= 0; --p) {
        const long long lo = bound(p), hi = bound(p + 1);
        if (hi <= ts) break;  // (no SK CTA shares a tile with the data-parallel ones)
        if (lo == hi) continue;
        if (threadIdx.x == 0) {
          unsigned f = 0;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(f) : "l"(flags + p) : "memory");
          } while (f == 0);
        }
        __syncthreads();
        const double *src = part + (size_t)p * (CF::BM * CF::BN) + threadIdx.x;
        double v[TE];
#pragma unroll
        for (int j = 0; j < TE; ++j) v[j] = __ldcg(src + j * CF::NT);
#pragma unroll
        for (int mi = 0; mi < CF::MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < CF::NI; ++ni)
#pragma unroll
            for (int e = 0; e < 2; ++e) acc[0][mi][ni][e] += v[(mi * CF::NI + ni) * 2 + e];
        __syncthreads();
        if (threadIdx.x == 0) flags[p] = 0u;  // consumed (read again only by the next launch)
        if (lo <= ts) break;
      }
    }
    if (NSMALL > 0 && K == 0) {  // no main loop waited for the small-K group
      cp_async_wait<0>();
      __syncthreads();
    }
    epi_f<CF, 1, NSMALL>(D, op, acc, sA, sB, M, N, m0, n0, vmax, bad);
  }
  epi_scale(vmax, bad, scale_bits, nonfinite);
}

template <class CF, int NSMALL>
inline void set_attr_sk() {
  cudaFuncSetAttribute(gemm_sk_kernel<CF, NSMALL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem_bytes<CF, NSMALL>());
}

// co-resident CTAs of the stream-K kernel (its persistent grid and partial-slot count)
template <class CF, int NSMALL>
inline int sk_grid() {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gemm_sk_kernel<CF, NSMALL>, CF::NT, smem_bytes<CF, NSMALL>());
  return sms * (per > 0 ? per : 1);
}

template <class CF, int NSMALL>
inline void launch_sk(const GemmDesc *d, int grid, const FOp &op, unsigned long long *sb, int *nf, double *part,
                      unsigned *flags, unsigned long long *ticket, int nsk, cudaStream_t st) {
  gemm_sk_kernel<CF, NSMALL><<<grid, CF::NT, smem_bytes<CF, NSMALL>(), st>>>(d, op, sb, nf, part, flags, ticket, nsk);
}

}  // namespace gemmk
