// Launchers for the FP64 DMMA GEMMs of the 2-site update (kernels in gemm_kernel.cuh).
// Tile shapes were chosen by tools/gemm_bench.cu on a B200:
//   Pi = f(A^1 B^1, ...):        64x64 CTA tile, 8 warps of 32x16, BK 16, 3 stages (19.7 TF/s at
//                                the configs[3] chi=256 shape 1024 x 1024 x 256, 53% of DMMA peak)
//   A = L X, B = X R, C = S - AB: 64x32 CTA tile, 4 warps of 32x16 (more CTAs for the 512-row
//                                shapes)
#include <cstdio>
#include <mutex>

#include "gemm_kernel.cuh"

namespace {
using namespace gemmk;
// ACI_GEMM_VEC (default 1): tiles staged with 16-byte cp.async in global order (Cfg::VEC); measured
// 28.4 -> 26.9 us on the full-size Pi, bit-identical results (tools/gemm_bench2.cu,
// profiles/r02m_gemm_variants.txt)
#ifndef ACI_GEMM_VEC
#define ACI_GEMM_VEC 1
#endif
// ACI_PI_WN / ACI_PI_MINB (A/B switches): warp-tile width and min CTAs per SM of the Pi tile
#ifndef ACI_PI_WN
#define ACI_PI_WN 16
#endif
#ifndef ACI_PI_MINB
#define ACI_PI_MINB 2
#endif
using CfgPi = Cfg<64, 64, 32, ACI_PI_WN, 16, 3, ACI_PI_MINB, ACI_GEMM_VEC>;
using CfgAB = Cfg<64, 32, 32, 16, 16, 3, 4, ACI_GEMM_VEC>;
// Small problems: 32x32 tiles of 4 warps. A 64x64-tile grid of fewer than ~2 CTAs per SM leaves
// SMs idle and runs the K loop serially on the busy ones; measured per launch (tools/gemm_latency.cu,
// f fused, K = 64..256): 64^2 6.5 -> 3.7 us, 256^2 9.7 -> 5.0 us, 512^2 16.0 -> 9.4 us, but
// 1024^2 25.4 -> 28.1 us, so the 64x64 tiles stay for grids of >= 256 of them.
using CfgS = Cfg<32, 32, 16, 16, 16, 3, 4, ACI_GEMM_VEC>;
inline bool small_grid(int max_m, int max_n) { return ((max_m + 63) / 64) * ((max_n + 63) / 64) < 256; }

template <int NB, int NS>
void launch_pi(const GemmDesc *d, int ndesc, int max_m, int max_n, const FOp &op, unsigned long long *sb, int *nf,
               cudaStream_t st) {
  if (small_grid(max_m, max_n)) launch<CfgS, NB, NS, EPI_F>(d, ndesc, max_m, max_n, op, sb, nf, st);
  else launch<CfgPi, NB, NS, EPI_F>(d, ndesc, max_m, max_n, op, sb, nf, st);
}
template <int EPI>
void launch_ab(const GemmDesc *d, int ndesc, int max_m, int max_n, const FOp &op, unsigned long long *sb, int *nf,
               cudaStream_t st) {
  if (small_grid(max_m, max_n)) launch<CfgS, 1, 0, EPI>(d, ndesc, max_m, max_n, op, sb, nf, st);
  else launch<CfgAB, 1, 0, EPI>(d, ndesc, max_m, max_n, op, sb, nf, st);
}
template <int NB>
void launch_fz(const GemmDesc *d, int ndesc, int max_m, int max_n, const FOp &op, unsigned long long *sb, int *nf,
               cudaStream_t st) {
  if (small_grid(max_m, max_n)) launch<CfgS, NB, 0, EPI_FZ>(d, ndesc, max_m, max_n, op, sb, nf, st);
  else launch<CfgPi, NB, 0, EPI_FZ>(d, ndesc, max_m, max_n, op, sb, nf, st);
}
// ---- streamed Pi (PiStreamArgs, aci_common.cuh). A persistent grid of ntmax x P CTAs: CTA q owns
// the 32-column tile j = q % ntmax of Pi_{b+1} and the chunks c = q / ntmax + P t (32 rows each).
// Its column panel of every DMMA input's B^n_{b+1} (K_n x 32) is loaded into shared memory once;
// per chunk it waits until the pivot rows the chunk needs are published (or the final rank says
// the chunk is past the end), gathers the chunk's A rows (one cp.async pass: all of K at once)
// and runs the DMMA k-steps from shared memory, then the EPI_F epilogue. So the work left when the
// prrLU ends is one chunk: one A gather + 32 x 32 x K of DMMA per CTA. The column-0 CTA of a chunk
// also stores the gathered rows to A^n_{b+1}. k-steps in the tile kernels' order: Pi is
// bit-identical to the unstreamed path (up to the sign of exact zeros).
constexpr int kStBM = 32, kStBN = 32, kStNT = 128, kStPB = kStBN + 4;
struct CfgSt {  // the epilogue's view (epi_f): 4 warps of 16 x 16
  static constexpr int BM = kStBM, BN = kStBN, WM = 16, WN = 16, NT = kStNT, WARPS_N = 2, MI = 2, NI = 2;
};
constexpr int kStreamMaxK = 256;  // sum of the DMMA inputs' K (shared-memory panels)

__host__ __device__ constexpr int st_k4(int K) { return (K + 3) & ~3; }
__host__ __device__ constexpr int st_pa(int K) { return st_k4(K) + 4; }  // A row pitch (doubles)

__device__ __forceinline__ int ld_vol(const int *p) { return *reinterpret_cast<const volatile int *>(p); }
#ifdef ACI_STREAM_TS
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

template <int NBIG, int NSMALL>
__global__ void __launch_bounds__(kStNT) pi_stream_kernel(PiStreamArgs S, FOp op) {
  using CF = CfgSt;
  constexpr int NI_ = NBIG + NSMALL;
  extern __shared__ __align__(16) double sdyn[];
  __shared__ const double *rowp[NI_][kStBM];
  __shared__ int s_r;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, c4 = lane & 3;
  const int wm = (w / CF::WARPS_N) * CF::WM, wn = (w % CF::WARPS_N) * CF::WN;
  const int nn = S.db2 * S.rk[S.b + 3];
  const int ntn = (nn + kStBN - 1) / kStBN;
  const int j = blockIdx.x % S.ntmax, P = gridDim.x / S.ntmax;
  // s as Pi_b left it, for bond b's index kernel (this stream merges Pi_{b+1}'s max only at its end;
  // every CTA of the prrLU read s for its threshold before the rank this stream waits for exists)
  if (blockIdx.x == 0 && tid == 0) *reinterpret_cast<unsigned long long *>(S.info + 4) = *S.scale;
  const bool active = j < ntn;
  double vmax = 0.0;
  bool bad = false;
  if (active) {
    const int n0 = j * kStBN;
    // shared layout: per DMMA input B panel [K4][kStPB] then A rows [32][pa]; small-K operands last
    double *Bs[NBIG > 0 ? NBIG : 1], *As[NBIG > 0 ? NBIG : 1];
    double *q = sdyn;
#pragma unroll
    for (int i = 0; i < NBIG; ++i) {
      Bs[i] = q;
      q += st_k4(S.c2[i]) * kStPB;
      As[i] = q;
      q += kStBM * st_pa(S.c2[i]);
    }
    double *sA = q, *sB = sA + NSMALL * kStBM * kSmallK;
    // B panels (zero-filled past n' and past K up to the k-step multiple of 4)
    const bool vecB = !(nn & 1);
#pragma unroll
    for (int i = 0; i < NBIG; ++i) {
      const int K = S.c2[i], K4 = st_k4(K);
      const double *B = S.B[i];
      if (vecB && !(reinterpret_cast<uintptr_t>(B) & 15)) {
        for (int t = tid; t < K4 * (kStBN / 2); t += kStNT) {
          const int k = t / (kStBN / 2), col = 2 * (t - k * (kStBN / 2));
          const bool v = k < K && n0 + col < nn;  // nn even: both columns or neither
          unsigned sd = (unsigned)__cvta_generic_to_shared(Bs[i] + k * kStPB + col);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sd),
                       "l"(v ? B + (size_t)k * nn + n0 + col : B), "r"(v ? 16 : 0));
        }
      } else {
        for (int t = tid; t < K4 * kStBN; t += kStNT) {
          const int k = t / kStBN, col = t - k * kStBN;
          const bool v = k < K && n0 + col < nn;
          cp_async8(Bs[i] + k * kStPB + col, v ? B + (size_t)k * nn + n0 + col : B, v);
        }
      }
    }
    cp_async_commit();
    GemmDesc D;  // the epilogue's view of Pi_{b+1}
    D.C = S.Pi;
    D.ldc = nn;
#pragma unroll
    for (int i = 0; i < NI_; ++i) D.K[i] = S.c2[i];
#ifdef ACI_STREAM_TS
    unsigned long long *ts = S.ts + 16 * S.b;
    if (tid == 0) atomicMax(ts + 0, ~gtime());
    unsigned long long tp[6];
#endif
    for (int c = blockIdx.x / S.ntmax;; c += P) {
      const int m0 = c * kStBM;
      if (tid == 0) {
        // the last pivot this chunk needs; past the buffer (kcap pivots at most) only r can tell
        const int kneed = (m0 + kStBM - 1) / S.d1, kpoll = kneed < S.kcap ? kneed : S.kcap - 1;
        int r;
        while ((r = ld_vol(S.r_in)) < 0 && (kneed >= S.kcap || ld_vol(S.rows + kpoll) < 0)) __nanosleep(S.poll_ns);
        s_r = r;
      }
      __syncthreads();
      const int r = s_r;
#ifdef ACI_STREAM_TS
      if (tid == 0) {
        if (r >= 0) atomicMax(ts + 1, ~gtime());
        if (r >= 0 && m0 < r * S.d1) atomicMax(ts + 2, gtime());
        atomicMax(ts + 3, gtime());
      }
#endif
      const int M = r >= 0 ? r * S.d1 : m0 + kStBM;  // rows known so far (all of Pi once r is)
      if (m0 >= M) break;  // past the final rank: so is every later chunk of this CTA
#ifdef ACI_STREAM_TS
      tp[0] = gtime();
#endif
      for (int t = tid; t < NI_ * kStBM; t += kStNT) {
        const int i = t / kStBM, row = t - i * kStBM, R = m0 + row;
        const double *p = nullptr;
        if (R < M) {
          const int k = R / S.d1, sg = R - k * S.d1;
          int pr;
          while ((pr = ld_vol(S.rows + k)) < 0) __nanosleep(64);  // published stores are unordered
          p = S.Ahat[i] + ((size_t)pr * S.d1 + sg) * S.c2[i];
        }
        rowp[i][row] = p;
      }
      __syncthreads();
#ifdef ACI_STREAM_TS
      tp[1] = gtime();
#endif
      // the chunk's A rows, all of K in one pass (zero rows past M, zero columns K..K4)
#pragma unroll
      for (int i = 0; i < NBIG; ++i) {
        const int K = S.c2[i], K4 = st_k4(K), pa = st_pa(K);
        if (!(K & 1) && !(reinterpret_cast<uintptr_t>(S.Ahat[i]) & 15)) {
          for (int t = tid; t < kStBM * (K4 / 2); t += kStNT) {
            const int row = t / (K4 / 2), kc = 2 * (t - row * (K4 / 2));
            const double *src = rowp[i][row];
            const bool v = src && kc < K;  // K even: both k or neither
            unsigned sd = (unsigned)__cvta_generic_to_shared(As[i] + row * pa + kc);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sd), "l"(v ? src + kc : S.Ahat[i]),
                         "r"(v ? 16 : 0));
          }
        } else {
          for (int t = tid; t < kStBM * K4; t += kStNT) {
            const int row = t / K4, kc = t - row * K4;
            const double *src = rowp[i][row];
            const bool v = src && kc < K;
            cp_async8(As[i] + row * pa + kc, v ? src + kc : S.Ahat[i], v);
          }
        }
      }
#pragma unroll
      for (int s_ = 0; s_ < NSMALL; ++s_) {
        const int i = NBIG + s_, K = S.c2[i];
        for (int t = tid; t < kStBM * kSmallK; t += kStNT) {
          const int row = t / kSmallK, kk = t - row * kSmallK;
          const double *src = rowp[i][row];
          const bool v = src && kk < K;
          cp_async8(&sA[s_ * kStBM * kSmallK + t], v ? src + kk : S.Ahat[i], v);
        }
        for (int t = tid; t < kSmallK * kStBN; t += kStNT) {
          const int kk = t / kStBN, col = t - kk * kStBN;
          const bool v = kk < K && n0 + col < nn;
          cp_async8(&sB[s_ * kSmallK * kStBN + t], v ? S.B[i] + (size_t)kk * nn + n0 + col : S.B[i], v);
        }
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
#ifdef ACI_STREAM_TS
      tp[2] = gtime();
#endif
      constexpr int NB = NBIG > 0 ? NBIG : 1;
      double acc[NB][CF::MI][CF::NI][2];
#pragma unroll
      for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int mi = 0; mi < CF::MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < CF::NI; ++ni) acc[i][mi][ni][0] = acc[i][mi][ni][1] = 0.0;
#pragma unroll
      for (int i = 0; i < NBIG; ++i) {
        const int K4 = st_k4(S.c2[i]), pa = st_pa(S.c2[i]);
        const double *Ai = As[i], *Bi = Bs[i];
#pragma unroll 4
        for (int ks = 0; ks < K4 / 4; ++ks) {
          double a[CF::MI], bv[CF::NI];
#pragma unroll
          for (int mi = 0; mi < CF::MI; ++mi) a[mi] = Ai[(wm + mi * 8 + g) * pa + 4 * ks + c4];
#pragma unroll
          for (int ni = 0; ni < CF::NI; ++ni) bv[ni] = Bi[(4 * ks + c4) * kStPB + wn + ni * 8 + g];
#pragma unroll
          for (int mi = 0; mi < CF::MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < CF::NI; ++ni) dmma(acc[i][mi][ni], a[mi], bv[ni]);
        }
      }
#ifdef ACI_STREAM_TS
      tp[3] = gtime();
#endif
      epi_f<CF, NBIG, NSMALL>(D, op, acc, sA, sB, M, nn, m0, n0, vmax, bad);
#ifdef ACI_STREAM_TS
      tp[4] = gtime();
#endif
      // A^n_{b+1} rows of this chunk, split over the chunk's ntn column-tile CTAs (rows j, j + ntn, ...)
#pragma unroll
      for (int i = 0; i < NI_; ++i) {
        if (!S.Anext[i]) continue;
        const int K = S.c2[i];
        for (int row = j; row < kStBM && m0 + row < M; row += ntn) {
          double *dst = S.Anext[i] + (size_t)(m0 + row) * K;
          if (i < NBIG) {
            const double *src = As[i < NBIG ? i : 0] + row * st_pa(K);
            for (int kk = tid; kk < K; kk += kStNT) dst[kk] = src[kk];
          } else {
            for (int kk = tid; kk < K; kk += kStNT) dst[kk] = rowp[i][row][kk];
          }
        }
      }
      __syncthreads();  // rowp / A rows / small operands are rewritten by the next chunk
#ifdef ACI_STREAM_TS
      tp[5] = gtime();
      if (tid == 0)
        for (int x = 0; x < 5; ++x) atomicMax(ts + 8 + x, tp[x + 1] - tp[x]);
#endif
    }
  }
  epi_scale(vmax, bad, S.sp, S.nonfinite);
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(S.done, 1u) == gridDim.x - 1) {  // the last CTA: every max |Pi_{b+1}| is in sp
      __threadfence();
      const unsigned long long v = *reinterpret_cast<volatile unsigned long long *>(S.sp);
      if (v > *reinterpret_cast<volatile unsigned long long *>(S.scale)) atomicMax(S.scale, v);
      *S.sp = 0ull;
      *S.done = 0u;
    }
  }
#ifdef ACI_STREAM_TS
  if (tid == 0 && active) atomicMax(S.ts + 16 * S.b + 4, gtime());
#endif
}

template <int NB, int NS>
void launch_stream_t(const PiStreamArgs &a, const FOp &op, int grid, cudaStream_t st) {
  size_t smem = sizeof(double) * (size_t)NS * (kStBM * kSmallK + kSmallK * kStBN);
  for (int i = 0; i < NB; ++i) smem += sizeof(double) * ((size_t)st_k4(a.c2[i]) * kStPB + (size_t)kStBM * st_pa(a.c2[i]));
  pi_stream_kernel<NB, NS><<<grid, kStNT, smem, st>>>(a, op);
}
template <int NB, int NS>
void set_attr_stream() {
  cudaFuncSetAttribute(pi_stream_kernel<NB, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}
}  // namespace

bool pi_stream_supported(int nbig, int nsmall, const int *c2, int ntmax) {
  if (nbig + nsmall < 1 || nbig + nsmall > 3 || ntmax < 1 || ntmax > 64) return false;
  int ks = 0;
  for (int i = 0; i < nbig; ++i) ks += st_k4(c2[i]);
  return ks <= kStreamMaxK;
}

void launch_pi_stream(const PiStreamArgs &a, int nsmall, const FOp &op, int grid, cudaStream_t st) {
  switch (a.nbig * 10 + nsmall) {
    case 10: launch_stream_t<1, 0>(a, op, grid, st); break;
    case 20: launch_stream_t<2, 0>(a, op, grid, st); break;
    case 30: launch_stream_t<3, 0>(a, op, grid, st); break;
    case 1: launch_stream_t<0, 1>(a, op, grid, st); break;
    case 11: launch_stream_t<1, 1>(a, op, grid, st); break;
    case 21: launch_stream_t<2, 1>(a, op, grid, st); break;
    case 2: launch_stream_t<0, 2>(a, op, grid, st); break;
    case 12: launch_stream_t<1, 2>(a, op, grid, st); break;
    case 3: launch_stream_t<0, 3>(a, op, grid, st); break;
    default: break;
  }
}

static void gemm_init_once() {
  set_attr_stream<1, 0>();
  set_attr_stream<2, 0>();
  set_attr_stream<3, 0>();
  set_attr_stream<0, 1>();
  set_attr_stream<1, 1>();
  set_attr_stream<2, 1>();
  set_attr_stream<0, 2>();
  set_attr_stream<1, 2>();
  set_attr_stream<0, 3>();
  set_attr<CfgAB, 1, 0, EPI_STORE>();
  set_attr<CfgAB, 1, 0, EPI_SUB>();
  set_attr<CfgPi, 1, 0, EPI_F>();
  set_attr<CfgPi, 2, 0, EPI_F>();
  set_attr<CfgPi, 3, 0, EPI_F>();
  set_attr<CfgPi, 4, 0, EPI_F>();
  set_attr<CfgPi, 0, 1, EPI_F>();
  set_attr<CfgPi, 1, 1, EPI_F>();
  set_attr<CfgPi, 2, 1, EPI_F>();
  set_attr<CfgPi, 0, 2, EPI_F>();
  set_attr<CfgPi, 1, 2, EPI_F>();
  set_attr<CfgPi, 0, 3, EPI_F>();
  set_attr<CfgAB, 1, 0, EPI_STORE_X>();
  set_attr<CfgPi, 1, 0, EPI_FZ>();
  set_attr<CfgPi, 2, 0, EPI_FZ>();
  set_attr<CfgPi, 3, 0, EPI_FZ>();
  set_attr<CfgPi, 4, 0, EPI_FZ>();
  set_attr<CfgS, 1, 0, EPI_STORE>();
  set_attr<CfgS, 1, 0, EPI_STORE_X>();
  set_attr<CfgS, 1, 0, EPI_F>();
  set_attr<CfgS, 2, 0, EPI_F>();
  set_attr<CfgS, 3, 0, EPI_F>();
  set_attr<CfgS, 4, 0, EPI_F>();
  set_attr<CfgS, 0, 1, EPI_F>();
  set_attr<CfgS, 1, 1, EPI_F>();
  set_attr<CfgS, 2, 1, EPI_F>();
  set_attr<CfgS, 0, 2, EPI_F>();
  set_attr<CfgS, 1, 2, EPI_F>();
  set_attr<CfgS, 0, 3, EPI_F>();
  set_attr<CfgS, 1, 0, EPI_FZ>();
  set_attr<CfgS, 2, 0, EPI_FZ>();
  set_attr<CfgS, 3, 0, EPI_FZ>();
  set_attr<CfgS, 4, 0, EPI_FZ>();
}

void gemm_init() {
  // kernel attributes are set once (thread-safe), outside any stream capture
  static std::once_flag once;
  std::call_once(once, gemm_init_once);
}

int gemm_small_k() { return kSmallK; }

void launch_gemm_sub(const GemmDesc *d, int ndesc, int max_m, int max_n, cudaStream_t st) {
  if (max_m <= 0 || max_n <= 0 || ndesc <= 0) return;
  FOp op = {};
  launch<CfgAB, 1, 0, EPI_SUB>(d, ndesc, max_m, max_n, op, nullptr, nullptr, st);
}

void launch_gemm_split(const GemmDesc *d, int ndesc, int max_m, int max_n, int nbig, int nsmall, bool fuse,
                       const FOp &op, unsigned long long *sb, int *nf, cudaStream_t st) {
  if (max_m <= 0 || max_n <= 0 || ndesc <= 0) return;
  if (!fuse) {
    launch_ab<EPI_STORE>(d, ndesc, max_m, max_n, op, sb, nf, st);
    return;
  }
  if (nbig + nsmall >= 4) {  // rare shape: every input through DMMA (descriptor order unchanged)
    launch_pi<4, 0>(d, ndesc, max_m, max_n, op, sb, nf, st);
    return;
  }
  switch (nbig * 10 + nsmall) {
    case 10: launch_pi<1, 0>(d, ndesc, max_m, max_n, op, sb, nf, st); break;
    case 20: launch_pi<2, 0>(d, ndesc, max_m, max_n, op, sb, nf, st); break;
    case 30: launch_pi<3, 0>(d, ndesc, max_m, max_n, op, sb, nf, st); break;
    case 1: launch_pi<0, 1>(d, ndesc, max_m, max_n, op, sb, nf, st); break;
    case 11: launch_pi<1, 1>(d, ndesc, max_m, max_n, op, sb, nf, st); break;
    case 21: launch_pi<2, 1>(d, ndesc, max_m, max_n, op, sb, nf, st); break;
    case 2: launch_pi<0, 2>(d, ndesc, max_m, max_n, op, sb, nf, st); break;
    case 12: launch_pi<1, 2>(d, ndesc, max_m, max_n, op, sb, nf, st); break;
    case 3: launch_pi<0, 3>(d, ndesc, max_m, max_n, op, sb, nf, st); break;
    default: break;
  }
}

void launch_gemm_z(const GemmDesc *d, int ndesc, int max_m, int max_n, int mode, int nin, const FOp &op,
                   unsigned long long *sb, int *nf, cudaStream_t st) {
  if (max_m <= 0 || max_n <= 0 || ndesc <= 0) return;
  if (mode == 0) {
    launch_ab<EPI_STORE>(d, ndesc, max_m, max_n, op, sb, nf, st);
  } else if (mode == 1) {
    launch_ab<EPI_STORE_X>(d, ndesc, max_m, max_n, op, sb, nf, st);
  } else {
    switch (nin) {
      case 1: launch_fz<1>(d, ndesc, max_m, max_n, op, sb, nf, st); break;
      case 2: launch_fz<2>(d, ndesc, max_m, max_n, op, sb, nf, st); break;
      case 3: launch_fz<3>(d, ndesc, max_m, max_n, op, sb, nf, st); break;
      default: launch_fz<4>(d, ndesc, max_m, max_n, op, sb, nf, st); break;
    }
  }
}

void launch_gemm(const GemmDesc *d_descs, int ndesc, int max_m, int max_n, int nin, bool fuse, const FOp &op,
                 unsigned long long *scale_bits, int *nonfinite, cudaStream_t st) {
  launch_gemm_split(d_descs, ndesc, max_m, max_n, fuse ? nin : 1, 0, fuse, op, scale_bits, nonfinite, st);
}
