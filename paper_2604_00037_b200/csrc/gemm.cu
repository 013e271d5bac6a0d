// Launchers for the FP64 DMMA GEMMs of the 2-site update (kernels in gemm_kernel.cuh).
// Tile shapes were chosen by tools/gemm_bench.cu on a B200:
//   Pi = f(A^1 B^1, ...):        64x64 CTA tile, 8 warps of 32x16, BK 16, 3 stages (19.7 TF/s at
//                                the configs[3] chi=256 shape 1024 x 1024 x 256, 53% of DMMA peak)
//   A = L X, B = X R, C = S - AB: 64x32 CTA tile, 4 warps of 32x16 (more CTAs for the 512-row
//                                shapes)
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
using CfgPi = Cfg<64, 64, 32, 16, 16, 3, 2, ACI_GEMM_VEC>;
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
}  // namespace

static void gemm_init_once() {
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
