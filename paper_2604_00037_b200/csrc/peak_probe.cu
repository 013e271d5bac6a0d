// libaci_peak.so — FP64 roofline denominators measured in the same process as the bench
// (measurement infrastructure, not part of the ACI path; MEASURED_PEAKS.json has no FP64 entry).
//   kind 0: DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4) register-only loop, 4 x 2 independent
//           accumulator tiles per warp, 8 warps per CTA, 2 CTAs per SM: the FP64 tensor-pipe peak
//           the contraction kernels (a1-a4) are held against;
//   kind 1: DFMA register-only loop (8 independent chains per thread): the FP64 ALU peak the
//           prrLU's rank-1 updates (a5) are held against.
// Each launch covers every SM (148 x 2 CTAs); the result is the best of `reps` CUDA-event-timed
// launches after one warm-up launch, in TFLOP/s (2 flops per FMA).
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

constexpr int kMI = 4, kNI = 2, kKS = 4;

__global__ void __launch_bounds__(256) dmma_loop(double *out, int iters) {
  double acc[kMI][kNI][2] = {};
  double a[kKS][kMI], b[kKS][kNI];
  for (int k = 0; k < kKS; ++k) {
    for (int i = 0; i < kMI; ++i) a[k][i] = 1e-3 * (threadIdx.x + i + k);
    for (int j = 0; j < kNI; ++j) b[k][j] = 1e-3 * (blockIdx.x + j + k);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < kKS; ++k)
#pragma unroll
      for (int i = 0; i < kMI; ++i)
#pragma unroll
        for (int j = 0; j < kNI; ++j) dmma(acc[i][j], a[k][i], b[k][j]);
  }
  double s = 0;
  for (int i = 0; i < kMI; ++i)
    for (int j = 0; j < kNI; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 12345.0) out[0] = s;  // keeps the loop; never true
}

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) dfma_loop(double *out, int iters) {
  double x[kChains];
  const double y = 1.0 + 1e-9 * threadIdx.x, z = 1e-12 * blockIdx.x;
  for (int c = 0; c < kChains; ++c) x[c] = 1e-3 * (threadIdx.x + c);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], y, z);
  }
  double s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.0) out[0] = s;
}

}  // namespace

extern "C" int aci_peak_fp64(int kind, int reps, double *tflops) {
  if (!tflops || (kind != 0 && kind != 1)) return -1;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -5;
  double *out = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess || cudaMallocAsync(&out, 64, st) != cudaSuccess ||
      cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)
    return -5;
  const int grid = 2 * sms, threads = 256;
  const int iters = kind == 0 ? 4000 : 20000;
  // flops per launch: DMMA 8x8x4 = 256 FMA per warp instruction; DFMA 1 FMA per thread
  const double fl = kind == 0 ? 2.0 * 256 * kMI * kNI * kKS * (double)iters * (threads / 32) * grid
                              : 2.0 * 8 * kChains * (double)iters * threads * grid;
  auto launch = [&](int it) {
    if (kind == 0) dmma_loop<<<grid, threads, 0, st>>>(out, it);
    else dfma_loop<<<grid, threads, 0, st>>>(out, it);
  };
  launch(iters);
  double best = 0.0;
  for (int r = 0; r < (reps > 0 ? reps : 5); ++r) {
    cudaEventRecord(e0, st);
    launch(iters);
    cudaEventRecord(e1, st);
    if (cudaEventSynchronize(e1) != cudaSuccess) break;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms > 0.f && fl / (ms * 1e9) > best) best = fl / (ms * 1e9);
  }
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(out, st);
  cudaStreamSynchronize(st);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  if (e != cudaSuccess) return -5;
  *tflops = best;
  return 0;
}

// ---------------------------------------------------------------------------------------------
// prrLU latency probes (roofline.latency in bench.py): the library's own prrLU (csrc/prrlu.cu,
// compiled here twice) on a seeded m x m block — with the work (the real per-pivot time of the
// tier that block selects) and with ACI_PRRLU_NOWORK (no rank-1 update, no rescan: every step
// exchanges the same winner, so what is left is the exchange chain — the per-pivot floor of the
// design: CTA argmax, cluster key exchange, cross-cluster leg, column read).
#include <cstdlib>

#include "aci_common.cuh"
namespace probe_work {
#include "prrlu.cu"
}
#undef ACI_PRRLU_NOWORK
#define ACI_PRRLU_NOWORK 1
namespace probe_nowork {
#include "prrlu.cu"
}

namespace {
__global__ void fill_kernel(double *M, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long x = seed + 0x9E3779B97F4A7C15ull * (i + 1);
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x ^= x >> 31;
    M[i] = (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
}
}  // namespace

// Per-pivot time of the library's prrLU on a seeded live m x n block (ld = n, at most kmax pivots)
// inside a launch sized for the static sm x sn block, as the product launches it (tier choice and
// hand-off included); nowork = 1: the ACI_PRRLU_NOWORK build (the exchange chain alone).
extern "C" int aci_peak_prrlu_shape(int m, int n, int kmax, int sm, int sn, int nowork, int reps,
                                    double *us_per_pivot, int *pivots);
extern "C" int aci_peak_prrlu(int m, int nowork, int reps, double *us_per_pivot, int *pivots) {
  if (m < 32 || m > 1024) return -1;
  return aci_peak_prrlu_shape(m, m, m > 512 ? 512 : m, m, m, nowork, reps, us_per_pivot, pivots);
}

extern "C" int aci_peak_prrlu_shape(int m, int n, int kmax, int sm, int sn, int nowork, int reps,
                                    double *us_per_pivot, int *pivots) {
  if (!us_per_pivot || m < 1 || n < 1 || m > sm || n > sn || sm > 1024 || sn > 1184 || kmax < 1) return -1;
  double *M = nullptr, *U = nullptr, *eps = nullptr;
  unsigned long long *colpub = nullptr, *keys = nullptr, *scale = nullptr;
  int *rows = nullptr, *cols = nullptr, *r = nullptr;
  unsigned *ctr = nullptr, *epoch = nullptr;
  LuDims *dims = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const size_t colpub_words = (size_t)2 * 148 * 1024 * 2;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&M, sizeof(double) * m * n) != cudaSuccess || cudaMalloc(&U, sizeof(double) * kmax * n) != cudaSuccess ||
      cudaMalloc(&eps, 8) != cudaSuccess || cudaMalloc(&colpub, 8 * colpub_words) != cudaSuccess ||
      cudaMalloc(&keys, 8 * 2 * 148 * 4) != cudaSuccess || cudaMalloc(&scale, 8) != cudaSuccess ||
      cudaMalloc(&rows, 4 * 1024) != cudaSuccess || cudaMalloc(&cols, 4 * 1024) != cudaSuccess ||
      cudaMalloc(&r, 4) != cudaSuccess || cudaMalloc(&ctr, 4) != cudaSuccess || cudaMalloc(&epoch, 4) != cudaSuccess ||
      cudaMalloc(&dims, sizeof(LuDims)) != cudaSuccess || cudaEventCreate(&e0) != cudaSuccess ||
      cudaEventCreate(&e1) != cudaSuccess)
    return -5;
  fill_kernel<<<296, 256, 0, st>>>(M, (size_t)m * n, 12345ull + m + 7919ull * n);
  cudaMemsetAsync(colpub, 0, 8 * colpub_words, st);
  cudaMemsetAsync(keys, 0, 8 * 2 * 148 * 4, st);
  cudaMemsetAsync(epoch, 0, 4, st);
  cudaMemsetAsync(scale, 0, 8, st);
  LuDims D{m, n, n, kmax, n};
  cudaMemcpyAsync(dims, &D, sizeof(D), cudaMemcpyHostToDevice, st);
  LuArgs a = {};
  a.M = M; a.dims = dims; a.tol = 0.0; a.thr_mode = 2; a.scale_bits = scale;
  a.rows = rows; a.cols = cols; a.r_out = r; a.eps_out = eps; a.U = U;
  a.colpub = colpub; a.colcap = 1024; a.keys = keys; a.counter = ctr; a.epoch = epoch;
  if (nowork) probe_nowork::prrlu_init();
  else probe_work::prrlu_init();
  auto launch = [&]() {
    return nowork ? probe_nowork::launch_prrlu(a, sm, sn, st, false, false, nullptr, false)
                  : probe_work::launch_prrlu(a, sm, sn, st, false, false, nullptr, false);
  };
  cudaError_t le = launch();
  double best = 1e30;
  for (int t = 0; t < (reps > 0 ? reps : 3) && le == cudaSuccess; ++t) {
    cudaEventRecord(e0, st);
    le = launch();
    cudaEventRecord(e1, st);
    if (cudaEventSynchronize(e1) != cudaSuccess) break;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  int hr = 0;
  cudaMemcpyAsync(&hr, r, 4, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  for (void *p : {(void *)M, (void *)U, (void *)eps, (void *)colpub, (void *)keys, (void *)scale, (void *)rows,
                  (void *)cols, (void *)r, (void *)ctr, (void *)epoch, (void *)dims})
    cudaFree(p);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  if (e != cudaSuccess || le != cudaSuccess || hr <= 0) return -5;
  *us_per_pivot = best * 1e3 / hr;
  if (pivots) *pivots = hr;
  return 0;
}
