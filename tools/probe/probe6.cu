// DMMA issue probe: register-only warp tiles shaped like the GEMM (MI x NI accumulators, fresh
// A/B fragments each k-step from registers) vs. the fixed-operand loop. Not product code.
#include <cstdio>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int MI, int NI, int KS>
__global__ void tile(double *out, int iters) {
  double acc[MI][NI][2] = {};
  double a[KS][MI], b[KS][NI];
  for (int k = 0; k < KS; ++k) {
    for (int i = 0; i < MI; ++i) a[k][i] = 1e-3 * (threadIdx.x + i + k);
    for (int j = 0; j < NI; ++j) b[k][j] = 1e-3 * (blockIdx.x + j + k);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < KS; ++k)
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma(acc[i][j], a[k][i], b[k][j]);
  }
  double s = 0;
  for (int i = 0; i < MI; ++i) for (int j = 0; j < NI; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 12345.0) out[0] = s;
}
template <int MI, int NI, int KS>
void run(double *out, int warps, int ctas_per_sm) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4000;
  tile<MI, NI, KS><<<148 * ctas_per_sm, warps * 32>>>(out, 10);
  cudaEventRecord(e0);
  tile<MI, NI, KS><<<148 * ctas_per_sm, warps * 32>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 256 * MI * NI * KS * (double)iters * warps * 148 * ctas_per_sm;
  printf("MI=%d NI=%d KS=%d warps/CTA=%2d CTAs/SM=%d: %.2f TF/s %s\n", MI, NI, KS, warps, ctas_per_sm, fl / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  double *out; CK(cudaMalloc(&out, 64));
  run<1, 4, 1>(out, 8, 2);   // probe1-like: fixed a, 4 chains
  run<4, 2, 1>(out, 8, 2);
  run<4, 2, 4>(out, 8, 2);
  run<4, 4, 4>(out, 4, 2);
  run<4, 4, 4>(out, 8, 1);
  run<2, 2, 4>(out, 16, 1);
  run<4, 2, 4>(out, 16, 1);
  run<4, 2, 2>(out, 8, 3);
  run<2, 4, 2>(out, 8, 3);
  return 0;
}
