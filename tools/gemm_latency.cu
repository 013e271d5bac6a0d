// Per-launch time of the Pi GEMM (CfgPi, f fused, one DMMA input + a K = 2 input) for small live
// sizes inside a large static grid, as the sweep launches it (development tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/gemm_latency.cu -o tools/gemm_latency
#include "../paper_2604_00037_b200/csrc/gemm_kernel.cuh"
#include <cstdio>
#include <vector>
using namespace gemmk;
using CfgPi = Cfg<64, 64, 32, 16, 16, 3, 2>;
using C32 = Cfg<32, 32, 16, 16, 16, 3, 4>;
using C3264 = Cfg<32, 64, 16, 32, 16, 3, 4>;
using C6432 = Cfg<64, 32, 32, 16, 16, 3, 4>;
using C32b = Cfg<32, 32, 16, 16, 32, 3, 4>;
using C32w8 = Cfg<32, 64, 16, 16, 16, 3, 4>;   // 8 warps of 16x16
using C64w8s4 = Cfg<64, 64, 32, 16, 16, 4, 2>;
using C32s4 = Cfg<32, 32, 16, 16, 16, 4, 4>;
using C32x16 = Cfg<32, 32, 16, 8, 16, 3, 4>;  // 8 warps of 16x8

__global__ void empty_kernel(int *p) { if (p && threadIdx.x == 1023) *p = 0; }

int main() {
  const int MX = 1024, NX = 1024, KX = 256;
  double *A, *B, *A2, *B2, *C;
  cudaMalloc(&A, 8 * MX * KX); cudaMalloc(&B, 8 * KX * NX); cudaMalloc(&A2, 8 * MX * 2); cudaMalloc(&B2, 8 * 2 * NX);
  cudaMalloc(&C, 8 * MX * NX);
  std::vector<double> h(MX * KX, 0.001);
  cudaMemcpy(A, h.data(), 8 * MX * KX, cudaMemcpyHostToDevice);
  cudaMemcpy(B, h.data(), 8 * KX * NX, cudaMemcpyHostToDevice);
  cudaMemset(A2, 0, 8 * MX * 2); cudaMemset(B2, 0, 8 * 2 * NX);
  GemmDesc *dd; cudaMalloc(&dd, sizeof(GemmDesc));
  FOp op = {}; op.T = 1; op.N = 2; op.coef[0] = 1.0; op.expo[0] = 1; op.expo[1] = 1; op.monomial_all_ones = 1;
  unsigned long long *sb; int *nf; cudaMalloc(&sb, 8); cudaMalloc(&nf, 4);
  set_attr<CfgPi, 1, 1, EPI_F>();
  set_attr<C32, 1, 1, EPI_F>();
  set_attr<C3264, 1, 1, EPI_F>();
  set_attr<C6432, 1, 1, EPI_F>();
  set_attr<C32b, 1, 1, EPI_F>();
  set_attr<C32w8, 1, 1, EPI_F>();
  set_attr<C64w8s4, 1, 1, EPI_F>();
  set_attr<C32s4, 1, 1, EPI_F>();
  set_attr<C32x16, 1, 1, EPI_F>();
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto fn, int n) {
    float best = 1e9, ms;
    for (int rep = 0; rep < 3; ++rep) {
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
      for (int i = 0; i < n; ++i) fn();
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(e0, st);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms / n < best ? ms / n : best;
      cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
    return best * 1e3;
  };
  printf("empty kernel (1 CTA)        %7.2f us\n", timeit([&] { empty_kernel<<<1, 32, 0, st>>>(nullptr); }, 200));
  printf("empty kernel (256x256 thr)  %7.2f us\n", timeit([&] { empty_kernel<<<256, 256, 0, st>>>(nullptr); }, 200));
  const int sizes[][3] = {{16, 16, 64}, {64, 64, 64}, {128, 128, 64}, {256, 256, 128}, {512, 512, 256}, {1024, 1024, 256}};
  for (auto &sz : sizes) {
    GemmDesc d = {};
    d.C = C; d.M = sz[0]; d.N = sz[1]; d.ldc = sz[1]; d.nin = 2;
    d.A[0] = A; d.lda[0] = sz[2]; d.K[0] = sz[2]; d.B[0] = B; d.ldb[0] = sz[1];
    d.A[1] = A2; d.lda[1] = 2; d.K[1] = 2; d.B[1] = B2; d.ldb[1] = sz[1];
    cudaMemcpy(dd, &d, sizeof(d), cudaMemcpyHostToDevice);
    const float tstat = timeit([&] { launch<CfgPi, 1, 1, EPI_F>(dd, 1, MX, NX, op, sb, nf, st); }, 100);
    const float tfit = timeit([&] { launch<CfgPi, 1, 1, EPI_F>(dd, 1, sz[0], sz[1], op, sb, nf, st); }, 100);
    const float t32 = timeit([&] { launch<C32, 1, 1, EPI_F>(dd, 1, sz[0], sz[1], op, sb, nf, st); }, 100);
    const float t3264 = timeit([&] { launch<C3264, 1, 1, EPI_F>(dd, 1, sz[0], sz[1], op, sb, nf, st); }, 100);
    const float t6432 = timeit([&] { launch<C6432, 1, 1, EPI_F>(dd, 1, sz[0], sz[1], op, sb, nf, st); }, 100);
    const float t32b = timeit([&] { launch<C32b, 1, 1, EPI_F>(dd, 1, sz[0], sz[1], op, sb, nf, st); }, 100);
    const float ta = timeit([&] { launch<C32w8, 1, 1, EPI_F>(dd, 1, sz[0], sz[1], op, sb, nf, st); }, 100);
    const float tb = timeit([&] { launch<C64w8s4, 1, 1, EPI_F>(dd, 1, sz[0], sz[1], op, sb, nf, st); }, 100);
    const float tc = timeit([&] { launch<C32s4, 1, 1, EPI_F>(dd, 1, sz[0], sz[1], op, sb, nf, st); }, 100);
    const float td = timeit([&] { launch<C32x16, 1, 1, EPI_F>(dd, 1, sz[0], sz[1], op, sb, nf, st); }, 100);
    printf("Pi %4d x %4d x %3d: 64x64 %7.2f | 32x32 %7.2f | 32x64 %7.2f | 64x32 %7.2f | 32x32bk32 %7.2f | 32x64w8 %7.2f | 64x64s4 %7.2f | 32x32s4 %7.2f | 32x32w8 %7.2f us | %s\n",
           sz[0], sz[1], sz[2], tfit, t32, t3264, t6432, t32b, ta, tb, tc, td, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
