// Where the time of the full-size Pi GEMM goes (development tool): the configs[3] chi = 256 shape
// (1024 x 1024, K = 256 plus a K = 2 input, f = product) with the epilogue variants.
#include "../paper_2604_00037_b200/csrc/gemm_kernel.cuh"
#include <cstdio>
#include <vector>
using namespace gemmk;
using CfgPi = Cfg<64, 64, 32, 16, 16, 3, 2>;
using CfgV = Cfg<64, 64, 32, 16, 16, 3, 2, 1>;
using CfgV32 = Cfg<64, 64, 32, 16, 32, 2, 2, 1>;
using CfgV4 = Cfg<64, 64, 32, 16, 16, 4, 2, 1>;

int main() {
  const int M = 1024, N = 1024, K = 256;
  double *A, *B, *A2, *B2, *C;
  cudaMalloc(&A, 8 * M * K); cudaMalloc(&B, 8 * K * N); cudaMalloc(&A2, 8 * M * 2); cudaMalloc(&B2, 8 * 2 * N);
  cudaMalloc(&C, 8 * M * N);
  std::vector<double> h(M * K, 0.001);
  cudaMemcpy(A, h.data(), 8 * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(B, h.data(), 8 * K * N, cudaMemcpyHostToDevice);
  cudaMemset(A2, 0, 8 * M * 2); cudaMemset(B2, 0, 8 * 2 * N);
  GemmDesc d = {};
  d.C = C; d.M = M; d.N = N; d.ldc = N; d.nin = 2;
  d.A[0] = A; d.lda[0] = K; d.K[0] = K; d.B[0] = B; d.ldb[0] = N;
  d.A[1] = A2; d.lda[1] = 2; d.K[1] = 2; d.B[1] = B2; d.ldb[1] = N;
  GemmDesc *dd;
  cudaMalloc(&dd, sizeof(GemmDesc) * 4);
  cudaMemcpy(dd, &d, sizeof(d), cudaMemcpyHostToDevice);
  GemmDesc dk = d;  // K = 16: launch + epilogue with a minimal main loop
  dk.K[0] = 16;
  cudaMemcpy(dd + 1, &dk, sizeof(d), cudaMemcpyHostToDevice);
  FOp op = {};
  op.T = 1; op.N = 2; op.coef[0] = 1.0; op.expo[0] = 1; op.expo[1] = 1; op.monomial_all_ones = 1;
  FOp op1 = op; op1.N = 1;
  unsigned long long *sb; int *nf;
  cudaMalloc(&sb, 8); cudaMalloc(&nf, 4);
  set_attr<CfgPi, 1, 1, EPI_F>();
  set_attr<CfgPi, 1, 0, EPI_F>();
  set_attr<CfgPi, 1, 0, EPI_STORE>();
  set_attr<CfgV, 1, 1, EPI_F>();
  set_attr<CfgV32, 1, 1, EPI_F>();
  set_attr<CfgV4, 1, 1, EPI_F>();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char *name, auto fn, double flops) {
    float best = 1e9, ms;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      for (int i = 0; i < 20; ++i) fn();
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      best = ms / 20 < best ? ms / 20 : best;
    }
    printf("%-48s %7.2f us %6.2f TF/s | %s\n", name, best * 1e3, flops / best / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  const double f = 2.0 * M * N * K;
  timeit("Pi: EPI_F, K=256 + rank-2 input (product path)", [&] { launch<CfgPi, 1, 1, EPI_F>(dd, 1, M, N, op, sb, nf, 0); }, f);
  timeit("VEC 16B bk16 s3: EPI_F + rank-2 input", [&] { launch<CfgV, 1, 1, EPI_F>(dd, 1, M, N, op, sb, nf, 0); }, f);
  timeit("VEC 16B bk32 s2: EPI_F + rank-2 input", [&] { launch<CfgV32, 1, 1, EPI_F>(dd, 1, M, N, op, sb, nf, 0); }, f);
  timeit("VEC 16B bk16 s4: EPI_F + rank-2 input", [&] { launch<CfgV4, 1, 1, EPI_F>(dd, 1, M, N, op, sb, nf, 0); }, f);
  timeit("EPI_F, K=256, no small input", [&] { launch<CfgPi, 1, 0, EPI_F>(dd, 1, M, N, op1, sb, nf, 0); }, f);
  timeit("EPI_STORE, K=256", [&] { launch<CfgPi, 1, 0, EPI_STORE>(dd, 1, M, N, op1, sb, nf, 0); }, f);
  timeit("EPI_F + rank-2 input, K=16 (launch + epilogue)", [&] { launch<CfgPi, 1, 1, EPI_F>(dd + 1, 1, M, N, op, sb, nf, 0); }, f / 16);
  timeit("EPI_STORE, K=16", [&] { launch<CfgPi, 1, 0, EPI_STORE>(dd + 1, 1, M, N, op1, sb, nf, 0); }, f / 16);
  // the VEC result equals the k-permuted kernel's bit for bit (same per-thread k order)
  std::vector<double> r0(M * N), r1(M * N);
  std::vector<double> hr(M * K);
  for (int i = 0; i < M * K; ++i) hr[i] = ((i * 2654435761u) % 1000) * 1e-3 - 0.5;
  cudaMemcpy(A, hr.data(), 8 * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hr.data(), 8 * K * N, cudaMemcpyHostToDevice);
  launch<CfgPi, 1, 1, EPI_F>(dd, 1, M, N, op, sb, nf, 0);
  cudaMemcpy(r0.data(), C, 8 * M * N, cudaMemcpyDeviceToHost);
  launch<CfgV, 1, 1, EPI_F>(dd, 1, M, N, op, sb, nf, 0);
  cudaMemcpy(r1.data(), C, 8 * M * N, cudaMemcpyDeviceToHost);
  size_t diff = 0;
  for (int i = 0; i < M * N; ++i) diff += r0[i] != r1[i];
  printf("VEC vs k-permuted: %zu differing entries of %d\n", diff, M * N);
  return 0;
}
