// Standalone DMMA GEMM microbenchmark (development tool): the a3+f shape of configs[3] chi=256
// (1024 x 1024, K = 256 and K = 2, f = product) and the a1 shape (512 x 512, K = 256).
#include "../paper_2604_00037_b200/csrc/gemm.cu"
#include <cstdio>
#include <vector>
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
  GemmDesc *dd; cudaMalloc(&dd, sizeof(GemmDesc) * 2);
  cudaMemcpy(dd, &d, sizeof(d), cudaMemcpyHostToDevice);
  GemmDesc d1 = {};
  d1.C = C; d1.M = 512; d1.N = 512; d1.ldc = 512; d1.nin = 1;
  d1.A[0] = A; d1.lda[0] = K; d1.K[0] = K; d1.B[0] = B; d1.ldb[0] = 512;
  cudaMemcpy(dd + 1, &d1, sizeof(d1), cudaMemcpyHostToDevice);
  FOp op = {};
  op.T = 1; op.N = 2; op.coef[0] = 1.0; op.expo[0] = 1; op.expo[1] = 1;
  unsigned long long *sb; int *nf;
  cudaMalloc(&sb, 8); cudaMalloc(&nf, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch_gemm(dd, 1, M, N, 2, true, op, sb, nf, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * M * N * (K + 2);
    printf("pi  1024x1024 K=256+2: %.2f us  %.2f TF/s\n", ms * 1e3 / 20, fl * 20 / ms / 1e9);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch_gemm(dd + 1, 1, 512, 512, 1, false, op, sb, nf, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 512 * 512 * K;
    printf("a1  512x512 K=256:     %.2f us  %.2f TF/s\n", ms * 1e3 / 20, fl * 20 / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
