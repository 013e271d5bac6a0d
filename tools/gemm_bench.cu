// Tile-shape sweep for the DMMA GEMM templates (development tool): the a3+f shape of configs[3]
// chi=256 (1024 x 1024, K = 256 plus a K = 2 input, f = product) and the a1 shape (512 x 512).
#include "../paper_2604_00037_b200/csrc/gemm_kernel.cuh"
#include <cstdio>
#include <vector>
using namespace gemmk;

static GemmDesc *dd;
static FOp op;
static unsigned long long *sb;
static int *nf;

template <class CF>
void run(const char *name) {
  set_attr<CF, 1, 1, EPI_F>();
  set_attr<CF, 1, 0, EPI_STORE>();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms, best_pi = 1e9, best_a1 = 1e9;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch<CF, 1, 1, EPI_F>(dd, 1, 1024, 1024, op, sb, nf, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    best_pi = ms / 20 < best_pi ? ms / 20 : best_pi;
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch<CF, 1, 0, EPI_STORE>(dd + 1, 1, 512, 512, op, sb, nf, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    best_a1 = ms / 20 < best_a1 ? ms / 20 : best_a1;
  }
  double fpi = 2.0 * 1024 * 1024 * 256, fa1 = 2.0 * 512 * 512 * 256;
  printf("%-34s pi %7.2f us %6.2f TF/s | a1 %7.2f us %6.2f TF/s | %s\n", name, best_pi * 1e3, fpi / best_pi / 1e9,
         best_a1 * 1e3, fa1 / best_a1 / 1e9, cudaGetErrorString(cudaGetLastError()));
}

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
  cudaMalloc(&dd, sizeof(GemmDesc) * 2);
  cudaMemcpy(dd, &d, sizeof(d), cudaMemcpyHostToDevice);
  GemmDesc d1 = {};
  d1.C = C; d1.M = 512; d1.N = 512; d1.ldc = 512; d1.nin = 1;
  d1.A[0] = A; d1.lda[0] = K; d1.K[0] = K; d1.B[0] = B; d1.ldb[0] = 512;
  cudaMemcpy(dd + 1, &d1, sizeof(d1), cudaMemcpyHostToDevice);
  op.T = 1; op.N = 2; op.coef[0] = 1.0; op.expo[0] = 1; op.expo[1] = 1; op.monomial_all_ones = 1;
  cudaMalloc(&sb, 8); cudaMalloc(&nf, 4);
  //                 BM   BN  WM  WN  BK ST MINB
  run<Cfg<64, 64, 32, 16, 16, 3, 2>>("64x64 w32x16 bk16 s3 (8w) mb2");
  run<Cfg<64, 64, 32, 32, 16, 3, 2>>("64x64 w32x32 bk16 s3 (4w) mb2");
  run<Cfg<64, 64, 32, 32, 16, 3, 3>>("64x64 w32x32 bk16 s3 (4w) mb3");
  run<Cfg<64, 64, 32, 32, 16, 4, 3>>("64x64 w32x32 bk16 s4 (4w) mb3");
  run<Cfg<64, 64, 32, 32, 16, 2, 3>>("64x64 w32x32 bk16 s2 (4w) mb3");
  run<Cfg<64, 64, 32, 16, 16, 4, 2>>("64x64 w32x16 bk16 s4 (8w) mb2");
  run<Cfg<128, 64, 32, 32, 16, 3, 1>>("128x64 w32x32 bk16 s3 (8w)");
  run<Cfg<64, 32, 32, 16, 16, 3, 4>>("64x32 w32x16 bk16 s3 (4w) mb4");
  run<Cfg<32, 64, 16, 32, 16, 3, 4>>("32x64 w16x32 bk16 s3 (4w) mb4");
  run<Cfg<64, 64, 32, 32, 32, 2, 2>>("64x64 w32x32 bk32 s2 (4w) mb2");
  return 0;
}
