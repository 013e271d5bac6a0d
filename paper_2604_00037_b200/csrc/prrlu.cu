// prrLU with full pivoting (Alg. 2) — the latency-critical step a5 of the 2-site
// update. Readings: R1 (relative threshold), R2 (stop rule, eps = first rejected candidate),
// R3 (ties -> smallest (row, col)), R4 (l_i = S_iq/S_pq, S_ij <- fma(-l_i, S_pj, S_ij)), R17.
//
// Design: the Schur complement lives in REGISTERS for the whole factorisation.
// Each thread owns an EA x EB register tile (rows tr + a*TR, columns c0 + tc + b*TC). Per pivot:
// local argmax -> block argmax (shuffles + smem) -> [grid tier: one inter-CTA exchange] ->
// pivot column (l) and pivot row (u) to smem -> rank-1 update in registers.
//   * CTA tier (GRID = false): one CTA holds the whole matrix (<= 128 x 128); per pivot cost is
//     three __syncthreads.
//   * grid tier (GRID = true): G co-resident CTAs (cooperative launch), column-partitioned. Each
//     CTA publishes its candidate (value, index) AND its candidate's column to global memory
//     before the exchange, so after ONE counter barrier every CTA can read the winner's column
//     directly: one global synchronisation per pivot.
// Eliminated rows/columns are kept as exact zeros (the oracle skips them; for every active
// entry the arithmetic is identical, so identical Pi gives bit-identical pivots).
#include <cooperative_groups.h>

#include "aci_common.cuh"

namespace {

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned *p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// candidate ordering (R3): larger |v| wins; on equal |v| the smaller flat index (row*n + col) wins
__device__ __forceinline__ bool better(double a, int ia, double b, int ib) {
  return a > b || (a == b && ia < ib);
}

template <int TR, int TC, int EA, int EB, bool GRID>
__global__ void __launch_bounds__(TR *TC) prrlu_kernel(LuArgs A) {
  constexpr int T = TR * TC;
  constexpr int NW = T / 32;
  constexpr int MROWS = TR * EA;
  constexpr int CB = TC * EB;  // columns per CTA
  __shared__ double s_l[MROWS];
  __shared__ double s_u[CB];
  __shared__ double s_wv[NW], s_wa[NW];
  __shared__ int s_wi[NW];
  __shared__ double s_cval;
  __shared__ int s_cidx;

  const int tid = threadIdx.x;
  const int tr = tid / TC, tc = tid % TC;
  const int lane = tid & 31, wid = tid >> 5;
  const int G = GRID ? gridDim.x : 1;
  const int g = GRID ? blockIdx.x : 0;
  const int c0 = g * CB;

  const int m = A.dims->m, n = A.dims->n, ldm = A.dims->ldm, kmax = A.dims->kmax, ldu = A.dims->ldu;
  const int mn = m < n ? m : n;
  double thr = A.tol;
  if (A.thr_mode == 0) thr = A.tol * __longlong_as_double((long long)*A.scale_bits);

  // ---- load the register tile; padding = 0 and excluded from the argmax
  double v[EA][EB];
  unsigned rowok = 0, colok = 0;
#pragma unroll
  for (int a = 0; a < EA; ++a)
    if (tr + a * TR < m) rowok |= 1u << a;
#pragma unroll
  for (int b = 0; b < EB; ++b)
    if (c0 + tc + b * TC < n) colok |= 1u << b;
#pragma unroll
  for (int a = 0; a < EA; ++a)
#pragma unroll
    for (int b = 0; b < EB; ++b) {
      const int i = tr + a * TR, j = c0 + tc + b * TC;
      v[a][b] = ((rowok >> a) & 1) && ((colok >> b) & 1) ? A.M[(size_t)i * ldm + j] : 0.0;
    }
  for (int i = tid; i < MROWS; i += T) s_l[i] = 0.0;
  for (int j = tid; j < CB; j += T) s_u[j] = 0.0;

  double first = 0.0, eps = 0.0;
  int k = 0;
  for (;;) {
    if (k == mn) { eps = 0.0; break; }
    // ---- local argmax over the register tile
    double ba = -1.0, bv = 0.0;
    int bi = 0x7fffffff;
#pragma unroll
    for (int a = 0; a < EA; ++a)
#pragma unroll
      for (int b = 0; b < EB; ++b) {
        if (((rowok >> a) & 1) && ((colok >> b) & 1)) {
          const double x = fabs(v[a][b]);
          const int idx = (tr + a * TR) * n + (c0 + tc + b * TC);
          if (better(x, idx, ba, bi)) { ba = x; bi = idx; bv = v[a][b]; }
        }
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double oa = __shfl_xor_sync(0xffffffffu, ba, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      if (better(oa, oi, ba, bi)) { ba = oa; bi = oi; bv = ov; }
    }
    if (lane == 0) { s_wa[wid] = ba; s_wi[wid] = bi; s_wv[wid] = bv; }
    __syncthreads();
    if (wid == 0) {
      ba = lane < NW ? s_wa[lane] : -1.0;
      bi = lane < NW ? s_wi[lane] : 0x7fffffff;
      bv = lane < NW ? s_wv[lane] : 0.0;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double oa = __shfl_xor_sync(0xffffffffu, ba, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        if (better(oa, oi, ba, bi)) { ba = oa; bi = oi; bv = ov; }
      }
      if (lane == 0) { s_cval = ba < 0 ? -1.0 : bv; s_cidx = ba < 0 ? -1 : bi; }
    }
    __syncthreads();

    if (GRID) {
      // ---- publish this CTA's candidate and its column, then one counter barrier
      const int par = k & 1;
      const int cidx = s_cidx;
      if (cidx >= 0) {
        const int jc = cidx % n - c0;  // local column of the candidate
        if ((jc % TC) == tc) {
          const int bc = jc / TC;
          double *dst = A.colpub + ((size_t)par * G + g) * A.colcap;
#pragma unroll
          for (int a = 0; a < EA; ++a)
#pragma unroll
            for (int b = 0; b < EB; ++b)
              if (b == bc && ((rowok >> a) & 1)) __stcg(dst + tr + a * TR, v[a][b]);
        }
      }
      if (tid == 0) {
        __stcg(A.keyval + par * G + g, s_cval);
        __stcg(A.keyidx + par * G + g, cidx);
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        red_release_add(A.counter, 1u);
        const unsigned target = (unsigned)(k + 1) * (unsigned)G;
        while (ld_acquire_u32(A.counter) < target) {
        }
      }
      __syncthreads();
      // ---- every CTA reduces all G keys (deterministic, no atomics on the values)
      if (tid < ((G + 31) & ~31)) {
        double xa = -1.0, xv = 0.0;
        int xi = 0x7fffffff;
        if (tid < G) {
          const double val = __ldcg(A.keyval + par * G + tid);
          const int idx = __ldcg(A.keyidx + par * G + tid);
          if (idx >= 0) { xa = fabs(val); xi = idx; xv = val; }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const double oa = __shfl_xor_sync(0xffffffffu, xa, o);
          const int oi = __shfl_xor_sync(0xffffffffu, xi, o);
          const double ov = __shfl_xor_sync(0xffffffffu, xv, o);
          if (better(oa, oi, xa, xi)) { xa = oa; xi = oi; xv = ov; }
        }
        if (lane == 0) { s_wa[wid] = xa; s_wi[wid] = xi; s_wv[wid] = xv; }
      }
      __syncthreads();
      if (tid == 0) {
        double xa = s_wa[0], xv = s_wv[0];
        int xi = s_wi[0];
        for (int w = 1; w < (G + 31) / 32; ++w)
          if (better(s_wa[w], s_wi[w], xa, xi)) { xa = s_wa[w]; xi = s_wi[w]; xv = s_wv[w]; }
        s_cval = xv;
        s_cidx = xi;
      }
      __syncthreads();
    }

    // ---- stop rule (R2), uniform across the grid
    const double c = s_cval;
    const int cidx = s_cidx;
    const double absc = fabs(c);
    if (k == 0) {
      first = absc;
      if (A.thr_mode == 1) thr = A.tol * first;
    }
    if (k == kmax) { eps = absc; break; }
    if (k > 0 && absc <= thr) { eps = absc; break; }
    const int p = cidx / n, q = cidx % n;
    if (g == 0 && tid == 0) { A.rows[k] = p; A.cols[k] = q; }
    if (k == 0 && c == 0.0) {
      // R17: zero block -> rank 1, dummy pivot (0,0), U row e_q, eps 0
      if (A.U)
        for (int j = c0 + tid; j < c0 + CB && j < n; j += T) A.U[(size_t)k * ldu + j] = (j == q) ? 1.0 : 0.0;
      eps = 0.0;
      k = 1;
      break;
    }

    // ---- pivot column l_i = S_iq / c (R4) and pivot row u_j = S_pj to shared memory
    if (GRID) {
      const double *src = A.colpub + ((size_t)(k & 1) * G + q / CB) * A.colcap;
      for (int i = tid; i < m; i += T) s_l[i] = __ldcg(src + i) / c;
    } else {
      const int jc = q - c0;
      if ((jc % TC) == tc) {
        const int bc = jc / TC;
#pragma unroll
        for (int a = 0; a < EA; ++a)
#pragma unroll
          for (int b = 0; b < EB; ++b)
            if (b == bc && ((rowok >> a) & 1)) s_l[tr + a * TR] = v[a][b] / c;
      }
    }
    if ((p % TR) == tr) {
      const int ap = p / TR;
#pragma unroll
      for (int a = 0; a < EA; ++a)
        if (a == ap)
#pragma unroll
          for (int b = 0; b < EB; ++b) s_u[tc + b * TC] = v[a][b];
    }
    __syncthreads();
    if (A.U)
      for (int jj = tid; jj < CB; jj += T) {
        const int j = c0 + jj;
        if (j < n) A.U[(size_t)k * ldu + j] = s_u[jj] / c;
      }
    // ---- rank-1 Schur update in registers; row p and column q become exact zeros
#pragma unroll
    for (int a = 0; a < EA; ++a) {
      const int i = tr + a * TR;
      const double li = s_l[i];
#pragma unroll
      for (int b = 0; b < EB; ++b) {
        const int j = c0 + tc + b * TC;
        double x = fma(-li, s_u[tc + b * TC], v[a][b]);
        if (i == p || j == q) x = 0.0;
        v[a][b] = x;
      }
    }
    ++k;
    __syncthreads();  // s_l / s_u / s_w* reuse
  }
  if (g == 0 && tid == 0) {
    *A.r_out = k;
    *A.eps_out = eps;
  }
}

struct Tier {
  int tr, tc, ea, eb;
  bool grid;
};

// CTA tiers (one block) and grid tiers (cooperative), smallest first.
template <int TR, int TC, int EA, int EB, bool GRID>
void launch_one(const LuArgs &a, int max_n, cudaStream_t st) {
  auto kern = prrlu_kernel<TR, TC, EA, EB, GRID>;
  if (!GRID) {
    kern<<<1, TR * TC, 0, st>>>(a);
    return;
  }
  int G = (max_n + TC * EB - 1) / (TC * EB);
  if (G < 1) G = 1;
  LuArgs args = a;
  void *params[] = {&args};
  cudaLaunchCooperativeKernel((const void *)kern, dim3(G), dim3(TR * TC), params, 0, st);
}

constexpr int kGridRowsSmall = 256, kGridRowsLarge = 1024;
constexpr int kGridColsSmall = 16, kGridColsLarge = 8;  // columns per CTA
constexpr int kMaxCTAs = 148;

}  // namespace

bool prrlu_supported(int max_m, int max_n) {
  if (max_m <= 128 && max_n <= 128) return true;
  if (max_m <= kGridRowsSmall) return (max_n + kGridColsSmall - 1) / kGridColsSmall <= kMaxCTAs;
  if (max_m <= kGridRowsLarge) return (max_n + kGridColsLarge - 1) / kGridColsLarge <= kMaxCTAs;
  return false;
}

void prrlu_envelope(int *max_rows, int *max_cols) {
  *max_rows = kGridRowsLarge;
  *max_cols = kMaxCTAs * kGridColsLarge;
}

size_t prrlu_exchange_bytes(int max_m, int max_n) {
  int G = kMaxCTAs;
  (void)max_n;
  int cap = max_m < 1024 ? 1024 : max_m;
  return (size_t)2 * G * cap * sizeof(double) + 2 * G * (sizeof(double) + sizeof(int)) + 256;
}

void launch_prrlu(const LuArgs &a, int max_m, int max_n, cudaStream_t st) {
  if (max_m <= 32 && max_n <= 32) return launch_one<8, 16, 4, 2, false>(a, max_n, st);
  if (max_m <= 64 && max_n <= 64) return launch_one<16, 16, 4, 4, false>(a, max_n, st);
  if (max_m <= 128 && max_n <= 128) return launch_one<16, 32, 8, 4, false>(a, max_n, st);
  cudaMemsetAsync(a.counter, 0, sizeof(unsigned), st);
  if (max_m <= kGridRowsSmall) return launch_one<32, 16, 8, 1, true>(a, max_n, st);
  return launch_one<64, 8, 16, 1, true>(a, max_n, st);
}
