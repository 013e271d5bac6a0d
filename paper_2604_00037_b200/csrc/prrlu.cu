// prrLU with full pivoting (Alg. 2) — the latency-critical step a5 of the 2-site
// update. Readings: R1 (relative threshold), R2 (stop rule, eps = first rejected candidate),
// R3 (ties -> smallest (row, col)), R4 (l_i = S_iq * [S_pq]^{-1} — P:535 multiplies by the
// inverse pivot, so one IEEE reciprocal per pivot —, S_ij <- fma(-l_i, S_pj, S_ij)), R17.
//
// Design. The Schur complement lives in REGISTERS for the whole factorisation.
// Rows run across the 32 lanes of a warp and columns across warps: thread (lane, w) holds
// S[lane + 32 a][c0 + w + NW b] for a < EA, b < EB. So one warp owns whole columns, which
// makes the pivot-column publication a coalesced single-warp store and lets that warp do the
// release itself. Per pivot:
//   rank-1 update, then a branch-free running (value, slot) max per thread
//   -> warp argmax: 3 x redux.sync on the exact key (|v| bits hi, lo; flat index)
//   -> CTA argmax: per-warp keys in smem, every warp reduces them itself
//   -> [grid tier: the owner warp of the CTA candidate publishes key + column, arrives on a
//       counter (red.release); one poll; every warp reduces the G published keys itself]
//   -> pivot column l = S_iq * (1/c) (R4) and pivot row u through smem.
// The pivot's sign comes from the (published) pivot column, so keys carry only |v|.
// Row p is zeroed exactly by l_p = 1 (fma(-1, u_j, u_j) = 0); column q by the owner warp.
// Eliminated entries are exact zeros: for every active entry the arithmetic equals the
// oracle's, so identical Pi gives bit-identical pivots.
//   * CTA tier (GRID = false): one CTA (up to 32 register entries per thread), three
//     __syncthreads per pivot.
//   * grid tier (GRID = true): G co-resident CTAs (cooperative launch), column-partitioned.
// The tier is chosen per launch on the device from the live block size (prrlu_kernel).
#include "aci_common.cuh"

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr unsigned BAD_ID = 0xffffffffu;

// Development instrumentation (tools/prrlu_bench.cu defines ACI_PRRLU_TIMING): cycles per phase
// of one pivot step, accumulated by thread 0 of CTA 0 into LuArgs::dbg[0..7].
#ifdef ACI_PRRLU_TIMING
#define PHASE(n)                        \
  do {                                  \
    if (tid == 0 && g == 0) {           \
      long long now_ = clock64();       \
      ph_[n] += now_ - ph_t_;           \
      ph_t_ = now_;                     \
    }                                   \
  } while (0)
#else
#define PHASE(n) \
  do {           \
  } while (0)
#endif

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned *p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct Key {
  unsigned hi, lo, id;  // |v| bits (hi, lo); id = flat index (row * n + col)
};

__device__ __forceinline__ bool better(const Key &a, const Key &b) {
  if (a.hi != b.hi) return a.hi > b.hi;
  if (a.lo != b.lo) return a.lo > b.lo;
  return a.id < b.id;
}

__device__ __forceinline__ Key warp_argmax(const Key &k) {
  const unsigned mh = __reduce_max_sync(FULL, k.hi);
  const unsigned ml = __reduce_max_sync(FULL, k.hi == mh ? k.lo : 0u);
  const unsigned mi = __reduce_min_sync(FULL, (k.hi == mh && k.lo == ml) ? k.id : BAD_ID);
  return Key{mh, ml, mi};
}

__device__ __forceinline__ double key_abs(const Key &k) {
  return __longlong_as_double((long long)(((unsigned long long)k.hi << 32) | k.lo));
}

constexpr int kNW = 16;          // warps per CTA (512 threads) for every variant
constexpr int kMaxRows = 1024;   // 32 * EA_max
constexpr int kMaxCB = 512;      // NW * EB_max

struct PrrluSmem {
  double l[kMaxRows];    // l_i (R4), l[p] = 1
  double raw[kMaxRows];  // CTA tier: raw pivot column
  double u[kMaxCB];      // pivot row segment
  unsigned hi[32], lo[32], id[32];
};

// One factorisation, register tile EA x EB per thread, NW warps per CTA. GRID: G CTAs (this is
// CTA g) cooperate through the exchange buffers; otherwise one CTA does everything.
template <int EA, int EB, int NW, bool GRID>
__device__ __forceinline__ void prrlu_body(const LuArgs &A, PrrluSmem &S, const int G, const int g) {
  constexpr int T = NW * 32;
  constexpr int MROWS = 32 * EA;
  constexpr int CB = NW * EB;  // columns per CTA
  static_assert(MROWS <= kMaxRows && CB <= kMaxCB, "tile exceeds the shared scratch");
  double *s_l = S.l, *s_raw = S.raw, *s_u = S.u;
  unsigned *s_hi = S.hi, *s_lo = S.lo, *s_id = S.id;
  const int tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const int c0 = g * CB;

  const int m = A.dims->m, n = A.dims->n, ldm = A.dims->ldm, kmax = A.dims->kmax, ldu = A.dims->ldu;
  const int mn = m < n ? m : n;
  double thr = A.tol;
  if (A.thr_mode == 0) thr = A.tol * __longlong_as_double((long long)*A.scale_bits);

  // ---- load; padding = 0 and never a candidate
  double v[EA][EB];
  bool rok[EA], cok[EB];
#pragma unroll
  for (int a = 0; a < EA; ++a) rok[a] = lane + 32 * a < m;
#pragma unroll
  for (int b = 0; b < EB; ++b) cok[b] = c0 + w + NW * b < n;
#pragma unroll
  for (int a = 0; a < EA; ++a)
#pragma unroll
    for (int b = 0; b < EB; ++b)
      v[a][b] = (rok[a] && cok[b]) ? A.M[(size_t)(lane + 32 * a) * ldm + c0 + w + NW * b] : 0.0;
  for (int i = tid; i < MROWS; i += T) s_l[i] = 0.0;
  for (int j = tid; j < CB; j += T) s_u[j] = 0.0;

  // Flat candidate index = row * NC + col with the PADDED width NC (>= every column of the
  // grid), so padding entries (always exact zeros) never alias a real index and never need a
  // mask: a zero can only win when every active entry is zero, and then the factorisation stops
  // (R2) — except at k = 0, where (0, 0) (a real entry) wins the R3 tie-break.
  const unsigned NC = (unsigned)(G * CB);
  // per-thread max over the register tile: NCH independent chains (slot e -> chain e % NCH),
  // strict '>' within a chain; chains merged with the slot (== flat-index) tie-break.
  double bx = 0.0;
  int be = 0;
  auto scan = [&]() {
    constexpr int NE = EA * EB;
    constexpr int NCH = NE < 4 ? NE : 4;
    double cx[NCH];
    int ce[NCH];
#pragma unroll
    for (int t = 0; t < NCH; ++t) { cx[t] = fabs(v[t / EB][t % EB]); ce[t] = t; }
#pragma unroll
    for (int e = NCH; e < NE; ++e) {
      const double ax = fabs(v[e / EB][e % EB]);
      const bool take = ax > cx[e % NCH];
      cx[e % NCH] = take ? ax : cx[e % NCH];
      ce[e % NCH] = take ? e : ce[e % NCH];
    }
    double bm = cx[0];
    int bi = ce[0];
#pragma unroll
    for (int t = 1; t < NCH; ++t) {
      const bool take = cx[t] > bm || (cx[t] == bm && ce[t] < bi);
      bm = take ? cx[t] : bm;
      bi = take ? ce[t] : bi;
    }
    bx = bm;
    be = bi;
  };
  auto thread_key = [&]() -> Key {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(bx);
    const int a = be / EB, b = be % EB;
    const unsigned flat = (unsigned)(lane + 32 * a) * NC + (unsigned)(c0 + w + NW * b);
    return Key{(unsigned)(bits >> 32), (unsigned)bits, flat};
  };
  scan();

  double first = 0.0, eps = 0.0;
  int k = 0;
#ifdef ACI_PRRLU_TIMING
  long long ph_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long ph_t_ = clock64();
#endif
  for (;;) {
    if (k == mn) { eps = 0.0; break; }
    // ---- warp -> CTA argmax
    const Key wk = warp_argmax(thread_key());
    if (lane == 0) { s_hi[w] = wk.hi; s_lo[w] = wk.lo; s_id[w] = wk.id; }
    __syncthreads();  // S1
    PHASE(0);
    const Key ck = warp_argmax(lane < NW ? Key{s_hi[lane], s_lo[lane], s_id[lane]} : Key{0u, 0u, BAD_ID});
    Key win = ck;
    PHASE(1);
    if (GRID) {
      const int par = k & 1;
      // the owner warp of the CTA candidate's column publishes column + key and arrives
      const int jc = (int)(ck.id % NC) - c0;
      const int pw = jc % NW;  // the warp that arrives for this CTA
      if (w == pw) {
        {
          const int bc = jc / NW;
          double *dst = A.colpub + ((size_t)par * G + g) * A.colcap;
#pragma unroll
          for (int b = 0; b < EB; ++b)
            if (b == bc)
#pragma unroll
              for (int a = 0; a < EA; ++a)
                if (rok[a]) __stcg(dst + lane + 32 * a, v[a][b]);
        }
        __syncwarp();
        if (lane == 0) {
          __stcg(reinterpret_cast<uint4 *>(A.keys) + par * G + g, make_uint4(ck.hi, ck.lo, ck.id, 0u));
          red_release_add(A.counter, 1u);
          const unsigned target = (unsigned)(k + 1) * (unsigned)G;
          while (ld_acquire_u32(A.counter) < target) {
          }
        }
      }
      PHASE(2);
      __syncthreads();  // S2: counter passed
      PHASE(3);
      Key gk{0u, 0u, BAD_ID};
      const uint4 *keys = reinterpret_cast<const uint4 *>(A.keys) + par * G;
      for (int t = lane; t < G; t += 32) {
        const uint4 qk = __ldcg(keys + t);
        const Key kq{qk.x, qk.y, qk.z};
        if (better(kq, gk)) gk = kq;
      }
      win = warp_argmax(gk);
      PHASE(4);
    }

    // ---- stop rule (R2), uniform across the grid
    const double absc = key_abs(win);
    if (k == 0) {
      first = absc;
      if (A.thr_mode == 1) thr = A.tol * first;
    }
    if (k == kmax) { eps = absc; break; }
    if (k > 0 && absc <= thr) { eps = absc; break; }
    const int p = (int)(win.id / NC), q = (int)(win.id % NC);
    if (g == 0 && tid == 0) { A.rows[k] = p; A.cols[k] = q; }
    if (k == 0 && absc == 0.0) {
      // R17: zero block -> rank 1, dummy pivot (0,0), U row e_q, eps 0
      if (A.U)
        for (int j = c0 + tid; j < c0 + CB && j < n; j += T) A.U[(size_t)k * ldu + j] = (j == q) ? 1.0 : 0.0;
      eps = 0.0;
      k = 1;
      break;
    }

    // ---- pivot row u_j = S_pj (lane p%32 of every warp) and pivot column l_i = S_iq / S_pq
    const int ap = p >> 5, lp = p & 31;
    if (lane == lp) {
#pragma unroll
      for (int a = 0; a < EA; ++a)
        if (a == ap)
#pragma unroll
          for (int b = 0; b < EB; ++b) s_u[w + NW * b] = v[a][b];
    }
    double inv;
    if (GRID) {
      const double *src = A.colpub + ((size_t)(k & 1) * G + q / CB) * A.colcap;
      inv = 1.0 / __ldcg(src + p);
#pragma unroll 4
      for (int i = tid; i < m; i += T) s_l[i] = (i == p) ? 1.0 : __ldcg(src + i) * inv;
    } else {
      const int jq = q - c0;
      if ((jq % NW) == w) {
        const int bq = jq / NW;
#pragma unroll
        for (int b = 0; b < EB; ++b)
          if (b == bq)
#pragma unroll
            for (int a = 0; a < EA; ++a) s_raw[lane + 32 * a] = v[a][b];
      }
      __syncthreads();  // S2 (CTA tier)
      inv = 1.0 / s_raw[p];
      for (int i = tid; i < m; i += T) s_l[i] = (i == p) ? 1.0 : s_raw[i] * inv;
    }
    __syncthreads();  // S3
    PHASE(5);
    if (A.U)
      for (int jj = tid; jj < CB; jj += T) {
        const int j = c0 + jj;
        if (j < n) A.U[(size_t)k * ldu + j] = (j == q) ? 1.0 : s_u[jj] * inv;
      }
    // ---- rank-1 Schur update in registers
    double ub[EB];
#pragma unroll
    for (int b = 0; b < EB; ++b) ub[b] = s_u[w + NW * b];
#pragma unroll
    for (int a = 0; a < EA; ++a) {
      const double li = s_l[lane + 32 * a];
#pragma unroll
      for (int b = 0; b < EB; ++b) v[a][b] = fma(-li, ub[b], v[a][b]);
    }
    // column q -> exact zeros (owner warp; warp-uniform branch)
    {
      const int jq = q - c0;
      if (jq >= 0 && jq < CB && (jq % NW) == w) {
        const int bq = jq / NW;
#pragma unroll
        for (int b = 0; b < EB; ++b)
          if (b == bq)
#pragma unroll
            for (int a = 0; a < EA; ++a) v[a][b] = 0.0;
      }
    }
    scan();
    PHASE(6);
    ++k;
    // s_l / s_u / s_raw are rewritten only after the next S1; every thread finished reading
    // them before arriving there.
  }
  if (g == 0 && tid == 0) {
    *A.r_out = k;
    *A.eps_out = eps;
#ifdef ACI_PRRLU_TIMING
    for (int t = 0; t < 8; ++t) A.dbg[t] = ph_[t];
#endif
  }
}

// Runtime tier selection from the LIVE sizes (device-resident ranks): the launch is sized for
// the static capacity, and CTAs beyond what the live block needs exit immediately.
__global__ void __launch_bounds__(kNW * 32) prrlu_kernel(LuArgs A) {
  __shared__ PrrluSmem S;
  const int m = A.dims->m, n = A.dims->n;
  const int g = blockIdx.x;
#define ACI_CTA_VARIANT(EA, EB)                                        \
  if (m <= 32 * (EA) && n <= kNW * (EB)) {                              \
    if (g == 0) prrlu_body<(EA), (EB), kNW, false>(A, S, 1, 0);        \
    return;                                                            \
  }
#define ACI_GRID_VARIANT(EA)                                           \
  if (m <= 32 * (EA)) {                                                \
    const int Gl = (n + kNW - 1) / kNW;                                \
    if (g < Gl) prrlu_body<(EA), 1, kNW, true>(A, S, Gl, g);           \
    return;                                                            \
  }
  ACI_CTA_VARIANT(1, 2)    //   32 x   32
  ACI_CTA_VARIANT(2, 4)    //   64 x   64
  ACI_CTA_VARIANT(4, 2)    //  128 x   32
  ACI_CTA_VARIANT(1, 8)    //   32 x  128
  ACI_CTA_VARIANT(4, 8)    //  128 x  128
  ACI_CTA_VARIANT(2, 16)   //   64 x  256
  ACI_CTA_VARIANT(8, 4)    //  256 x   64
  ACI_CTA_VARIANT(1, 32)   //   32 x  512
  ACI_CTA_VARIANT(16, 2)   //  512 x   32
  ACI_GRID_VARIANT(4)      //  128 x 16 per CTA
  ACI_GRID_VARIANT(8)      //  256 x 16 per CTA
  ACI_GRID_VARIANT(16)     //  512 x 16 per CTA
  ACI_GRID_VARIANT(32)     // 1024 x 16 per CTA
#undef ACI_CTA_VARIANT
#undef ACI_GRID_VARIANT
}

constexpr int kMaxCTAs = 148;

bool fits_one_cta(int m, int n) {
  const int v[][2] = {{1, 2}, {2, 4}, {4, 2}, {1, 8}, {4, 8}, {2, 16}, {8, 4}, {1, 32}, {16, 2}};
  for (auto &e : v)
    if (m <= 32 * e[0] && n <= kNW * e[1]) return true;
  return false;
}

}  // namespace

bool prrlu_supported(int max_m, int max_n) {
  if (fits_one_cta(max_m, max_n)) return true;
  return max_m <= kMaxRows && (max_n + kNW - 1) / kNW <= kMaxCTAs;
}

void prrlu_envelope(int *max_rows, int *max_cols) {
  *max_rows = kMaxRows;
  *max_cols = kMaxCTAs * kNW;
}

size_t prrlu_exchange_bytes(int max_m, int max_n) {
  (void)max_n;
  int cap = max_m < kMaxRows ? kMaxRows : max_m;
  return (size_t)2 * kMaxCTAs * cap * sizeof(double) + 2 * kMaxCTAs * 16 + 256;
}

void launch_prrlu(const LuArgs &a, int max_m, int max_n, cudaStream_t st) {
  if (fits_one_cta(max_m, max_n)) {
    prrlu_kernel<<<1, kNW * 32, 0, st>>>(a);
    return;
  }
  cudaMemsetAsync(a.counter, 0, sizeof(unsigned), st);
  int G = (max_n + kNW - 1) / kNW;
  LuArgs args = a;
  void *params[] = {&args};
  cudaLaunchCooperativeKernel((const void *)prrlu_kernel, dim3(G), dim3(kNW * 32), params, 0, st);
}
