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
//   -> [grid tier: the owner warp of the CTA candidate publishes key + column as tagged
//       packets (each 8-byte word carries epoch|step, so no release/acquire fence is needed),
//       arrives on a counter; one poll; every warp reads the G keys with all loads in flight]
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

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_relaxed_add(unsigned *p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Counter poll with NP loads in flight, issued ~kPollGap cycles apart and checked in issue
// order: completion is seen ~one L2 latency after it lands instead of up to two, which also
// shrinks the skew between CTAs at the next pivot.
#ifndef ACI_KEYPOLL_MAXG
#define ACI_KEYPOLL_MAXG 16
#endif
#ifndef ACI_POLL_NP
#define ACI_POLL_NP 1  // measured: more loads in flight only add contention on the counter line
#endif
constexpr int kPollGap = 160;
__device__ __forceinline__ void poll_counter(const unsigned *ctr, unsigned target) {
  constexpr int NP = ACI_POLL_NP;
  unsigned v[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    v[i] = ld_relaxed_u32(ctr);
    if (NP > 1) {
      const long long t0 = clock64();
      while (clock64() - t0 < kPollGap) {
      }
    }
  }
  for (;;) {
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      if (v[i] >= target) return;
      v[i] = ld_relaxed_u32(ctr);
    }
  }
}

// 16-byte packet = two independently single-copy-atomic 8-byte words, each tagged
__device__ __forceinline__ void st_pkt(unsigned long long *p, unsigned long long w0, unsigned long long w1) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
__device__ __forceinline__ void ld_pkt(const unsigned long long *p, unsigned long long &w0, unsigned long long &w1) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
}
__device__ __forceinline__ unsigned long long tagged(unsigned tag, unsigned v) {
  return ((unsigned long long)tag << 32) | v;
}
__device__ __forceinline__ double pkt_double(unsigned long long w0, unsigned long long w1) {
  return __longlong_as_double((long long)(((w1 & 0xffffffffull) << 32) | (w0 & 0xffffffffull)));
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

// columns per warp of the 8-warp grid tiers, measured (tools/prrlu_bench.cu): 16 CTAs with the
// key-poll barrier beat more CTAs with the counter barrier up to 512 rows
#ifndef ACI_W8_EB128
#define ACI_W8_EB128 4
#endif
#ifndef ACI_W8_EB256
#define ACI_W8_EB256 2
#endif
#ifndef ACI_W8_EB512
#define ACI_W8_EB512 4
#endif
#ifndef ACI_BIG_EB
#define ACI_BIG_EB 2  // columns per warp for the 1024-row grid tier (64 CTAs for 1024 columns)
#endif
constexpr int kNW = 16;          // warps per CTA (512 threads) for every variant
constexpr int kMaxRows = 1024;   // 32 * EA_max
constexpr int kMaxCB = 512;      // NW * EB_max

struct PrrluSmem {
  double l[kMaxRows];    // l_i (R4), l[p] = 1
  double raw[kMaxRows];  // CTA tier: raw pivot column
  double u[kMaxCB];      // pivot row segment
  unsigned hi[32], lo[32], id[32];
  unsigned win[4];  // grid winner broadcast (key-poll mode)
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
  const unsigned ep = GRID ? (*A.epoch & 0xfffffu) : 0u;  // read by every CTA before any arrival
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
      const unsigned tag = (ep << 12) | (unsigned)(k + 1);
      // the owner warp of the CTA candidate's column publishes the column (tagged packets, no
      // fence) and lane 0 publishes the key and arrives on the counter
      const int jc = (int)(ck.id % NC) - c0;
      const int pw = jc % NW;
      if (w == pw) {
        const int bc = jc / NW;
        unsigned long long *dst = A.colpub + (((size_t)par * G + g) * A.colcap) * 2;
#pragma unroll
        for (int b = 0; b < EB; ++b)
          if (b == bc)
#pragma unroll
            for (int a = 0; a < EA; ++a)
              if (rok[a]) {
                const unsigned long long bits = (unsigned long long)__double_as_longlong(v[a][b]);
                st_pkt(dst + 2 * (lane + 32 * a), tagged(tag, (unsigned)bits), tagged(tag, (unsigned)(bits >> 32)));
              }
        if (lane == 0) {
          unsigned long long *kd = A.keys + ((size_t)par * G + g) * 4;
          st_pkt(kd, tagged(tag, ck.hi), tagged(tag, ck.lo));
          st_pkt(kd + 2, tagged(tag, ck.id), 0ull);
          if (G > ACI_KEYPOLL_MAXG) red_relaxed_add(A.counter, 1u);
        }
      }
      PHASE(2);
      // small grids: the tagged keys themselves are the barrier (warp 0 polls them, no counter);
      // larger grids: one counter poll then every warp reads the keys (measured crossover ~16)
      const bool keypoll = G <= ACI_KEYPOLL_MAXG;
      if (!keypoll) {
        if (tid == 0) poll_counter(A.counter, (unsigned)(k + 1) * (unsigned)G);
        __syncthreads();  // S2: every CTA has arrived
      }
      PHASE(3);
      // read all G keys: independent loads in flight, stale packets re-read until their tag is
      // this step's
      constexpr int KPL = (148 + 31) / 32;  // keys per lane
      Key gk{0u, 0u, BAD_ID};
      if (!keypoll || w == 0) {
        unsigned long long kw[KPL][4];
#pragma unroll
        for (int t = 0; t < KPL; ++t) {
          const int s_ = lane + 32 * t;
          if (s_ < G) {
            const unsigned long long *kp = A.keys + ((size_t)par * G + s_) * 4;
            ld_pkt(kp, kw[t][0], kw[t][1]);
            ld_pkt(kp + 2, kw[t][2], kw[t][3]);
          }
        }
#pragma unroll
        for (int t = 0; t < KPL; ++t) {
          const int s_ = lane + 32 * t;
          if (s_ < G) {
            const unsigned long long *kp = A.keys + ((size_t)par * G + s_) * 4;
            while ((unsigned)(kw[t][0] >> 32) != tag || (unsigned)(kw[t][1] >> 32) != tag ||
                   (unsigned)(kw[t][2] >> 32) != tag) {
              ld_pkt(kp, kw[t][0], kw[t][1]);
              ld_pkt(kp + 2, kw[t][2], kw[t][3]);
            }
            const Key kq{(unsigned)kw[t][0], (unsigned)kw[t][1], (unsigned)kw[t][2]};
            if (better(kq, gk)) gk = kq;
          }
        }
      }
      win = warp_argmax(gk);
      if (keypoll) {
        if (tid == 0) { S.win[0] = win.hi; S.win[1] = win.lo; S.win[2] = win.id; }
        __syncthreads();  // S2: the winner, known only after every CTA's key arrived
        win = Key{S.win[0], S.win[1], S.win[2]};
      }
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
      const unsigned tag = (ep << 12) | (unsigned)(k + 1);
      const unsigned long long *src = A.colpub + (((size_t)(k & 1) * G + q / CB) * A.colcap) * 2;
      constexpr int PPT = (MROWS + T - 1) / T;  // column packets per thread
      unsigned long long cw[PPT + 1][2];
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int i = tid + T * t;
        if (i < m) ld_pkt(src + 2 * i, cw[t][0], cw[t][1]);
      }
      ld_pkt(src + 2 * p, cw[PPT][0], cw[PPT][1]);
      while ((unsigned)(cw[PPT][0] >> 32) != tag || (unsigned)(cw[PPT][1] >> 32) != tag)
        ld_pkt(src + 2 * p, cw[PPT][0], cw[PPT][1]);
      inv = 1.0 / pkt_double(cw[PPT][0], cw[PPT][1]);
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int i = tid + T * t;
        if (i < m) {
          while ((unsigned)(cw[t][0] >> 32) != tag || (unsigned)(cw[t][1] >> 32) != tag)
            ld_pkt(src + 2 * i, cw[t][0], cw[t][1]);
          s_l[i] = (i == p) ? 1.0 : pkt_double(cw[t][0], cw[t][1]) * inv;
        }
      }
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
    // every CTA read the epoch before its first arrival, and CTA 0 only gets here after the
    // last exchange, so the increment cannot race with a reader of this launch
    if (GRID) atomicAdd(A.epoch, 1u);
#ifdef ACI_PRRLU_TIMING
    for (int t = 0; t < 8; ++t) A.dbg[t] = ph_[t];
#endif
  }
}

// Runtime tier selection from the LIVE sizes (device-resident ranks): the launch is sized for
// the static capacity, and CTAs beyond what the live block needs exit immediately. Two
// instantiations: 16 warps (static rows <= 512) and 8 warps (static rows <= 1024: 8 columns per
// CTA and up to 255 registers, so the 32-row-slot tiles do not spill).
template <int NWT>
__global__ void __launch_bounds__(NWT * 32) prrlu_kernel(LuArgs A) {
  __shared__ PrrluSmem S;
  const int m = A.dims->m, n = A.dims->n;
  const int g = blockIdx.x;
#define ACI_CTA_VARIANT(EA, EB)                                        \
  if (m <= 32 * (EA) && n <= NWT * (EB)) {                              \
    if (g == 0) prrlu_body<(EA), (EB), NWT, false>(A, S, 1, 0);        \
    return;                                                            \
  }
#define ACI_GRID_VARIANT(EA) ACI_GRID_VARIANT2(EA, 1)
#define ACI_GRID_VARIANT2(EA, EB)                                      \
  if (m <= 32 * (EA)) {                                                \
    const int Gl = (n + NWT * (EB) - 1) / (NWT * (EB));                \
    if (g < Gl) prrlu_body<(EA), (EB), NWT, true>(A, S, Gl, g);        \
    return;                                                            \
  }
  if (NWT == 16) {
    ACI_CTA_VARIANT(1, 2)    //   32 x   32
    ACI_CTA_VARIANT(2, 4)    //   64 x   64
    ACI_CTA_VARIANT(4, 2)    //  128 x   32
    ACI_CTA_VARIANT(1, 8)    //   32 x  128
    ACI_CTA_VARIANT(4, 8)    //  128 x  128
    ACI_CTA_VARIANT(2, 16)   //   64 x  256
    ACI_CTA_VARIANT(8, 4)    //  256 x   64
    ACI_CTA_VARIANT(1, 32)   //   32 x  512
    ACI_CTA_VARIANT(16, 2)   //  512 x   32
    ACI_GRID_VARIANT2(4, 2)  //  128 x 32 per CTA (key-poll barrier for <= 16 CTAs)
    ACI_GRID_VARIANT2(8, 2)  //  256 x 32 per CTA
    ACI_GRID_VARIANT(16)     //  512 x 16 per CTA (counter barrier)
  } else {
    ACI_CTA_VARIANT(1, 4)    //   32 x   32
    ACI_CTA_VARIANT(2, 8)    //   64 x   64
    ACI_CTA_VARIANT(4, 4)    //  128 x   32
    ACI_CTA_VARIANT(1, 16)   //   32 x  128
    ACI_CTA_VARIANT(4, 16)   //  128 x  128
    ACI_CTA_VARIANT(8, 8)    //  256 x   64
    ACI_CTA_VARIANT(2, 32)   //   64 x  256
    ACI_CTA_VARIANT(32, 2)   // 1024 x   16
    ACI_GRID_VARIANT2(4, ACI_W8_EB128)   //  128 x 8*EB per CTA
    ACI_GRID_VARIANT2(8, ACI_W8_EB256)   //  256 x 8*EB per CTA
    ACI_GRID_VARIANT2(16, ACI_W8_EB512)  //  512 x 8*EB per CTA
    ACI_GRID_VARIANT2(32, ACI_BIG_EB)  // 1024 x 8*EB per CTA
  }
#undef ACI_CTA_VARIANT
#undef ACI_GRID_VARIANT
#undef ACI_GRID_VARIANT2
}

constexpr int kMaxCTAs = 148;
constexpr int kRowsSmall = 512;  // static rows handled by the 16-warp instantiation

bool fits_one_cta(int m, int n, int nwt) {
  const int v16[][2] = {{1, 2}, {2, 4}, {4, 2}, {1, 8}, {4, 8}, {2, 16}, {8, 4}, {1, 32}, {16, 2}};
  const int v8[][2] = {{1, 4}, {2, 8}, {4, 4}, {1, 16}, {4, 16}, {8, 8}, {2, 32}, {32, 2}};
  if (nwt == 16) {
    for (auto &e : v16)
      if (m <= 32 * e[0] && n <= 16 * e[1]) return true;
  } else {
    for (auto &e : v8)
      if (m <= 32 * e[0] && n <= 8 * e[1]) return true;
  }
  return false;
}

}  // namespace

bool prrlu_supported(int max_m, int max_n) {
  return fits_one_cta(max_m, max_n, 8) || (max_m <= kMaxRows && (max_n + 7) / 8 <= kMaxCTAs);
}

void prrlu_envelope(int *max_rows, int *max_cols) {
  *max_rows = kMaxRows;
  *max_cols = kMaxCTAs * 8;
}

size_t prrlu_exchange_bytes(int max_m, int max_n) {
  (void)max_n;
  int cap = max_m < kMaxRows ? kMaxRows : max_m;
  return (size_t)2 * kMaxCTAs * cap * 16 + 2 * kMaxCTAs * 32 + 256;
}

void launch_prrlu(const LuArgs &a, int max_m, int max_n, cudaStream_t st) {
  // the 8-warp instantiation measured faster than the 16-warp one at every block size
  constexpr int nwt = 8;
  const void *kern = (const void *)prrlu_kernel<nwt>;
  if (fits_one_cta(max_m, max_n, nwt)) {
    void *params[] = {const_cast<LuArgs *>(&a)};
    cudaLaunchKernel(kern, dim3(1), dim3(nwt * 32), params, 0, st);
    return;
  }
  cudaMemsetAsync(a.counter, 0, sizeof(unsigned), st);
  const int G = (max_n + nwt - 1) / nwt;  // enough for every variant the live size may select
  LuArgs args = a;
  void *params[] = {&args};
  cudaLaunchCooperativeKernel(kern, dim3(G), dim3(nwt * 32), params, 0, st);
}
