// prrLU with full pivoting (Alg. 2) — the latency-critical step a5 of the 2-site
// update. Readings: R1 (relative threshold), R2 (stop rule, eps = first rejected candidate),
// R3 (ties -> smallest (row, col)), R4 (l_i = S_iq * [S_pq]^{-1} — P:535 multiplies by the
// inverse pivot, so one IEEE reciprocal per pivot —, S_ij <- fma(-l_i, S_pj, S_ij)), R17;
// complex entries: RZ1-RZ4.
//
// Design. The Schur complement lives in REGISTERS for the whole factorisation.
// Rows run across the 32 lanes of a warp and columns across warps: thread (lane, w) holds
// S[lane + 32 a][c0 + w + NW b] for a < EA, b < EB. So one warp owns whole columns, which
// makes the pivot-column publication a coalesced single-warp store. Per pivot:
//   rank-1 update, then a branch-free running (value, slot) max per thread
//   -> warp argmax: 3 x redux.sync on the exact key (|v| bits hi, lo; flat index)
//   -> CTA argmax: per-warp keys in smem, every warp reduces them itself
//   -> cross-CTA exchange of the tier (below)
//   -> pivot column l = S_iq * (1/c) (R4) and pivot row u through smem.
// The pivot's sign comes from the pivot column, so keys carry only |v| (complex: w = |z|^2).
// Row p is zeroed exactly by l_p = 1 (fma(-1, u_j, u_j) = 0); column q by the owner warp.
// Eliminated entries are exact zeros: for every active entry the arithmetic equals the
// oracle's, so identical Pi gives bit-identical pivots.
// Tiers (chosen per launch on the device from the live block size, prrlu_kernel):
//   * CTA tier (XM = 0): one CTA (up to 32 register entries per thread), two barriers per pivot.
//   * cluster tier (XM = 2, default): whole 16-CTA clusters; keys pushed through DSMEM
//     (st.async + mbarrier), the candidate column published to L2 as tagged packets (each
//     8-byte word carries epoch|step, so no release/acquire fence is needed); several clusters
//     exchange cluster winners through L2 (one poller per cluster + DSMEM broadcast).
//   * push tier (XM = 3, prrlu_kernel_push, real blocks of <= 128 static rows): one 8-CTA cluster;
//     every CTA pushes its candidate column with its key into every peer's shared memory
//     (cp.async.bulk over DSMEM), so the winner's column is local when the keys are in.
//   * L2 grid tier (XM = 1): cooperative launch, tagged key packets with a key-poll or counter
//     barrier — used only when 16- and 8-CTA clusters cannot all be co-resident.
//   * single-cluster mode (prrlu_kernel_one, aci_options.concurrent): at most one cluster.
// All tiers use the same keys, tie-break and arithmetic, so they take identical decisions
// (tests/test_gpu_parity.py::test_prrlu_tiers_identical_pivots).
#include <cstdlib>

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
#ifndef ACI_LEADER_NP
#define ACI_LEADER_NP 1  // cluster-leader key poll: loads in flight (measured: 3 is not faster)
#endif
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

// ---- cluster (DSMEM) exchange primitives: keys are pushed into every CTA's shared memory with
// st.async, whose complete_tx lands on the destination CTA's mbarrier (measured 0.2-0.25 us per
// 8/16-CTA key exchange vs ~0.7-0.8 us for an L2 poll, profiles/r01_probe7_cluster_push.txt)
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa_u32(unsigned a, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(unsigned a, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_arm(unsigned a, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_async_key(unsigned raddr, unsigned a, unsigned b, unsigned c, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
               "r"(a), "r"(b), "r"(c), "r"(0u), "r"(rbar)
               : "memory");
}

// DSMEM bulk copy (async proxy) from this CTA's shared memory into a cluster peer's, completing
// `bytes` of transaction on the peer's mbarrier; 16-byte aligned, size a multiple of 16
__device__ __forceinline__ void bulk_push(unsigned rdst, unsigned src, unsigned bytes, unsigned rbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rdst),
               "r"(src), "r"(bytes), "r"(rbar)
               : "memory");
}

// push tier (XM = 3): one 8-CTA cluster; every CTA's candidate column is pushed into every
// cluster CTA's shared memory (dynamic: [2 parities][8 ranks][kPushRows] + 2 staging columns)
constexpr int kPushCS = 8;
constexpr int kPushRows = 128;
constexpr size_t kPushSmem = sizeof(double) * (2 * kPushCS * kPushRows + 2 * kPushRows);
extern __shared__ __align__(16) double push_dyn[];

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

// Rook mode (prrlu_rook.cuh): per-row values (l_i, the raw pivot column) in a paired shared layout,
// row i = lane + 32 a at (a / 2) * 64 + 2 lane + a % 2 (a warp's reads are 512 contiguous bytes).
__device__ __forceinline__ int lpair2(int i) { return ((i >> 6) << 6) | ((i & 31) << 1) | ((i >> 5) & 1); }

// columns per warp of the 8-warp grid tiers, measured (tools/prrlu_bench.cu): 16 CTAs with the
// key-poll barrier beat more CTAs with the counter barrier up to 512 rows
#ifndef ACI_W8_EB128
#define ACI_W8_EB128 4
#endif
#ifndef ACI_W8_EB256
#define ACI_W8_EB256 2
#endif
#ifndef ACI_NARROW512
#define ACI_NARROW512 1
#endif
#ifndef ACI_NARROW128
#define ACI_NARROW128 1
#endif
#ifndef ACI_W8_EB512
#define ACI_W8_EB512 4
#endif
#ifndef ACI_BIG_EB
#define ACI_BIG_EB 2  // columns per warp for the 1024-row grid tier (64 CTAs for 1024 columns)
#endif
// Column-slot stride factor of the exchange buffer (kept at 1: a spread layout over L2 slices was
// measured without gain, profiles/r02_prrlu_bench_variants.txt); packet i sits at u64 offset 2 i
constexpr int kColSpread = 1;
__device__ __forceinline__ int cpk(int i) { return 2 * i; }
// ACI_PRRLU_NOWORK (measurement builds only, csrc/peak_probe.cu): skip the rank-1 update, the
// column zeroing and the rescan, so every step exchanges the same winner — the per-pivot latency
// of the exchange alone, the floor the real kernel is reported against (bench.py roofline.latency)
#ifndef ACI_PRRLU_NOWORK
#define ACI_PRRLU_NOWORK 0
#endif
constexpr bool kNoWork = ACI_PRRLU_NOWORK != 0;
constexpr int kMaxRows = 1024;   // 32 * EA_max
constexpr int kMaxCTAs = 148;
static_assert(ACI_W8_EB128 >= 2 && ACI_W8_EB256 >= 2 && ACI_W8_EB512 >= 2 && ACI_BIG_EB >= 2,
              "launch_prrlu sizes grids for >= 16 columns per CTA");
constexpr int kMaxCB = 512;      // NW * EB_max

struct PrrluSmem {
  // complex factorisations keep real parts in [0, kMax) and imaginary parts in [kMax, 2 kMax)
  double l[2 * kMaxRows];    // l_i (R4), l[p] = 1
  double raw[2 * kMaxRows];  // CTA tier: raw pivot column
  double u[2 * kMaxCB];      // pivot row segment
  unsigned hi[32], lo[32], id[32];
  unsigned win[4];  // grid winner broadcast (key-poll mode)
  uint4 ck[2][16];                // cluster tier: CTA keys pushed by the cluster's CTAs (by parity)
  uint4 gw[2];                    // cluster tier, several clusters: global winner pushed by rank 0
  unsigned long long mb[4];       // cluster tier: key mbarrier and winner mbarrier per parity
};
// rook mode (prrlu_rook.cuh): the same scratch plus a bitmap of eliminated columns
struct RookSmem : PrrluSmem {
  unsigned cdone[48];  // up to 1536 columns
};

// One factorisation, register tile EA x EB per thread, NW warps per CTA. GRID: G CTAs (this is
// CTA g) cooperate through the exchange buffers; otherwise one CTA does everything.
// XM: exchange mode. 0 = one CTA; 1 = grid of co-resident CTAs exchanging through L2 (tagged
// packets, counter or key-poll barrier); 2 = grid of whole thread-block clusters: CTA keys are
// pushed through DSMEM (st.async + mbarrier), cluster winners (if more than one cluster) and
// candidate columns go through L2 as tagged packets.
// CPLX: complex entries (interleaved (re, im) in A.M and A.U; ldm, ldu count complex elements),
// readings RZ1-RZ4: the key is w = fl(re^2) + fl(im^2), |c| = sqrt(w),
// inv = (c_re / w, -c_im / w), l_i = S_iq * inv and u-row products as RZ3 (no FMA contraction),
// the Schur update as the RZ4 fma sequence. Bit-identical to oracle/aci_oracle_z.c for equal Pi.
// ---- Hand-off (HO) of a multi-cluster factorisation to ONE cluster (ACI_HANDOFF). A block that
// needs two 16-CTA clusters (the 512 x 1024 blocks of configs[3] at chi = 256: 512 pivots with a
// cross-cluster L2 leg each) shrinks as it is factorised: after K pivots the live Schur complement
// is (m - K) x (n - K). At k = K every CTA writes its live entries, compacted (eliminated rows and
// columns dropped, order kept), to a scratch area; the first cluster reloads the compacted block
// into a one-cluster register layout and continues from pivot K with the same threshold, first
// candidate and tie-break (the compacted (row, col) order is the original one: the maps are
// increasing), so the pivots and the arithmetic are exactly those of the uninterrupted run.
// Phase 1 (HO = 1) keeps bitmaps of the eliminated rows / columns; phase 2 (HO = 2) maps its
// compacted pivot indices and U columns back. Shared scratch (S.raw, unused by the real grid
// tiers), as 32-bit words:
constexpr int kHoDeadR = 0;      // 32 words: eliminated rows (<= 1024)
constexpr int kHoDeadC = 32;     // 48 words: eliminated columns (<= 1536)
constexpr int kHoPrefR = 80;     // exclusive prefix of the popcounts of kHoDeadR
constexpr int kHoPrefC = 112;    // exclusive prefix of the popcounts of kHoDeadC
constexpr int kHoRowMap = 160;   // compacted row -> original row (<= 1024)
constexpr int kHoColMap = 1184;  // compacted column -> original column (<= 1536)
constexpr int kHoDeadList = 2720;  // eliminated columns in increasing order (<= 1024)
constexpr int kHoFlags = 1024;   // grid barrier flags in A.keys (u64 words [1024, 1024 + 2 G))
constexpr int kHoEA = 8, kHoEB = 6;  // phase-2 register tile: 256 rows x 16 CTAs x 48 columns
#ifndef ACI_HANDOFF
#define ACI_HANDOFF 1
#endif
struct HoState {
  int k;         // pivots done before the hand-off (phase 2 starts at pivot k)
  double first;  // |first candidate| (R8 threshold mode)
  double thr;
  bool handed;
};
__device__ __forceinline__ unsigned *ho_words(PrrluSmem &S) { return reinterpret_cast<unsigned *>(S.raw); }
// compacted index of original index i: i minus the eliminated ones below it
__device__ __forceinline__ int ho_rank(const unsigned *dead, const unsigned *pref, int i) {
  return i - (int)(pref[i >> 5] + __popc(dead[i >> 5] & ((1u << (i & 31)) - 1u)));
}

template <int EA, int EB, int NW, int XM, bool CPLX = false, int HO = 0>
__device__ __forceinline__ void prrlu_body(const LuArgs &A, PrrluSmem &S, const int G, const int g,
                                           HoState *hs = nullptr) {
  static_assert(HO == 0 || (XM == 2 && !CPLX), "hand-off: real cluster tier only");
  constexpr bool GRID = XM != 0;
  constexpr int Z = CPLX ? 2 : 1;  // doubles per entry
  constexpr int T = NW * 32;
  constexpr int MROWS = 32 * EA;
  constexpr int CB = NW * EB;  // columns per CTA
  static_assert(MROWS <= kMaxRows && CB <= kMaxCB, "tile exceeds the shared scratch");
  double *s_l = S.l, *s_raw = S.raw, *s_u = S.u;
  unsigned *s_hi = S.hi, *s_lo = S.lo, *s_id = S.id;
  const int tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const int c0 = g * CB;

  // phase 2 of a hand-off works on the compacted (m - K) x (n - K) block, pivots numbered from K
  const int k0 = HO == 2 ? hs->k : 0;
  const int m = A.dims->m - k0, n = A.dims->n - k0, kmax = A.dims->kmax, ldu = A.dims->ldu;
  const int ldm = HO == 2 ? n : A.dims->ldm;
  const unsigned ep = GRID ? (*A.epoch & 0xfffffu) : 0u;  // read by every CTA before any arrival
  const int mn = (m < n ? m : n) + k0;
  double thr = A.tol;
  if (A.thr_mode == 0) thr = A.tol * __longlong_as_double((long long)*A.scale_bits);
  // hand-off scratch: the compacted live block, behind the exchange slots of a 64-CTA grid
  double *const hbuf = reinterpret_cast<double *>(A.colpub + (size_t)2 * 64 * A.colcap * 2);
  const double *const Msrc = HO == 2 ? hbuf : A.M;
  unsigned *const hw = ho_words(S);
  if constexpr (HO == 1)
    for (int i = tid; i < kHoPrefR; i += T) hw[i] = 0u;  // eliminated-row / -column bitmaps

  // ---- load; padding = 0 and never a candidate
  double v[EA][EB][Z];
  bool rok[EA], cok[EB];
#pragma unroll
  for (int a = 0; a < EA; ++a) rok[a] = lane + 32 * a < m;
#pragma unroll
  for (int b = 0; b < EB; ++b) cok[b] = c0 + w + NW * b < n;
#pragma unroll
  for (int a = 0; a < EA; ++a)
#pragma unroll
    for (int b = 0; b < EB; ++b)
#pragma unroll
      for (int z = 0; z < Z; ++z)
        v[a][b][z] = (rok[a] && cok[b])
                         ? (HO == 2 ? __ldcg(Msrc + (size_t)(lane + 32 * a) * ldm + c0 + w + NW * b)
                                    : Msrc[((size_t)(lane + 32 * a) * ldm + c0 + w + NW * b) * Z + z])
                         : 0.0;
  for (int i = tid; i < Z * kMaxRows; i += T) s_l[i] = 0.0;
  for (int j = tid; j < Z * kMaxCB; j += T) s_u[j] = 0.0;

  // Flat candidate index = row * NC + col with the PADDED width NC (>= every column of the
  // grid), so padding entries (always exact zeros) never alias a real index and never need a
  // mask: a zero can only win when every active entry is zero, and then the factorisation stops
  // (R2) — except at k = 0, where (0, 0) (a real entry) wins the R3 tie-break.
  // NC is rounded up to a power of two (2^ncs): the flat index splits into (row, col) with a
  // shift and a mask instead of a runtime integer division on the per-pivot critical path; the
  // lexicographic (row, col) order of the flat indices (R3) holds for any NC >= the live width.
  constexpr unsigned kLogCB = CB <= 1 ? 0u : (unsigned)(31 - __builtin_clz((unsigned)CB));
  const unsigned ncs = (XM == 0) ? kLogCB : (unsigned)(32 - __clz(G * CB - 1));
  static_assert(XM != 0 || (CB & (CB - 1)) == 0, "one-CTA tiers: columns per CTA a power of two");
  const unsigned NC = 1u << ncs;
  // per-thread max over the register tile: NCH independent chains (slot e -> chain e % NCH),
  // strict '>' within a chain; chains merged with the slot (== flat-index) tie-break.
  double bx = 0.0;
  int be = 0;
  auto scan = [&]() {
    constexpr int NE = EA * EB;
    constexpr int NCH = NE < 4 ? NE : 4;
    // chains keep the SIGNED value and compare magnitudes (|.| operand modifiers of DSETP), so
    // no FP64-pipe instruction is spent materialising |v|
    double cx[NCH];
    int ce[NCH];
    // complex: the chains hold w = fl(re^2) + fl(im^2) (RZ1), compared directly
    auto mag = [&](int e) -> double {
      const double *x = v[e / EB][e % EB];
      return CPLX ? __dadd_rn(__dmul_rn(x[0], x[0]), __dmul_rn(x[Z - 1], x[Z - 1])) : x[0];
    };
#pragma unroll
    for (int t = 0; t < NCH; ++t) { cx[t] = mag(t); ce[t] = t; }
#pragma unroll
    for (int e = NCH; e < NE; ++e) {
      const double x = mag(e);
      const bool take = fabs(x) > fabs(cx[e % NCH]);
      cx[e % NCH] = take ? x : cx[e % NCH];
      ce[e % NCH] = take ? e : ce[e % NCH];
    }
    double bm = cx[0];
    int bi = ce[0];
#pragma unroll
    for (int t = 1; t < NCH; ++t) {
      const bool take = fabs(cx[t]) > fabs(bm) || (fabs(cx[t]) == fabs(bm) && ce[t] < bi);
      bm = take ? cx[t] : bm;
      bi = take ? ce[t] : bi;
    }
    bx = fabs(bm);
    be = bi;
  };
  auto thread_key = [&]() -> Key {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(bx);
    const int a = be / EB, b = be % EB;
    const unsigned flat = ((unsigned)(lane + 32 * a) << ncs) | (unsigned)(c0 + w + NW * b);
    return Key{(unsigned)(bits >> 32), (unsigned)bits, flat};
  };
  scan();
  if constexpr (XM == 3) {
    // keys (16 B) and candidate columns (MROWS doubles) of every cluster CTA land on one
    // mbarrier per parity, armed for steps 0 and 1 before any CTA pushes
    if (tid == 0) {
      const unsigned CS = cluster_size();
      for (int t = 0; t < 2; ++t) mbar_init(smem_u32(&S.mb[t]), 1u);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_arm(smem_u32(&S.mb[0]), CS * (16u + 8u * MROWS));
      mbar_arm(smem_u32(&S.mb[1]), CS * (16u + 8u * MROWS));
    }
    cluster_sync_all();
  }
  if (XM == 2) {
    // one mbarrier per parity, armed for steps 0 and 1 before any CTA of the cluster pushes
    if (tid == 0) {
      const unsigned CS = cluster_size();
      for (int t = 0; t < 4; ++t) mbar_init(smem_u32(&S.mb[t]), 1u);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_arm(smem_u32(&S.mb[0]), CS * 16u);
      mbar_arm(smem_u32(&S.mb[1]), CS * 16u);
      mbar_arm(smem_u32(&S.mb[2]), 16u);
      mbar_arm(smem_u32(&S.mb[3]), 16u);
    }
    cluster_sync_all();
  }

  double first = HO == 2 ? hs->first : 0.0, eps = 0.0;
  if constexpr (HO == 2) thr = hs->thr;
  int k = k0;
  bool handed = false;
#ifdef ACI_PRRLU_TIMING
  long long ph_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long ph_t_ = clock64();
#endif
  for (;;) {
    if (k == mn) { eps = 0.0; break; }
    if constexpr (HO == 1) {
      if (k == hs->k) {
        // ---- hand-off: write the live entries, compacted, then publish this CTA's flag
        __syncthreads();  // the bitmaps of pivots 0..K-1 (thread 0) are complete
        if (w == 0) {
          // exclusive prefix of the popcounts: rows (32 words) and columns (48 words)
          const unsigned pr = __popc(hw[kHoDeadR + lane]);
          unsigned xr = pr;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(FULL, xr, o);
            if (lane >= o) xr += t;
          }
          hw[kHoPrefR + lane] = xr - pr;
          const unsigned c_lo = __popc(hw[kHoDeadC + lane]);
          const unsigned c_hi = lane < 16 ? __popc(hw[kHoDeadC + 32 + lane]) : 0u;
          unsigned xl = c_lo, xh = c_hi;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned tl = __shfl_up_sync(FULL, xl, o), th = __shfl_up_sync(FULL, xh, o);
            if (lane >= o) { xl += tl; xh += th; }
          }
          const unsigned tot_lo = __shfl_sync(FULL, xl, 31);
          hw[kHoPrefC + lane] = xl - c_lo;
          if (lane < 16) hw[kHoPrefC + 32 + lane] = tot_lo + xh - c_hi;
        }
        __syncthreads();
        const int ldh = n - k;  // compacted width
#pragma unroll
        for (int a = 0; a < EA; ++a) {
          const int i = lane + 32 * a;
          if (i < m && !((hw[kHoDeadR + (i >> 5)] >> (i & 31)) & 1u)) {
            const int ri = ho_rank(hw + kHoDeadR, hw + kHoPrefR, i);
#pragma unroll
            for (int b = 0; b < EB; ++b) {
              const int j = c0 + w + NW * b;
              if (j < n && !((hw[kHoDeadC + (j >> 5)] >> (j & 31)) & 1u))
                hbuf[(size_t)ri * ldh + ho_rank(hw + kHoDeadC, hw + kHoPrefC, j)] = v[a][b][0];
            }
          }
        }
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          st_pkt(A.keys + 2 * (kHoFlags / 2 + g), tagged(ep, 0xfffu), 0ull);
        }
        hs->first = first;
        hs->thr = thr;
        hs->handed = true;
        handed = true;
        break;
      }
    }
    // ---- warp -> CTA argmax
    const Key wk = warp_argmax(thread_key());
    if (lane == 0) { s_hi[w] = wk.hi; s_lo[w] = wk.lo; s_id[w] = wk.id; }
    __syncthreads();  // S1
    PHASE(0);
    const Key ck = warp_argmax(lane < NW ? Key{s_hi[lane], s_lo[lane], s_id[lane]} : Key{0u, 0u, BAD_ID});
    Key win = ck;
    PHASE(1);
    if constexpr (XM == 3) {
      // ---- push tier: key + candidate column into every cluster CTA (DSMEM), one wait
      const int par = k & 1;
      const unsigned CS = cluster_size(), crank = cluster_rank();
      const int jc = (int)(ck.id & (NC - 1u)) - c0;
      const int pw = jc % NW;
      if (w == 0 && lane < (int)CS)
        st_async_key(mapa_u32(smem_u32(&S.ck[par][crank]), (unsigned)lane), ck.hi, ck.lo, ck.id,
                     mapa_u32(smem_u32(&S.mb[par]), (unsigned)lane));
      if (w == pw) {
        double *stg = push_dyn + 2 * kPushCS * kPushRows + par * kPushRows;
        const int bc = jc / NW;
#pragma unroll
        for (int b = 0; b < EB; ++b)
          if (b == bc)
#pragma unroll
            for (int a = 0; a < EA; ++a) stg[lane + 32 * a] = v[a][b][0];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane < (int)CS) {
          double *dst = push_dyn + ((size_t)par * kPushCS + crank) * kPushRows;
          bulk_push(mapa_u32(smem_u32(dst), (unsigned)lane), smem_u32(stg), 8u * MROWS,
                    mapa_u32(smem_u32(&S.mb[par]), (unsigned)lane));
          asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
        }
      }
      PHASE(2);
      const unsigned mbp = smem_u32(&S.mb[par]);
      mbar_wait(mbp, (unsigned)(k >> 1) & 1u);
      PHASE(3);
      if (tid == 0) mbar_arm(mbp, CS * (16u + 8u * MROWS));  // for step k + 2
      const uint4 q4 = S.ck[par][lane < (int)CS ? lane : 0];
      win = warp_argmax(lane < (int)CS ? Key{q4.x, q4.y, q4.z} : Key{0u, 0u, BAD_ID});
      PHASE(4);
    } else if (GRID) {
      const int par = k & 1;
      const unsigned tag = (ep << 12) | (unsigned)(k + 1);
      // the owner warp of the CTA candidate's column publishes the column (tagged packets, no
      // fence) and lane 0 publishes the key and arrives on the counter
      const int jc = (int)(ck.id & (NC - 1u)) - c0;
      const int pw = jc % NW;
      if (XM == 2 && w == 0) {
        // cluster tier: the key goes out first (st.async into every cluster CTA's smem), the
        // column store follows; readers only touch it after the key exchange
        const unsigned CS = cluster_size();
        if (lane < (int)CS)
          st_async_key(mapa_u32(smem_u32(&S.ck[par][cluster_rank()]), (unsigned)lane), ck.hi, ck.lo, ck.id,
                       mapa_u32(smem_u32(&S.mb[par]), (unsigned)lane));
      }
      if (w == pw) {
        const int bc = jc / NW;
        unsigned long long *dst = A.colpub + (((size_t)par * G + g) * A.colcap) * 2;
#pragma unroll
        for (int b = 0; b < EB; ++b)
          if (b == bc)
#pragma unroll
            for (int a = 0; a < EA; ++a)
              if (rok[a])
#pragma unroll
                for (int z = 0; z < Z; ++z) {
                  const unsigned long long bits = (unsigned long long)__double_as_longlong(v[a][b][z]);
                  st_pkt(dst + 2 * (Z * (lane + 32 * a) + z), tagged(tag, (unsigned)bits),
                         tagged(tag, (unsigned)(bits >> 32)));
                }
        if (XM == 1 && lane == 0) {
          unsigned long long *kd = A.keys + ((size_t)par * G + g) * 4;
          st_pkt(kd, tagged(tag, ck.hi), tagged(tag, ck.lo));
          st_pkt(kd + 2, tagged(tag, ck.id), 0ull);
          if (G > ACI_KEYPOLL_MAXG) red_relaxed_add(A.counter, 1u);
        }
      }
      PHASE(2);
      if (XM == 2) {
        // ---- cluster key exchange: push this CTA's key into every cluster CTA's smem
        const unsigned CS = cluster_size(), crank = cluster_rank();
        const unsigned mbp = smem_u32(&S.mb[par]);
        mbar_wait(mbp, (unsigned)(k >> 1) & 1u);
        PHASE(3);
        if (tid == 0) mbar_arm(mbp, CS * 16u);  // re-arm this parity for step k + 2
        const uint4 q4 = S.ck[par][lane < (int)CS ? lane : 0];
        const Key cw = warp_argmax(lane < (int)CS ? Key{q4.x, q4.y, q4.z} : Key{0u, 0u, BAD_ID});
        const int NCL = G / (int)CS;
        if (NCL == 1) {
          win = cw;
        } else {
          // cluster winners through L2: warp 0 of each cluster's rank-0 CTA publishes its
          // cluster's winner (slots 256 B apart), polls the NCL tagged keys and pushes the
          // global winner to its cluster peers through DSMEM (one poller per cluster keeps the
          // L2 lines uncontended)
          const int cid = g / (int)CS;
          const unsigned mwp = smem_u32(&S.mb[2 + par]);
          if (crank == 0 && w == 0) {
            if (lane == 0) {
              unsigned long long *kd = A.keys + ((size_t)par * kMaxCTAs / 8 + cid) * 32;
              st_pkt(kd, tagged(tag, cw.hi), tagged(tag, cw.lo));
              st_pkt(kd + 2, tagged(tag, cw.id), 0ull);
            }
            Key gk{0u, 0u, BAD_ID};
            if (lane < NCL) {
              // rolling poll: ACI_LEADER_NP loads in flight, issued ~kPollGap cycles apart, so a
              // packet is seen about one L2 round trip after it lands
              const unsigned long long *kp = A.keys + ((size_t)par * kMaxCTAs / 8 + lane) * 32;
              constexpr int NP = ACI_LEADER_NP;
              unsigned long long kw[NP][4];
#pragma unroll
              for (int i = 0; i < NP; ++i) {
                ld_pkt(kp, kw[i][0], kw[i][1]);
                ld_pkt(kp + 2, kw[i][2], kw[i][3]);
                if (NP > 1 && i + 1 < NP) {
                  const long long t0 = clock64();
                  while (clock64() - t0 < kPollGap) {
                  }
                }
              }
              bool got = false;
              while (!got) {
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                  if (!got) {
                    if ((unsigned)(kw[i][0] >> 32) == tag && (unsigned)(kw[i][1] >> 32) == tag &&
                        (unsigned)(kw[i][2] >> 32) == tag) {
                      gk = Key{(unsigned)kw[i][0], (unsigned)kw[i][1], (unsigned)kw[i][2]};
                      got = true;
                    } else {
                      ld_pkt(kp, kw[i][0], kw[i][1]);
                      ld_pkt(kp + 2, kw[i][2], kw[i][3]);
                    }
                  }
                }
              }
            }
            const Key gw = warp_argmax(gk);
            if (lane < (int)CS)
              st_async_key(mapa_u32(smem_u32(&S.gw[par]), (unsigned)lane), gw.hi, gw.lo, gw.id, mapa_u32(mwp, (unsigned)lane));
          }
          mbar_wait(mwp, (unsigned)(k >> 1) & 1u);
          if (tid == 0) mbar_arm(mwp, 16u);
          win = Key{S.gw[par].x, S.gw[par].y, S.gw[par].z};
        }
      } else {
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
      }
      PHASE(4);
    }

    // ---- stop rule (R2), uniform across the grid; complex keys carry w = |c|^2 (RZ1)
    const double wkey = key_abs(win);
    const double absc = CPLX ? __dsqrt_rn(wkey) : wkey;
    if (k == 0) {
      first = absc;
      if (A.thr_mode == 1) thr = A.tol * first;
    }
    if (k == kmax) { eps = absc; break; }
    if (k > 0 && absc <= thr) { eps = absc; break; }
    const int p = (int)(win.id >> ncs), q = (int)(win.id & (NC - 1u));
    if (g == 0 && tid == 0) {
      if constexpr (HO == 2) {
        A.rows[k] = (int)hw[kHoRowMap + p];
        A.cols[k] = (int)hw[kHoColMap + q];
      } else {
        A.rows[k] = p;
        A.cols[k] = q;
      }
    }
    if constexpr (HO == 1)
      if (tid == 0) {  // eliminated row p and column q (the hand-off's compaction)
        hw[kHoDeadR + (p >> 5)] |= 1u << (p & 31);
        hw[kHoDeadC + (q >> 5)] |= 1u << (q & 31);
      }
    if (k == 0 && absc == 0.0) {
      // R17: zero block -> rank 1, dummy pivot (0,0), U row e_q, eps 0
      if (A.U)
        for (int j = c0 + tid; j < c0 + CB && j < n; j += T)
#pragma unroll
          for (int z = 0; z < Z; ++z) A.U[((size_t)k * ldu + j) * Z + z] = (j == q && z == 0) ? 1.0 : 0.0;
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
          for (int b = 0; b < EB; ++b)
#pragma unroll
            for (int z = 0; z < Z; ++z) s_u[z * kMaxCB + w + NW * b] = v[a][b][z];
    }
    if constexpr (!CPLX) {
    // 1/|c| from the key, off the column's critical path; the sign arrives with the column
    // (1/(-x) = -(1/x) exactly). CTA tier: l_i = S_iq * (1/S_pq) (R4) is applied as
    // fma(l'_i, -/+u_j, v) with l'_i = S_iq * (1/|c|): negation is exact, so this is
    // bit-identical to fma(-l_i, u_j, v).
    // __drcp_rn is the correctly rounded reciprocal, i.e. the same bits as 1.0 / |c|; the empty
    // asm pins its evaluation here, ahead of the column loads it would otherwise trail
    // (grid tiers: computed right after the column loads are issued, so it runs under their latency)
    double inv_abs = 0.0;
    if constexpr (!GRID || XM == 3) {
      inv_abs = __drcp_rn(absc);
      asm volatile("" : "+d"(inv_abs));
    }
    double inv;       // signed 1/S_pq
    double ub[EB];    // pivot row (CTA tier: sign-folded, -u_j (c > 0) or +u_j (c < 0))
    if constexpr (XM == 3) {
      // the winner's column is already in this CTA's shared memory (pushed with its key)
      const double *col = push_dyn + ((size_t)(k & 1) * kPushCS + q / CB) * kPushRows;
      const bool neg = col[p] < 0.0;
      inv = neg ? -inv_abs : inv_abs;
      __syncthreads();  // S3: pivot row in smem
      PHASE(5);
      if (A.U)
        for (int jj = tid; jj < CB; jj += T) {
          const int j = c0 + jj;
          if (j < n) A.U[(size_t)k * ldu + j] = (j == q) ? 1.0 : s_u[jj] * inv;
        }
#pragma unroll
      for (int b = 0; b < EB; ++b) ub[b] = s_u[w + NW * b];
      if constexpr (!kNoWork) {
#pragma unroll
      for (int a = 0; a < EA; ++a) {
        const int i = lane + 32 * a;
        const double li = i < m ? ((i == p) ? 1.0 : col[i] * inv) : 0.0;
#pragma unroll
        for (int b = 0; b < EB; ++b) v[a][b][0] = fma(-li, ub[b], v[a][b][0]);
      }
      }
    } else if (GRID) {
      const unsigned tag = (ep << 12) | (unsigned)(k + 1);
      PHASE(7);
      const unsigned long long *src = A.colpub + (((size_t)(k & 1) * G + q / CB) * A.colcap) * 2;
      constexpr int PPT = (MROWS + T - 1) / T;  // column packets per thread
      unsigned long long cw[PPT + 1][2];
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int i = tid + T * t;
        if (i < m) ld_pkt(src + 2 * i, cw[t][0], cw[t][1]);
      }
      ld_pkt(src + 2 * p, cw[PPT][0], cw[PPT][1]);  // the pivot itself, for its sign
      inv_abs = __drcp_rn(absc);
      asm volatile("" : "+d"(inv_abs));
      while ((unsigned)(cw[PPT][0] >> 32) != tag || (unsigned)(cw[PPT][1] >> 32) != tag)
        ld_pkt(src + 2 * p, cw[PPT][0], cw[PPT][1]);
      const bool neg = (cw[PPT][1] & 0x80000000ull) != 0;
      inv = neg ? -inv_abs : inv_abs;
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int i = tid + T * t;
        if (i < m) {
          while ((unsigned)(cw[t][0] >> 32) != tag || (unsigned)(cw[t][1] >> 32) != tag)
            ld_pkt(src + 2 * i, cw[t][0], cw[t][1]);
          s_l[i] = (i == p) ? 1.0 : pkt_double(cw[t][0], cw[t][1]) * inv;
        }
      }
      __syncthreads();  // S3
      PHASE(5);
      if (A.U) {
        for (int jj = tid; jj < CB; jj += T) {
          const int j = c0 + jj;
          if (j < n) {
            const int jo = HO == 2 ? (int)hw[kHoColMap + j] : j;
            A.U[(size_t)k * ldu + jo] = (j == q) ? 1.0 : s_u[jj] * inv;
          }
        }
        if constexpr (HO == 2) {
          // columns eliminated before the hand-off: their pivot-row entries are exact +0, so U = 0 * inv
          const int per = (k0 + G - 1) / G;
          for (int t = tid; t < per; t += T) {
            const int d = g * per + t;
            if (d < k0) A.U[(size_t)k * ldu + (int)hw[kHoDeadList + d]] = 0.0 * inv;
          }
        }
      }
#pragma unroll
      for (int b = 0; b < EB; ++b) ub[b] = s_u[w + NW * b];
      if constexpr (!kNoWork) {
#pragma unroll
      for (int a = 0; a < EA; ++a) {
        const double li = s_l[lane + 32 * a];
#pragma unroll
        for (int b = 0; b < EB; ++b) v[a][b][0] = fma(-li, ub[b], v[a][b][0]);
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
            for (int a = 0; a < EA; ++a) s_raw[lane + 32 * a] = v[a][b][0];
      }
      __syncthreads();  // S2 (CTA tier): raw pivot column and pivot row in smem
      const bool neg = s_raw[p] < 0.0;
      inv = neg ? -inv_abs : inv_abs;
#pragma unroll
      for (int b = 0; b < EB; ++b) ub[b] = neg ? s_u[w + NW * b] : -s_u[w + NW * b];
      PHASE(5);
      if (A.U)
        for (int jj = tid; jj < CB; jj += T) {
          const int j = c0 + jj;
          if (j < n) A.U[(size_t)k * ldu + j] = (j == q) ? 1.0 : s_u[jj] * inv;
        }
      // every thread forms its own l'_i (no third barrier)
      if constexpr (!kNoWork) {
#pragma unroll
      for (int a = 0; a < EA; ++a) {
        const int i = lane + 32 * a;
        const double li = (i == p) ? (neg ? -1.0 : 1.0) : s_raw[i] * inv_abs;
#pragma unroll
        for (int b = 0; b < EB; ++b) v[a][b][0] = fma(li, ub[b], v[a][b][0]);
      }
      }
    }
    } else {
    // ---- complex (RZ2-RZ4): inv = conj(c) / w with w the key's |c|^2
    double cr, ci;
    if (GRID) {
      const unsigned tag = (ep << 12) | (unsigned)(k + 1);
      const unsigned long long *src = A.colpub + (((size_t)(k & 1) * G + q / CB) * A.colcap) * 2;
      constexpr int PPT = (MROWS + T - 1) / T;  // column entries per thread (2 packets each)
      unsigned long long cw[PPT + 1][2][2];
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int i = tid + T * t;
        if (i < m)
#pragma unroll
          for (int z = 0; z < 2; ++z) ld_pkt(src + 2 * (2 * i + z), cw[t][z][0], cw[t][z][1]);
      }
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        ld_pkt(src + 2 * (2 * p + z), cw[PPT][z][0], cw[PPT][z][1]);
        while ((unsigned)(cw[PPT][z][0] >> 32) != tag || (unsigned)(cw[PPT][z][1] >> 32) != tag)
          ld_pkt(src + 2 * (2 * p + z), cw[PPT][z][0], cw[PPT][z][1]);
      }
      cr = pkt_double(cw[PPT][0][0], cw[PPT][0][1]);
      ci = pkt_double(cw[PPT][1][0], cw[PPT][1][1]);
      const double ir = __ddiv_rn(cr, wkey), ii = __ddiv_rn(-ci, wkey);
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int i = tid + T * t;
        if (i < m) {
#pragma unroll
          for (int z = 0; z < 2; ++z)
            while ((unsigned)(cw[t][z][0] >> 32) != tag || (unsigned)(cw[t][z][1] >> 32) != tag)
              ld_pkt(src + 2 * (2 * i + z), cw[t][z][0], cw[t][z][1]);
          const double xr = pkt_double(cw[t][0][0], cw[t][0][1]), xi = pkt_double(cw[t][1][0], cw[t][1][1]);
          double lr = 1.0, li = 0.0;
          if (i != p) {  // RZ3
            lr = __dsub_rn(__dmul_rn(xr, ir), __dmul_rn(xi, ii));
            li = __dadd_rn(__dmul_rn(xr, ii), __dmul_rn(xi, ir));
          }
          s_l[i] = lr;
          s_l[kMaxRows + i] = li;
        }
      }
      __syncthreads();  // S3
    } else {
      const int jq = q - c0;
      if ((jq % NW) == w) {
        const int bq = jq / NW;
#pragma unroll
        for (int b = 0; b < EB; ++b)
          if (b == bq)
#pragma unroll
            for (int a = 0; a < EA; ++a) {
              s_raw[lane + 32 * a] = v[a][b][0];
              s_raw[kMaxRows + lane + 32 * a] = v[a][b][Z - 1];
            }
      }
      __syncthreads();  // S2 (CTA tier)
      cr = s_raw[p];
      ci = s_raw[kMaxRows + p];
    }
    const double ir = __ddiv_rn(cr, wkey), ii = __ddiv_rn(-ci, wkey);
    PHASE(5);
    if (A.U)
      for (int jj = tid; jj < CB; jj += T) {
        const int j = c0 + jj;
        if (j < n) {
          double yr = 1.0, yi = 0.0;
          if (j != q) {  // RZ3
            const double ur = s_u[jj], ui = s_u[kMaxCB + jj];
            yr = __dsub_rn(__dmul_rn(ur, ir), __dmul_rn(ui, ii));
            yi = __dadd_rn(__dmul_rn(ur, ii), __dmul_rn(ui, ir));
          }
          A.U[((size_t)k * ldu + j) * 2] = yr;
          A.U[((size_t)k * ldu + j) * 2 + 1] = yi;
        }
      }
    double ubr[EB], ubi[EB];
#pragma unroll
    for (int b = 0; b < EB; ++b) {
      ubr[b] = s_u[w + NW * b];
      ubi[b] = s_u[kMaxCB + w + NW * b];
    }
#pragma unroll
    for (int a = 0; a < EA; ++a) {
      const int i = lane + 32 * a;
      double lr, li;
      if (GRID) {
        lr = s_l[i];
        li = s_l[kMaxRows + i];
      } else {  // every thread forms its own l_i (RZ3)
        const double xr = s_raw[i], xi = s_raw[kMaxRows + i];
        lr = __dsub_rn(__dmul_rn(xr, ir), __dmul_rn(xi, ii));
        li = __dadd_rn(__dmul_rn(xr, ii), __dmul_rn(xi, ir));
        if (i == p) { lr = 1.0; li = 0.0; }
      }
#pragma unroll
      for (int b = 0; b < EB; ++b) {  // RZ4
        const double tr = fma(-lr, ubr[b], v[a][b][0]);
        const double ti = fma(-lr, ubi[b], v[a][b][Z - 1]);
        v[a][b][0] = fma(li, ubi[b], tr);
        v[a][b][Z - 1] = fma(-li, ubr[b], ti);
      }
    }
    }
    // column q -> exact zeros (owner warp; warp-uniform branch)
    if constexpr (!kNoWork) {
      const int jq = q - c0;
      if (jq >= 0 && jq < CB && (jq % NW) == w) {
        const int bq = jq / NW;
#pragma unroll
        for (int b = 0; b < EB; ++b)
          if (b == bq)
#pragma unroll
            for (int a = 0; a < EA; ++a)
#pragma unroll
              for (int z = 0; z < Z; ++z) v[a][b][z] = 0.0;
      }
    }
    if constexpr (!kNoWork) scan();
    PHASE(6);
    ++k;
    // s_l / s_u / s_raw are rewritten only after the next S1; every thread finished reading
    // them before arriving there.
  }
  if (g == 0 && tid == 0 && !handed) {
    *A.r_out = k;
    *A.eps_out = eps;
    // every CTA read the epoch before its first arrival, and CTA 0 only gets here after the
    // last exchange, so the increment cannot race with a reader of this launch
    if (GRID) atomicAdd(A.epoch, 1u);
#ifdef ACI_PRRLU_TIMING
    for (int t = 0; t < 8; ++t) A.dbg[t] = ph_[t];
#endif
  }
  if (XM >= 2) cluster_sync_all();  // no CTA leaves while a cluster peer may still push to it
}

#include "prrlu_rook.cuh"

// Rook mode (LuArgs::rook): the prrlu_kernel_one envelope (one CTA or one 16-CTA cluster), real
// values; the same variant list as prrlu_kernel_one.
template <int NWT>
__global__ void __launch_bounds__(NWT * 32) prrlu_kernel_rook(LuArgs A) {
  __shared__ RookSmem S;
  const int m = A.dims->m, n = A.dims->n;
  const int g = blockIdx.x;
#define ACI_CTA_VARIANT(EA, EB)                                        \
  if (m <= 32 * (EA) && n <= NWT * (EB)) {                              \
    if (g == 0) prrlu_body_rook<(EA), (EB), NWT, 0>(A, S, 1, 0);       \
    return;                                                            \
  }
#define ACI_ONE_VARIANT(EA, EB)                                        \
  if (m <= 32 * (EA) && n <= 16 * NWT * (EB)) {                         \
    prrlu_body_rook<(EA), (EB), NWT, 2>(A, S, 16, g);                  \
    return;                                                            \
  }
  ACI_CTA_VARIANT(1, 4)
  ACI_CTA_VARIANT(2, 8)
  ACI_CTA_VARIANT(4, 4)
  ACI_CTA_VARIANT(1, 16)
  ACI_CTA_VARIANT(4, 16)
  ACI_CTA_VARIANT(8, 8)
  ACI_CTA_VARIANT(2, 32)
  ACI_ONE_VARIANT(4, 8)    //  128 x 1024
  ACI_ONE_VARIANT(8, 4)    //  256 x  512
  ACI_ONE_VARIANT(16, 4)   //  512 x  512
#undef ACI_CTA_VARIANT
#undef ACI_ONE_VARIANT
}

// Runtime tier selection from the LIVE sizes (device-resident ranks): the launch is sized for
// the static capacity, and CTAs beyond what the live block needs exit immediately. 8 warps per
// CTA (up to 255 registers, so the 32-row-slot tiles do not spill; measured faster than 16).
// XM = 1: cooperative grid, L2 exchange. XM = 2: cluster launch; the participating CTAs are
// rounded up to whole clusters (CTAs past the live columns hold padding only).
// ACI_CLUSTER_CTA_MAXE: in the cluster kernel (XM = 2, real), one-CTA variants with more register
// entries per thread than this are skipped, so such live blocks (e.g. 128 x 128 inside a 256-wide
// launch) spread over the cluster's CTAs instead of one SM (A/B switch; 64 = every variant).
// 32 measured faster on products (chi = 64/128/256: 20.9/35.6/56.9 -> 20.5/35.3/56.6 ms, identical
// pivots, profiles/r02zg_cta_maxe_ab.txt)
#ifndef ACI_CLUSTER_CTA_MAXE
#define ACI_CLUSTER_CTA_MAXE 32
#endif
// The hand-off pivot is a multiple of 4: phase 2 re-initialises the key mbarriers, and the body
// waits on mbarrier (k & 1) with parity (k >> 1) & 1, so its first two waits (steps K, K + 1) are
// on phase 0 of fresh mbarriers only if K % 4 == 0
__device__ __forceinline__ int ho_round(int K) { return (K + 3) & ~3; }
// Hand-off eligibility: K pivots before it, some after it, and room for the compacted block
__device__ __forceinline__ bool ho_ok(const LuArgs &A, int m, int n, int K) {
  const int mn = m < n ? m : n, kx = A.dims->kmax < mn ? A.dims->kmax : mn;
  return K > 0 && K < kx &&
         (size_t)(m - K) * (size_t)(n - K) <= (size_t)(2 * kMaxCTAs - 64) * (size_t)A.colcap * 2;
}
// Phase 1 on Gl CTAs with an EA1 x EB1 tile, then (if it reached pivot K) phase 2 on the first 16
// CTAs (one cluster) with an EA2 x EB2 tile (hand-off comment above prrlu_body)
template <int EA1, int EB1, int EA2, int EB2, int NWT>
__device__ __forceinline__ void ho_run(const LuArgs &A, PrrluSmem &S, int m, int n, int g, int Gl, int K) {
  constexpr int CS = 16;
  HoState hs{K, 0.0, 0.0, false};
  prrlu_body<EA1, EB1, NWT, 2, false, 1>(A, S, Gl, g, &hs);
  if (!hs.handed || g >= CS) return;
  const int tid = threadIdx.x;
  if (tid < Gl) {  // every CTA's compacted entries are out
    const unsigned long long want = tagged(*A.epoch & 0xfffffu, 0xfffu);
    unsigned long long w0, w1;
    do {
      ld_pkt(A.keys + 2 * (kHoFlags / 2 + tid), w0, w1);
    } while (w0 != want);
    __threadfence();
  }
  unsigned *hw = ho_words(S);
  for (int i = tid; i < m; i += NWT * 32)
    if (!((hw[kHoDeadR + (i >> 5)] >> (i & 31)) & 1u)) hw[kHoRowMap + ho_rank(hw + kHoDeadR, hw + kHoPrefR, i)] = i;
  for (int j = tid; j < n; j += NWT * 32) {
    const int rj = ho_rank(hw + kHoDeadC, hw + kHoPrefC, j);
    if ((hw[kHoDeadC + (j >> 5)] >> (j & 31)) & 1u) hw[kHoDeadList + (j - rj)] = j;
    else hw[kHoColMap + rj] = j;
  }
  if (tid < 4) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&S.mb[tid])) : "memory");
  __syncthreads();
  prrlu_body<EA2, EB2, NWT, 2, false, 2>(A, S, CS, g, &hs);
}

template <int NWT, int XM, bool CPLX>
__global__ void __launch_bounds__(NWT * 32) prrlu_kernel(LuArgs A) {
  __shared__ PrrluSmem S;
  const int m = A.dims->m, n = A.dims->n;
  const int g = blockIdx.x;
#define ACI_CTA_VARIANT(EA, EB)                                        \
  if (!(XM == 2 && !CPLX && (EA) * (EB) > ACI_CLUSTER_CTA_MAXE) &&     \
      m <= 32 * (EA) && n <= NWT * (EB)) {                              \
    if (g == 0) prrlu_body<(EA), (EB), NWT, 0, CPLX>(A, S, 1, 0);      \
    return;                                                            \
  }
#define ACI_GRID_VARIANT2(EA, EB)                                      \
  if (m <= 32 * (EA)) {                                                \
    int Gl = (n + NWT * (EB) - 1) / (NWT * (EB));                      \
    if (XM == 2) {                                                     \
      const int CS = (int)cluster_size();                              \
      Gl = (Gl + CS - 1) / CS * CS;                                    \
    }                                                                  \
    if (g < Gl) prrlu_body<(EA), (EB), NWT, XM, CPLX>(A, S, Gl, g);    \
    return;                                                            \
  }
  if constexpr (!CPLX) {
    ACI_CTA_VARIANT(1, 4)    //   32 x   32
    ACI_CTA_VARIANT(2, 8)    //   64 x   64
    ACI_CTA_VARIANT(4, 4)    //  128 x   32
    ACI_CTA_VARIANT(1, 16)   //   32 x  128
    ACI_CTA_VARIANT(4, 16)   //  128 x  128
    ACI_CTA_VARIANT(8, 8)    //  256 x   64
    ACI_CTA_VARIANT(2, 32)   //   64 x  256
    ACI_CTA_VARIANT(32, 2)   // 1024 x   16
#if ACI_NARROW128
    // 128-row blocks no wider than one cluster of 16-column CTAs (configs[3]: 128 x 256): 16 CTAs x
    // 8 entries per thread instead of 8 CTAs x 16
    if (n <= 16 * NWT * 2) {
      ACI_GRID_VARIANT2(4, 2)
    }
#endif
    ACI_GRID_VARIANT2(4, ACI_W8_EB128)   //  128 x 8*EB per CTA
    ACI_GRID_VARIANT2(8, ACI_W8_EB256)   //  256 x 8*EB per CTA
#if ACI_NARROW512
    // 512-row blocks no wider than one cluster of 16-column CTAs (configs[3]: 512 x 256, r = 256):
    // 16 CTAs x 32 entries per thread instead of 8 CTAs x 64 (the update + scan halves)
    if (n <= 16 * NWT * 2) {
#if ACI_HANDOFF
      // one cluster, 32 entries per thread: once the live block fits 384 x 128 (e.g. 512 x 256 at
      // pivot 128) it continues on 12 x 1 entries per thread
      if constexpr (XM == 2 && !CPLX) {
        const int K = ho_round(max(m - 384, n - 128));
        if (m > 256 && m <= 512 && cluster_size() == 16 && ho_ok(A, m, n, K)) {
          if (g < 16) ho_run<16, 2, 12, 1, NWT>(A, S, m, n, g, 16, K);
          return;
        }
      }
#endif
      ACI_GRID_VARIANT2(16, 2)
    }
#endif
#if ACI_HANDOFF
    // 257..512-row blocks that need two or more 16-CTA clusters: hand off to one cluster once the
    // live block fits kHoEA x kHoEB per thread (hand-off comment above prrlu_body)
    if constexpr (XM == 2 && !CPLX) {
      if (m > 256 && m <= 512) {
        const int CS = (int)cluster_size();
        int Gl = (n + NWT * ACI_W8_EB512 - 1) / (NWT * ACI_W8_EB512);
        Gl = (Gl + CS - 1) / CS * CS;
        const int K = ho_round(max(m - 32 * kHoEA, n - 16 * NWT * kHoEB));
        if (CS == 16 && Gl > CS && Gl <= 64 && ho_ok(A, m, n, K)) {
          if (g < Gl) ho_run<16, ACI_W8_EB512, kHoEA, kHoEB, NWT>(A, S, m, n, g, Gl, K);
          return;
        }
      }
    }
#endif
    ACI_GRID_VARIANT2(16, ACI_W8_EB512)  //  512 x 8*EB per CTA
    ACI_GRID_VARIANT2(32, ACI_BIG_EB)    // 1024 x 8*EB per CTA
  } else {
    // complex entries take two registers: at most 32 entries per thread
    ACI_CTA_VARIANT(1, 8)    //   32 x   64
    ACI_CTA_VARIANT(2, 8)    //   64 x   64
    ACI_CTA_VARIANT(4, 4)    //  128 x   32
    ACI_CTA_VARIANT(1, 16)   //   32 x  128
    ACI_CTA_VARIANT(4, 8)    //  128 x   64
    ACI_CTA_VARIANT(2, 16)   //   64 x  128
    ACI_CTA_VARIANT(8, 4)    //  256 x   32
    ACI_CTA_VARIANT(16, 2)   //  512 x   16
    ACI_GRID_VARIANT2(4, 4)  //  128 x 32 per CTA
    ACI_GRID_VARIANT2(8, 2)  //  256 x 16 per CTA
    ACI_GRID_VARIANT2(16, 2) //  512 x 16 per CTA
  }
#undef ACI_CTA_VARIANT
#undef ACI_GRID_VARIANT2
}

// Single-cluster mode (aci_options.concurrent): every grid variant uses
// exactly one 16-CTA cluster (gang-scheduled by the hardware), so prrLU launches of products
// running concurrently on other streams can never hold part of each other's participants while
// spinning. More columns per CTA than the default tiers where needed to fit 16 CTAs.
template <int NWT, bool CPLX>
__global__ void __launch_bounds__(NWT * 32) prrlu_kernel_one(LuArgs A) {
  __shared__ PrrluSmem S;
  const int m = A.dims->m, n = A.dims->n;
  const int g = blockIdx.x;
#define ACI_CTA_VARIANT(EA, EB)                                        \
  if (m <= 32 * (EA) && n <= NWT * (EB)) {                              \
    if (g == 0) prrlu_body<(EA), (EB), NWT, 0, CPLX>(A, S, 1, 0);      \
    return;                                                            \
  }
#define ACI_ONE_VARIANT(EA, EB)                                        \
  if (m <= 32 * (EA) && n <= 16 * NWT * (EB)) {                         \
    prrlu_body<(EA), (EB), NWT, 2, CPLX>(A, S, 16, g);                 \
    return;                                                            \
  }
  if constexpr (!CPLX) {
    ACI_CTA_VARIANT(1, 4)
    ACI_CTA_VARIANT(2, 8)
    ACI_CTA_VARIANT(4, 4)
    ACI_CTA_VARIANT(1, 16)
    ACI_CTA_VARIANT(4, 16)
    ACI_CTA_VARIANT(8, 8)
    ACI_CTA_VARIANT(2, 32)
    ACI_CTA_VARIANT(32, 2)
    ACI_ONE_VARIANT(4, 8)    //  128 x 1024
    ACI_ONE_VARIANT(8, 4)    //  256 x  512
    ACI_ONE_VARIANT(16, 4)   //  512 x  512
    ACI_ONE_VARIANT(32, 2)   // 1024 x  256
  } else {
    ACI_CTA_VARIANT(1, 8)
    ACI_CTA_VARIANT(2, 8)
    ACI_CTA_VARIANT(4, 4)
    ACI_CTA_VARIANT(1, 16)
    ACI_CTA_VARIANT(4, 8)
    ACI_CTA_VARIANT(2, 16)
    ACI_CTA_VARIANT(8, 4)
    ACI_CTA_VARIANT(16, 2)
    ACI_ONE_VARIANT(4, 8)    //  128 x 1024
    ACI_ONE_VARIANT(8, 4)    //  256 x  512
    ACI_ONE_VARIANT(16, 2)   //  512 x  256
  }
#undef ACI_CTA_VARIANT
#undef ACI_ONE_VARIANT
}

// Push tier (real blocks up to 128 x 256, one 8-CTA cluster): every CTA pushes its candidate
// column into every cluster CTA's shared memory together with its key (cp.async.bulk DSMEM copy,
// complete_tx on the receiver's mbarrier), so the winner's column is local once the keys are in —
// no L2 round trip per pivot. Columns per CTA = 8 warps x EB. Measured per pivot
// (tools/prrlu_bench): 128 x 128 1.21 us against 1.49 us in one CTA; at 256 rows the 8 x 2 KB
// DSMEM pushes per CTA take ~1000 cycles and it loses to the 16-CTA L2 tier (1.88 vs 1.39 us).
template <int NWT>
__global__ void __launch_bounds__(NWT * 32) prrlu_kernel_push(LuArgs A) {
  __shared__ PrrluSmem S;
  const int m = A.dims->m, n = A.dims->n;
  const int g = blockIdx.x;
#define ACI_CTA_VARIANT(EA, EB)                                        \
  if (m <= 32 * (EA) && n <= NWT * (EB)) {                              \
    if (g == 0) prrlu_body<(EA), (EB), NWT, 0, false>(A, S, 1, 0);     \
    return;                                                            \
  }
#define ACI_PUSH_VARIANT(EA, EB)                                       \
  if (m <= 32 * (EA) && n <= kPushCS * NWT * (EB)) {                    \
    prrlu_body<(EA), (EB), NWT, 3, false>(A, S, kPushCS, g);           \
    return;                                                            \
  }
  ACI_CTA_VARIANT(1, 4)    //  32 x  32
  ACI_CTA_VARIANT(2, 8)    //  64 x  64
  ACI_PUSH_VARIANT(4, 2)   // 128 x 128
  ACI_PUSH_VARIANT(2, 4)   //  64 x 256
  ACI_PUSH_VARIANT(4, 4)   // 128 x 256
#undef ACI_CTA_VARIANT
#undef ACI_PUSH_VARIANT
}

constexpr int kNWT = 8;

static bool push_enabled() {
  static const bool on = [] {
    const char *e = getenv("ACI_PRRLU_PUSH");
    return !e || atoi(e) != 0;
  }();
  return on;
}

// A cooperative launch would gang-schedule a multi-cluster grid: tools/probe/coop_spin.cu measured
// (profiles/r02_coop_spin.txt) that a cooperative cluster launch larger than the co-resident
// cluster count is refused rather than split into waves. But the multi-cluster prrLU launched
// cooperatively inside the captured iteration crashed the host process (SIGSEGV,
// profiles/r02d_ab.txt, chi = 256), so it is not used: multi-cluster grids stay plain cluster
// launches, serialised across host threads by the library (aci.cu) and checked for co-residency
// once (cluster_choice).
bool fits_one_cta(int m, int n, bool cplx) {
  const int v8[][2] = {{1, 4}, {2, 8}, {4, 4}, {1, 16}, {4, 16}, {8, 8}, {2, 32}, {32, 2}};
  const int z8[][2] = {{1, 8}, {2, 8}, {4, 4}, {1, 16}, {4, 8}, {2, 16}, {8, 4}, {16, 2}};
  for (int t = 0; t < 8; ++t) {
    const int *e = cplx ? z8[t] : v8[t];
    if (m <= 32 * e[0] && n <= kNWT * e[1]) return true;
  }
  return false;
}

// Cluster size of the XM = 2 launch, chosen once. Every participating cluster spins on the others
// (cross-cluster exchange), so ALL clusters a live block can use must be co-resident: the widest
// grid variant uses ceil(kMaxCTAs * 8 / 16) = 74 CTAs (16 columns per CTA at the envelope's 1184
// columns). 16-CTA clusters (non-portable) if ceil(74 / 16) of them fit at once for both the real
// and the complex kernel, else 8-CTA clusters under the same rule, else 0 = the cooperative L2
// tier (co-residency guaranteed by the cooperative launch). ACI_PRRLU_CLUSTER=0/8/16 restricts
// the choice (measurements). Measured on this pool: 7 co-resident 16-CTA clusters, 15 8-CTA ones.
constexpr int kWidestGrid = (kMaxCTAs * 8 + 15) / 16;

static int cluster_choice_once() {
  int cs = -1;
  auto active = [&](const void *kern, int c) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c * 8);
    cfg.blockDim = dim3(kNWT * 32);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return n;
  };
  auto fits = [&](int c) {
    const int need = (kWidestGrid + c - 1) / c;
    return active((const void *)prrlu_kernel<kNWT, 2, false>, c) >= need &&
           active((const void *)prrlu_kernel<kNWT, 2, true>, c) >= need;
  };
  const char *env = getenv("ACI_PRRLU_CLUSTER");
  int want = env ? atoi(env) : 16;
  cs = 0;
  if (want >= 16 && fits(16)) cs = 16;
  else if (want >= 8 && fits(8)) cs = 8;
  return cs;
}

// thread-safe one-time choice (C++11 function-local static initialisation)
int cluster_choice() {
  static const int cs = cluster_choice_once();
  return cs;
}

}  // namespace

bool prrlu_coop_multicluster() { return true; }  // the cooperative L2 grid tier serves concurrent mode

bool prrlu_supported_one(int m, int n, bool cplx) {
  if (fits_one_cta(m, n, cplx)) return true;
  const int v[][2] = {{128, 1024}, {256, 512}, {512, 512}, {1024, 256}};
  const int z[][2] = {{128, 1024}, {256, 512}, {512, 256}};
  if (cplx) {
    for (auto &e : z)
      if (m <= e[0]) return n <= e[1];
  } else {
    for (auto &e : v)
      if (m <= e[0]) return n <= e[1];
  }
  return false;
}

// rook envelope: prrlu_kernel_rook's variants (one CTA, or one 16-CTA cluster up to 512 rows)
static bool rook_fits_cta(int m, int n) {
  const int cta[][2] = {{32, 32}, {64, 64}, {128, 32}, {32, 128}, {128, 128}, {256, 64}, {64, 256}};
  for (auto &e : cta)
    if (m <= e[0] && n <= e[1]) return true;
  return false;
}
bool prrlu_supported_rook(int m, int n) {
  if (rook_fits_cta(m, n)) return true;
  const int one[][2] = {{128, 1024}, {256, 512}, {512, 512}};
  for (auto &e : one)
    if (m <= e[0]) return n <= e[1];
  return false;
}

bool prrlu_supported(int max_m, int max_n, bool cplx) {
  if (fits_one_cta(max_m, max_n, cplx)) return true;
  if (cplx) return max_m <= 512 && (max_n + 15) / 16 <= 64;
  return max_m <= kMaxRows && (max_n + 7) / 8 <= kMaxCTAs;
}

void prrlu_envelope(int *max_rows, int *max_cols) {
  *max_rows = kMaxRows;
  *max_cols = kMaxCTAs * 8;
}

int prrlu_col_spread() { return kColSpread; }

size_t prrlu_exchange_bytes(int max_m, int max_n) {
  (void)max_n;
  int cap = max_m < kMaxRows ? kMaxRows : max_m;
  return (size_t)2 * kMaxCTAs * cap * 16 + 2 * kMaxCTAs * 32 + 256;
}

// Kernel attributes, set once before any stream capture: the push tier's static + dynamic shared
// memory exceeds the 48 KB default; 16-CTA clusters need the non-portable size.
static int attr_once() {
  cudaFuncSetAttribute((const void *)prrlu_kernel_push<kNWT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kPushSmem);
  // 16-CTA clusters are a non-portable size
  const void *k16[] = {(const void *)prrlu_kernel<kNWT, 2, false>, (const void *)prrlu_kernel<kNWT, 2, true>,
                       (const void *)prrlu_kernel_one<kNWT, false>, (const void *)prrlu_kernel_one<kNWT, true>,
                       (const void *)prrlu_kernel_rook<kNWT>};
  for (const void *f : k16) cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return 0;
}

void prrlu_init() {
  cluster_choice();
  static const int once = attr_once();
  (void)once;
}

// Every variant goes through cudaLaunchKernelEx so that a launch-completion event (fired once all
// CTAs have begun executing) can be attached: the sweep forks its look-ahead GEMM off it, onto the
// SMs the prrLU does not hold (aci.cu bond_update).
template <bool CPLX>
static cudaError_t launch_prrlu_t(const LuArgs &a, int max_m, int max_n, cudaStream_t st, bool one, cudaEvent_t started,
                                  bool rook) {
  LuArgs args = a;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kNWT * 32);
  cfg.stream = st;
  cudaLaunchAttribute at[3];
  int na = 0;
  auto cluster = [&](int cs) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cs;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  };
  if (started) {
    at[na].id = cudaLaunchAttributeLaunchCompletionEvent;
    at[na].val.launchCompletionEvent.event = started;
    at[na].val.launchCompletionEvent.flags = 0;
    ++na;
  }
  cfg.attrs = at;
  if (rook) {  // NEXT-4: one CTA or one 16-CTA cluster (prrlu_supported_one), real values
    if (CPLX || !prrlu_supported_rook(max_m, max_n)) return cudaErrorNotSupported;
    const bool cta = rook_fits_cta(max_m, max_n);
    cfg.gridDim = dim3(cta ? 1 : 16);
    if (!cta) cluster(16);
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, prrlu_kernel_rook<kNWT>, args);
  }
  if (!CPLX && !fits_one_cta(max_m, max_n, CPLX) && max_m <= kPushRows && max_n <= kPushCS * kNWT * 4 &&
      push_enabled()) {
    cfg.gridDim = dim3(kPushCS);
    cfg.dynamicSmemBytes = kPushSmem;
    cluster(kPushCS);
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, prrlu_kernel_push<kNWT>, args);
  }
  if (one && !fits_one_cta(max_m, max_n, CPLX) && prrlu_supported_one(max_m, max_n, CPLX)) {
    cfg.gridDim = dim3(16);
    cluster(16);
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, prrlu_kernel_one<kNWT, CPLX>, args);
  }
  if (fits_one_cta(max_m, max_n, CPLX)) {
    cfg.gridDim = dim3(1);
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, prrlu_kernel<kNWT, 1, CPLX>, args);
  }
  // every grid variant holds at least 8 warps x 2 columns per CTA (ACI_W8_EB* / ACI_BIG_EB >= 2;
  // complex: EB >= 2), so ceil(max_n / 16) CTAs cover any live block (ACI_PRRLU_G8=1: the round-1
  // sizing of 8 columns per CTA, for A/B)
  static const int cols_per_cta = [] {
    const char *e = getenv("ACI_PRRLU_G8");
    return (e && atoi(e) != 0) ? kNWT : 2 * kNWT;
  }();
  int G = (max_n + cols_per_cta - 1) / cols_per_cta;
  // concurrent mode beyond one cluster: the L2 grid tier, launched cooperatively (gang-scheduled:
  // the whole grid is resident or none of it), so products running concurrently cannot hold part
  // of each other's spinning CTAs; multi-cluster launches are not gang-scheduled
  const int cs = one ? 0 : cluster_choice();
  if (cs > 0) {
    G = (G + cs - 1) / cs * cs;
    cfg.gridDim = dim3(G);
    cluster(cs);
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, prrlu_kernel<kNWT, 2, CPLX>, args);
  }
  cudaMemsetAsync(a.counter, 0, sizeof(unsigned), st);
  cfg.gridDim = dim3(G);
  at[na].id = cudaLaunchAttributeCooperative;
  at[na].val.cooperative = 1;
  ++na;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, prrlu_kernel<kNWT, 1, CPLX>, args);
}

cudaError_t launch_prrlu(const LuArgs &a, int max_m, int max_n, cudaStream_t st, bool cplx, bool one,
                         cudaEvent_t started, bool rook) {
  return cplx ? launch_prrlu_t<true>(a, max_m, max_n, st, one, started, rook)
              : launch_prrlu_t<false>(a, max_m, max_n, st, one, started, rook);
}
