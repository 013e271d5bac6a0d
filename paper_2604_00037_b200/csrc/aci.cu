// libaci.so: TT objects, the ACI sweep controller (Alg. 1) and the small kernels of
// the 2-site update (planning, index-set / frame update, convergence, output cores, evaluation).
// The GEMMs are in gemm.cu, the prrLU in prrlu.cu. The host code below only computes static
// capacities and enqueues kernels: live ranks chi'_l never leave the device during a sweep
// (one word per iteration is read back for the convergence test).
//
// Streams per call: the caller's stream carries the critical path of every bond (Pi GEMM ->
// prrLU -> update kernel); a side stream runs the look-ahead GEMM that produces the next bond's
// operand beside the prrLU (forked off the prrLU's launch-completion event, joined by the
// update) and, for large L->R bonds, the streamed Pi of the next bond (pi_stream_kernel: rows of
// Pi_{b+1} as the prrLU publishes the pivot rows they need); a third stream runs the index-set /
// log kernel of each bond (joined before the convergence test). One iteration of all three is
// captured as one CUDA graph and cached.
// Memory: a persistent per-stream workspace (stable address -> graph-cache hits) and a
// stream-ordered pool for TT cores.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <atomic>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: named host ranges for profilers (ncu --nvtx)

#include "../../include/aci.h"
#include "aci_common.cuh"

// RAII NVTX range over host enqueue phases (the device work they enqueue shows up under them in
// ncu --nvtx / nsys); no effect without a profiler attached
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

// ============================================================================ errors
static thread_local std::string g_err;
static int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}
#define CUDA_TRY(x)                                                                                 \
  do {                                                                                              \
    cudaError_t e_ = (x);                                                                           \
    if (e_ != cudaSuccess) return fail(ACI_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

extern "C" const char *aci_last_error(void) { return g_err.c_str(); }
extern "C" const char *aci_version(void) { return "aci-b200 0.1 (sm_100a, FP64 DMMA + register-resident prrLU)"; }

// ============================================================================ TT objects
struct tt_s {
  int L = 0;
  int cplx = 0;             // 1: complex cores, interleaved (re, im) doubles
  std::vector<int> d, ranks;
  std::vector<size_t> off;  // L+1 offsets (doubles; 2 per complex entry)
  double *dcores = nullptr;
  size_t total = 0;
  int dev = 0;              // device the cores live on
  int pooled = 0;           // 1: dcores came from core_pool()
};

// The library's own stream (per host thread), used when the caller passes NULL.
static cudaStream_t lib_stream() {
  static thread_local cudaStream_t s = nullptr;
  if (!s) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  return s;
}

// Core storage comes from a library-owned stream-ordered pool per device that never returns
// memory to the driver (release threshold = max): an output reuses the pages of the TT destroyed
// before it instead of paying for fresh page mappings (a fresh cudaMalloc of the 160 MB
// chi = 256 output measured 0-95 ms on top of a 72 ms product).
static cudaMemPool_t core_pool() {
  constexpr int kMaxDev = 64;
  static std::mutex mu;
  static cudaMemPool_t pools[kMaxDev] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev) return nullptr;
  std::lock_guard<std::mutex> g(mu);
  if (!pools[dev]) {
    cudaMemPoolProps pp = {};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = dev;
    if (cudaMemPoolCreate(&pools[dev], &pp) != cudaSuccess) { pools[dev] = nullptr; cudaGetLastError(); return nullptr; }
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
  }
  return pools[dev];
}

static cudaError_t core_alloc(tt_s *t, size_t bytes, cudaStream_t st) {
  cudaGetDevice(&t->dev);
  cudaMemPool_t pool = core_pool();
  t->pooled = pool != nullptr;
  if (!pool) return cudaMalloc(&t->dcores, bytes);
  return cudaMallocFromPoolAsync((void **)&t->dcores, bytes, pool, st);
}

// Back to the pool, stream-ordered on the library stream. Every library call that touches a TT
// has completed its work on it before returning, so nothing of ours can still read the cores;
// work the caller enqueued on tt_device_cores() must be complete (aci.h). No device-wide
// synchronisation: from a host thread it breaks stream captures running in other threads
// (measured: driver crashes in concurrent-mode stress, tools/conc_stress.py).
static void core_free(tt_s *t) {
  if (!t->dcores) return;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != t->dev) cudaSetDevice(t->dev);
  if (t->pooled) {
    cudaFreeAsync(t->dcores, lib_stream());
    cudaStreamSynchronize(lib_stream());
  } else {
    cudaFree(t->dcores);
  }
  if (cur != t->dev) cudaSetDevice(cur);
  t->dcores = nullptr;
}

static int check_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return fail(ACI_ERR_CUDA, "no CUDA device (libaci has no CPU fallback)");
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) return fail(ACI_ERR_CUDA, "libaci is built for sm_100a only");
  return ACI_OK;
}

static int validate_shape(int L, const int *d, const int *ranks) {
  if (L < 1 || !d || !ranks) return fail(ACI_ERR_INVALID, "tt: L < 1 or null shape");
  if (ranks[0] != 1 || ranks[L] != 1) return fail(ACI_ERR_INVALID, "tt: boundary ranks must be 1");
  for (int s = 0; s < L; ++s) {
    if (d[s] < 1 || d[s] > 255) return fail(ACI_ERR_INVALID, "tt: local dimension out of 1..255");
    if (ranks[s] < 1) return fail(ACI_ERR_INVALID, "tt: rank < 1");
  }
  return ACI_OK;
}

static tt_s *tt_alloc_shape(int L, const int *d, const int *ranks, int cplx = 0) {
  tt_s *t = new tt_s;
  t->L = L;
  t->cplx = cplx;
  t->d.assign(d, d + L);
  t->ranks.assign(ranks, ranks + L + 1);
  t->off.resize(L + 1);
  size_t o = 0;
  for (int s = 0; s < L; ++s) {
    t->off[s] = o;
    o += (size_t)ranks[s] * d[s] * ranks[s + 1] * (cplx ? 2 : 1);
  }
  t->off[L] = o;
  t->total = o;
  return t;
}

// NaN/Inf scan of a device buffer (flag |= 1), so tt_create validates on the device after the
// upload instead of walking every host element before it.
__global__ void nonfinite_scan_kernel(const double *x, size_t n, int *flag) {
  int bad = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

static int tt_create_impl(int L, const int *d, const int *ranks, const double *const *cores, int cplx,
                          tt_t **out) {
  if (!out || !cores) return fail(ACI_ERR_INVALID, "tt_create: null argument");
  int st = validate_shape(L, d, ranks);
  if (st) return st;
  if ((st = check_device())) return st;
  for (int s = 0; s < L; ++s)
    if (!cores[s]) return fail(ACI_ERR_INVALID, "tt_create: null core");
  tt_s *t = tt_alloc_shape(L, d, ranks, cplx);
  // all cores enqueued back to back on the library stream (asynchronous DMA from pinned host
  // memory), then one device-side NaN/Inf scan and a single synchronisation
  cudaStream_t strm = lib_stream();
  if (core_alloc(t, sizeof(double) * std::max<size_t>(t->total, 1) + sizeof(int), strm) != cudaSuccess) {
    cudaGetLastError();
    delete t;
    return fail(ACI_ERR_OOM, "tt_create: device allocation failed");
  }
  int *flag = reinterpret_cast<int *>(t->dcores + std::max<size_t>(t->total, 1));
  cudaMemsetAsync(flag, 0, sizeof(int), strm);
  for (int s = 0; s < L; ++s)
    cudaMemcpyAsync(t->dcores + t->off[s], cores[s], sizeof(double) * (t->off[s + 1] - t->off[s]),
                    cudaMemcpyHostToDevice, strm);
  const size_t n = t->total;
  if (n) nonfinite_scan_kernel<<<(int)std::min<size_t>(1184, (n + 255) / 256), 256, 0, strm>>>(t->dcores, n, flag);
  int bad = 0;
  cudaMemcpyAsync(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost, strm);
  cudaError_t e = cudaStreamSynchronize(strm);
  if (e != cudaSuccess || bad) {
    core_free(t);
    delete t;
    if (e != cudaSuccess) return fail(ACI_ERR_CUDA, std::string("tt_create: ") + cudaGetErrorString(e));
    return fail(ACI_ERR_NONFINITE, "tt_create: NaN/Inf in core");
  }
  *out = t;
  return ACI_OK;
}

extern "C" int tt_create(int L, const int *d, const int *ranks, const double *const *cores, tt_t **out) {
  return tt_create_impl(L, d, ranks, cores, 0, out);
}

extern "C" int tt_create_z(int L, const int *d, const int *ranks, const double *const *cores, tt_t **out) {
  return tt_create_impl(L, d, ranks, cores, 1, out);
}

extern "C" int tt_is_complex(const tt_t *t) { return t ? t->cplx : 0; }

static int tt_create_device_impl(int L, const int *d, const int *ranks, const double *dev_cores, void *stream,
                                 int cplx, tt_t **out) {
  if (!out || !dev_cores) return fail(ACI_ERR_INVALID, "tt_create_device: null argument");
  int st = validate_shape(L, d, ranks);
  if (st) return st;
  if ((st = check_device())) return st;
  tt_s *t = tt_alloc_shape(L, d, ranks, cplx);
  cudaStream_t s = (cudaStream_t)stream;
  if (core_alloc(t, sizeof(double) * std::max<size_t>(t->total, 1), s) != cudaSuccess) {
    cudaGetLastError();
    delete t;
    return fail(ACI_ERR_OOM, "tt_create_device: device allocation failed");
  }
  cudaMemcpyAsync(t->dcores, dev_cores, sizeof(double) * t->total, cudaMemcpyDeviceToDevice, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    core_free(t);
    delete t;
    return fail(ACI_ERR_CUDA, std::string("tt_create_device: ") + cudaGetErrorString(e));
  }
  *out = t;
  return ACI_OK;
}

extern "C" int tt_create_device(int L, const int *d, const int *ranks, const double *dev_cores, void *stream,
                                tt_t **out) {
  return tt_create_device_impl(L, d, ranks, dev_cores, stream, 0, out);
}

extern "C" int tt_create_device_z(int L, const int *d, const int *ranks, const double *dev_cores, void *stream,
                                  tt_t **out) {
  return tt_create_device_impl(L, d, ranks, dev_cores, stream, 1, out);
}

extern "C" int tt_destroy(tt_t *t) {
  if (!t) return ACI_OK;
  core_free(t);
  delete t;
  return ACI_OK;
}

extern "C" int tt_shape(const tt_t *t, int *L, int *d, int *ranks) {
  if (!t || !L) return fail(ACI_ERR_INVALID, "tt_shape: null argument");
  *L = t->L;
  if (d) std::copy(t->d.begin(), t->d.end(), d);
  if (ranks) std::copy(t->ranks.begin(), t->ranks.end(), ranks);
  return ACI_OK;
}

extern "C" const double *tt_device_cores(const tt_t *t) { return t ? t->dcores : nullptr; }

extern "C" int tt_get_cores(const tt_t *t, double *const *host_cores) {
  if (!t || !host_cores) return fail(ACI_ERR_INVALID, "tt_get_cores: null argument");
  for (int s = 0; s < t->L; ++s)
    if (!host_cores[s]) return fail(ACI_ERR_INVALID, "tt_get_cores: null core buffer");
  cudaStream_t strm = lib_stream();
  for (int s = 0; s < t->L; ++s)
    cudaMemcpyAsync(host_cores[s], t->dcores + t->off[s], sizeof(double) * (t->off[s + 1] - t->off[s]),
                    cudaMemcpyDeviceToHost, strm);
  CUDA_TRY(cudaStreamSynchronize(strm));
  return ACI_OK;
}

// ============================================================================ small kernels

// V'[p][beta] = W[p][sigma_p * r1 + beta]  (selection after W = V * X_s viewed r0 x (d r1))
__global__ void eval_select_kernel(const double *W, double *V, const uint8_t *idx, int L, int s, int d, int r1,
                                   int64_t np) {
  const int64_t tot = np * r1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = t / r1;
    int b = (int)(t - p * r1);
    int sg = idx[p * L + s];
    V[t] = W[p * (int64_t)d * r1 + (int64_t)sg * r1 + b];
  }
}

__global__ void eval_first_kernel(const double *X0, double *V, const uint8_t *idx, int L, int r1, int64_t np) {
  const int64_t tot = np * r1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = t / r1;
    int b = (int)(t - p * r1);
    V[t] = X0[(int64_t)idx[p * L] * r1 + b];
  }
}

__global__ void eval_desc_kernel(GemmDesc *desc, const double *V, const double *X, double *W, int np, int r0,
                                 int dr1) {
  GemmDesc D = {};
  D.C = W; D.M = np; D.N = dr1; D.ldc = dr1; D.nin = 1;
  D.A[0] = V; D.lda[0] = r0; D.K[0] = r0;
  D.B[0] = X; D.ldb[0] = dr1;
  *desc = D;
}

// ---------------------------------------------------------------------------- sweep state
// Static (host-known) pointers and dims of one bond for one input.
struct InBond {
  const double *Xb, *Xb1;
  const double *Rnext;  // R^n_{b+2} (chi_{b+2} x rmax[b+1], ld ldR) of the canonicalisation; null at
                        // b == L-2 (R_L = [1]); read once, for the first L->R half-sweep's B^n_b
  int ldR;
  double *Ast, *Bst;    // this bond's Pi operands A^n_b (null at b == 0: X^n_0) and B^n_b (null at
                        // b == L-2: X^n_{L-1}), kept across half-sweeps
  double *Ahat, *Bhat;  // look-ahead scratch (A^n_b X^n_{b+1} in L->R, X^n_b B^n_b in R->L)
  const double *Xeb, *Xeb1;  // complex runs: expanded cores of sites b, b+1 (right operands)
  int c0, c1, c2;       // chi^n_b, chi^n_{b+1}, chi^n_{b+2}
};
struct alignas(8) BondStatic {
  int b, L, N, dir, db, db1;
  int Z;                // 1 real, 2 complex (interleaved left operands, expanded right operands)
  int ldu;              // static ld of the U store (nmax[b])
  int maxrank;
  InBond in[ACI_GEMM_MAX_IN];
  double *Pi;
};

// Complex runs (S.Z = 2) use the same real GEMMs: a complex left operand (M x K) is read as the
// real M x 2K matrix of its interleaved storage, a right operand is stored 2x2-block expanded
// (2K x 2N), so K and N double; a2's result is written expanded (EPI_STORE_X, xd = d_{b+1}).
// a2: B^n = X^n_{b+1} R^n_{b+2} : (c1 db1 x c2) (c2 x rr) -> (c1 db1) x rr == c1 x (db1 rr)
__device__ __forceinline__ GemmDesc desc_b(const BondStatic &S, const InBond &I, int rr, double *C) {
  GemmDesc bb = {};
  if (!I.Rnext) return bb;
  const int z = S.Z;
  bb.C = C; bb.M = I.c1 * S.db1; bb.N = z * rr; bb.nin = 1;
  bb.ldc = z == 2 ? 2 * S.db1 * rr : rr;  // expanded c1 x (db1 rr) block matrix
  bb.xd = S.db1;
  bb.A[0] = I.Xb1; bb.lda[0] = z * I.c2; bb.K[0] = z * I.c2; bb.B[0] = I.Rnext; bb.ldb[0] = z * I.ldR;
  return bb;
}

// Live sizes -> the a3+a4 descriptor, the prrLU dims and the look-ahead GEMM of one bond update.
// Pi's operands are stored per bond: A^n_b is written by the L->R update of bond b-1, B^n_b by the
// R->L update of bond b+1 (before the first iteration: by a one-time launch from the canonical R
// frames, plan_pre_kernel). The look-ahead computes, while this bond's prrLU runs on its own SMs,
// the product whose rows (L->R) or columns (R->L) the new pivots select as the next bond's operand:
//   L->R: A^n_{b+1} = L^n_b X^n_{b+1} = (A^n_b X^n_{b+1})[I_b rows]       (L^n_b = A^n_b[I_b])
//   R->L: B^n_{b-1} = X^n_b R^n_{b+1} = (X^n_b B^n_b)[:, J_{b+1} cols]     (R^n_{b+1} = B^n_b[:, J])
// so no GEMM sits between the update of one bond and the Pi of the next. An L->R bond reads B^n_b
// of the previous R->L half-sweep and an R->L bond A^n_b of this iteration's L->R (R20).
__device__ void plan_bond_r(const BondStatic &S, int rl, int rr, GemmDesc *ab, GemmDesc *pi, LuDims *lu) {
  const int b = S.b;
  const int m = rl * S.db, n = S.db1 * rr;
  const int z = S.Z;
  GemmDesc P = {};
  P.C = S.Pi; P.M = m; P.N = z * n; P.ldc = z * n; P.nin = S.N;
  for (int i = 0; i < S.N; ++i) {
    const InBond &I = S.in[i];
    // a3: Pi^n = A^n B^n : (m x c1) (c1 x n)
    P.A[i] = b > 0 ? I.Ast : I.Xb;
    P.lda[i] = z * I.c1;
    P.K[i] = z * I.c1;
    P.B[i] = b + 2 < S.L ? I.Bst : (z == 2 ? I.Xeb1 : I.Xb1);
    P.ldb[i] = z * n;
    GemmDesc h = {};
    if (S.dir == 0 && b + 2 < S.L) {
      // (m x c1) (c1 x db1 c2) -> m x (db1 c2); complex: interleaved rows, expanded X
      h.C = I.Ahat; h.M = m; h.N = z * S.db1 * I.c2; h.ldc = h.N; h.nin = 1;
      h.A[0] = P.A[i]; h.lda[0] = z * I.c1; h.K[0] = z * I.c1;
      h.B[0] = z == 2 ? I.Xeb1 : I.Xb1; h.ldb[0] = z * S.db1 * I.c2;
    } else if (S.dir == 1 && b > 0) {
      // (c0 db x c1) (c1 x n) -> (c0 db) x n == c0 x (db n); complex: written expanded (xd = db)
      h.C = I.Bhat; h.M = I.c0 * S.db; h.N = z * n; h.ldc = z == 2 ? 2 * S.db * n : n; h.xd = S.db; h.nin = 1;
      h.A[0] = I.Xb; h.lda[0] = z * I.c1; h.K[0] = z * I.c1;
      h.B[0] = P.B[i]; h.ldb[0] = z * n;
    }
    ab[i] = h;
  }
  *pi = P;
  LuDims D;
  D.m = m; D.n = n; D.ldm = n;
  D.kmax = min(S.maxrank, min(m, n));
  D.ldu = S.ldu;
  *lu = D;
}

__device__ __forceinline__ void plan_bond(const BondStatic &S, const int *rk, GemmDesc *ab, GemmDesc *pi, LuDims *lu) {
  plan_bond_r(S, rk[S.b], rk[S.b + 2], ab, pi, lu);
}

__global__ void plan_bond_kernel(const BondStatic *S, const int *rk, GemmDesc *ab, GemmDesc *pi, LuDims *lu) {
  plan_bond(*S, rk, ab, pi, lu);
}

// Descriptors of B^n_b = X^n_{b+1} R^n_{b+2} for every bond b = 0..L-3 from the canonical R frames
// (once per product, before the first L->R half-sweep), one thread per (bond, input).
__global__ void plan_pre_kernel(const BondStatic *S, int nb, int N, const int *rk, GemmDesc *pre) {
  for (int t = threadIdx.x; t < nb * N; t += blockDim.x) {
    const int b = t / N, i = t % N;
    const BondStatic &B = S[b];
    const InBond &I = B.in[i];
    pre[t] = desc_b(B, I, rk[b + 2], I.Bst);
  }
}


struct UpdateArgs {
  int b, dir, L, N, db, db1;
  const int *rows, *cols;     // pivots of this bond
  const int *r_in;            // accepted pivots
  const double *eps_in;
  int *rk;
  uint8_t *Iprev, *Inew;      // Imi[b-1] (rmax[b-1] x b), Imi[b] (rmax[b] x (b+1))
  uint8_t *Jnext, *Jnew;      // Jmi[b+2] (x (L-b-2)), Jmi[b+1] (x (L-b-1))
  const double *Ahat[ACI_GEMM_MAX_IN];  // L->R: A^n_b X^n_{b+1} (m x W doubles)
  double *Anext[ACI_GEMM_MAX_IN];       // A^n_{b+1} = Ahat[I_b rows] (r x W); null at b == L-2
  int W[ACI_GEMM_MAX_IN];               // Z d_{b+1} chi^n_{b+2}
  const double *Bhat[ACI_GEMM_MAX_IN];  // R->L: X^n_b B^n_b ((c0 d_b) x n; complex expanded, ld 2 d_b n)
  double *Bprev[ACI_GEMM_MAX_IN];       // B^n_{b-1} = Bhat[:, J cols] (c0 x d_b r); null at b == 0
  int c0[ACI_GEMM_MAX_IN];
  const double *Pi;           // for Y_0 at b == 0 (R->L)
  double *Y0;                 // d_0 x rmax[0], ld = r
  unsigned long long *maxeps_bits;
  const unsigned long long *scale_bits;
  // per-update log (slot = iteration * per_iter + step; the iteration counter lives on the
  // device so one captured CUDA graph serves every iteration)
  int *log_info;              // 5 ints per slot
  double *log_es;             // 2 doubles per slot
  int *log_rows, *log_cols;   // cap_piv per slot
  const int *iter;
  int step, per_iter, cap_piv;
  int Z;                      // 2: complex (L frames / A^n interleaved, R frames / B^n expanded)
  // plan of the next bond update (fused; null for the last update of an iteration)
  const BondStatic *next;
  GemmDesc *ab, *pi;
  LuDims *lu;
  int *info;                  // 8 ints: this bond's (rl, rr, r, -, s bits) for index_bond_kernel
  int next_b;                 // bond index of `next` (-1: none)
  // streamed Pi: non-null = the stream of Pi_{b+1} took the snapshot of s and merges its max |Pi|
  // (this kernel runs beside it and leaves s alone)
  unsigned long long *sp;
  unsigned long long *ts;  // development timestamps (ACI_STREAM_TS builds only)
};

// Index-set update (a6, R21) and frame update (a7: the rows/columns of A^n / B^n the
// new pivots select — the same numbers Alg. 5 recomputes).
// ACI_PDL_UPDATE (A/B switch): the update kernel is launched as a programmatic dependent of the
// prrLU (it may be scheduled before the prrLU grid ends and waits in griddepcontrol.wait, which
// returns once the prrLU grid has completed and its memory is visible)
#ifndef ACI_PDL_UPDATE
#define ACI_PDL_UPDATE 0
#endif
__global__ void update_bond_kernel(UpdateArgs U) {
#if ACI_PDL_UPDATE
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
#ifdef ACI_STREAM_TS
  if (U.ts && U.dir == 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    U.ts[16 * U.b + 5] = t;  // update start
    U.ts[16 * U.b + 6] = *U.r_in;
  }
#endif
  const int r = *U.r_in;
  const int b = U.b, L = U.L;
  const int rl = U.rk[b], rr = U.rk[b + 2];
  const int n = U.db1 * rr;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  const size_t slot = (size_t)(*U.iter) * U.per_iter + U.step;
  // warp 0 stages the next update's static description in shared memory with one coalesced pass
  // (the planner's field-by-field reads from global memory were a ~15k-cycle dependent chain)
  __shared__ BondStatic s_next;
  if (blockIdx.x == 0 && threadIdx.x < 32 && U.next) {
    const unsigned long long *src = reinterpret_cast<const unsigned long long *>(U.next);
    unsigned long long *dst = reinterpret_cast<unsigned long long *>(&s_next);
    for (int t = threadIdx.x; t < (int)(sizeof(BondStatic) / 8); t += 32) dst[t] = src[t];
    __syncwarp();
  }
  // the next bond's ranks, loaded together with r (rk[b+1], which this kernel writes, is r)
  const int nb = U.next_b;
  const int rl2 = nb >= 0 ? (nb == b + 1 ? r : U.rk[nb]) : 0;
  const int rr2 = nb >= 0 ? (nb + 2 == b + 1 ? r : U.rk[nb + 2]) : 0;
  if (gt == 0) {
    U.rk[b + 1] = r;
    if (U.next) plan_bond_r(s_next, rl2, rr2, U.ab, U.pi, U.lu);
    // sizes and s as this bond saw them, for index_bond_kernel (which may trail the sweep while
    // later bonds rewrite rk and s)
    U.info[0] = rl; U.info[1] = rr; U.info[2] = r;
    if (!U.sp) *reinterpret_cast<unsigned long long *>(U.info + 4) = *U.scale_bits;
  }
  (void)L;
  (void)slot;
  if (U.dir == 0) {
    // A^n_{b+1}[k][:] = Ahat[rows[k]][:] (a row of the look-ahead product is (sigma', beta) of
    // the next bond's (k, sigma') x beta operand)
    for (int i = 0; i < U.N; ++i) {
      if (!U.Anext[i]) continue;
      const int W = U.W[i];
      for (int t = gt; t < r * W; t += gs) {
        const int k = t / W, j = t - k * W;
        U.Anext[i][t] = U.Ahat[i][(size_t)U.rows[k] * W + j];
      }
    }
  } else {
    const int db = U.db;
    for (int i = 0; i < U.N; ++i) {
      if (!U.Bprev[i]) continue;
      const int c0 = U.c0[i];
      if (U.Z == 1) {
        // B^n_{b-1}[alpha][sigma r + k] = Bhat[alpha db + sigma][cols[k]]
        for (int t = gt; t < c0 * db * r; t += gs) {
          const int row = t / r, k = t - row * r;
          U.Bprev[i][t] = U.Bhat[i][(size_t)row * n + U.cols[k]];
        }
      } else {
        // expanded 2x2 blocks: rows 2 alpha + {0,1}, columns 2 (sigma x + k) + {0,1}
        for (int t = gt; t < 2 * c0 * db * r; t += gs) {
          const int a2 = t / (db * r), rem = t - a2 * (db * r), sg = rem / r, k = rem - sg * r;
          const double *src = U.Bhat[i] + (size_t)a2 * 2 * db * n + 2 * ((size_t)sg * n + U.cols[k]);
          double *dst = U.Bprev[i] + (size_t)a2 * 2 * db * r + 2 * ((size_t)sg * r + k);
          dst[0] = src[0];
          dst[1] = src[1];
        }
      }
    }
    if (b == 0) {
      const int m = rl * U.db;
      if (U.Z == 1) {
        for (int t = gt; t < m * r; t += gs) {
          const int ii = t / r, k = t % r;
          U.Y0[t] = U.Pi[(size_t)ii * n + U.cols[k]];
        }
      } else {
        for (int t = gt; t < m * r; t += gs) {
          const int ii = t / r, k = t % r;
          U.Y0[2 * t] = U.Pi[((size_t)ii * n + U.cols[k]) * 2];
          U.Y0[2 * t + 1] = U.Pi[((size_t)ii * n + U.cols[k]) * 2 + 1];
        }
      }
    }
  }
}


// Index-set update (a6, R21), the error bookkeeping (a9) and the pivot log of one bond.
// Nothing on the sweep's critical path reads them, so this runs on a side stream after the
// bond's update kernel (whose snapshot of the bond's sizes and s it reads) and overlaps the next
// bonds; the iteration joins it before the convergence test.
struct IndexArgs {
  int b, dir, L, db;
  const int *rows, *cols, *info;
  const double *eps_in;
  uint8_t *Iprev, *Inew, *Jnext, *Jnew;
  unsigned long long *maxeps_bits;
  int *log_info;
  double *log_es;
  int *log_rows, *log_cols;
  const int *iter;
  int step, per_iter, cap_piv;
};
__global__ void index_bond_kernel(IndexArgs U) {
  const int rl = U.info[0], rr = U.info[1], r = U.info[2];
  const int b = U.b, L = U.L;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  const size_t slot = (size_t)(*U.iter) * U.per_iter + U.step;
  if (gt == 0) {
    const double eps = *U.eps_in;
    atomicMax(U.maxeps_bits, (unsigned long long)__double_as_longlong(eps));
    int *li = U.log_info + slot * 5;
    li[0] = b; li[1] = U.dir; li[2] = rl; li[3] = rr; li[4] = r;
    U.log_es[slot * 2] = eps;
    U.log_es[slot * 2 + 1] = __longlong_as_double(*reinterpret_cast<const long long *>(U.info + 4));
  }
  for (int k = gt; k < r; k += gs) {
    U.log_rows[slot * U.cap_piv + k] = U.rows[k];
    U.log_cols[slot * U.cap_piv + k] = U.cols[k];
  }
  // multi-indices: I_b[k] = (I_{b-1}[row / d_b], row % d_b); J_{b+1}[k] = (col / rr, J_{b+2}[col % rr])
  for (int t = gt; t < r * (b + 1); t += gs) {
    const int k = t / (b + 1), pos = t % (b + 1);
    const int row = U.rows[k];
    U.Inew[t] = pos == b ? (uint8_t)(row % U.db) : U.Iprev[(row / U.db) * b + pos];
  }
  const int wJ = L - b - 1;
  for (int t = gt; t < r * wJ; t += gs) {
    const int k = t / wJ, pos = t % wJ;
    const int col = U.cols[k];
    U.Jnew[t] = pos == 0 ? (uint8_t)(col / rr) : U.Jnext[(col % rr) * (wJ - 1) + pos - 1];
  }
}

// Convergence test after a full iteration (R10).
__global__ void converge_kernel(int *rk, int *prev, int L, unsigned long long *maxeps_bits,
                                const unsigned long long *scale_bits, double tol, int tol_mode, int *flag,
                                double *err_out, int *iter) {
  if (threadIdx.x != 0) return;
  *iter += 1;
  int grew = 0;
  for (int b = 0; b < L - 1; ++b) {
    if (rk[b + 1] > prev[b]) grew = 1;
    prev[b] = rk[b + 1];
  }
  const double s = __longlong_as_double((long long)*scale_bits);
  const double me = __longlong_as_double((long long)*maxeps_bits);
  const double thr = tol_mode == ACI_TOL_RELATIVE ? tol * s : tol;
  *flag = (!grew && me <= thr) ? 1 : 0;
  *err_out = tol_mode == ACI_TOL_RELATIVE ? (s > 0 ? me / s : 0.0) : me;
  *maxeps_bits = 0ull;
}

// ---- canonicalisation of y_init
struct CanonArgs {
  int s, L, N, ds;
  int yr_s;                       // rows of M (y_init left bond of site s)
  const double *M;                // Yabs[s] (or the original core at s = L-1), yr_s x (ds * rk[s+1])
  LuDims *lu;
  int maxrank;
  // R-frame temp GEMMs: T^n = X^n_s (c0 ds x c1) * R^n_{s+1} (c1 x rk[s+1], ld ldR) -> c0 x (ds rk[s+1])
  const double *Xs[ACI_GEMM_MAX_IN];
  const double *Rnext[ACI_GEMM_MAX_IN];  // null at s = L-1
  int ldR;
  double *Tbuf[ACI_GEMM_MAX_IN];
  int c0[ACI_GEMM_MAX_IN], c1[ACI_GEMM_MAX_IN];
  GemmDesc *tdesc;                // N descriptors
  int Z;                          // 2: complex (R frames expanded, T interleaved)
};

__global__ void plan_canon_kernel(CanonArgs C, const int *rk) {
  const int jn = rk[C.s + 1];
  LuDims D;
  D.m = C.yr_s; D.n = C.ds * jn; D.ldm = D.n;
  D.kmax = min(C.maxrank, min(D.m, D.n));
  D.ldu = 0;
  *C.lu = D;
  for (int i = 0; i < C.N; ++i) {
    GemmDesc g = {};
    if (C.Rnext[i]) {
      g.C = C.Tbuf[i]; g.M = C.c0[i] * C.ds; g.N = C.Z * jn; g.ldc = C.Z * jn; g.nin = 1;
      g.A[0] = C.Xs[i]; g.lda[0] = C.Z * C.c1[i]; g.K[0] = C.Z * C.c1[i];
      g.B[0] = C.Rnext[i]; g.ldb[0] = C.Z * C.ldR;
    }
    C.tdesc[i] = g;
  }
}

struct CanonUpd {
  int s, L, N, ds, yr_s, yr_prev_rows;   // yr_prev_rows = yr[s-1] * d[s-1]
  const int *cols, *r_in;
  int *rk;
  uint8_t *Jnext, *Jnew;                 // Jmi[s+1] (x (L-s-1)), Jmi[s] (x (L-s))
  const double *M;                       // yr_s x (ds * jn)
  double *Mp;                            // gather M[:, J] -> yr_s x r
  const double *T[ACI_GEMM_MAX_IN];      // T^n (c0 x ds*jn), or X^n_s itself at s = L-1
  double *Rnew[ACI_GEMM_MAX_IN];         // R^n_s (c0 x rmax[s-1]), ld ldRnew
  int ldRnew;
  int c0[ACI_GEMM_MAX_IN];
  const double *Yin_prev;                // y_init core s-1 : (yr[s-1] d) x yr_s
  double *Yabs_prev;                     // out: (yr[s-1] d) x r
  GemmDesc *ydesc;
  int *canon_n;                          // log
  int *canon_cols;
  int Z;                                 // 2: complex (Mp and R frames written expanded)
};

__global__ void canon_update_kernel(CanonUpd U) {
  const int r = *U.r_in;
  const int s = U.s, L = U.L;
  const int jn = U.rk[s + 1];
  const int n = U.ds * jn;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  if (gt == 0) {
    U.rk[s] = r;  // |J_s| = rank of bond s-1; this kernel only reads rk[s+1]
    *U.canon_n = r;
    GemmDesc g = {};
    g.C = U.Yabs_prev; g.M = U.yr_prev_rows; g.N = U.Z * r; g.ldc = U.Z * r; g.nin = 1;
    g.A[0] = U.Yin_prev; g.lda[0] = U.Z * U.yr_s; g.K[0] = U.Z * U.yr_s;
    g.B[0] = U.Mp; g.ldb[0] = U.Z * r;
    *U.ydesc = g;
  }
  for (int k = gt; k < r; k += gs) U.canon_cols[k] = U.cols[k];
  const int wJ = L - s;
  for (int t = gt; t < r * wJ; t += gs) {
    const int k = t / wJ, pos = t % wJ;
    const int col = U.cols[k];
    U.Jnew[t] = pos == 0 ? (uint8_t)(col / jn) : U.Jnext[(col % jn) * (wJ - 1) + pos - 1];
  }
  if (U.Z == 1) {
    for (int t = gt; t < U.yr_s * r; t += gs) {
      const int a = t / r, k = t % r;
      U.Mp[t] = U.M[(size_t)a * n + U.cols[k]];
    }
    for (int i = 0; i < U.N; ++i) {
      const int c0 = U.c0[i];
      for (int t = gt; t < c0 * r; t += gs) {
        const int a = t / r, k = t % r;
        U.Rnew[i][(size_t)a * U.ldRnew + k] = U.T[i][(size_t)a * n + U.cols[k]];
      }
    }
    return;
  }
  // complex: gathered entries (re, im) written as 2x2 blocks [[re, im], [-im, re]]
  auto put = [](double *E, size_t ld, int a, int k, double re, double im) {
    E[(size_t)(2 * a) * ld + 2 * k] = re;
    E[(size_t)(2 * a) * ld + 2 * k + 1] = im;
    E[(size_t)(2 * a + 1) * ld + 2 * k] = -im;
    E[(size_t)(2 * a + 1) * ld + 2 * k + 1] = re;
  };
  for (int t = gt; t < U.yr_s * r; t += gs) {
    const int a = t / r, k = t % r;
    const double *x = U.M + ((size_t)a * n + U.cols[k]) * 2;
    put(U.Mp, 2 * (size_t)r, a, k, x[0], x[1]);
  }
  for (int i = 0; i < U.N; ++i) {
    const int c0 = U.c0[i];
    for (int t = gt; t < c0 * r; t += gs) {
      const int a = t / r, k = t % r;
      const double *x = U.T[i] + ((size_t)a * n + U.cols[k]) * 2;
      put(U.Rnew[i], 2 * (size_t)U.ldRnew, a, k, x[0], x[1]);
    }
  }
}

// ---- output cores (a8): Y_{b+1} = U_J^{-1} U (Alg. 3 right branch, R5)
// Step 1 gathers the unit-upper pivot block U_J[k][i] = U[k][q_i] densely (one launch, all
// bonds). Step 2: one CTA per (bond, 32-column block) keeps B[:, block] in shared memory and runs
// the back substitution B_k = U_k - sum_{i>k} U_J[k][i] B_i; each column's dot product is split
// over 8 lanes of one warp and reduced with shuffles, so a row costs one __syncthreads.
struct TrsmArgs {
  const double *U;  // U store of bond b (r x n), ld ldu
  int ldu;
  const int *cols;  // pivot columns q_0..q_{r-1}
  int b, d1;        // bond, d_{b+1}
  double *UJ;       // dense r x r gather of U_J, ld ldj
  int ldj;
  double *out;      // output core b+1, r x n row-major
};

__global__ void gather_uj_kernel(const TrsmArgs *args, const int *rk) {
  const TrsmArgs A = args[blockIdx.y];
  const int r = rk[A.b + 1];
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < r * r; t += gridDim.x * blockDim.x) {
    const int k = t / r, i = t % r;
    A.UJ[(size_t)k * A.ldj + i] = A.U[(size_t)k * A.ldu + A.cols[i]];
  }
}

// Unit-upper solve of one diagonal block: x = U_J[R,R]^{-1} x for the rows R = [r0, r0 + nr) of
// every column of the bond (x already holds U[R] - U_J[R, below] B[below]). One thread per column.
struct TriArgs {
  const double *UJ;
  int ldj;
  double *out;  // output core (r x n), rows R updated in place
  int n, r0, nr;
};
// Right-looking substitution with the block's x in registers: once x_k is final, every x_i
// (i < k) takes its fma independently, so a thread has up to k FMAs in flight instead of one
// dependent chain per row; U_J[R,R] is read from shared memory as warp-uniform broadcasts.
constexpr int kTriNB = 64, kTriThreads = 128;
__global__ void __launch_bounds__(kTriThreads) tri_block_kernel(const TriArgs *args) {
  __shared__ double su[kTriNB][kTriNB];  // su[i][k] = U_J[r0 + i][r0 + k]
  const TriArgs A = args[blockIdx.y];
  const int j = blockIdx.x * kTriThreads + threadIdx.x;
  if (blockIdx.x * kTriThreads >= A.n) return;
  const int nr = A.nr;
  for (int t = threadIdx.x; t < nr * nr; t += kTriThreads) {
    const int i = t / nr, k = t % nr;
    su[i][k] = A.UJ[(size_t)(A.r0 + i) * A.ldj + A.r0 + k];
  }
  const bool live = j < A.n;
  double x[kTriNB];
#pragma unroll
  for (int k = 0; k < kTriNB; ++k) x[k] = (live && k < nr) ? A.out[(size_t)(A.r0 + k) * A.n + j] : 0.0;
  __syncthreads();
#pragma unroll
  for (int k = kTriNB - 1; k > 0; --k) {
    if (k < nr) {
      const double xk = x[k];
#pragma unroll
      for (int i = 0; i < k; ++i) x[i] = fma(-su[i][k], xk, x[i]);
    }
  }
  if (live)
#pragma unroll
    for (int k = 0; k < kTriNB; ++k)
      if (k < nr) A.out[(size_t)(A.r0 + k) * A.n + j] = x[k];
}

__global__ void copy_prev_kernel(const int *rk, int *prev, int L) {
  for (int b = threadIdx.x; b < L - 1; b += blockDim.x) prev[b] = rk[b + 1];
}

// ---- complex output cores: Y_{b+1} = U_J^{-1} U (Alg. 3 right branch, R5; products
// as RZ5). One launch for every bond: a CTA owns 16 columns of one bond and keeps them in shared
// memory; 8 lanes share each column's dot products (shuffle reduction), one barrier per row.
struct ZTrsmArgs {
  const double *U;  // complex U store (r x n, ld ldu complex)
  int ldu;
  const int *cols;
  double *out;      // complex output core (r x n)
  int r, n;
};
constexpr int kZTrsmCols = 16;
__global__ void __launch_bounds__(128) ztrsm_kernel(const ZTrsmArgs *args) {
  extern __shared__ double zb[];  // [r][kZTrsmCols][2]
  const ZTrsmArgs A = args[blockIdx.y];
  const int j0 = blockIdx.x * kZTrsmCols;
  if (j0 >= A.n) return;
  const int c = threadIdx.x >> 3, t = threadIdx.x & 7;
  const int j = j0 + c;
  for (int e = threadIdx.x; e < A.r * kZTrsmCols; e += blockDim.x) {
    const int i = e / kZTrsmCols, cc = e % kZTrsmCols;
    const bool ok = j0 + cc < A.n;
    zb[2 * e] = ok ? A.U[((size_t)i * A.ldu + j0 + cc) * 2] : 0.0;
    zb[2 * e + 1] = ok ? A.U[((size_t)i * A.ldu + j0 + cc) * 2 + 1] : 0.0;
  }
  __syncthreads();
  for (int k = A.r - 1; k >= 0; --k) {
    double sr = 0.0, si = 0.0;
    for (int i = k + 1 + t; i < A.r; i += 8) {
      const double *u = A.U + ((size_t)k * A.ldu + A.cols[i]) * 2;
      const double br = zb[2 * (i * kZTrsmCols + c)], bi = zb[2 * (i * kZTrsmCols + c) + 1];
      sr += u[0] * br - u[1] * bi;
      si += u[0] * bi + u[1] * br;
    }
#pragma unroll
    for (int o = 4; o; o >>= 1) {
      sr += __shfl_xor_sync(0xffffffffu, sr, o);
      si += __shfl_xor_sync(0xffffffffu, si, o);
    }
    if (t == 0) {
      zb[2 * (k * kZTrsmCols + c)] -= sr;
      zb[2 * (k * kZTrsmCols + c) + 1] -= si;
    }
    __syncthreads();
  }
  if (j < A.n)
    for (int k = t; k < A.r; k += 8) {
      A.out[((size_t)k * A.n + j) * 2] = zb[2 * (k * kZTrsmCols + c)];
      A.out[((size_t)k * A.n + j) * 2 + 1] = zb[2 * (k * kZTrsmCols + c) + 1];
    }
}

// 2x2-block expansion of a complex (rows x cols) matrix for use as a right GEMM operand.
__global__ void expand_kernel(const double *X, double *E, int rows, int cols) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < rows * cols; t += gridDim.x * blockDim.x) {
    const int a = t / cols, k = t % cols;
    const double re = X[2 * (size_t)t], im = X[2 * (size_t)t + 1];
    const size_t ld = 2 * (size_t)cols;
    E[(2 * a) * ld + 2 * k] = re;
    E[(2 * a) * ld + 2 * k + 1] = im;
    E[(2 * a + 1) * ld + 2 * k] = -im;
    E[(2 * a + 1) * ld + 2 * k + 1] = re;
  }
}

// ============================================================================ host: workspace
namespace {

struct Carver {
  char *base = nullptr;
  size_t off = 0;
  template <class T>
  T *take(size_t count) {
    off = (off + 255) & ~(size_t)255;
    T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
    off += std::max<size_t>(count, 1) * sizeof(T);
    return p;
  }
};

// Launch accounting and optional per-class CUDA-event timing (aci_options.profile).
struct Prof {
  bool on = false;
  cudaStream_t st = nullptr;
  int64_t launches[ACI_PROF_NCLASS] = {};
  int64_t total = 0;
  int64_t per_iter_launches = 0;
  struct Span { int cls; cudaEvent_t a, b; };
  std::vector<Span> spans;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  int cur = -1;
  cudaEvent_t cur_a = nullptr;
  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  void begin(int cls) {
    cur = cls;
    if (on) {
      cur_a = get();
      cudaEventRecord(cur_a, st);
    }
  }
  void end(int nlaunch) {
    launches[cur] += nlaunch;
    total += nlaunch;
    if (on) {
      cudaEvent_t b = get();
      cudaEventRecord(b, st);
      spans.push_back({cur, cur_a, b});
    }
  }
  void collect(aci_profile *out) {
    for (int c = 0; c < ACI_PROF_NCLASS; ++c) { out->ms[c] = 0.0; out->launches[c] = launches[c]; }
    for (auto &sp : spans) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, sp.a, sp.b);
      out->ms[sp.cls] += ms;
    }
  }
  ~Prof() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

struct Run {
  Prof *P = nullptr;
  // Per-bond pivot outputs are kept PER SWEEP DIRECTION (index dir * L + b): the index/log kernel of
  // an L->R update trails the sweep on a side stream, and the first R->L update is the same bond
  // (L-2); with one buffer per direction nothing on the main stream overwrites what it still reads
  // (the iteration joins the side stream before the next iteration reuses them).
  int *binfo = nullptr;         // 8 ints per (dir, bond): the update's snapshot for index_bond_kernel
  cudaError_t launch_err = cudaSuccess;  // first rejected prrLU launch (eager launches)
  int cplx = 0, Z = 1, ZE = 1;  // complex run: Z = 2 doubles per entry, ZE = 4 for expanded operands
  int one = 0;                  // aci_options.concurrent: single-cluster prrLU launches
  int rook = 0;                 // aci_options.pivoting == ACI_PIVOT_ROOK (R23, NEXT-4)
  // streamed Pi: the Pi of L->R bond b+1 is computed while the prrLU of bond b
  // runs (pi_stream_kernel on the look-ahead stream), so neither that GEMM nor the row gather
  // sits between the two factorisations. Pi is double-buffered by bond parity (PiB[b & 1]): the
  // streamed Pi_{b+1} is written while the prrLU of bond b may still be loading Pi_b.
  int stream = 0;
  double *PiB[2] = {nullptr, nullptr};
  unsigned long long *sp = nullptr;  // max |Pi_{b+1}| of the stream, merged into s by its last CTA
  unsigned *sdone = nullptr;         // the stream's CTA exit counter
  int *prow0 = nullptr;              // the L->R pivot-row buffers (one block: reset to -1 per iteration)
  unsigned long long *ts = nullptr;  // ACI_STREAM_TS builds: per-bond timestamps of the last iteration
  size_t prow0_ints = 0;
  int L = 0, N = 0, maxrank = 0, max_sweeps = 0, log_cap_upd = 0, log_cap_piv = 0, colcap = 0;
  std::vector<int> d, yr;
  std::vector<std::vector<int>> xr;      // [n][s], s = 0..L
  std::vector<const double *> xcore0;    // device base of input n
  std::vector<std::vector<size_t>> xoff; // [n][s]
  std::vector<std::vector<double *>> Xe; // [n][s]: complex runs, 2x2-block expanded cores (GemmDesc::xd)
  std::vector<int> rmax, mmax, nmax;     // per bond
  // device
  int *rk = nullptr, *prev = nullptr, *rout = nullptr, *nonfinite = nullptr, *conv = nullptr, *iter = nullptr;
  double *epsb = nullptr, *err = nullptr;
  unsigned long long *scale = nullptr, *maxeps = nullptr;
  std::vector<int *> prow, pcol;
  std::vector<std::vector<double *>> Rf;  // [n][s]: R frames of the canonicalisation
  std::vector<double *> Abuf, Bbuf, Ust, Yin, Yabs;  // Abuf/Bbuf: look-ahead scratch per input
  std::vector<std::vector<double *>> Ast, Bst;  // [n][b]: Pi operands A^n_b, B^n_b (plan_bond)
  BondStatic *dStat = nullptr;   // [dir * (L-1) + b], uploaded once per call
  GemmDesc *dPre = nullptr;      // (L-1) * N descriptors of the one-time B^n_b launch
  std::vector<BondStatic> hStat;
  std::vector<int> nbig, nsmall; // [dir * (L-1) + b]: Pi kernel input split
  std::vector<FOp> opb;          // [dir * (L-1) + b]: op with exponents in Pi input order
  double *Pi = nullptr, *Y0 = nullptr, *Mp = nullptr;
  std::vector<uint8_t *> Imi, Jmi;
  GemmDesc *dAB = nullptr, *dPi = nullptr, *dT = nullptr, *dY = nullptr;
  LuDims *dLu = nullptr;
  int *log_info = nullptr, *log_rows = nullptr, *log_cols = nullptr, *canon_n = nullptr, *canon_cols = nullptr;
  double *log_es = nullptr;
  unsigned long long *colpub = nullptr;
  unsigned long long *keys = nullptr;
  unsigned *epoch = nullptr;
  unsigned *counter = nullptr;
  TrsmArgs *dtrsm = nullptr;
  GemmDesc *dtgemm = nullptr;
  struct TriArgs *dtri = nullptr;
  std::vector<double *> UJ;
};

static long long capped_prod(const std::vector<int> &d, int lo, int hi) {  // prod d[lo..hi], capped
  long long p = 1;
  for (int s = lo; s <= hi; ++s) {
    p *= d[s];
    if (p > (1 << 20)) return 1 << 20;
  }
  return p;
}

static void plan_capacities(Run &R) {
  const int L = R.L;
  R.rmax.assign(std::max(L - 1, 0), 0);
  R.mmax.assign(std::max(L - 1, 0), 0);
  R.nmax.assign(std::max(L - 1, 0), 0);
  for (int b = 0; b < L - 1; ++b)
    R.rmax[b] = (int)std::min<long long>(R.maxrank, std::min(capped_prod(R.d, 0, b), capped_prod(R.d, b + 1, L - 1)));
  for (int b = 0; b < L - 1; ++b) {
    R.mmax[b] = R.d[b] * (b == 0 ? 1 : R.rmax[b - 1]);
    R.nmax[b] = R.d[b + 1] * (b == L - 2 ? 1 : R.rmax[b + 1]);
  }
}

static size_t carve(Run &R, char *base) {
  Carver c;
  c.base = base;
  const int L = R.L, N = R.N;
  R.rk = c.take<int>(L + 1);
  R.prev = c.take<int>(L);
  R.rout = c.take<int>(2 * L);
  R.nonfinite = c.take<int>(1);
  R.conv = c.take<int>(1);
  R.iter = c.take<int>(1);
  R.epsb = c.take<double>(2 * L);
  R.err = c.take<double>(1);
  R.scale = c.take<unsigned long long>(1);
  R.maxeps = c.take<unsigned long long>(1);
  R.prow.resize(2 * L);
  R.pcol.resize(2 * L);
  // the L->R pivot rows in one block (streamed Pi: one memset sets them to -1 per iteration)
  R.prow0_ints = 0;
  for (int s = 0; s < L; ++s) R.prow0_ints += (size_t)(s < L - 1 ? R.rmax[s] : 1) + 1;
  R.prow0 = c.take<int>(R.prow0_ints);
  for (int t = 0, off = 0; t < 2 * L; ++t) {  // [dir * L + b], bonds 0..L-2; canon uses the dir-0 arrays of bond s-1
    const int s = t % L;
    int cap = s < L - 1 ? R.rmax[s] : 1;
    if (t < L) {
      R.prow[t] = R.prow0 ? R.prow0 + off : nullptr;
      off += cap + 1;
    } else {
      R.prow[t] = c.take<int>(cap + 1);
    }
    R.pcol[t] = c.take<int>(cap + 1);
  }
  R.sp = c.take<unsigned long long>(1);
  R.sdone = c.take<unsigned>(1);
#ifdef ACI_STREAM_TS
  R.ts = c.take<unsigned long long>(16 * (size_t)L);
#endif
  R.Rf.assign(N, std::vector<double *>(L + 1, nullptr));
  R.Abuf.assign(N, nullptr);
  R.Bbuf.assign(N, nullptr);
  for (int n = 0; n < N; ++n) {
    size_t acap = 1, bcap = 1;
    // complex: left operands (A^n) interleaved (x Z), right operands (R frames, B^n) in 2x2-block
    // expanded form (x ZE). Abuf: A^n_b X^n_{b+1} (L->R look-ahead); Bbuf: X^n_b B^n_b (R->L
    // look-ahead) and the canonicalisation's X_s R_{s+1}
    for (int b = 0; b < L - 1; ++b) {
      if (b + 2 < L) acap = std::max(acap, (size_t)R.mmax[b] * R.d[b + 1] * R.xr[n][b + 2]);
      if (b > 0) bcap = std::max(bcap, (size_t)R.xr[n][b] * R.d[b] * R.nmax[b]);
      bcap = std::max(bcap, (size_t)R.xr[n][b + 1] * R.nmax[b]);
    }
    for (int s = 1; s < L; ++s) R.Rf[n][s] = c.take<double>((size_t)R.xr[n][s] * R.rmax[s - 1] * R.ZE);
    R.Abuf[n] = c.take<double>(acap * R.Z);
    R.Bbuf[n] = c.take<double>(bcap * R.ZE);
  }
  R.Ast.assign(N, std::vector<double *>(L, nullptr));
  R.Bst.assign(N, std::vector<double *>(L, nullptr));
  for (int n = 0; n < N; ++n) {
    for (int b = 1; b < L - 1; ++b)
      R.Ast[n][b] = c.take<double>((size_t)R.rmax[b - 1] * R.d[b] * R.xr[n][b + 1] * R.Z);
    for (int b = 0; b + 2 < L; ++b)
      R.Bst[n][b] = c.take<double>((size_t)R.xr[n][b + 1] * R.d[b + 1] * R.rmax[b + 1] * R.ZE);
  }
  R.Xe.assign(N, std::vector<double *>(L, nullptr));
  for (int n = 0; n < N && R.cplx; ++n) {
    for (int s = 0; s < L; ++s) R.Xe[n][s] = c.take<double>((size_t)R.xr[n][s] * R.d[s] * R.xr[n][s + 1] * 4);
  }
  size_t picap = 1;
  for (int b = 0; b < L - 1; ++b) picap = std::max(picap, (size_t)R.mmax[b] * R.nmax[b]);
  R.Pi = c.take<double>(picap * R.Z);
  R.PiB[0] = R.Pi;
  R.PiB[1] = R.stream ? c.take<double>(picap * R.Z) : R.Pi;
  R.Ust.assign(L, nullptr);
  for (int b = 0; b < L - 1; ++b) R.Ust[b] = c.take<double>((size_t)R.rmax[b] * R.nmax[b] * R.Z);
  R.Y0 = c.take<double>(L > 1 ? (size_t)R.mmax[0] * R.rmax[0] * R.Z : 1);
  R.Imi.assign(L, nullptr);
  R.Jmi.assign(L + 1, nullptr);
  for (int b = 0; b < L - 1; ++b) R.Imi[b] = c.take<uint8_t>((size_t)R.rmax[b] * (b + 1));
  for (int s = 1; s < L; ++s) R.Jmi[s] = c.take<uint8_t>((size_t)R.rmax[s - 1] * (L - s));
  R.Yin.assign(L, nullptr);
  R.Yabs.assign(L, nullptr);
  size_t mpcap = 1;
  for (int s = 0; s < L; ++s) {
    R.Yin[s] = c.take<double>((size_t)R.yr[s] * R.d[s] * R.yr[s + 1] * R.Z);
    if (s < L - 1) R.Yabs[s] = c.take<double>((size_t)R.yr[s] * R.d[s] * R.rmax[s] * R.Z);
    if (s >= 1) mpcap = std::max(mpcap, (size_t)R.yr[s] * R.rmax[s - 1]);
  }
  R.Mp = c.take<double>(mpcap * R.ZE);
  R.dAB = c.take<GemmDesc>(2 * ACI_GEMM_MAX_IN);
  R.dStat = c.take<BondStatic>(2 * std::max(L - 1, 1));
  R.dPre = c.take<GemmDesc>((size_t)std::max(L - 1, 1) * N);
  R.dPi = c.take<GemmDesc>(1);
  R.dT = c.take<GemmDesc>(ACI_GEMM_MAX_IN);
  R.dY = c.take<GemmDesc>(1);
  R.dLu = c.take<LuDims>(1);
  R.log_info = c.take<int>((size_t)R.log_cap_upd * 5);
  R.log_es = c.take<double>((size_t)R.log_cap_upd * 2);
  R.log_rows = c.take<int>((size_t)R.log_cap_upd * R.log_cap_piv);
  R.log_cols = c.take<int>((size_t)R.log_cap_upd * R.log_cap_piv);
  R.canon_n = c.take<int>(L + 1);
  R.canon_cols = c.take<int>((size_t)(L + 1) * R.log_cap_piv);
  R.colpub = c.take<unsigned long long>((size_t)2 * 148 * R.colcap * 2 * prrlu_col_spread());
  R.keys = c.take<unsigned long long>(2 * 148 * 4);
  R.epoch = c.take<unsigned>(1);
  R.counter = c.take<unsigned>(1);
  R.dtrsm = c.take<TrsmArgs>(L);
  R.binfo = c.take<int>((size_t)16 * std::max(L - 1, 1));
  R.UJ.assign(L, nullptr);
  size_t nblk = 0;
  for (int b = 0; b < L - 1; ++b) {
    R.UJ[b] = c.take<double>((size_t)R.rmax[b] * R.rmax[b] * R.Z);
    nblk += (R.rmax[b] + 63) / 64;
  }
  R.dtgemm = c.take<GemmDesc>(nblk);
  R.dtri = c.take<TriArgs>(nblk);
  return c.off + 256;
}

struct Inputs {
  std::vector<const tt_s *> tts;   // distinct
  FOp op;
};

static int prepare(aci_op op, const tt_t *const *inputs, int n_inputs, Inputs &I) {
  if (!inputs || n_inputs < 1) return fail(ACI_ERR_INVALID, "aci: no inputs");
  if (op.n_terms < 1 || op.n_terms > ACI_MAX_TERMS || !op.coef || !op.expo)
    return fail(ACI_ERR_INVALID, "aci: op must have 1..8 terms and non-null coef/expo");
  std::vector<int> map(n_inputs);
  for (int i = 0; i < n_inputs; ++i) {
    if (!inputs[i]) return fail(ACI_ERR_INVALID, "aci: null input");
    int u = -1;
    for (size_t j = 0; j < I.tts.size(); ++j)
      if (I.tts[j] == inputs[i]) u = (int)j;
    if (u < 0) {
      u = (int)I.tts.size();
      I.tts.push_back(inputs[i]);
    }
    map[i] = u;
  }
  const int N = (int)I.tts.size();
  if (N > ACI_MAX_INPUTS) return fail(ACI_ERR_INVALID, "aci: more than 4 distinct inputs");
  const tt_s *t0 = I.tts[0];
  for (int j = 1; j < N; ++j) {
    if (I.tts[j]->L != t0->L || I.tts[j]->d != t0->d) return fail(ACI_ERR_SHAPE, "aci: inputs differ in L or d (S:253)");
    if (I.tts[j]->cplx != t0->cplx) return fail(ACI_ERR_SHAPE, "aci: inputs mix real and complex TTs");
  }
  std::memset(&I.op, 0, sizeof(I.op));
  I.op.T = op.n_terms;
  I.op.N = N;
  for (int t = 0; t < op.n_terms; ++t) {
    if (!std::isfinite(op.coef[t])) return fail(ACI_ERR_INVALID, "aci: non-finite coefficient");
    I.op.coef[t] = op.coef[t];
    for (int i = 0; i < n_inputs; ++i) {
      int e = op.expo[t * n_inputs + i];
      if (e < 0 || e > ACI_MAX_EXPO) return fail(ACI_ERR_INVALID, "aci: exponent out of 0..4");
      I.op.expo[t * N + map[i]] += e;
    }
    for (int u = 0; u < N; ++u)
      if (I.op.expo[t * N + u] > 3 * ACI_MAX_EXPO) return fail(ACI_ERR_INVALID, "aci: merged exponent too large");
  }
  I.op.monomial_all_ones = I.op.T == 1 ? 1 : 0;
  for (int u = 0; u < N && I.op.T == 1; ++u)
    if (I.op.expo[u] != 1) I.op.monomial_all_ones = 0;
  return ACI_OK;
}

// counter-based N(0,1) (splitmix64 + Box-Muller) for the default y_init (R9)
static uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
static double normal_at(uint64_t seed, uint64_t i) {
  double u1 = ((splitmix(seed ^ (2 * i)) >> 11) + 1) * (1.0 / 9007199254740993.0);
  double u2 = (splitmix(seed ^ (2 * i + 1)) >> 11) * (1.0 / 9007199254740992.0);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

}  // namespace

// ---------------------------------------------------------------------------- workspaces
// One persistent workspace per stream, grown on demand: calls on a stream are serialised (each
// returns after synchronising it), and a stable address lets repeated products hit the graph
// cache (the captured iteration embeds workspace pointers). At most kWsCap idle workspaces are
// kept (least recently used freed first); a workspace in use by a running call is never freed.
struct WsEntry {
  cudaStream_t st;
  char *ptr;
  size_t size;
  int inuse;
  uint64_t last_use;
};
static std::mutex g_ws_mu;
static std::vector<WsEntry> g_ws;
static uint64_t g_ws_clock = 0;
constexpr size_t kWsCap = 16;

// A stream carries one call at a time: a second call on a stream whose workspace is in use (a
// concurrent-mode call and a default-tier call from two host threads on one stream) is refused
// (*busy = true) instead of sharing — or reallocating under — the running call's workspace.
static char *stream_workspace_acquire(cudaStream_t st, size_t need, bool *busy) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  *busy = false;
  for (auto &e : g_ws)
    if (e.st == st) {
      if (e.inuse > 0) {
        *busy = true;
        return nullptr;
      }
      if (e.size < need) {
        cudaFree(e.ptr);
        e.ptr = nullptr;
        e.size = 0;
        if (cudaMalloc((void **)&e.ptr, need) != cudaSuccess) return nullptr;
        e.size = need;
      }
      ++e.inuse;
      e.last_use = ++g_ws_clock;
      return e.ptr;
    }
  while (g_ws.size() >= kWsCap) {
    auto lru = g_ws.end();
    for (auto it = g_ws.begin(); it != g_ws.end(); ++it)
      if (it->inuse == 0 && (lru == g_ws.end() || it->last_use < lru->last_use)) lru = it;
    if (lru == g_ws.end()) break;
    cudaFree(lru->ptr);
    g_ws.erase(lru);
  }
  char *p = nullptr;
  if (cudaMalloc((void **)&p, need) != cudaSuccess) return nullptr;
  g_ws.push_back({st, p, need, 1, ++g_ws_clock});
  return p;
}

static void stream_workspace_release(cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  for (auto &e : g_ws)
    if (e.st == st) {
      --e.inuse;
      return;
    }
}

// ---------------------------------------------------------------------------- graph cache
// Instantiated iteration graphs keyed by every host value the capture reads: capture plus
// instantiation of ~1500 nodes costs ~10 ms of host time per call, the replay is free.
struct GraphEntry {
  std::vector<uint64_t> key;
  cudaGraphExec_t exec;
  int64_t launches;
  uint64_t last_use;
  int inuse;  // calls currently replaying it (concurrent calls on other streams): never evicted
};
static std::mutex g_cache_mu;
static std::vector<GraphEntry> g_cache;
static uint64_t g_cache_clock = 0;
constexpr size_t kGraphCacheCap = 8;

// A hit is pinned (inuse) until graph_cache_release.
static cudaGraphExec_t graph_cache_acquire(const std::vector<uint64_t> &key, int64_t *launches) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  for (auto &e : g_cache)
    if (e.key == key) {
      e.last_use = ++g_cache_clock;
      ++e.inuse;
      *launches = e.launches;
      return e.exec;
    }
  return nullptr;
}
// Insert a freshly instantiated graph, pinned; evicts the least recently used idle entry when
// full. Returns false (the caller keeps ownership) if every entry is in use.
static bool graph_cache_insert(const std::vector<uint64_t> &key, cudaGraphExec_t exec, int64_t launches) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (g_cache.size() >= kGraphCacheCap) {
    auto lru = g_cache.end();
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it)
      if (it->inuse == 0 && (lru == g_cache.end() || it->last_use < lru->last_use)) lru = it;
    if (lru == g_cache.end()) return false;
    cudaGraphExecDestroy(lru->exec);
    g_cache.erase(lru);
  }
  g_cache.push_back({key, exec, launches, ++g_cache_clock, 1});
  return true;
}
// End of a call: unpin a cached graph (drop: also remove and destroy it, after a failure), or
// destroy an uncached one.
static void graph_cache_release(cudaGraphExec_t exec, bool cached, bool drop) {
  if (!exec) return;
  if (!cached) {
    cudaGraphExecDestroy(exec);
    return;
  }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  for (size_t i = 0; i < g_cache.size(); ++i)
    if (g_cache[i].exec == exec) {
      --g_cache[i].inuse;
      if (drop && g_cache[i].inuse == 0) {
        cudaGraphExecDestroy(exec);
        g_cache.erase(g_cache.begin() + i);
      }
      return;
    }
}
static std::vector<uint64_t> graph_key(const Run &R, const FOp &op, double tol, int tol_mode, const void *ws,
                                       size_t need, cudaStream_t st) {
  std::vector<uint64_t> k;
  auto u = [&](uint64_t v) { k.push_back(v); };
  auto dbl = [&](double v) {
    uint64_t b;
    std::memcpy(&b, &v, 8);
    u(b);
  };
  u((uint64_t)(uintptr_t)ws); u(need); u((uint64_t)(uintptr_t)st);
  u(R.L); u(R.N); u(R.maxrank); u(R.log_cap_upd); u(R.log_cap_piv); u(R.colcap); u(R.cplx); u(R.one); u(R.rook); u(R.stream);
  dbl(tol); u(tol_mode);
  for (int x : R.d) u(x);
  for (int x : R.yr) u(x);
  for (int n = 0; n < R.N; ++n) {
    u((uint64_t)(uintptr_t)R.xcore0[n]);
    for (int x : R.xr[n]) u(x);
  }
  u(op.T); u(op.N); u(op.monomial_all_ones);
  for (int t = 0; t < op.T; ++t) dbl(op.coef[t]);
  for (int t = 0; t < op.T * op.N; ++t) u(op.expo[t]);
  return k;
}

// ============================================================================ host: the sweep
namespace {

static void launch_update(Run &R, int b, int dir, int logslot, const BondStatic *next, cudaStream_t st,
                          bool streamed = false) {
  UpdateArgs U = {};
  if (streamed) {  // the stream gathered A^n_{b+1}: only the ranks, the plan and the s merge remain
    U.sp = R.sp;
  }
  U.next = next; U.ab = R.dAB; U.pi = R.dPi; U.lu = R.dLu;
  U.next_b = next ? (int)((next - R.dStat) % (R.L - 1)) : -1;
  U.b = b; U.dir = dir; U.L = R.L; U.N = R.N; U.db = R.d[b]; U.db1 = R.d[b + 1];
  const int pv = dir * R.L + b;  // per-direction pivot buffers (Run::binfo)
  U.rows = R.prow[pv]; U.cols = R.pcol[pv]; U.r_in = R.rout + pv; U.eps_in = R.epsb + pv;
  U.rk = R.rk;
  U.Iprev = b > 0 ? R.Imi[b - 1] : nullptr;
  U.Inew = R.Imi[b];
  U.Jnext = b + 2 < R.L ? R.Jmi[b + 2] : nullptr;
  U.Jnew = R.Jmi[b + 1];
  for (int n = 0; n < R.N; ++n) {
    U.Ahat[n] = R.Abuf[n];
    U.Anext[n] = dir == 0 && b + 2 < R.L && !streamed ? R.Ast[n][b + 1] : nullptr;
    U.W[n] = b + 2 < R.L ? R.Z * R.d[b + 1] * R.xr[n][b + 2] : 0;
    U.Bhat[n] = R.Bbuf[n];
    U.Bprev[n] = dir == 1 && b > 0 ? R.Bst[n][b - 1] : nullptr;
    U.c0[n] = R.xr[n][b];
  }
  U.Z = R.Z;
  U.Pi = R.PiB[b & 1];
  U.Y0 = R.Y0;
  U.maxeps_bits = R.maxeps;
  U.scale_bits = R.scale;
  U.log_info = R.log_info;
  U.log_es = R.log_es;
  U.log_rows = R.log_rows;
  U.log_cols = R.log_cols;
  U.iter = R.iter;
  U.step = logslot;
  U.per_iter = 2 * (R.L - 1);
  U.cap_piv = R.log_cap_piv;
  U.info = R.binfo + 8 * (dir * (R.L - 1) + b);
  U.ts = R.ts;
  size_t work = streamed ? 1 : (size_t)R.rmax[b] * 256;
  int blocks = (int)std::min<size_t>(592, std::max<size_t>(1, (work + 255) / 256));
#if ACI_PDL_UPDATE
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, update_bond_kernel, U);
#else
  update_bond_kernel<<<blocks, 256, 0, st>>>(U);
#endif
}

static void launch_index(Run &R, int b, int dir, int logslot, cudaStream_t st) {
  IndexArgs U = {};
  U.b = b; U.dir = dir; U.L = R.L; U.db = R.d[b];
  const int pv = dir * R.L + b;
  U.rows = R.prow[pv]; U.cols = R.pcol[pv]; U.info = R.binfo + 8 * (dir * (R.L - 1) + b); U.eps_in = R.epsb + pv;
  U.Iprev = b > 0 ? R.Imi[b - 1] : nullptr;
  U.Inew = R.Imi[b];
  U.Jnext = b + 2 < R.L ? R.Jmi[b + 2] : nullptr;
  U.Jnew = R.Jmi[b + 1];
  U.maxeps_bits = R.maxeps;
  U.log_info = R.log_info; U.log_es = R.log_es; U.log_rows = R.log_rows; U.log_cols = R.log_cols;
  U.iter = R.iter; U.step = logslot; U.per_iter = 2 * (R.L - 1); U.cap_piv = R.log_cap_piv;
  const size_t work = (size_t)R.rmax[b] * (size_t)std::max(b + 1, R.L - b - 1);
  const int blocks = (int)std::min<size_t>(148, std::max<size_t>(1, (work + 255) / 256));
  index_bond_kernel<<<blocks, 256, 0, st>>>(U);
}

// Static description of every bond update (both directions), built once per call on the host
// and uploaded to the workspace: the planner kernels read it together with the live ranks.
static void build_statics(Run &R, const FOp &op) {
  const int L = R.L, N = R.N, nb = L - 1;
  R.hStat.assign(2 * nb, BondStatic{});
  R.nbig.assign(2 * nb, 0);
  R.nsmall.assign(2 * nb, 0);
  R.opb.assign(2 * nb, op);
  for (int dir = 0; dir < 2; ++dir)
    for (int b = 0; b < nb; ++b) {
      BondStatic &S = R.hStat[dir * nb + b];
      S.b = b; S.L = L; S.N = N; S.dir = dir; S.db = R.d[b]; S.db1 = R.d[b + 1];
      S.Z = R.Z;
      S.ldu = R.nmax[b];
      S.maxrank = R.maxrank;
      S.Pi = R.PiB[b & 1];
      // Pi kernel input order: inputs whose inner dimension chi^n_{b+1} is large run the DMMA
      // main loop (first), tiny ones (e.g. rank-2 inputs) are evaluated in the epilogue; the op's
      // exponents are permuted to the same order.
      int order[ACI_GEMM_MAX_IN], nbig = 0, nsmall = 0;
      // (complex runs: every input through the DMMA main loop)
      for (int n = 0; n < N; ++n)
        if (R.cplx || R.xr[n][b + 1] > gemm_small_k()) order[nbig++] = n;
      for (int n = 0; n < N; ++n)
        if (!R.cplx && R.xr[n][b + 1] <= gemm_small_k()) order[nbig + nsmall++] = n;
      R.nbig[dir * nb + b] = nbig;
      R.nsmall[dir * nb + b] = nsmall;
      FOp &ob = R.opb[dir * nb + b];
      for (int t = 0; t < op.T; ++t)
        for (int k = 0; k < N; ++k) ob.expo[t * N + k] = op.expo[t * N + order[k]];
      for (int kk = 0; kk < N; ++kk) {
        const int n = order[kk];
        InBond &I = S.in[kk];
        I.c0 = R.xr[n][b]; I.c1 = R.xr[n][b + 1]; I.c2 = R.xr[n][b + 2];
        I.Xb = R.xcore0[n] + R.xoff[n][b];
        I.Xb1 = R.xcore0[n] + R.xoff[n][b + 1];
        I.Rnext = b + 2 < L ? R.Rf[n][b + 2] : nullptr;
        I.ldR = b + 2 < L ? R.rmax[b + 1] : 1;
        I.Ahat = R.Abuf[n];
        I.Bhat = R.Bbuf[n];
        I.Ast = R.Ast[n][b];
        I.Bst = R.Bst[n][b];
        I.Xeb = R.Xe[n][b];
        I.Xeb1 = R.Xe[n][b + 1];
      }
    }
}

static const BondStatic *dstat(const Run &R, int dir, int b) { return R.dStat + dir * (R.L - 1) + b; }

// B^n_b = X^n_{b+1} R^n_{b+2} of every bond from the canonical R frames, in one launch (once per
// product; afterwards every B^n_b is written by the R->L update of bond b+1).
static void pre_launch(Run &R, cudaStream_t st) {
  const int L = R.L, N = R.N;
  int pm = 0, pn = 0;
  for (int b = 0; b + 2 < L; ++b)
    for (int n = 0; n < N; ++n) {
      pm = std::max(pm, R.xr[n][b + 1] * R.d[b + 1]);
      pn = std::max(pn, R.rmax[b + 1]);
    }
  if (pm == 0) return;
  R.P->begin(ACI_PROF_GEMM_AB);
  plan_pre_kernel<<<1, 256, 0, st>>>(dstat(R, 0, 0), L - 1, N, R.rk, R.dPre);
  FOp dummy = {};
  if (R.cplx)
    launch_gemm_z(R.dPre, (L - 1) * N, pm, 2 * pn, 1, 1, dummy, nullptr, nullptr, st);
  else
    launch_gemm(R.dPre, (L - 1) * N, pm, pn, 1, false, dummy, nullptr, nullptr, st);
  R.P->end(2);
}

// The look-ahead GEMM runs on a second stream (per host thread) forked off the prrLU's
// launch-completion event, so it starts once every prrLU CTA is resident and fills the SMs the
// prrLU leaves idle; the update of the bond joins it.
// Created by side_stream_init() at the start of every call, before any stream capture (creating
// streams or events inside a capture is refused, which left null events behind).
struct SideStream {
  cudaStream_t st = nullptr, ix = nullptr;  // look-ahead GEMMs; index/log kernels
  cudaEvent_t started = nullptr, done = nullptr, upd = nullptr, ix_done = nullptr;
  cudaEvent_t la = nullptr;  // streamed Pi: the look-ahead GEMM done (its descriptors may be re-planned)
};
static SideStream &side_stream() {
  static thread_local SideStream s;
  return s;
}
static bool side_stream_init() {
  SideStream &s = side_stream();
  if (s.st && s.ix && s.started && s.done && s.upd && s.ix_done && s.la) return true;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (!s.st && cudaStreamCreateWithPriority(&s.st, cudaStreamNonBlocking, lo) != cudaSuccess) s.st = nullptr;
  if (!s.ix && cudaStreamCreateWithPriority(&s.ix, cudaStreamNonBlocking, lo) != cudaSuccess) s.ix = nullptr;
  for (cudaEvent_t *e : {&s.started, &s.done, &s.upd, &s.ix_done, &s.la})
    if (!*e && cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) *e = nullptr;
  return s.st && s.ix && s.started && s.done && s.upd && s.ix_done && s.la;
}

// ACI_STREAM_SERIAL=1: the stream runs after the prrLU instead of beside it (A/B)
static bool serial_stream() {
  static const bool s = [] {
    const char *e = getenv("ACI_STREAM_SERIAL");
    return e && atoi(e) != 0;
  }();
  return s;
}

// Does the prrLU of L->R bond b stream the Pi of bond b+1 (Run::stream)?
// Only large Pi are streamed (static m' n' sum K >= ACI_STREAM_MIN, default 2^26 multiply-adds, e.g.
// 512 x 512 x 256): for the small ones the stream's last chunk costs about what the Pi GEMM and
// the gather cost.
static bool streams_next(const Run &R, int b, int dir) {
  if (!R.stream || dir != 0 || b + 2 >= R.L) return false;
  static const double min_fma = [] {
    const char *e = getenv("ACI_STREAM_MIN");
    return e ? atof(e) : 67108864.0;
  }();
  int c2[ACI_GEMM_MAX_IN];
  double ksum = 0;
  for (int kk = 0; kk < R.N; ++kk) {
    c2[kk] = R.hStat[b + 1].in[kk].c1;
    if (kk < R.nbig[b + 1]) ksum += c2[kk];
  }
  if ((double)R.mmax[b + 1] * R.nmax[b + 1] * ksum < min_fma) return false;
  return pi_stream_supported(R.nbig[b + 1], R.nsmall[b + 1], c2, (R.nmax[b + 1] + 31) / 32);
}

// Pi_{b+1} while the prrLU of bond b runs, on the look-ahead stream after the look-ahead GEMM
// (whose rows it gathers): inputs in bond b+1's Pi order.
static void launch_stream(Run &R, int b, cudaStream_t st) {
  static const int ctas = [] {  // ~CTAs of the stream (ntmax x P, P >= 1); it runs beside the prrLU
    const char *e = getenv("ACI_STREAM_GRID");
    const int g = e ? atoi(e) : 64;
    return g > 0 ? g : 64;
  }();
  const int ntmax = (R.nmax[b + 1] + 31) / 32;
  const int grid = ntmax * std::max(1, ctas / ntmax);
  const int L = R.L, N = R.N, k1 = b + 1;
  const BondStatic &S1 = R.hStat[k1];  // dir 0
  PiStreamArgs A = {};
  static const unsigned poll_ns = [] {
    const char *e = getenv("ACI_STREAM_POLL_NS");
    return e ? (unsigned)atoi(e) : 128u;
  }();
  A.rows = R.prow[b]; A.r_in = R.rout + b; A.rk = R.rk; A.kcap = R.rmax[b]; A.poll_ns = poll_ns; A.ntmax = ntmax;
  A.b = b; A.d1 = R.d[b + 1]; A.db2 = R.d[b + 2]; A.N = N; A.nbig = R.nbig[k1];
  for (int kk = 0; kk < N; ++kk) {
    const InBond &I = S1.in[kk];
    A.Ahat[kk] = I.Ahat;
    A.Anext[kk] = I.Ast;
    A.B[kk] = k1 + 2 < L ? I.Bst : I.Xb1;
    A.c2[kk] = I.c1;
  }
  A.Pi = R.PiB[k1 & 1];
  A.ts = R.ts;
  A.sp = R.sp;
  A.scale = R.scale;
  A.done = R.sdone;
  A.info = R.binfo + 8 * b;  // dir 0
  A.nonfinite = R.nonfinite;
  launch_pi_stream(A, R.nsmall[k1], R.opb[k1], grid, st);
}

// One 2-site update (Alg. 1): [plan] -> a3+a4 -> a5 (|| look-ahead GEMM) -> a6/a7 (+ the
// plan of the next bond, fused into the update kernel when `next` is given).
static void bond_update(Run &R, double tol, int tol_mode, int b, int dir, int logslot, bool plan_here,
                        const BondStatic *next, cudaStream_t st) {
  const int L = R.L, N = R.N, k = dir * (L - 1) + b;
  int la_m = 0, la_n = 0;  // look-ahead GEMM bounds (complex: in complex columns)
  for (int n = 0; n < N; ++n) {
    if (dir == 0 && b + 2 < L) { la_m = R.mmax[b]; la_n = std::max(la_n, R.d[b + 1] * R.xr[n][b + 2]); }
    if (dir == 1 && b > 0) { la_m = std::max(la_m, R.xr[n][b] * R.d[b]); la_n = R.nmax[b]; }
  }
  if (plan_here) {
    R.P->begin(ACI_PROF_UPDATE);
    plan_bond_kernel<<<1, 1, 0, st>>>(dstat(R, dir, b), R.rk, R.dAB, R.dPi, R.dLu);
    R.P->end(1);
  }
  // streamed_in: Pi_b was computed beside the previous bond's prrLU; stream_out: this prrLU
  // streams Pi_{b+1}
  const bool streamed_in = b > 0 && streams_next(R, b - 1, dir), stream_out = streams_next(R, b, dir);
  if (!streamed_in) {
    R.P->begin(ACI_PROF_GEMM_PI);
    if (R.cplx)
      launch_gemm_z(R.dPi, 1, R.mmax[b], 2 * R.nmax[b], 2, N, R.opb[k], R.scale, R.nonfinite, st);
    else
      launch_gemm_split(R.dPi, 1, R.mmax[b], R.nmax[b], R.nbig[k], R.nsmall[k], true, R.opb[k], R.scale, R.nonfinite,
                        st);
    R.P->end(1);
  }
  LuArgs a = {};
  a.M = R.PiB[b & 1]; a.dims = R.dLu; a.tol = tol; a.thr_mode = tol_mode == ACI_TOL_RELATIVE ? 0 : 2;
  a.scale_bits = R.scale;
  const int pv = dir * L + b;
  a.rows = R.prow[pv]; a.cols = R.pcol[pv]; a.r_out = R.rout + pv; a.eps_out = R.epsb + pv;
  a.U = dir == 1 ? R.Ust[b] : nullptr;
  a.colpub = R.colpub; a.colcap = R.colcap; a.keys = R.keys; a.counter = R.counter; a.epoch = R.epoch;
  SideStream &sd = side_stream();
  const bool look = la_m > 0 && la_n > 0;
  R.P->begin(ACI_PROF_PRRLU);
  const cudaError_t le = launch_prrlu(a, R.mmax[b], R.nmax[b], st, R.cplx != 0, R.one != 0, look ? sd.started : nullptr,
                                      R.rook != 0);
  if (le != cudaSuccess && R.launch_err == cudaSuccess) R.launch_err = le;
  R.P->end(1);
  if (look) {
    cudaStreamWaitEvent(sd.st, sd.started, 0);
    cudaStream_t mine = R.P->st;
    R.P->st = sd.st;
    R.P->begin(ACI_PROF_GEMM_AB);
    FOp dummy = {};
    if (R.cplx)
      launch_gemm_z(R.dAB, N, la_m, 2 * la_n, dir == 0 ? 0 : 1, 1, dummy, nullptr, nullptr, sd.st);
    else
      launch_gemm(R.dAB, N, la_m, la_n, 1, false, dummy, nullptr, nullptr, sd.st);
    R.P->end(1);
    const bool serial = serial_stream();
    if (stream_out && !serial) {
      cudaEventRecord(sd.la, sd.st);
      R.P->begin(ACI_PROF_GEMM_PI);
      launch_stream(R, b, sd.st);
      R.P->end(1);
    }
    R.P->st = mine;
    cudaEventRecord(sd.done, sd.st);
    if (stream_out && !serial) {  // the ranks and the next plan beside the stream's last chunk
      cudaStreamWaitEvent(st, sd.la, 0);  // (the plan rewrites the look-ahead GEMM's descriptors)
      R.P->begin(ACI_PROF_UPDATE);
      launch_update(R, b, dir, logslot, next, st, true);
      R.P->end(1);
    }
    cudaStreamWaitEvent(st, sd.done, 0);
    if (stream_out && serial) {
      R.P->begin(ACI_PROF_GEMM_PI);
      launch_stream(R, b, st);
      R.P->end(1);
    }
  }
  if (!(stream_out && look && !serial_stream())) {
    R.P->begin(ACI_PROF_UPDATE);
    launch_update(R, b, dir, logslot, next, st, stream_out && look);
    R.P->end(1);
  }
  cudaEventRecord(sd.upd, st);
  cudaStreamWaitEvent(sd.ix, sd.upd, 0);
  cudaStream_t mine = R.P->st;
  R.P->st = sd.ix;
  R.P->begin(ACI_PROF_UPDATE);
  launch_index(R, b, dir, logslot, sd.ix);
  R.P->end(1);
  R.P->st = mine;
}

// End of an iteration's sweeps: the index/log stream joins the main stream (the convergence test
// reads the error bookkeeping).
static void index_join(cudaStream_t st) {
  SideStream &sd = side_stream();
  cudaEventRecord(sd.ix_done, sd.ix);
  cudaStreamWaitEvent(st, sd.ix_done, 0);
}

// ACI_DEBUG_PENDING=1 (debugging): report a pending runtime error at points of a call
static void dbg_pending(const char *where) {
  static const bool on = [] {
    const char *e = getenv("ACI_DEBUG_PENDING");
    return e && atoi(e) != 0;
  }();
  if (!on) return;
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) fprintf(stderr, "[aci] pending %s at %s\n", cudaGetErrorString(e), where);
}

static void canon_step(Run &R, double tol, int tol_mode, int s, cudaStream_t st) {
  const int L = R.L, N = R.N;
  CanonArgs C = {};
  C.s = s; C.L = L; C.N = N; C.ds = R.d[s]; C.yr_s = R.yr[s];
  C.M = s == L - 1 ? R.Yin[s] : R.Yabs[s];
  C.lu = R.dLu;
  C.maxrank = R.rmax[s - 1];  // R9': canonical J_s never exceeds the full-tensor bond bound
  C.ldR = s + 1 < L ? R.rmax[s] : 1;
  C.tdesc = R.dT;
  C.Z = R.Z;
  int tm = 0, tn = 0;
  for (int n = 0; n < N; ++n) {
    C.Xs[n] = R.xcore0[n] + R.xoff[n][s];
    C.Rnext[n] = s + 1 < L ? R.Rf[n][s + 1] : nullptr;
    C.Tbuf[n] = R.Bbuf[n];
    C.c0[n] = R.xr[n][s];
    C.c1[n] = R.xr[n][s + 1];
    if (C.Rnext[n]) { tm = std::max(tm, C.c0[n] * C.ds); tn = std::max(tn, R.rmax[s]); }
  }
  R.P->begin(ACI_PROF_CANON);
  plan_canon_kernel<<<1, 1, 0, st>>>(C, R.rk);
  FOp dummy = {};
  const int max_m = R.yr[s], max_n = R.nmax[s - 1];
  LuArgs a = {};
  a.M = C.M; a.dims = R.dLu; a.tol = tol; a.thr_mode = tol_mode == ACI_TOL_RELATIVE ? 1 : 2;
  a.scale_bits = R.scale;
  a.rows = R.prow[s - 1]; a.cols = R.pcol[s - 1]; a.r_out = R.rout + (s - 1); a.eps_out = R.epsb + (s - 1);
  a.U = nullptr;
  a.colpub = R.colpub; a.colcap = R.colcap; a.keys = R.keys; a.counter = R.counter; a.epoch = R.epoch;
  // the R-frame product T^n = X^n_s R^n_{s+1} is only gathered after the factorisation: it runs on
  // the side stream beside the prrLU (forked off its launch-completion event, as in the sweep)
  SideStream &sd = side_stream();
  const cudaError_t le = launch_prrlu(a, max_m, max_n, st, R.cplx != 0, R.one != 0, tm > 0 ? sd.started : nullptr,
                                      R.rook != 0);
  if (le != cudaSuccess && R.launch_err == cudaSuccess) R.launch_err = le;
  if (tm > 0) {
    cudaStreamWaitEvent(sd.st, sd.started, 0);
    if (R.cplx) launch_gemm_z(R.dT, N, tm, 2 * tn, 0, 1, dummy, nullptr, nullptr, sd.st);
    else launch_gemm(R.dT, N, tm, tn, 1, false, dummy, nullptr, nullptr, sd.st);
    cudaEventRecord(sd.done, sd.st);
    cudaStreamWaitEvent(st, sd.done, 0);
  }
  CanonUpd U = {};
  U.s = s; U.L = L; U.N = N; U.ds = R.d[s]; U.yr_s = R.yr[s]; U.yr_prev_rows = R.yr[s - 1] * R.d[s - 1];
  U.cols = R.pcol[s - 1]; U.r_in = R.rout + (s - 1);
  U.rk = R.rk;
  U.Jnext = s + 1 < L ? R.Jmi[s + 1] : nullptr;
  U.Jnew = R.Jmi[s];
  U.M = C.M;
  U.Mp = R.Mp;
  for (int n = 0; n < N; ++n) {
    U.T[n] = C.Rnext[n] ? R.Bbuf[n] : C.Xs[n];
    U.Rnew[n] = R.Rf[n][s];
    U.c0[n] = R.xr[n][s];
  }
  U.ldRnew = R.rmax[s - 1];
  U.Yin_prev = R.Yin[s - 1];
  U.Yabs_prev = R.Yabs[s - 1];
  U.ydesc = R.dY;
  U.canon_n = R.canon_n + s;
  U.canon_cols = R.canon_cols + (size_t)s * R.log_cap_piv;
  U.Z = R.Z;
  canon_update_kernel<<<64, 256, 0, st>>>(U);
  if (R.cplx)
    launch_gemm_z(R.dY, 1, R.yr[s - 1] * R.d[s - 1], 2 * R.rmax[s - 1], 0, 1, dummy, nullptr, nullptr, st);
  else
    launch_gemm(R.dY, 1, R.yr[s - 1] * R.d[s - 1], R.rmax[s - 1], 1, false, dummy, nullptr, nullptr, st);
  R.P->end(4 + (tm > 0 ? 1 : 0));
}

}  // namespace

extern "C" int aci_limits(int *max_rows, int *max_cols) {
  if (!max_rows || !max_cols) return fail(ACI_ERR_INVALID, "aci_limits: null");
  prrlu_envelope(max_rows, max_cols);
  return ACI_OK;
}

static int build_run(const Inputs &I, const tt_s *y, int maxrank, int max_sweeps, Run &R, int one = 0,
                     int rook = 0) {
  const tt_s *t0 = I.tts[0];
  R.L = t0->L;
  R.N = (int)I.tts.size();
  R.d = t0->d;
  R.maxrank = maxrank;
  R.max_sweeps = max_sweeps;
  R.xr.resize(R.N);
  R.xcore0.resize(R.N);
  R.xoff.resize(R.N);
  for (int n = 0; n < R.N; ++n) {
    R.xr[n] = I.tts[n]->ranks;
    R.xcore0[n] = I.tts[n]->dcores;
    R.xoff[n] = I.tts[n]->off;
  }
  R.yr = y->ranks;
  R.cplx = t0->cplx;
  R.Z = R.cplx ? 2 : 1;
  R.ZE = R.cplx ? 4 : 1;
  plan_capacities(R);
  R.log_cap_upd = 2 * std::max(R.L - 1, 1) * max_sweeps;
  R.log_cap_piv = 1;
  for (int b = 0; b < R.L - 1; ++b) R.log_cap_piv = std::max(R.log_cap_piv, R.rmax[b]);
  R.colcap = 32;
  for (int b = 0; b < R.L - 1; ++b) R.colcap = std::max(R.colcap, R.mmax[b]);
  for (int s = 0; s < R.L; ++s) R.colcap = std::max(R.colcap, R.yr[s]);
  R.colcap *= R.Z;
  // envelope (rook mode: the single-cluster envelope, real values)
  R.one = one;
  R.rook = rook;
  // streamed Pi: real values, full pivoting, default tiers (ACI_STREAM_PI=0: off, for A/B)
  static const bool stream_env = [] {
    const char *e = getenv("ACI_STREAM_PI");
    return !e || atoi(e) != 0;
  }();
  R.stream = stream_env && !R.cplx && !rook && !one && R.L >= 3 ? 1 : 0;
  if (rook && R.cplx) return fail(ACI_ERR_UNSUPPORTED, "aci: rook pivoting is implemented for real values only");
  auto ok = [&](int m, int n) {
    if (rook) return prrlu_supported_rook(m, n);
    if (one && !prrlu_coop_multicluster()) return prrlu_supported_one(m, n, R.cplx != 0);
    return prrlu_supported(m, n, R.cplx != 0);
  };
  for (int b = 0; b < R.L - 1; ++b)
    if (!ok(R.mmax[b], R.nmax[b]))
      return fail(ACI_ERR_UNSUPPORTED, "aci: 2-site block " + std::to_string(R.mmax[b]) + "x" +
                                           std::to_string(R.nmax[b]) + " exceeds the prrLU envelope");
  for (int s = 1; s < R.L; ++s)
    if (!ok(R.yr[s], R.nmax[s - 1]))
      return fail(ACI_ERR_UNSUPPORTED, "aci: y_init bond too large for the prrLU envelope");
  return ACI_OK;
}

// multi-cluster prrLU launches of different host threads are serialised (aci_elementwise_ex)
static std::mutex multi_cluster_mu;

extern "C" int aci_elementwise_ex(aci_op op, const tt_t *const *inputs, int n_inputs, double tol, int maxrank,
                                  int max_sweeps, tt_t **out, aci_report *rep, const aci_options *opts) {
  NvtxRange nv_call("aci_elementwise");
  dbg_pending("entry");
  // a successful call leaves the thread's last-error state as it found it: runtime calls that
  // returned success may still leave a pending error behind (seen under ncu for launches with a
  // launch-completion event), which the caller's next CUDA call would report as its own
  const bool clean_entry = cudaPeekAtLastError() == cudaSuccess;
  auto t_start = std::chrono::steady_clock::now();
  if (!out) return fail(ACI_ERR_INVALID, "aci: out is null");
  *out = nullptr;
  if (!(tol >= 0) || maxrank < 1 || max_sweeps < 1) return fail(ACI_ERR_INVALID, "aci: tol < 0, maxrank < 1 or max_sweeps < 1");
  aci_options o = {};
  if (opts) o = *opts;
  if (o.tol_mode != ACI_TOL_RELATIVE && o.tol_mode != ACI_TOL_ABSOLUTE) return fail(ACI_ERR_INVALID, "aci: bad tol_mode");
  // Default-tier calls may launch prrLU grids of several clusters that spin on each other; two
  // such launches co-scheduled from different host threads could each hold part of their
  // clusters and wait forever, so those calls are serialised within the process. Calls with
  // aci_options.concurrent use single-cluster launches and run concurrently.
  std::unique_lock<std::mutex> serial(multi_cluster_mu, std::defer_lock);
  if (!o.concurrent) serial.lock();
  Inputs I;
  int st = prepare(op, inputs, n_inputs, I);
  if (st) return st;
  if ((st = check_device())) return st;
  const tt_s *t0 = I.tts[0];
  const int L = t0->L;
  if (L < 2) return fail(ACI_ERR_INVALID, "aci: L must be >= 2 (the 2-site update needs two sites)");
  cudaStream_t strm = o.stream ? (cudaStream_t)o.stream : lib_stream();
  gemm_init();
  prrlu_init();
  if (!side_stream_init()) {
    cudaGetLastError();
    return fail(ACI_ERR_CUDA, "aci: could not create the look-ahead stream");
  }

  // ---- y_init (R9)
  tt_s *ygen = nullptr;
  const tt_s *y = o.y_init;
  if (y) {
    if (y->L != L || y->d != t0->d) return fail(ACI_ERR_SHAPE, "aci: y_init shape differs from the inputs");
    if (y->cplx != t0->cplx) return fail(ACI_ERR_SHAPE, "aci: y_init must be complex iff the inputs are");
  } else {
    std::vector<int> yr(L + 1, 1);
    for (int s = 1; s < L; ++s) {
      int r = maxrank;
      for (auto *t : I.tts) r = std::min(r, t->ranks[s]);
      yr[s] = (int)std::min<long long>(r, std::min(capped_prod(t0->d, 0, s - 1), capped_prod(t0->d, s, L - 1)));
    }
    std::vector<std::vector<double>> cores(L);
    std::vector<const double *> ptr(L);
    uint64_t cnt = 0;
    for (int s = 0; s < L; ++s) {
      cores[s].resize((size_t)yr[s] * t0->d[s] * yr[s + 1] * (t0->cplx ? 2 : 1));
      for (auto &x : cores[s]) x = normal_at(o.seed, cnt++);
      ptr[s] = cores[s].data();
    }
    st = t0->cplx ? tt_create_z(L, t0->d.data(), yr.data(), ptr.data(), &ygen)
                  : tt_create(L, t0->d.data(), yr.data(), ptr.data(), &ygen);
    if (st) return st;
    y = ygen;
  }

  Run R;
  if (o.pivoting != ACI_PIVOT_FULL && o.pivoting != ACI_PIVOT_ROOK) {
    tt_destroy(ygen);
    return fail(ACI_ERR_INVALID, "aci: bad pivoting mode");
  }
  st = build_run(I, y, maxrank, max_sweeps, R, o.concurrent ? 1 : 0, o.pivoting == ACI_PIVOT_ROOK ? 1 : 0);
  if (st) { tt_destroy(ygen); return st; }
  size_t need = carve(R, nullptr);
  char *ws = nullptr;
  bool own_ws = false;
  if (o.workspace) {
    if (o.workspace_bytes < need) { tt_destroy(ygen); return fail(ACI_ERR_OOM, "aci: caller workspace too small"); }
    // 16-byte packet stores/loads and cp.async tiles need aligned carve offsets: the carver aligns
    // offsets to 256 bytes, so the base must be 256-byte aligned too (aci.h)
    if (reinterpret_cast<uintptr_t>(o.workspace) & 255u) {
      tt_destroy(ygen);
      return fail(ACI_ERR_INVALID, "aci: caller workspace must be 256-byte aligned");
    }
    ws = (char *)o.workspace;
  } else {
    bool busy = false;
    ws = stream_workspace_acquire(strm, need, &busy);  // pinned until cleanup()
    own_ws = ws != nullptr;
    if (!ws) {
      tt_destroy(ygen);
      if (busy) return fail(ACI_ERR_INVALID, "aci: another call is running on this stream (use one stream per concurrent call)");
      return fail(ACI_ERR_OOM, "aci: workspace allocation failed");
    }
  }
  carve(R, ws);
  auto cleanup = [&]() {
    if (own_ws) stream_workspace_release(strm);
    tt_destroy(ygen);
  };

  Prof prof;
  prof.on = o.profile != nullptr;
  prof.st = strm;
  R.P = &prof;

  // ---- initial state
  cudaMemsetAsync(R.rk, 0, sizeof(int) * (L + 1), strm);
  {
    std::vector<int> rk0(L + 1, 0);
    rk0[0] = 1; rk0[L] = 1;
    // host->device copies of state: boundary ranks and the static bond table (pointers and
    // input ranks of every bond update; no data)
    cudaMemcpyAsync(R.rk, rk0.data(), sizeof(int) * (L + 1), cudaMemcpyHostToDevice, strm);
    build_statics(R, I.op);
    cudaMemcpyAsync(R.dStat, R.hStat.data(), sizeof(BondStatic) * R.hStat.size(), cudaMemcpyHostToDevice, strm);
    cudaStreamSynchronize(strm);
  }
  cudaMemsetAsync(R.scale, 0, sizeof(unsigned long long), strm);
  cudaMemsetAsync(R.sp, 0, sizeof(unsigned long long), strm);
  cudaMemsetAsync(R.sdone, 0, sizeof(unsigned), strm);
  cudaMemsetAsync(R.maxeps, 0, sizeof(unsigned long long), strm);
  cudaMemsetAsync(R.nonfinite, 0, sizeof(int), strm);
  cudaMemsetAsync(R.iter, 0, sizeof(int), strm);
  // tags in the exchange buffers must never match stale data: clear them once per call
  cudaMemsetAsync(R.keys, 0, sizeof(unsigned long long) * 2 * 148 * 4, strm);
  cudaMemsetAsync(R.colpub, 0, sizeof(unsigned long long) * 2 * 148 * R.colcap * 2 * prrlu_col_spread(), strm);
  cudaMemsetAsync(R.epoch, 0, sizeof(unsigned), strm);
  for (int s = 0; s < L; ++s)
    cudaMemcpyAsync(R.Yin[s], y->dcores + y->off[s], sizeof(double) * (y->off[s + 1] - y->off[s]),
                    cudaMemcpyDeviceToDevice, strm);
  if (R.cplx) {
    // right-operand copies of the input cores (core s viewed chi_s x (d_s chi_{s+1}))
    prof.begin(ACI_PROF_CANON);
    for (int n = 0; n < R.N; ++n)
      for (int s = 0; s < L; ++s)
        expand_kernel<<<64, 256, 0, strm>>>(R.xcore0[n] + R.xoff[n][s], R.Xe[n][s], R.xr[n][s], R.d[s] * R.xr[n][s + 1]);
    prof.end(R.N * L);
  }

  // ---- a0: CI-canonicalise y_init, right-to-left
  {
    NvtxRange nv("aci: canonicalise y_init (a0)");
    for (int s = L - 1; s >= 1; --s) canon_step(R, tol, o.tol_mode, s, strm);
  }
  prof.begin(ACI_PROF_CANON);
  copy_prev_kernel<<<1, 64, 0, strm>>>(R.rk, R.prev, L);
  prof.end(1);
  pre_launch(R, strm);  // B^n_b of the first L->R half-sweep

  // ---- main loop. One iteration (L->R and R->L half-sweeps + convergence test)
  // is a fixed sequence of launches whose live sizes are read on the device, so it is captured
  // once as a CUDA graph and replayed; only the convergence flag comes back to the host.
  auto one_iteration = [&]() {
    int step = 0;
#ifdef ACI_STREAM_TS
    cudaMemsetAsync(R.ts, 0, sizeof(unsigned long long) * 16 * L, strm);
#endif
    if (R.stream) {  // the streams poll the L->R pivot rows and ranks: -1 = not written yet
      cudaMemsetAsync(R.prow0, 0xff, sizeof(int) * R.prow0_ints, strm);
      cudaMemsetAsync(R.rout, 0xff, sizeof(int) * L, strm);
    }
    for (int b = 0; b < L - 1; ++b)
      bond_update(R, tol, o.tol_mode, b, 0, step++, b == 0, b + 1 < L - 1 ? dstat(R, 0, b + 1) : dstat(R, 1, L - 2), strm);
    for (int b = L - 2; b >= 0; --b)
      bond_update(R, tol, o.tol_mode, b, 1, step++, false, b > 0 ? dstat(R, 1, b - 1) : nullptr, strm);
    index_join(strm);
    prof.begin(ACI_PROF_CONV);
    converge_kernel<<<1, 32, 0, strm>>>(R.rk, R.prev, L, R.maxeps, R.scale, tol, o.tol_mode, R.conv, R.err,
                                        R.iter);
    prof.end(1);
  };
  cudaGraphExec_t gexec = nullptr;
  bool gcached = false;
  int graph_iters = 0;
  auto tg0 = std::chrono::steady_clock::now();
  static const bool graphs = [] {  // ACI_NO_GRAPH=1: direct launches (debugging)
    const char *e = getenv("ACI_NO_GRAPH");
    return !e || atoi(e) == 0;
  }();
  if (!prof.on && strm != nullptr && graphs) {
    // the captured iteration depends only on host values (shapes, pointers, op, tol), so a call
    // that repeats them (same workspace address and inputs) replays the instantiated graph
    const std::vector<uint64_t> key = graph_key(R, I.op, tol, o.tol_mode, ws, need, strm);
    gexec = graph_cache_acquire(key, &prof.per_iter_launches);
    gcached = gexec != nullptr;
    if (!gexec) {
      cudaGraph_t graph = nullptr;
      const int64_t before = prof.total;
      if (cudaStreamBeginCapture(strm, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
        one_iteration();
        if (cudaStreamEndCapture(strm, &graph) != cudaSuccess || !graph ||
            cudaGraphInstantiate(&gexec, graph, 0) != cudaSuccess)
          gexec = nullptr;
        if (graph) cudaGraphDestroy(graph);
      }
      cudaGetLastError();  // a failed capture falls back to direct launches
      if (!gexec) R.launch_err = cudaSuccess;  // (their launch results are what counts)
      prof.per_iter_launches = prof.total - before;
      prof.total = before;
      if (gexec) gcached = graph_cache_insert(key, gexec, prof.per_iter_launches);
    }
  }
  const float ms_graph = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - tg0).count();
  int it = 0, converged = 0;
  cudaEvent_t ev_it[2] = {nullptr, nullptr};
  if (o.iter_ms) {
    cudaEventCreate(&ev_it[0]);
    cudaEventCreate(&ev_it[1]);
  }
  for (it = 1; it <= max_sweeps; ++it) {
    NvtxRange nv("aci: iteration (L->R + R->L half-sweeps, convergence test)");
    if (ev_it[0]) cudaEventRecord(ev_it[0], strm);
    if (gexec && cudaGraphLaunch(gexec, strm) != cudaSuccess) {
      // a rejected replay (seen under ncu for graphs instantiated by an earlier call) ran nothing:
      // drop the graph and run this and the remaining iterations as direct launches, leaving no
      // pending runtime error behind for the caller's next CUDA call
      cudaGetLastError();
      graph_cache_release(gexec, gcached, true);
      gexec = nullptr;
      gcached = false;
    }
    if (gexec) {
      prof.total += prof.per_iter_launches;
      ++graph_iters;
    } else {
      one_iteration();
    }
    if (ev_it[1]) cudaEventRecord(ev_it[1], strm);
    int flag = 0;
    cudaMemcpyAsync(&flag, R.conv, sizeof(int), cudaMemcpyDeviceToHost, strm);
    cudaError_t e = cudaStreamSynchronize(strm);
    if (e != cudaSuccess) {
      graph_cache_release(gexec, gcached, true);
      cleanup();
      return fail(ACI_ERR_CUDA, std::string("aci sweep: ") + cudaGetErrorString(e));
    }
    if (ev_it[0]) cudaEventElapsedTime(&o.iter_ms[it - 1], ev_it[0], ev_it[1]);
    if (flag) { converged = 1; break; }
  }
  for (auto ev : ev_it)
    if (ev) cudaEventDestroy(ev);
  graph_cache_release(gexec, gcached, false);  // every replay of this call is complete (synchronised)
  gexec = nullptr;
  if (it > max_sweeps) it = max_sweeps;
  const int slot = it * 2 * (L - 1);

  // ---- results: ranks, flags, log
  std::vector<int> rk(L + 1);
  int nonfinite = 0;
  double err = 0, scale = 0;
  unsigned long long scale_bits = 0;
  cudaMemcpyAsync(rk.data(), R.rk, sizeof(int) * (L + 1), cudaMemcpyDeviceToHost, strm);
  cudaMemcpyAsync(&nonfinite, R.nonfinite, sizeof(int), cudaMemcpyDeviceToHost, strm);
  cudaMemcpyAsync(&err, R.err, sizeof(double), cudaMemcpyDeviceToHost, strm);
  cudaMemcpyAsync(&scale_bits, R.scale, sizeof(double), cudaMemcpyDeviceToHost, strm);
  cudaError_t e = cudaStreamSynchronize(strm);
  if (e == cudaSuccess) e = R.launch_err;  // a rejected launch leaves the results unwritten
  if (e != cudaSuccess) { cleanup(); return fail(ACI_ERR_CUDA, std::string("aci: ") + cudaGetErrorString(e)); }
  std::memcpy(&scale, &scale_bits, sizeof(double));
  if (nonfinite) { cleanup(); return fail(ACI_ERR_NONFINITE, "aci: f produced NaN/Inf (S:255)"); }

  // ---- a8: output cores from the last right-to-left half-sweep (R5)
  NvtxRange nv_out("aci: output cores (a8)");
  tt_s *res = tt_alloc_shape(L, t0->d.data(), rk.data(), R.cplx);
  if (core_alloc(res, sizeof(double) * std::max<size_t>(res->total, 1), strm) != cudaSuccess) {
    cudaGetLastError();
    delete res;
    cleanup();
    return fail(ACI_ERR_OOM, "aci: output allocation failed");
  }
  cudaMemcpyAsync(res->dcores, R.Y0, sizeof(double) * (res->off[1] - res->off[0]), cudaMemcpyDeviceToDevice, strm);
  if (R.cplx) {
    std::vector<ZTrsmArgs> za(L - 1);
    int nmx = 1, rmx = 1;
    for (int b = 0; b < L - 1; ++b) {
      za[b] = ZTrsmArgs{R.Ust[b], R.nmax[b], R.pcol[L + b], res->dcores + res->off[b + 1], rk[b + 1], R.d[b + 1] * rk[b + 2]};
      nmx = std::max(nmx, za[b].n);
      rmx = std::max(rmx, za[b].r);
    }
    cudaMemcpyAsync(R.dtrsm, za.data(), sizeof(ZTrsmArgs) * za.size(), cudaMemcpyHostToDevice, strm);
    const int smem = rmx * kZTrsmCols * 2 * (int)sizeof(double);
    cudaFuncSetAttribute(ztrsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    prof.begin(ACI_PROF_TRSM);
    ztrsm_kernel<<<dim3((nmx + kZTrsmCols - 1) / kZTrsmCols, L - 1), 128, smem, strm>>>(
        reinterpret_cast<const ZTrsmArgs *>(R.dtrsm));
    prof.end(1);
    e = cudaStreamSynchronize(strm);
    if (e != cudaSuccess) {
      tt_destroy(res);
      cleanup();
      return fail(ACI_ERR_CUDA, std::string("aci output: ") + cudaGetErrorString(e));
    }
  } else {
    // Blocked back substitution B = U_J^{-1} U (64-row blocks from the bottom): per step one
    // batched DMMA GEMM B[R] = U[R] - U_J[R, below] B[below] over all bonds, then the diagonal
    // block solve. The final ranks are known on the host here, so descriptors are built here.
    constexpr int NB = kTriNB;
    std::vector<TrsmArgs> ta(L - 1);
    int nmx = 1, nsteps = 0;
    for (int b = 0; b < L - 1; ++b) {
      ta[b].U = R.Ust[b]; ta[b].ldu = R.nmax[b]; ta[b].cols = R.pcol[L + b]; ta[b].b = b; ta[b].d1 = R.d[b + 1];  // last R->L pivots
      ta[b].UJ = R.UJ[b]; ta[b].ldj = R.rmax[b];
      ta[b].out = res->dcores + res->off[b + 1];
      nmx = std::max(nmx, R.d[b + 1] * rk[b + 2]);
      nsteps = std::max(nsteps, (rk[b + 1] + NB - 1) / NB);
    }
    std::vector<GemmDesc> gd;
    std::vector<TriArgs> tr;
    std::vector<int> gcount(nsteps, 0), tcount(nsteps, 0);
    for (int s = 0; s < nsteps; ++s) {
      for (int b = 0; b < L - 1; ++b) {
        const int r = rk[b + 1], n = R.d[b + 1] * rk[b + 2];
        const int nbk = (r + NB - 1) / NB;
        const int blk = nbk - 1 - s;
        if (blk < 0) continue;
        const int r0 = blk * NB, nr = std::min(NB, r - r0), below = r0 + nr;
        GemmDesc g = {};
        g.C = ta[b].out + (size_t)r0 * n; g.M = nr; g.N = n; g.ldc = n; g.nin = 1;
        g.S = R.Ust[b] + (size_t)r0 * R.nmax[b]; g.lds = R.nmax[b];
        g.A[0] = R.UJ[b] + (size_t)r0 * R.rmax[b] + below; g.lda[0] = R.rmax[b]; g.K[0] = r - below;
        g.B[0] = ta[b].out + (size_t)below * n; g.ldb[0] = n;
        gd.push_back(g);
        gcount[s]++;
        tr.push_back(TriArgs{R.UJ[b], R.rmax[b], ta[b].out, n, r0, nr});
        tcount[s]++;
      }
    }
    // descriptors live in the workspace tail (sized for (L-1) * ceil(rmax/NB) entries)
    cudaMemcpyAsync(R.dtrsm, ta.data(), sizeof(TrsmArgs) * (L - 1), cudaMemcpyHostToDevice, strm);
    cudaMemcpyAsync(R.dtgemm, gd.data(), sizeof(GemmDesc) * gd.size(), cudaMemcpyHostToDevice, strm);
    cudaMemcpyAsync(R.dtri, tr.data(), sizeof(TriArgs) * tr.size(), cudaMemcpyHostToDevice, strm);
    prof.begin(ACI_PROF_TRSM);
    gather_uj_kernel<<<dim3(64, L - 1), 256, 0, strm>>>(R.dtrsm, R.rk);
    size_t go = 0;
    for (int s = 0; s < nsteps; ++s) {
      launch_gemm_sub(R.dtgemm + go, gcount[s], NB, nmx, strm);
      tri_block_kernel<<<dim3((nmx + kTriThreads - 1) / kTriThreads, tcount[s]), kTriThreads, 0, strm>>>(R.dtri + go);
      go += gcount[s];
    }
    prof.end(1 + 2 * nsteps);
    e = cudaStreamSynchronize(strm);
    if (e != cudaSuccess) {
      tt_destroy(res);
      cleanup();
      return fail(ACI_ERR_CUDA, std::string("aci output: ") + cudaGetErrorString(e));
    }
  }

  // ---- report + optional log / index sets
  const int nupd = slot;
  std::vector<int> info((size_t)nupd * 5);
  std::vector<double> es((size_t)nupd * 2);
  // stream-ordered copies (a synchronous cudaMemcpy would synchronise with the legacy stream,
  // which other host threads' stream captures forbid)
  cudaMemcpyAsync(info.data(), R.log_info, sizeof(int) * info.size(), cudaMemcpyDeviceToHost, strm);
  cudaMemcpyAsync(es.data(), R.log_es, sizeof(double) * es.size(), cudaMemcpyDeviceToHost, strm);
  cudaStreamSynchronize(strm);
  aci_report rp = {};
  rp.error_estimate = err;
  rp.scale = scale;
  rp.iterations = it;
  rp.converged = converged;
  rp.n_updates = nupd;
  for (int s = 0; s <= L; ++s) rp.max_rank = std::max(rp.max_rank, rk[s]);
  for (int u = 0; u < nupd; ++u) {
    const int b = info[u * 5], rl = info[u * 5 + 2], rr = info[u * 5 + 3], r = info[u * 5 + 4];
    const int m = rl * R.d[b], n = R.d[b + 1] * rr;
    for (int i = 0; i < R.N; ++i) {
      const double c0 = R.xr[i][b], c1 = R.xr[i][b + 1], c2 = R.xr[i][b + 2];
      // complex: 4 real products per complex product (RZ5)
      rp.flops_contraction +=
          R.ZE * (2.0 * rl * c0 * R.d[b] * c1 + 2.0 * c1 * R.d[b + 1] * c2 * rr + 2.0 * m * c1 * n);
    }
    for (int k = 0; k < r; ++k) rp.flops_prrlu += R.ZE * 2.0 * (m - k - 1) * (double)(n - k - 1);
    rp.pivot_steps += r;
  }
  for (int b = 0; b < L - 1; ++b) {
    const double r = rk[b + 1], n = R.d[b + 1] * rk[b + 2];
    rp.flops_trsm += R.ZE * r * r * (n - r);
  }
  if (o.log) {
    aci_pivot_log *lg = o.log;
    const int nw = std::min(nupd, lg->capacity_updates);
    for (int u = 0; u < nw; ++u) {
      if (lg->info) std::memcpy(lg->info + u * 5, &info[u * 5], sizeof(int) * 5);
      if (lg->eps_scale) std::memcpy(lg->eps_scale + u * 2, &es[u * 2], sizeof(double) * 2);
      const int r = std::min(info[u * 5 + 4], lg->capacity_pivots);
      if (lg->rows)
        cudaMemcpyAsync(lg->rows + (size_t)u * lg->capacity_pivots, R.log_rows + (size_t)u * R.log_cap_piv,
                        sizeof(int) * r, cudaMemcpyDeviceToHost, strm);
      if (lg->cols)
        cudaMemcpyAsync(lg->cols + (size_t)u * lg->capacity_pivots, R.log_cols + (size_t)u * R.log_cap_piv,
                        sizeof(int) * r, cudaMemcpyDeviceToHost, strm);
    }
    lg->n_written = nw;
    if (lg->canon_n) {
      std::vector<int> cn(L + 1, 0);
      cudaMemcpyAsync(cn.data(), R.canon_n, sizeof(int) * (L + 1), cudaMemcpyDeviceToHost, strm);
      cudaStreamSynchronize(strm);
      for (int s = 1; s < L; ++s) {
        lg->canon_n[s] = cn[s];
        if (lg->canon_cols)
          cudaMemcpyAsync(lg->canon_cols + (size_t)s * lg->capacity_pivots, R.canon_cols + (size_t)s * R.log_cap_piv,
                          sizeof(int) * std::min(cn[s], lg->capacity_pivots), cudaMemcpyDeviceToHost, strm);
      }
    }
  }
  if (o.I_sets)
    for (int b = 0; b < L - 1; ++b)
      if (o.I_sets[b])
        cudaMemcpyAsync(o.I_sets[b], R.Imi[b], (size_t)rk[b + 1] * (b + 1), cudaMemcpyDeviceToHost, strm);
  if (o.J_sets)
    for (int s = 1; s < L; ++s)
      if (o.J_sets[s])
        cudaMemcpyAsync(o.J_sets[s], R.Jmi[s], (size_t)rk[s] * (L - s), cudaMemcpyDeviceToHost, strm);
  e = cudaStreamSynchronize(strm);
#ifdef ACI_STREAM_TS
  {  // b, start, first-r-seen, last item start, exit, update start (ns, relative to the kernel start), r
    std::vector<unsigned long long> h(16 * (size_t)L);
    cudaMemcpy(h.data(), R.ts, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
    for (int b = 0; b + 2 < L; ++b) {
      const unsigned long long *t = &h[16 * b];
      const unsigned long long t0 = ~t[0], tr = ~t[1];
      if (!t[0]) continue;
      fprintf(stderr, "ts b=%d r=%lld start->r %.2f us | r->last item %.2f | r->exit %.2f | exit->update %.2f | item after r: %s\n",
              b, (long long)t[6], (tr - t0) * 1e-3, ((long long)t[3] - (long long)tr) * 1e-3,
              ((long long)t[4] - (long long)tr) * 1e-3, ((long long)t[5] - (long long)t[4]) * 1e-3, t[2] ? "yes" : "no");
      fprintf(stderr, "   max per item: rowp %.2f | A load %.2f | dmma %.2f | epilogue %.2f | A store %.2f us\n", t[8] * 1e-3,
              t[9] * 1e-3, t[10] * 1e-3, t[11] * 1e-3, t[12] * 1e-3);
    }
  }
#endif
  cleanup();
  if (e != cudaSuccess) { tt_destroy(res); return fail(ACI_ERR_CUDA, std::string("aci: ") + cudaGetErrorString(e)); }
  auto t_end = std::chrono::steady_clock::now();
  rp.ms = std::chrono::duration<float, std::milli>(t_end - t_start).count();
  rp.n_launches = prof.total;
  rp.graph_iterations = graph_iters;
  rp.ms_graph_setup = ms_graph;
  if (o.profile) prof.collect(o.profile);
  if (rep) *rep = rp;
  *out = res;
  dbg_pending("return");
  if (clean_entry) cudaGetLastError();
  return converged ? ACI_OK : ACI_NOT_CONVERGED;
}

extern "C" int aci_elementwise(aci_op op, const tt_t *const *inputs, int n_inputs, double tol, int maxrank,
                               int max_sweeps, tt_t **out, aci_report *rep) {
  return aci_elementwise_ex(op, inputs, n_inputs, tol, maxrank, max_sweeps, out, rep, nullptr);
}

extern "C" int aci_elementwise_batch(aci_job *jobs, int n_jobs, int max_parallel) {
  if (n_jobs < 0 || (n_jobs > 0 && !jobs)) return fail(ACI_ERR_INVALID, "aci_elementwise_batch: null jobs");
  if (n_jobs == 0) return ACI_OK;
  const int nt = std::max(1, std::min(n_jobs, max_parallel > 0 ? max_parallel : 8));
  std::atomic<int> next{0};
  auto worker = [&]() {
    for (int j = next.fetch_add(1); j < n_jobs; j = next.fetch_add(1)) {
      aci_job &J = jobs[j];
      aci_options o = J.options ? *J.options : aci_options{};
      o.concurrent = 1;
      o.stream = nullptr;  // the worker thread's library stream
      o.workspace = nullptr;
      o.workspace_bytes = 0;
      J.status = aci_elementwise_ex(J.op, J.inputs, J.n_inputs, J.tol, J.maxrank, J.max_sweeps, J.out, J.rep, &o);
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(worker);
  worker();
  for (auto &t : th) t.join();
  for (int j = 0; j < n_jobs; ++j)
    if (jobs[j].status < 0) return fail(jobs[j].status, "aci_elementwise_batch: job " + std::to_string(j) + " failed");
  return ACI_OK;
}

extern "C" int aci_workspace_query(const tt_t *const *inputs, int n_inputs, int maxrank, int max_sweeps,
                                   const tt_t *y_init, size_t *bytes) {
  if (!bytes || !inputs || n_inputs < 1 || maxrank < 1 || max_sweeps < 1)
    return fail(ACI_ERR_INVALID, "aci_workspace_query: bad args");
  std::vector<double> coef(1, 1.0);
  std::vector<int> expo(n_inputs, 1);
  aci_op op = {1, coef.data(), expo.data()};
  Inputs I;
  int st = prepare(op, inputs, n_inputs, I);
  if (st) return st;
  const tt_s *t0 = I.tts[0];
  tt_s tmp;
  if (!y_init) {
    tmp.L = t0->L;
    tmp.d = t0->d;
    tmp.ranks.assign(t0->L + 1, 1);
    for (int s = 1; s < t0->L; ++s) {
      int r = maxrank;
      for (auto *t : I.tts) r = std::min(r, t->ranks[s]);
      tmp.ranks[s] = (int)std::min<long long>(r, std::min(capped_prod(t0->d, 0, s - 1), capped_prod(t0->d, s, t0->L - 1)));
    }
    y_init = &tmp;
  }
  Run R;
  st = build_run(I, y_init, maxrank, max_sweeps, R);  // the pivot log holds max_sweeps iterations
  if (st) return st;
  *bytes = carve(R, nullptr);
  return ACI_OK;
}

// ============================================================================ evaluation (K6)
extern "C" int tt_evaluate_device(const tt_t *t, int64_t npts, const uint8_t *dev_idx, double *dev_out,
                                  void *stream) {
  if (!t || npts < 0 || (npts > 0 && (!dev_idx || !dev_out))) return fail(ACI_ERR_INVALID, "tt_evaluate: bad args");
  if (npts == 0) return ACI_OK;
  cudaStream_t st = stream ? (cudaStream_t)stream : lib_stream();  // never the legacy stream
  const int L = t->L;
  // complex TTs: the same real pipeline on interleaved vectors (ranks x 2) against 2x2-block
  // expanded cores
  const int z = t->cplx ? 2 : 1;
  int rmx = 1, wmx = 1;
  size_t emx = 1;
  for (int s = 0; s < L; ++s) {
    rmx = std::max(rmx, z * t->ranks[s + 1]);
    wmx = std::max(wmx, z * t->d[s] * t->ranks[s + 1]);
    emx = std::max(emx, (size_t)4 * t->ranks[s] * t->d[s] * t->ranks[s + 1]);
  }
  const int64_t P = 8192;
  double *V = nullptr, *W = nullptr, *E = nullptr;
  GemmDesc *desc = nullptr;
  if (cudaMallocAsync((void **)&V, sizeof(double) * P * rmx, st) != cudaSuccess ||
      cudaMallocAsync((void **)&W, sizeof(double) * P * wmx, st) != cudaSuccess ||
      cudaMallocAsync((void **)&desc, sizeof(GemmDesc), st) != cudaSuccess ||
      (t->cplx && cudaMallocAsync((void **)&E, sizeof(double) * emx * L, st) != cudaSuccess))
    return fail(ACI_ERR_OOM, "tt_evaluate: workspace");
  std::vector<size_t> eoff(L + 1, 0);
  for (int s = 0; s < L; ++s) eoff[s + 1] = eoff[s] + (t->cplx ? (size_t)4 * t->ranks[s] * t->d[s] * t->ranks[s + 1] : 0);
  if (t->cplx)
    for (int s = 1; s < L; ++s)
      expand_kernel<<<64, 256, 0, st>>>(t->dcores + t->off[s], E + eoff[s], t->ranks[s], t->d[s] * t->ranks[s + 1]);
  FOp dummy = {};
  for (int64_t p0 = 0; p0 < npts; p0 += P) {
    const int np = (int)std::min<int64_t>(P, npts - p0);
    const uint8_t *ix = dev_idx + p0 * L;
    eval_first_kernel<<<296, 256, 0, st>>>(t->dcores, V, ix, L, z * t->ranks[1], np);
    for (int s = 1; s < L; ++s) {
      const int r0 = t->ranks[s], r1 = t->ranks[s + 1];
      const double *X = t->cplx ? E + eoff[s] : t->dcores + t->off[s];
      eval_desc_kernel<<<1, 1, 0, st>>>(desc, V, X, W, np, z * r0, z * t->d[s] * r1);
      launch_gemm(desc, 1, np, z * t->d[s] * r1, 1, false, dummy, nullptr, nullptr, st);
      eval_select_kernel<<<592, 256, 0, st>>>(W, V, ix, L, s, t->d[s], z * r1, np);
    }
    cudaMemcpyAsync(dev_out + z * p0, V, sizeof(double) * np * z, cudaMemcpyDeviceToDevice, st);
  }
  cudaFreeAsync(V, st);
  cudaFreeAsync(W, st);
  cudaFreeAsync(desc, st);
  if (E) cudaFreeAsync(E, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(ACI_ERR_CUDA, std::string("tt_evaluate: ") + cudaGetErrorString(e));
  return ACI_OK;
}

// a5 alone (include/aci.h aci_prrlu): the library's prrLU on a caller's device block, launched for
// the static capacity static_m x static_n as a bond update launches it (tier and hand-off chosen on
// the device from the live m x n)
extern "C" int aci_prrlu(const double *dev_M, int m, int n, int maxrank, double tol, int tol_mode, int static_m,
                         int static_n, int *dev_rows, int *dev_cols, double *dev_U, int *rank, double *eps,
                         void *stream) {
  if (!dev_M || !dev_rows || !dev_cols || !rank || !eps || m < 1 || n < 1 || maxrank < 1 || !(tol >= 0.0) ||
      (tol_mode != ACI_TOL_RELATIVE && tol_mode != ACI_TOL_ABSOLUTE))
    return fail(ACI_ERR_INVALID, "aci_prrlu: bad args");
  int st_ = check_device();
  if (st_) return st_;
  const int sm = static_m > 0 ? static_m : m, sn = static_n > 0 ? static_n : n;
  if (sm < m || sn < n) return fail(ACI_ERR_INVALID, "aci_prrlu: static size below the live size");
  if (!prrlu_supported(sm, sn)) return fail(ACI_ERR_UNSUPPORTED, "aci_prrlu: block beyond aci_limits");
  prrlu_init();
  cudaStream_t st = stream ? (cudaStream_t)stream : lib_stream();
  const int colcap = std::max(sm, 1024);
  const size_t colwords = (size_t)2 * 148 * colcap * 2 * prrlu_col_spread(), keywords = (size_t)2 * 148 * 4;
  unsigned long long *colpub = nullptr, *keys = nullptr;
  unsigned *ctr = nullptr;
  LuDims *dims = nullptr;
  int *rout = nullptr;
  double *eout = nullptr;
  const size_t small = 64 + sizeof(LuDims) + 16;
  char *sb = nullptr;
  if (cudaMallocAsync((void **)&colpub, 8 * colwords, st) != cudaSuccess ||
      cudaMallocAsync((void **)&keys, 8 * keywords, st) != cudaSuccess ||
      cudaMallocAsync((void **)&sb, small, st) != cudaSuccess)
    return fail(ACI_ERR_OOM, "aci_prrlu: workspace");
  // small scratch: counter (4) | epoch (4) | scale (8) | r (4) | eps (8, at 24) | dims (at 64)
  ctr = reinterpret_cast<unsigned *>(sb);
  unsigned *epoch = ctr + 1;
  unsigned long long *scale = reinterpret_cast<unsigned long long *>(sb + 8);
  rout = reinterpret_cast<int *>(sb + 16);
  eout = reinterpret_cast<double *>(sb + 24);
  dims = reinterpret_cast<LuDims *>(sb + 64);
  cudaMemsetAsync(colpub, 0, 8 * colwords, st);
  cudaMemsetAsync(keys, 0, 8 * keywords, st);
  cudaMemsetAsync(sb, 0, small, st);
  const int kmax = std::min(maxrank, std::min(m, n));
  const LuDims D{m, n, n, kmax, n};
  cudaMemcpyAsync(dims, &D, sizeof(D), cudaMemcpyHostToDevice, st);
  LuArgs a = {};
  a.M = dev_M; a.dims = dims; a.tol = tol; a.thr_mode = tol_mode == ACI_TOL_RELATIVE ? 1 : 2; a.scale_bits = scale;
  a.rows = dev_rows; a.cols = dev_cols; a.r_out = rout; a.eps_out = eout; a.U = dev_U;
  a.colpub = colpub; a.colcap = colcap; a.keys = keys; a.counter = ctr; a.epoch = epoch;
  cudaError_t le;
  {
    std::lock_guard<std::mutex> serial(multi_cluster_mu);  // multi-cluster grids: one at a time (aci_elementwise_ex)
    le = launch_prrlu(a, sm, sn, st, false, false, nullptr, false);
  }
  int hr = 0;
  double he = 0.0;
  cudaMemcpyAsync(&hr, rout, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&he, eout, sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(colpub, st);
  cudaFreeAsync(keys, st);
  cudaFreeAsync(sb, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  if (le != cudaSuccess || e != cudaSuccess)
    return fail(ACI_ERR_CUDA, std::string("aci_prrlu: ") + cudaGetErrorString(le != cudaSuccess ? le : e));
  *rank = hr;
  *eps = he;
  return ACI_OK;
}

extern "C" int tt_evaluate(const tt_t *t, int64_t npts, const uint8_t *idx, double *out) {
  if (!t || npts < 0 || (npts > 0 && (!idx || !out))) return fail(ACI_ERR_INVALID, "tt_evaluate: bad args");
  if (npts == 0) return ACI_OK;
  const int L = t->L;
  for (int64_t p = 0; p < npts; ++p)
    for (int s = 0; s < L; ++s)
      if (idx[p * L + s] >= t->d[s]) return fail(ACI_ERR_INVALID, "tt_evaluate: index >= d_s");
  // stream-ordered on the library stream (a legacy-stream cudaMalloc/cudaMemcpy would synchronise
  // with, and break, stream captures running in other host threads)
  cudaStream_t st = lib_stream();
  uint8_t *di = nullptr;
  double *dout = nullptr;
  const size_t nout = (size_t)npts * (t->cplx ? 2 : 1);
  if (cudaMallocAsync((void **)&di, (size_t)npts * L, st) != cudaSuccess ||
      cudaMallocAsync((void **)&dout, sizeof(double) * nout, st) != cudaSuccess) {
    cudaGetLastError();
    if (di) cudaFreeAsync(di, st);
    cudaStreamSynchronize(st);
    return fail(ACI_ERR_OOM, "tt_evaluate: device buffers");
  }
  cudaMemcpyAsync(di, idx, (size_t)npts * L, cudaMemcpyHostToDevice, st);
  int rc = tt_evaluate_device(t, npts, di, dout, st);
  if (rc == ACI_OK) cudaMemcpyAsync(out, dout, sizeof(double) * nout, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(di, st);
  cudaFreeAsync(dout, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (rc == ACI_OK && e != cudaSuccess) rc = fail(ACI_ERR_CUDA, std::string("tt_evaluate: ") + cudaGetErrorString(e));
  return rc;
}
