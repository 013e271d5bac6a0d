// 2-D cluster tier (round 2; included by prrlu.cu after prrlu_body, whose keys, tie-break (R3),
// stop rule (R2, R17), elimination arithmetic (R4) and cluster primitives it reuses).
//
// One 16-CTA cluster holds the block as a 4 x 4 grid of CTA tiles: CTA (ri, ci) (cluster rank
// 4 ri + ci) owns rows [ri RB, ri RB + RB) and columns [ci CBK, ci CBK + CBK), thread (lane, w)
// entries (ri RB + lane + 32 a, ci CBK + w + NW b) in registers. Per pivot:
//   scan -> warp / CTA argmax -> cluster all-reduce of the 16 CTA keys over DSMEM (st.async +
//   mbarrier; the pivot's sign rides in the key's id, id = 2 flat + sign, which keeps the R3 order)
//   -> the owners of the winner's column segment (the 4 CTAs of its column block) push their RB
//   values to the 4 CTAs of their row block, and the owners of the pivot row (the 4 CTAs of its row
//   block) push their CBK values to the 4 CTAs of their column block (8-byte st.async straight from
//   registers; the pivot row is first spread over EB lanes with shuffles) -> one mbarrier wait ->
//   rank-1 update.
// So no column goes through L2 and every CTA receives RB + CBK values per pivot instead of a whole
// column. Blocks up to 4 RB x 4 CBK: (EA, EB) = (2, 8) for <= 256 x 256, (4, 16) for <= 512 x 512.
// Decisions and arithmetic are those of prrlu_body (identical pivots for equal Pi).
template <int EA, int EB, int NW>
__device__ __forceinline__ void prrlu_body_2d(const LuArgs &A, PrrluSmem &S) {
  constexpr int T = NW * 32;
  constexpr int RB = 32 * EA, CBK = NW * EB, PC = 4;
  static_assert(RB <= kMaxRows && 2 * CBK <= 2 * kMaxCB && EB <= 32, "2-D tile exceeds the shared scratch");
  const int tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const unsigned crank = cluster_rank();
  const int g = (int)crank;  // PHASE() instrumentation: rank 0
  const int ri = (int)crank / PC, ci = (int)crank % PC;
  const int r0 = ri * RB, c0 = ci * CBK;
  const int m = A.dims->m, n = A.dims->n, ldm = A.dims->ldm, kmax = A.dims->kmax, ldu = A.dims->ldu;
  const int mn = m < n ? m : n;
  double thr = A.tol;
  if (A.thr_mode == 0) thr = A.tol * __longlong_as_double((long long)*A.scale_bits);

  double v[EA][EB];
#pragma unroll
  for (int a = 0; a < EA; ++a)
#pragma unroll
    for (int b = 0; b < EB; ++b) {
      const int i = r0 + lane + 32 * a, j = c0 + w + NW * b;
      v[a][b] = (i < m && j < n) ? A.M[(size_t)i * ldm + j] : 0.0;
    }
  const unsigned NC = (unsigned)(PC * CBK);  // padded width of the flat index (R3 order unchanged)

  double bx = 0.0;
  int be = 0;
  auto scan = [&]() {
    constexpr int NE = EA * EB;
    constexpr int NCH = NE < 4 ? NE : 4;
    double cx[NCH];
    int ce[NCH];
#pragma unroll
    for (int t = 0; t < NCH; ++t) { cx[t] = v[t / EB][t % EB]; ce[t] = t; }
#pragma unroll
    for (int e = NCH; e < NE; ++e) {
      const double x = v[e / EB][e % EB];
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
    bx = bm;  // signed
    be = bi;
  };
  // key: |v| bits (hi, lo), id = 2 * flat + sign bit (the min over ids still picks the smallest flat
  // index among equal magnitudes, R3; the sign travels with the winner)
  auto thread_key = [&]() -> Key {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(bx));
    const int a = be / EB, b = be % EB;
    const unsigned flat = (unsigned)(r0 + lane + 32 * a) * NC + (unsigned)(c0 + w + NW * b);
    return Key{(unsigned)(bits >> 32), (unsigned)bits, 2u * flat + (bx < 0.0 ? 1u : 0u)};
  };
  scan();
  const unsigned seg_bytes = (unsigned)(RB + CBK) * 8u;
  if (tid == 0) {
    for (int t = 0; t < 4; ++t) mbar_init(smem_u32(&S.mb[t]), 1u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arm(smem_u32(&S.mb[0]), 16u * 16u);
    mbar_arm(smem_u32(&S.mb[1]), 16u * 16u);
    mbar_arm(smem_u32(&S.mb[2]), seg_bytes);
    mbar_arm(smem_u32(&S.mb[3]), seg_bytes);
  }
  cluster_sync_all();

  double first = 0.0, eps = 0.0;
  int k = 0;
#ifdef ACI_PRRLU_TIMING
  long long ph_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long ph_t_ = clock64();
#endif
  for (;;) {
    if (k == mn) { eps = 0.0; break; }
    const int par = k & 1;
    const unsigned ph = (unsigned)(k >> 1) & 1u;
    // ---- warp -> CTA argmax (key slots double-buffered by parity: no CTA barrier follows)
    const Key wk = warp_argmax(thread_key());
    if (lane == 0) { S.hi[16 * par + w] = wk.hi; S.lo[16 * par + w] = wk.lo; S.id[16 * par + w] = wk.id; }
    __syncthreads();
    PHASE(0);
    const Key ck = warp_argmax(lane < NW ? Key{S.hi[16 * par + lane], S.lo[16 * par + lane], S.id[16 * par + lane]}
                                         : Key{0u, 0u, BAD_ID});
    PHASE(1);
    // ---- cluster all-reduce of the CTA keys (DSMEM)
    if (w == 0 && lane < 16)
      st_async_key(mapa_u32(smem_u32(&S.ck[par][crank]), (unsigned)lane), ck.hi, ck.lo, ck.id,
                   mapa_u32(smem_u32(&S.mb[par]), (unsigned)lane));
    PHASE(2);
    mbar_wait(smem_u32(&S.mb[par]), ph);
    PHASE(3);
    if (tid == 0) mbar_arm(smem_u32(&S.mb[par]), 16u * 16u);
    const uint4 q4 = S.ck[par][lane < 16 ? lane : 0];
    const Key win = warp_argmax(lane < 16 ? Key{q4.x, q4.y, q4.z} : Key{0u, 0u, BAD_ID});
    PHASE(4);

    // ---- stop rule (R2), as prrlu_body
    const double absc = key_abs(win);
    if (k == 0) {
      first = absc;
      if (A.thr_mode == 1) thr = A.tol * first;
    }
    if (k == kmax) { eps = absc; break; }
    if (k > 0 && absc <= thr) { eps = absc; break; }
    const unsigned flat = win.id >> 1;
    const int p = (int)(flat / NC), q = (int)(flat % NC);
    if (crank == 0 && tid == 0) { A.rows[k] = p; A.cols[k] = q; }
    if (k == 0 && absc == 0.0) {
      if (A.U && ri == 0)
        for (int jj = tid; jj < CBK; jj += T)
          if (c0 + jj < n) A.U[(size_t)k * ldu + c0 + jj] = (c0 + jj == q) ? 1.0 : 0.0;
      eps = 0.0;
      k = 1;
      break;
    }
    const int rp = p / RB, cq = q / CBK;
    double *colseg = S.raw + par * kMaxRows;  // S[r0 + i][q], i < RB
    double *rowseg = S.u + par * kMaxCB;      // S[p][c0 + j], j < CBK
    const unsigned sbar = smem_u32(&S.mb[2 + par]);
    // ---- column segment: the 4 CTAs of column block cq push to the 4 CTAs of their row block
    if (ci == cq) {
      const int jq = q - c0;
      if (w == jq % NW) {
        const int bq = jq / NW;
#pragma unroll
        for (int a = 0; a < EA; ++a) {
          double x = v[a][0];
#pragma unroll
          for (int b = 1; b < EB; ++b) x = (b == bq) ? v[a][b] : x;
          const unsigned la = smem_u32(colseg + lane + 32 * a);
#pragma unroll
          for (int cj = 0; cj < PC; ++cj) {
            const unsigned dst = (unsigned)(ri * PC + cj);
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(mapa_u32(la, dst)),
                         "l"(__double_as_longlong(x)), "r"(mapa_u32(sbar, dst))
                         : "memory");
          }
        }
      }
    }
    // ---- pivot row segment: the 4 CTAs of row block rp push to the 4 CTAs of their column block;
    // lane (p - r0) % 32 of every warp spreads its EB row values over lanes 0..EB-1 first
    if (ri == rp) {
      const int ap = (p - r0) >> 5, lp = (p - r0) & 31;
      double mine = 0.0;
#pragma unroll
      for (int b = 0; b < EB; ++b) {
        double x = v[0][b];
#pragma unroll
        for (int a = 1; a < EA; ++a) x = (a == ap) ? v[a][b] : x;
        const double y = __shfl_sync(FULL, x, lp);
        if (lane == b) mine = y;
      }
      if (lane < EB) {
        const unsigned la = smem_u32(rowseg + w + NW * lane);
#pragma unroll
        for (int rk = 0; rk < PC; ++rk) {
          const unsigned dst = (unsigned)(rk * PC + ci);
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(mapa_u32(la, dst)),
                       "l"(__double_as_longlong(mine)), "r"(mapa_u32(sbar, dst))
                       : "memory");
        }
      }
    }
    mbar_wait(sbar, ph);
    if (tid == 0) mbar_arm(sbar, seg_bytes);
    PHASE(5);
    // R4: inv = [S_pq]^{-1} (|c| from the key, the sign from its id); l_p = 1, U_k[q] = 1
    const double inv_abs = __drcp_rn(absc);
    const double inv = (win.id & 1u) ? -inv_abs : inv_abs;
    if (A.U && ri == 0)
      for (int jj = tid; jj < CBK; jj += T) {
        const int j = c0 + jj;
        if (j < n) A.U[(size_t)k * ldu + j] = (j == q) ? 1.0 : rowseg[jj] * inv;
      }
    double ub[EB];
#pragma unroll
    for (int b = 0; b < EB; ++b) ub[b] = rowseg[w + NW * b];
#pragma unroll
    for (int a = 0; a < EA; ++a) {
      const int il = lane + 32 * a;
      const double li = (r0 + il == p) ? 1.0 : colseg[il] * inv;
#pragma unroll
      for (int b = 0; b < EB; ++b) v[a][b] = fma(-li, ub[b], v[a][b]);
    }
    // column q -> exact zeros (owner warp)
    {
      const int jq = q - c0;
      if (jq >= 0 && jq < CBK && (jq % NW) == w) {
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
  }
  if (crank == 0 && tid == 0) {
    *A.r_out = k;
    *A.eps_out = eps;
#ifdef ACI_PRRLU_TIMING
    for (int t = 0; t < 8; ++t) A.dbg[t] = ph_[t];
#endif
  }
  cluster_sync_all();  // no CTA leaves while a peer may still push to it
}
