// Rook-pivoting prrLU (B:5 "prrLU with full/rook pivoting"; reading R23 of
// the paper itself only uses full pivoting). Included by prrlu.cu after
// prrlu_body, whose register layout, keys, tie-break (R3), stop rule (R2), elimination arithmetic
// (R4) and exchange primitives it reuses; oracle/aci_oracle.c (rook_search) is the reference.
//
// Search per pivot (R23): start at the smallest active column c; r = the max |.| row of column c;
// then alternate the row maximum of row r and the column maximum of column c until an entry is the
// largest of both its active row and its active column (only a STRICTLY larger extremum moves the
// search; ties to the smallest index). The accepted (r, c) and its value feed the same stop rule
// and Schur update as full pivoting. No full-block scan per pivot: the rank-1 update is all the
// per-entry work.
//   * column maxima are warp-local (a warp owns whole columns): the owner warp reduces its lanes,
//     then one broadcast (one CTA: a shared-memory reduction; one cluster: the owner CTA's warp
//     pushes the key into every cluster CTA's shared memory, st.async + mbarrier);
//   * row maxima: the lane holding row r in every warp reduces its EB entries, then a CTA
//     reduction and (one cluster) a cluster all-reduce of the CTA keys over DSMEM;
//   * the pivot column: one CTA reads it from the owner warp's shared-memory copy; in a cluster the
//     owner CTA publishes every searched column to L2 as tagged packets (publication counter P,
//     two slots per CTA by parity) and the CTAs read the final one.
// Supported where the factorisation fits one CTA or one 16-CTA cluster (the prrlu_kernel_one
// envelope); real values only.
// (included once per prrlu.cu instance; csrc/peak_probe.cu instantiates prrlu.cu twice)

template <int EA, int EB, int NW, int XM>
__device__ __forceinline__ void prrlu_body_rook(const LuArgs &A, RookSmem &S, const int G, const int g) {
  static_assert(XM == 0 || XM == 2, "rook pivoting: one CTA or one cluster");
  constexpr bool GRID = XM != 0;
  constexpr int T = NW * 32;
  constexpr int MROWS = 32 * EA;
  constexpr int CB = NW * EB;
  static_assert(MROWS <= kMaxRows && CB <= kMaxCB && EA <= 32 && EB <= 32, "tile exceeds the shared scratch");
  double *s_l = S.l, *s_raw = S.raw, *s_u = S.u;
  const int tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const int c0 = g * CB;

  const int m = A.dims->m, n = A.dims->n, ldm = A.dims->ldm, kmax = A.dims->kmax, ldu = A.dims->ldu;
  const unsigned ep = GRID ? (*A.epoch & 0xfffffu) : 0u;
  const int mn = m < n ? m : n;
  double thr = A.tol;
  if (A.thr_mode == 0) thr = A.tol * __longlong_as_double((long long)*A.scale_bits);

  double v[EA][EB][1];
  bool rok[EA], cok[EB];
#pragma unroll
  for (int a = 0; a < EA; ++a) rok[a] = lane + 32 * a < m;
#pragma unroll
  for (int b = 0; b < EB; ++b) cok[b] = c0 + w + NW * b < n;
#pragma unroll
  for (int a = 0; a < EA; ++a)
#pragma unroll
    for (int b = 0; b < EB; ++b)
      v[a][b][0] = (rok[a] && cok[b]) ? A.M[(size_t)(lane + 32 * a) * ldm + c0 + w + NW * b] : 0.0;
  for (int i = tid; i < kMaxRows; i += T) s_l[i] = 0.0;
  for (int j = tid; j < kMaxCB; j += T) s_u[j] = 0.0;
  for (int i = tid; i < (int)(sizeof(S.cdone) / sizeof(unsigned)); i += T) S.cdone[i] = 0u;
  const unsigned NC = (unsigned)(G * CB);
  // done rows of this thread (bit a: row lane + 32 a) and done columns (bit b: col c0 + w + NW b)
  unsigned rdm = 0u, cdm = 0u;

  if (XM == 2) {
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
  } else {
    __syncthreads();
  }

  int xr = 0;      // CTA reductions (parity halves of S.hi/lo/id)
  int xa = 0;      // cluster all-reduces (S.ck, mb[0..1])
  int xb = 0;      // cluster broadcasts (S.gw, mb[2..3])
  unsigned P = 0;  // column publications (cluster): slot parity and tag
  auto ptag = [&](unsigned pub) -> unsigned { return (ep << 12) | (pub % 4095u + 1u); };

  // every thread of the CTA gets the CTA's best key (warp keys through shared memory)
  auto cta_reduce = [&](const Key &wk) -> Key {
    const int h = (xr & 1) * 16;
    ++xr;
    if (lane == 0) { S.hi[h + w] = wk.hi; S.lo[h + w] = wk.lo; S.id[h + w] = wk.id; }
    __syncthreads();
    return warp_argmax(lane < NW ? Key{S.hi[h + lane], S.lo[h + lane], S.id[h + lane]} : Key{0u, 0u, BAD_ID});
  };
  // cluster all-reduce of the CTA keys (every CTA pushes its key into every CTA's shared memory)
  auto cluster_allreduce = [&](const Key &ck) -> Key {
    const int par = xa & 1;
    const unsigned ph = (unsigned)(xa >> 1) & 1u;
    ++xa;
    const unsigned CS = cluster_size();
    if (w == 0 && lane < (int)CS)
      st_async_key(mapa_u32(smem_u32(&S.ck[par][cluster_rank()]), (unsigned)lane), ck.hi, ck.lo, ck.id,
                   mapa_u32(smem_u32(&S.mb[par]), (unsigned)lane));
    const unsigned mbp = smem_u32(&S.mb[par]);
    mbar_wait(mbp, ph);
    if (tid == 0) mbar_arm(mbp, CS * 16u);
    const uint4 q4 = S.ck[par][lane < (int)CS ? lane : 0];
    return warp_argmax(lane < (int)CS ? Key{q4.x, q4.y, q4.z} : Key{0u, 0u, BAD_ID});
  };

  // max |S[i][c]| over the active rows of column c (ties -> smallest row); the cluster owner also
  // publishes column c to L2 (publication P)
  auto colmax = [&](int c) -> Key {
    const int jc = c - c0;
    const bool own = jc >= 0 && jc < CB;
    const int ow = own ? jc % NW : -1, bc = own ? jc / NW : 0;
    Key wk{0u, 0u, BAD_ID};
    if (w == ow) {
      Key tk{0u, 0u, BAD_ID};
#pragma unroll
      for (int b = 0; b < EB; ++b)
        if (b == bc)
#pragma unroll
          for (int a = 0; a < EA; ++a) {
            const int i = lane + 32 * a;
            if (rok[a] && !((rdm >> a) & 1u)) {
              const unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(v[a][b][0]));
              const Key kk{(unsigned)(bits >> 32), (unsigned)bits, (unsigned)i * NC + (unsigned)c};
              if (better(kk, tk)) tk = kk;
            }
          }
      wk = warp_argmax(tk);
      if (GRID) {
        // publish column c (tagged packets) for the CTAs that may pivot on it
        const unsigned tag = ptag(P);
        unsigned long long *dst = A.colpub + (((size_t)(P & 1u) * G + g) * A.colcap) * 2 * kColSpread;
#pragma unroll
        for (int b = 0; b < EB; ++b)
          if (b == bc)
#pragma unroll
            for (int a = 0; a < EA; ++a)
              if (rok[a]) {
                const unsigned long long bits = (unsigned long long)__double_as_longlong(v[a][b][0]);
                st_pkt(dst + cpk(lane + 32 * a), tagged(tag, (unsigned)bits), tagged(tag, (unsigned)(bits >> 32)));
              }
      }
    }
    if (!GRID) return cta_reduce(wk);
    ++P;
    // cluster: the owner warp pushes its key into every CTA's broadcast slot
    const int par = xb & 1;
    const unsigned ph = (unsigned)(xb >> 1) & 1u;
    ++xb;
    const unsigned CS = cluster_size();
    if (w == ow && lane < (int)CS)
      st_async_key(mapa_u32(smem_u32(&S.gw[par]), (unsigned)lane), wk.hi, wk.lo, wk.id,
                   mapa_u32(smem_u32(&S.mb[2 + par]), (unsigned)lane));
    const unsigned mbp = smem_u32(&S.mb[2 + par]);
    mbar_wait(mbp, ph);
    if (tid == 0) mbar_arm(mbp, 16u);
    return Key{S.gw[par].x, S.gw[par].y, S.gw[par].z};
  };

  // max |S[r][j]| over the active columns of row r (ties -> smallest column)
  auto rowmax = [&](int r) -> Key {
    const int ar = r >> 5, lr = r & 31;
    Key tk{0u, 0u, BAD_ID};
    if (lane == lr) {
#pragma unroll
      for (int a = 0; a < EA; ++a)
        if (a == ar)
#pragma unroll
          for (int b = 0; b < EB; ++b)
            if (cok[b] && !((cdm >> b) & 1u)) {
              const unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(v[a][b][0]));
              const Key kk{(unsigned)(bits >> 32), (unsigned)bits, (unsigned)r * NC + (unsigned)(c0 + w + NW * b)};
              if (better(kk, tk)) tk = kk;
            }
    }
    const Key wk{__shfl_sync(FULL, tk.hi, lr), __shfl_sync(FULL, tk.lo, lr), __shfl_sync(FULL, tk.id, lr)};
    const Key ck = cta_reduce(wk);
    return GRID ? cluster_allreduce(ck) : ck;
  };
  auto gt = [](const Key &a, const Key &b) { return a.hi != b.hi ? a.hi > b.hi : a.lo > b.lo; };

  int cfirst = 0;  // smallest active column (uniform)
  double eps = 0.0;
  int k = 0;
#ifdef ACI_PRRLU_TIMING
  long long ph_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long ph_t_ = clock64();
#endif
  for (;;) {
    if (k == mn) { eps = 0.0; break; }
    // ---- rook search (R23)
    int c = cfirst;
    Key cur = colmax(c);
    unsigned Pc = P - 1u;  // cluster: publication of the current column
    int r = (int)(cur.id / NC);
    for (;;) {
      const Key rw = rowmax(r);
      if (!gt(rw, cur)) break;  // (r, c) is the max of its row and of its column
      c = (int)(rw.id % NC);
      cur = rw;
      const Key cn = colmax(c);
      Pc = P - 1u;
      if (!gt(cn, cur)) break;  // (r, c) is the max of its column and of its row
      r = (int)(cn.id / NC);
      cur = cn;
    }
    PHASE(4);
    const int p = r, q = c;
    const double absc = key_abs(cur);
    if (k == 0 && A.thr_mode == 1) thr = A.tol * absc;  // R8 reading for the rook search's first pivot
    if (k == kmax) { eps = absc; break; }
    if (k > 0 && absc <= thr) { eps = absc; break; }
    if (g == 0 && tid == 0) { A.rows[k] = p; A.cols[k] = q; }
    if (k == 0 && absc == 0.0) {
      // R17: zero block -> rank 1, dummy pivot (0,0) (the rook search lands there), U row e_q, eps 0
      if (A.U)
        for (int j = c0 + tid; j < c0 + CB && j < n; j += T) A.U[(size_t)k * ldu + j] = (j == q) ? 1.0 : 0.0;
      eps = 0.0;
      k = 1;
      break;
    }
    const int ap = p >> 5, lp = p & 31;
    if (lane == lp) {
#pragma unroll
      for (int a = 0; a < EA; ++a)
        if (a == ap)
#pragma unroll
          for (int b = 0; b < EB; ++b) s_u[w + NW * b] = v[a][b][0];
    }
    const double inv_abs = __drcp_rn(absc);  // 1/|c| (correctly rounded); the sign comes with the column
    double inv;
    if (GRID) {
      // the pivot column from L2: publication Pc of CTA q / CB
      const unsigned tag = ptag(Pc);
      const unsigned long long *src = A.colpub + (((size_t)(Pc & 1u) * G + q / CB) * A.colcap) * 2 * kColSpread;
      constexpr int PPT = (MROWS + T - 1) / T;
      unsigned long long cw[PPT + 1][2];
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int i = tid + T * t;
        if (i < m) ld_pkt(src + cpk(i), cw[t][0], cw[t][1]);
      }
      ld_pkt(src + cpk(p), cw[PPT][0], cw[PPT][1]);
      while ((unsigned)(cw[PPT][0] >> 32) != tag || (unsigned)(cw[PPT][1] >> 32) != tag)
        ld_pkt(src + cpk(p), cw[PPT][0], cw[PPT][1]);
      inv = (cw[PPT][1] & 0x80000000ull) ? -inv_abs : inv_abs;
#pragma unroll
      for (int t = 0; t < PPT; ++t) {
        const int i = tid + T * t;
        if (i < m) {
          while ((unsigned)(cw[t][0] >> 32) != tag || (unsigned)(cw[t][1] >> 32) != tag)
            ld_pkt(src + cpk(i), cw[t][0], cw[t][1]);
          s_l[lpair2(i)] = (i == p) ? 1.0 : pkt_double(cw[t][0], cw[t][1]) * inv;
        }
      }
      __syncthreads();
    } else {
      const int jq = q - c0;
      if ((jq % NW) == w) {
        const int bq = jq / NW;
#pragma unroll
        for (int b = 0; b < EB; ++b)
          if (b == bq)
#pragma unroll
            for (int a = 0; a < EA; ++a) s_raw[lpair2(lane + 32 * a)] = v[a][b][0];
      }
      __syncthreads();
      inv = s_raw[lpair2(p)] < 0.0 ? -inv_abs : inv_abs;
#pragma unroll
      for (int t = 0; t < (MROWS + T - 1) / T; ++t) {
        const int i = tid + T * t;
        if (i < MROWS) s_l[lpair2(i)] = (i == p) ? 1.0 : s_raw[lpair2(i)] * inv;
      }
      __syncthreads();
    }
    PHASE(5);
    if (A.U)
      for (int jj = tid; jj < CB; jj += T) {
        const int j = c0 + jj;
        if (j < n) A.U[(size_t)k * ldu + j] = (j == q) ? 1.0 : s_u[jj] * inv;
      }
    double ub[EB];
#pragma unroll
    for (int b = 0; b < EB; ++b) ub[b] = s_u[w + NW * b];
    // fma(-l_i, u_j, S_ij) (R4), l_p = 1 zeroes row p exactly
#pragma unroll
    for (int a = 0; a < EA; ++a) {
      const double li = s_l[lpair2(lane + 32 * a)];
#pragma unroll
      for (int b = 0; b < EB; ++b) v[a][b][0] = fma(-li, ub[b], v[a][b][0]);
    }
    {
      const int jq = q - c0;
      if (jq >= 0 && jq < CB && (jq % NW) == w) {
        const int bq = jq / NW;
#pragma unroll
        for (int b = 0; b < EB; ++b)
          if (b == bq)
#pragma unroll
            for (int a = 0; a < EA; ++a) v[a][b][0] = 0.0;
        cdm |= 1u << bq;
      }
      if (lp == lane) rdm |= 1u << ap;
    }
    // the smallest active column, from a per-warp view of the eliminated columns (each warp's lane 0
    // records q itself, so no cross-warp ordering is needed)
    if (lane == 0) atomicOr(&S.cdone[q >> 5], 1u << (q & 31));
    __syncwarp();
    while (cfirst < n && ((S.cdone[cfirst >> 5] >> (cfirst & 31)) & 1u)) ++cfirst;
    PHASE(6);
    ++k;
    // s_l / s_u / s_raw are rewritten only after this pivot's readers passed a later barrier
    // (the next pivot's first reduction)
  }
  if (g == 0 && tid == 0) {
    *A.r_out = k;
    *A.eps_out = eps;
    if (GRID) atomicAdd(A.epoch, 1u);
#ifdef ACI_PRRLU_TIMING
    for (int t = 0; t < 8; ++t) A.dbg[t] = ph_[t];
#endif
  }
  if (XM == 2) cluster_sync_all();
}
