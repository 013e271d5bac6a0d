"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU reference for the ACI hot path of
PAPER.md (arxiv 2604.00037). Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package. It shares no code with the CUDA path
(``paper_2604_00037_b200``), and the CUDA path never imports it.

Contents
--------
* ``aci``      — Alg. 1-5 as naive C loops (``aci_oracle.c``),
                 readings R1-R22 of DESIGN.md §2.
* ``aci_z``, ``ldu_z`` — the same for complex values (f: C^N -> C, P:84;
                 ``aci_oracle_z.c``), complex-arithmetic readings RZ1-RZ6.
* ``ldu``, ``ci_right``, ``assemble_pi`` — the sub-steps (Alg. 2, Alg. 3,
                 Eq. pifromframes), exported for the pin tests.
* ``tt_evaluate``, ``tt_dense`` — the plain definition of a TT.
* ``exact_product`` + ``tt_round`` — the textbook alternative: Kronecker-δ
                 (MPO-MPS) product of the inputs followed
                 by TT-SVD truncation; the "plain definition" of f(x¹..xᴺ)
                 where its rank is small enough (configs[0], [1], [3]).

Pinning status: every function above is pinned by a
``-m "not gpu"`` test against closed forms, brute force or exact rational
arithmetic (rook mode included). Rank-capped runs (configs[4]) have no exact
product to compare with; their last update is pinned against the definition
(the block built by direct evaluation of the inputs at the final index sets,
factorised by the pinned prrLU, gives the logged pivots) and the output's
interpolation identity on that cross; the earlier updates of such runs are
pinned only through their (individually pinned) sub-steps.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "aci_oracle.c")
_SRCZ = os.path.join(_HERE, "aci_oracle_z.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

STATUS = {0: "ok", -1: "invalid", -3: "nonfinite", -4: "oom"}


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (no fast-math, no FP contraction)."""
    if (force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC)
            or os.path.getmtime(_LIB) < os.path.getmtime(_SRCZ)):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
                               "-o", _LIB, _SRC, _SRCZ, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB)
        dp, ip, vp = C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_void_p
        lib.oracle_aci.restype = vp
        lib.oracle_aci.argtypes = [C.c_int, ip, C.c_int, ip, C.POINTER(dp), C.c_int, dp, ip, ip,
                                   C.POINTER(dp), C.c_double, C.c_int, C.c_int, C.c_int, ip]
        lib.oracle_free.argtypes = [vp]
        lib.oracle_report.argtypes = [vp, dp, dp, ip, ip, dp, dp, C.POINTER(C.c_longlong)]
        lib.oracle_out_ranks.argtypes = [vp, ip]
        lib.oracle_out_core.argtypes = [vp, C.c_int, dp]
        lib.oracle_log_count.argtypes = [vp]
        lib.oracle_log_entry.argtypes = [vp, C.c_int, ip, dp, ip, ip]
        lib.oracle_chi.argtypes = [vp, C.c_int]
        lib.oracle_jn.argtypes = [vp, C.c_int]
        lib.oracle_Iset.argtypes = [vp, C.c_int, C.c_void_p]
        lib.oracle_Jset.argtypes = [vp, C.c_int, C.c_void_p]
        lib.oracle_canon_jn.argtypes = [vp, C.c_int]
        lib.oracle_canon_Jset.argtypes = [vp, C.c_int, C.c_void_p]
        lib.oracle_canon_cols.argtypes = [vp, C.c_int, ip]
        lib.oracle_Lframe.argtypes = [vp, C.c_int, C.c_int, dp]
        lib.oracle_Rframe.argtypes = [vp, C.c_int, C.c_int, dp]
        lib.oracle_ldu.argtypes = [C.c_int, C.c_int, dp, C.c_double, C.c_int, C.c_int, ip, ip, ip, dp, dp, dp,
                                   C.c_int, dp]
        lib.oracle_ldu_p.argtypes = [C.c_int, C.c_int, dp, C.c_double, C.c_int, C.c_int, C.c_int, ip, ip, ip, dp,
                                     dp, dp, C.c_int, dp]
        lib.oracle_aci_p.restype = vp
        lib.oracle_aci_p.argtypes = lib.oracle_aci.argtypes[:-1] + [C.c_int, ip]
        lib.oracle_ci_right.argtypes = [C.c_int, C.c_int, dp, C.c_double, C.c_int, C.c_int, ip, ip, ip, dp, dp,
                                        C.c_int, dp]
        lib.oracle_assemble_pi.argtypes = [C.c_int, ip, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(dp),
                                           C.POINTER(dp), C.POINTER(dp), C.POINTER(dp), C.c_int, dp, ip, dp]
        lib.oraclez_aci.restype = vp
        lib.oraclez_aci.argtypes = lib.oracle_aci.argtypes
        lib.oraclez_free.argtypes = [vp]
        lib.oraclez_report.argtypes = lib.oracle_report.argtypes
        lib.oraclez_out_ranks.argtypes = [vp, ip]
        lib.oraclez_out_core.argtypes = [vp, C.c_int, dp]
        lib.oraclez_log_count.argtypes = [vp]
        lib.oraclez_log_entry.argtypes = [vp, C.c_int, ip, dp, ip, ip]
        lib.oraclez_log_gaps.argtypes = [vp, C.c_int, dp]
        lib.oraclez_canon_jn.argtypes = [vp, C.c_int]
        lib.oraclez_canon_cols.argtypes = [vp, C.c_int, ip]
        lib.oraclez_ldu.argtypes = [C.c_int, C.c_int, dp, C.c_double, C.c_int, C.c_int, ip, ip, ip, dp, dp,
                                    C.c_int, dp]
        _lib = lib
    return _lib


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _iptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _cores_of(x):
    return x.cores if hasattr(x, "cores") else list(x)


# --------------------------------------------------------------------------
# Alg. 2 / Alg. 3 / Eq. pifromframes (pin-test entry points)
# --------------------------------------------------------------------------
PIVOTING = {"full": 0, "rook": 1}


def ldu(M, thr: float, maxrank: int, relative_to_own_max: bool = False, pivoting: str = "full") -> dict:
    """Alg. 2 with R2-R4/R17; pivoting "full" or "rook" (R23, NEXT-4).
    Returns rows, cols, D, U (r x n), L (m x r), eps."""
    lib = _load()
    M = np.ascontiguousarray(M, dtype=np.float64)
    m, n = M.shape
    maxr = max(1, min(m, n, maxrank))
    r = C.c_int()
    eps = C.c_double()
    rows = np.zeros(maxr, np.int32)
    cols = np.zeros(maxr, np.int32)
    D = np.zeros(maxr)
    U = np.zeros((maxr, n))
    Lc = np.zeros((m, maxr))
    st = lib.oracle_ldu_p(m, n, _dptr(M), thr, 1 if relative_to_own_max else 0, maxrank, PIVOTING[pivoting],
                          C.byref(r), _iptr(rows), _iptr(cols), _dptr(D), _dptr(U), _dptr(Lc), maxr, C.byref(eps))
    if st != 0:
        raise ValueError(f"oracle_ldu: {STATUS.get(st, st)}")
    k = r.value
    return {"r": k, "rows": rows[:k].copy(), "cols": cols[:k].copy(), "D": D[:k].copy(), "U": U[:k].copy(),
            "L": Lc[:, :k].copy(), "eps": eps.value}


def ci_right(M, thr: float, maxrank: int, relative_to_own_max: bool = False) -> dict:
    """Alg. 3 right branch: A = M[:, J], B = U_J^{-1} U."""
    lib = _load()
    M = np.ascontiguousarray(M, dtype=np.float64)
    m, n = M.shape
    maxr = max(1, min(m, n, maxrank))
    r = C.c_int()
    eps = C.c_double()
    rows = np.zeros(maxr, np.int32)
    cols = np.zeros(maxr, np.int32)
    A = np.zeros((m, maxr))
    B = np.zeros((maxr, n))
    st = lib.oracle_ci_right(m, n, _dptr(M), thr, 1 if relative_to_own_max else 0, maxrank, C.byref(r), _iptr(rows),
                             _iptr(cols), _dptr(A), _dptr(B), maxr, C.byref(eps))
    if st != 0:
        raise ValueError(f"oracle_ci_right: {STATUS.get(st, st)}")
    k = r.value
    return {"r": k, "rows": rows[:k].copy(), "cols": cols[:k].copy(), "A": A[:, :k].copy(), "B": B[:k].copy(),
            "eps": eps.value}


def assemble_pi(Ls, X0s, X1s, Rs, op) -> np.ndarray:
    """Eq. pifromframes then f for explicit frames.

    Ls[n]: rl x c0 (None = [1]), X0s[n]: core of site b, X1s[n]: core of site b+1,
    Rs[n]: c2 x rr (None = [1]). Returns Pi as the (rl*d_b) x (d_{b+1}*rr) matricisation.
    """
    lib = _load()
    N = len(X0s)
    rl = 1 if Ls[0] is None else Ls[0].shape[0]
    rr = 1 if Rs[0] is None else Rs[0].shape[1]
    db, db1 = X0s[0].shape[1], X1s[0].shape[1]
    c = np.array([[X0s[i].shape[0], X0s[i].shape[2], X1s[i].shape[2]] for i in range(N)], np.int32)
    keep = []

    def arr(xs):
        out = (C.POINTER(C.c_double) * N)()
        for i, x in enumerate(xs):
            if x is None:
                out[i] = C.POINTER(C.c_double)()
            else:
                x = np.ascontiguousarray(x, dtype=np.float64)
                keep.append(x)
                out[i] = _dptr(x)
        return out

    coef = np.ascontiguousarray(op["coef"], dtype=np.float64)
    expo = np.ascontiguousarray(op["expo"], dtype=np.int32)
    Pi = np.zeros((rl * db, db1 * rr))
    lib.oracle_assemble_pi(N, _iptr(c), db, db1, rl, rr, arr(Ls), arr(X0s), arr(X1s), arr(Rs), len(coef),
                           _dptr(coef), _iptr(expo), _dptr(Pi))
    return Pi


# --------------------------------------------------------------------------
# Alg. 1 — full ACI run
# --------------------------------------------------------------------------
class AciResult:
    """Handle on an oracle ACI run; owns the C state until freed."""

    def __init__(self, h, L, N, d, xranks):
        self._h = h
        self.L, self.N, self.d, self.xranks = L, N, d, xranks
        lib = _load()
        sc, err, fc, fp = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        it, cv = C.c_int(), C.c_int()
        pv = C.c_longlong()
        lib.oracle_report(h, C.byref(sc), C.byref(err), C.byref(it), C.byref(cv), C.byref(fc), C.byref(fp),
                          C.byref(pv))
        self.report = {"scale": sc.value, "error_estimate": err.value, "iterations": it.value,
                       "converged": bool(cv.value), "flops_contraction": fc.value, "flops_prrlu": fp.value,
                       "pivot_steps": pv.value}
        ranks = np.zeros(L + 1, np.int32)
        lib.oracle_out_ranks(h, _iptr(ranks))
        self.ranks = [int(x) for x in ranks]
        self.cores = []
        for s in range(L):
            c = np.zeros((self.ranks[s], d[s], self.ranks[s + 1]))
            lib.oracle_out_core(h, s, _dptr(c))
            self.cores.append(c)
        self.log = []
        for u in range(lib.oracle_log_count(h)):
            info = np.zeros(5, np.int32)
            es = np.zeros(2)
            lib.oracle_log_entry(h, u, _iptr(info), _dptr(es), None, None)
            rows = np.zeros(info[4], np.int32)
            cols = np.zeros(info[4], np.int32)
            lib.oracle_log_entry(h, u, _iptr(info), _dptr(es), _iptr(rows), _iptr(cols))
            self.log.append({"bond": int(info[0]), "dir": int(info[1]), "rl": int(info[2]), "rr": int(info[3]),
                             "r": int(info[4]), "eps": float(es[0]), "scale": float(es[1]), "rows": rows,
                             "cols": cols})

    def chi(self, b):
        return _load().oracle_chi(self._h, b)

    def Iset(self, b):
        out = np.zeros((self.chi(b), b + 1), np.uint8)
        _load().oracle_Iset(self._h, b, out.ctypes.data)
        return out

    def Jset(self, s):
        n = _load().oracle_jn(self._h, s)
        out = np.zeros((n, self.L - s), np.uint8)
        _load().oracle_Jset(self._h, s, out.ctypes.data)
        return out

    def canon_Jset(self, s):
        n = _load().oracle_canon_jn(self._h, s)
        out = np.zeros((n, self.L - s), np.uint8)
        _load().oracle_canon_Jset(self._h, s, out.ctypes.data)
        return out

    def canon_cols(self, s):
        n = _load().oracle_canon_jn(self._h, s)
        out = np.zeros(n, np.int32)
        _load().oracle_canon_cols(self._h, s, _iptr(out))
        return out

    def Lframe(self, n, b):
        out = np.zeros((self.chi(b), self.xranks[n][b + 1]))
        _load().oracle_Lframe(self._h, n, b, _dptr(out))
        return out

    def Rframe(self, n, s):
        out = np.zeros((self.xranks[n][s], _load().oracle_jn(self._h, s)))
        _load().oracle_Rframe(self._h, n, s, _dptr(out))
        return out

    def free(self):
        if self._h:
            _load().oracle_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def aci(inputs, op, y_init, tol, maxrank, max_sweeps, relative=True, pivoting="full") -> AciResult:
    """Run Alg. 1. ``inputs`` are distinct TTs; ``op`` = {coef, expo} over them;
    ``pivoting`` "full" or "rook" (R23) for every prrLU of the run."""
    lib = _load()
    ins = [_cores_of(x) for x in inputs]
    N = len(ins)
    L = len(ins[0])
    d = [int(c.shape[1]) for c in ins[0]]
    xr = np.array([[int(c[0].shape[0])] + [int(cc.shape[2]) for cc in c] for c in ins], np.int32)
    keep = []
    cp = (C.POINTER(C.c_double) * (N * L))()
    for n in range(N):
        for s in range(L):
            a = np.ascontiguousarray(ins[n][s], dtype=np.float64)
            keep.append(a)
            cp[n * L + s] = _dptr(a)
    yc = _cores_of(y_init)
    yr = np.array([int(yc[0].shape[0])] + [int(c.shape[2]) for c in yc], np.int32)
    yp = (C.POINTER(C.c_double) * L)()
    for s in range(L):
        a = np.ascontiguousarray(yc[s], dtype=np.float64)
        keep.append(a)
        yp[s] = _dptr(a)
    coef = np.ascontiguousarray(op["coef"], dtype=np.float64)
    expo = np.ascontiguousarray(op["expo"], dtype=np.int32)
    dd = np.array(d, np.int32)
    st = C.c_int()
    h = lib.oracle_aci_p(L, _iptr(dd), N, _iptr(xr), cp, len(coef), _dptr(coef), _iptr(expo), _iptr(yr), yp,
                         float(tol), 0 if relative else 1, int(maxrank), int(max_sweeps), PIVOTING[pivoting],
                         C.byref(st))
    if not h:
        raise ValueError(f"oracle_aci: {STATUS.get(st.value, st.value)}")
    return AciResult(h, L, N, d, [list(map(int, r)) for r in xr])


# --------------------------------------------------------------------------
# Complex values (f: C^N -> C): aci_oracle_z.c, readings RZ1-RZ6
# --------------------------------------------------------------------------
def _zptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def ldu_z(M, thr: float, maxrank: int, relative_to_own_max: bool = False) -> dict:
    """Alg. 2 on a complex matrix (RZ1-RZ4). Returns rows, cols, D, U (r x n), eps."""
    lib = _load()
    M = np.ascontiguousarray(M, dtype=np.complex128)
    m, n = M.shape
    maxr = max(1, min(m, n, maxrank))
    r, eps = C.c_int(), C.c_double()
    rows = np.zeros(maxr, np.int32)
    cols = np.zeros(maxr, np.int32)
    D = np.zeros(maxr, np.complex128)
    U = np.zeros((maxr, n), np.complex128)
    st = lib.oraclez_ldu(m, n, _zptr(M), thr, 1 if relative_to_own_max else 0, maxrank, C.byref(r), _iptr(rows),
                         _iptr(cols), _zptr(D), _zptr(U), maxr, C.byref(eps))
    if st != 0:
        raise ValueError(f"oraclez_ldu: {STATUS.get(st, st)}")
    k = r.value
    return {"r": k, "rows": rows[:k].copy(), "cols": cols[:k].copy(), "D": D[:k].copy(), "U": U[:k].copy(),
            "eps": eps.value}


class AciResultZ:
    """Handle on a complex oracle ACI run (cores complex128)."""

    def __init__(self, h, L, N, d):
        self._h = h
        self.L, self.N, self.d = L, N, d
        lib = _load()
        sc, err, fc, fp = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        it, cv = C.c_int(), C.c_int()
        pv = C.c_longlong()
        lib.oraclez_report(h, C.byref(sc), C.byref(err), C.byref(it), C.byref(cv), C.byref(fc), C.byref(fp),
                           C.byref(pv))
        self.report = {"scale": sc.value, "error_estimate": err.value, "iterations": it.value,
                       "converged": bool(cv.value), "flops_contraction": fc.value, "flops_prrlu": fp.value,
                       "pivot_steps": pv.value}
        ranks = np.zeros(L + 1, np.int32)
        lib.oraclez_out_ranks(h, _iptr(ranks))
        self.ranks = [int(x) for x in ranks]
        self.cores = []
        for s in range(L):
            c = np.zeros((self.ranks[s], d[s], self.ranks[s + 1]), np.complex128)
            lib.oraclez_out_core(h, s, _zptr(c))
            self.cores.append(c)
        self.log = []
        for u in range(lib.oraclez_log_count(h)):
            info = np.zeros(5, np.int32)
            es = np.zeros(2)
            lib.oraclez_log_entry(h, u, _iptr(info), _dptr(es), None, None)
            rows = np.zeros(info[4], np.int32)
            cols = np.zeros(info[4], np.int32)
            lib.oraclez_log_entry(h, u, _iptr(info), _dptr(es), _iptr(rows), _iptr(cols))
            gap = np.zeros(info[4])
            lib.oraclez_log_gaps(h, u, _dptr(gap))
            self.log.append({"bond": int(info[0]), "dir": int(info[1]), "rl": int(info[2]), "rr": int(info[3]),
                             "r": int(info[4]), "eps": float(es[0]), "scale": float(es[1]), "rows": rows,
                             "cols": cols, "gap": gap})

    def canon_cols(self, s):
        n = _load().oraclez_canon_jn(self._h, s)
        out = np.zeros(n, np.int32)
        _load().oraclez_canon_cols(self._h, s, _iptr(out))
        return out

    def free(self):
        if self._h:
            _load().oraclez_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def aci_z(inputs, op, y_init, tol, maxrank, max_sweeps, relative=True) -> AciResultZ:
    """Complex Alg. 1 with RZ1-RZ6; inputs and y_init complex TTs."""
    lib = _load()
    ins = [_cores_of(x) for x in inputs]
    N, L = len(ins), len(ins[0])
    d = [int(c.shape[1]) for c in ins[0]]
    xr = np.array([[int(c[0].shape[0])] + [int(cc.shape[2]) for cc in c] for c in ins], np.int32)
    keep = []
    cp = (C.POINTER(C.c_double) * (N * L))()
    for n in range(N):
        for s in range(L):
            a = np.ascontiguousarray(ins[n][s], dtype=np.complex128)
            keep.append(a)
            cp[n * L + s] = _zptr(a)
    yc = _cores_of(y_init)
    yr = np.array([int(yc[0].shape[0])] + [int(c.shape[2]) for c in yc], np.int32)
    yp = (C.POINTER(C.c_double) * L)()
    for s in range(L):
        a = np.ascontiguousarray(yc[s], dtype=np.complex128)
        keep.append(a)
        yp[s] = _zptr(a)
    coef = np.ascontiguousarray(op["coef"], dtype=np.float64)
    expo = np.ascontiguousarray(op["expo"], dtype=np.int32)
    dd = np.array(d, np.int32)
    st = C.c_int()
    h = lib.oraclez_aci(L, _iptr(dd), N, _iptr(xr), cp, len(coef), _dptr(coef), _iptr(expo), _iptr(yr), yp,
                        float(tol), 0 if relative else 1, int(maxrank), int(max_sweeps), C.byref(st))
    if not h:
        raise ValueError(f"oraclez_aci: {STATUS.get(st.value, st.value)}")
    return AciResultZ(h, L, N, d)


# --------------------------------------------------------------------------
# Plain definitions (numpy): TT evaluation, dense tensor, exact product
# --------------------------------------------------------------------------
def tt_evaluate(cores, idx, chunk: int = 4096) -> np.ndarray:
    """x_sigma = X_1[sigma_1] X_2[sigma_2] ... X_L[sigma_L], per point."""
    cores = _cores_of(cores)
    idx = np.asarray(idx)
    dt = np.result_type(*cores)
    out = np.empty(idx.shape[0], dt)
    for p0 in range(0, idx.shape[0], chunk):
        sl = idx[p0:p0 + chunk]
        v = np.ones((sl.shape[0], 1), dt)
        for s, c in enumerate(cores):
            nv = np.empty((sl.shape[0], c.shape[2]), dt)
            for sg in range(c.shape[1]):
                sel = sl[:, s] == sg
                if np.any(sel):
                    nv[sel] = v[sel] @ c[:, sg, :]
            v = nv
        out[p0:p0 + chunk] = v[:, 0]
    return out


def tt_dense(cores) -> np.ndarray:
    """Materialise the full tensor (small L only), flattened with sigma_1 most significant."""
    cores = _cores_of(cores)
    v = cores[0].reshape(-1, cores[0].shape[2])
    for c in cores[1:]:
        v = (v @ c.reshape(c.shape[0], -1)).reshape(-1, c.shape[2])
    return v[:, 0]


def _kron_cores(factors):
    """Cores of the elementwise product of TTs (Kronecker-delta contraction):
    C[(a1..ak), s, (b1..bk)] = prod_i F_i[a_i, s, b_i]."""
    L = len(factors[0])
    out = []
    for s in range(L):
        c = factors[0][s]
        for f in factors[1:]:
            g = f[s]
            c = np.einsum("asb,csd->acsbd", c, g).reshape(c.shape[0] * g.shape[0], c.shape[1],
                                                         c.shape[2] * g.shape[2])
        out.append(c)
    return out


def exact_product(inputs, op) -> list:
    """f(x^1..x^N) for polynomial f as an exact TT (block sum of Kronecker products)."""
    ins = [_cores_of(x) for x in inputs]
    terms = []
    for coef, ex in zip(op["coef"], op["expo"]):
        factors = []
        for n, e in enumerate(ex):
            factors += [ins[n]] * int(e)
        cs = _kron_cores(factors) if len(factors) > 1 else [c.copy() for c in factors[0]]
        cs[0] = cs[0] * coef
        terms.append(cs)
    if len(terms) == 1:
        return terms[0]
    L = len(terms[0])
    out = []
    for s in range(L):
        parts = [t[s] for t in terms]
        if s == 0:
            out.append(np.concatenate(parts, axis=2))
        elif s == L - 1:
            out.append(np.concatenate(parts, axis=0))
        else:
            rl = sum(p.shape[0] for p in parts)
            rr = sum(p.shape[2] for p in parts)
            c = np.zeros((rl, parts[0].shape[1], rr), np.result_type(*parts))
            i = j = 0
            for p in parts:
                c[i:i + p.shape[0], :, j:j + p.shape[2]] = p
                i += p.shape[0]
                j += p.shape[2]
            out.append(c)
    return out


def tt_round(cores, tol: float) -> list:
    """Textbook TT-SVD rounding: left-to-right QR, then right-to-left truncated SVD with
    per-bond Frobenius budget tol*||C||_F/sqrt(L-1) (the step the paper leaves to the
    MPO-MPS baseline)."""
    cores = [np.array(c, dtype=np.result_type(c, np.float64)) for c in _cores_of(cores)]
    L = len(cores)
    for s in range(L - 1):
        r0, d, r1 = cores[s].shape
        Q, R = np.linalg.qr(cores[s].reshape(r0 * d, r1))
        cores[s] = Q.reshape(r0, d, Q.shape[1])
        cores[s + 1] = np.einsum("ab,bsc->asc", R, cores[s + 1])
    norm = np.linalg.norm(cores[-1])
    delta = tol * norm / np.sqrt(max(L - 1, 1))
    for s in range(L - 1, 0, -1):
        r0, d, r1 = cores[s].shape
        U, S, Vt = np.linalg.svd(cores[s].reshape(r0, d * r1), full_matrices=False)
        tail = np.sqrt(np.cumsum((S ** 2)[::-1]))[::-1]  # tail[k] = ||S[k:]||
        keep = int(np.sum(tail > delta)) if delta > 0 else len(S)
        keep = max(keep, 1)
        cores[s] = Vt[:keep].reshape(keep, d, r1)
        cores[s - 1] = np.einsum("asb,bc->asc", cores[s - 1], U[:, :keep] * S[:keep])
    return cores


def tt_axpby(alpha, a, beta, b) -> list:
    """alpha*a + beta*b as a TT (block-diagonal sum, rank r_a + r_b)."""
    a, b = _cores_of(a), _cores_of(b)
    L = len(a)
    out = []
    for s in range(L):
        x, y = a[s], b[s]
        if s == 0:
            x, y = alpha * x, beta * y
        if L == 1:
            out.append(x + y)
        elif s == 0:
            out.append(np.concatenate([x, y], axis=2))
        elif s == L - 1:
            out.append(np.concatenate([x, y], axis=0))
        else:
            c = np.zeros((x.shape[0] + y.shape[0], x.shape[1], x.shape[2] + y.shape[2]), np.result_type(x, y))
            c[:x.shape[0], :, :x.shape[2]] = x
            c[x.shape[0]:, :, x.shape[2]:] = y
            out.append(c)
    return out


def tt_norm(cores) -> float:
    """Frobenius norm by left-orthogonalisation (QR sweep): no cancellation, accurate even when
    the TT is a small difference of two large ones."""
    cores = [np.array(c, dtype=np.result_type(c, np.float64)) for c in _cores_of(cores)]
    R = np.ones((1, 1))
    for c in cores:
        c = np.einsum("ab,bsc->asc", R, c)
        r0, d, r1 = c.shape
        _, R = np.linalg.qr(c.reshape(r0 * d, r1))
    return float(np.linalg.norm(R))

