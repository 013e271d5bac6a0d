"""Pins for the oracle's prrLU (Alg. 2) and cross interpolation (Alg. 3).

Every check here is independent of the oracle's own arithmetic: hand-worked
golden cases (tests/golden/prrlu_hand.json), exact rational elimination
(fractions.Fraction), residuals recomputed from the returned factors, and
closed-form properties (rank-1 termination, interpolation identities).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "prrlu_hand.json")


def test_golden_hand_worked_cases():
    for case in json.load(open(GOLDEN))["cases"]:
        M = np.array(case["M"], dtype=np.float64)
        f = oracle.ldu(M, case["tol_abs"], case["maxrank"])
        assert list(f["rows"]) == case["rows"], case["name"]
        assert list(f["cols"]) == case["cols"], case["name"]
        assert np.allclose(f["D"], case["D"], rtol=1e-15, atol=0), case["name"]
        if "eps" in case:
            assert f["eps"] == case["eps"], case["name"]
        else:
            assert f["eps"] <= case["eps_max"], case["name"]


def _gecp_exact(M, maxrank):
    """Complete-pivoting Gaussian elimination in exact rational arithmetic (textbook GECP)."""
    m, n = len(M), len(M[0])
    S = [[Fraction(int(x)) for x in row] for row in M]
    rows_done, cols_done = set(), set()
    piv, D, gaps = [], [], []
    for _ in range(min(m, n, maxrank)):
        cand = sorted(((abs(S[i][j]), -i, -j) for i in range(m) if i not in rows_done
                       for j in range(n) if j not in cols_done), reverse=True)
        best = cand[0]
        if best[0] == 0:
            break
        p, q = -best[1], -best[2]
        gaps.append(float((best[0] - cand[1][0]) / best[0]) if len(cand) > 1 else 1.0)
        c = S[p][q]
        piv.append((p, q))
        D.append(c)
        for i in range(m):
            if i in rows_done or i == p:
                continue
            li = S[i][q] / c
            for j in range(n):
                if j in cols_done or j == q:
                    continue
                S[i][j] -= li * S[p][j]
        rows_done.add(p)
        cols_done.add(q)
    return piv, D, gaps


def test_pivots_match_exact_rational_gecp():
    """On random small integer matrices the float oracle picks the same pivots as exact GECP
    wherever the exact top-2 gap is not a near-tie, and the pivot values agree to ~1e-13."""
    rng = np.random.default_rng(7)
    checked = 0
    for trial in range(80):
        m, n = rng.integers(2, 7, size=2)
        M = rng.integers(-999, 1000, size=(m, n)).astype(float)
        piv, D, gaps = _gecp_exact(M.astype(int).tolist(), min(m, n))
        f = oracle.ldu(M, 0.0, min(m, n))
        k_ok = len(piv)
        for k, g in enumerate(gaps):
            if g < 1e-9:  # exact tie that float rounding may break either way
                k_ok = k
                break
        got = list(zip(f["rows"][:k_ok].tolist(), f["cols"][:k_ok].tolist()))
        assert got == piv[:k_ok], (trial, M)
        for k in range(k_ok):
            assert abs(f["D"][k] - float(D[k])) <= 1e-12 * abs(float(D[k]))
        checked += k_ok
    assert checked > 100


def _residual(M, f):
    return M - f["L"] @ np.diag(f["D"]) @ f["U"]


@pytest.mark.parametrize("seed", range(8))
def test_each_pivot_is_argmax_of_recomputed_residual(seed):
    """R18 replacement for 'pivots nonincreasing': pivot k is the max-|.| entry of
    M - L_{:k} D_{:k} U_{:k} recomputed from the returned factors (brute force)."""
    rng = np.random.default_rng(seed)
    m, n = rng.integers(3, 14, size=2)
    M = rng.standard_normal((m, n))
    f = oracle.ldu(M, 0.0, min(m, n))
    for k in range(f["r"]):
        R = M - f["L"][:, :k] @ np.diag(f["D"][:k]) @ f["U"][:k]
        R[list(f["rows"][:k]), :] = 0
        R[:, list(f["cols"][:k])] = 0
        i, j = np.unravel_index(np.argmax(np.abs(R)), R.shape)
        assert abs(abs(R[i, j]) - abs(R[f["rows"][k], f["cols"][k]])) <= 1e-12 * abs(R[i, j])
        assert abs(f["D"][k] - R[f["rows"][k], f["cols"][k]]) <= 1e-12 * abs(R[i, j])


@pytest.mark.parametrize("seed", range(6))
def test_eps_is_max_residual_and_full_rank_reconstructs(seed):
    rng = np.random.default_rng(100 + seed)
    m, n = rng.integers(4, 16, size=2)
    # numerically rank-deficient: rank 3 + tiny noise
    M = rng.standard_normal((m, 3)) @ rng.standard_normal((3, n)) + 1e-7 * rng.standard_normal((m, n))
    f = oracle.ldu(M, 1e-5, min(m, n))
    assert f["r"] == 3
    assert abs(f["eps"] - np.abs(_residual(M, f)).max()) <= 1e-12 * np.abs(M).max()
    g = oracle.ldu(M, 0.0, min(m, n))
    assert g["r"] == min(m, n) and g["eps"] == 0.0
    assert np.abs(_residual(M, g)).max() <= 1e-12 * np.abs(M).max()


def test_rank_one_terminates_after_one_pivot():
    rng = np.random.default_rng(3)
    for _ in range(20):
        u, v = rng.standard_normal(7), rng.standard_normal(5)
        M = np.outer(u, v)
        f = oracle.ldu(M, 1e-12, 5, relative_to_own_max=True)
        assert f["r"] == 1
        assert f["eps"] <= 1e-14 * np.abs(M).max()


def test_factor_structure():
    """L unit lower / U unit upper in pivot order (R4)."""
    rng = np.random.default_rng(11)
    M = rng.standard_normal((9, 7))
    f = oracle.ldu(M, 0.0, 7)
    LI = f["L"][f["rows"], :]
    UJ = f["U"][:, f["cols"]]
    assert np.allclose(np.diag(LI), 1) and np.allclose(np.triu(LI, 1), 0)
    assert np.allclose(np.diag(UJ), 1) and np.allclose(np.tril(UJ, -1), 0)
    assert np.abs(f["U"]).max() <= 1 + 1e-15  # full pivoting bounds |U| <= 1
    assert np.abs(f["L"]).max() <= 1 + 1e-15


@pytest.mark.parametrize("seed", range(5))
def test_cross_interpolation_identities(seed):
    """Alg. 3 right branch: B[:, J] = identity, A = M[:, J], AB exact on pivot rows/cols."""
    rng = np.random.default_rng(200 + seed)
    m, n = rng.integers(5, 12, size=2)
    M = rng.standard_normal((m, 4)) @ rng.standard_normal((4, n)) + 1e-9 * rng.standard_normal((m, n))
    f = oracle.ci_right(M, 1e-6, 10, relative_to_own_max=True)
    r = f["r"]
    assert r == 4
    assert np.abs(f["B"][:, f["cols"]] - np.eye(r)).max() <= 1e-14
    assert np.array_equal(f["A"], M[:, f["cols"]])
    AB = f["A"] @ f["B"]
    scale = np.abs(M).max()
    assert np.abs(AB[f["rows"], :] - M[f["rows"], :]).max() <= 1e-12 * scale
    assert np.abs(AB[:, f["cols"]] - M[:, f["cols"]]).max() <= 1e-12 * scale
    assert np.abs(AB - M).max() <= 10 * 1e-6 * scale


def test_nonfinite_rejected():
    M = np.ones((3, 3))
    M[1, 2] = np.nan
    with pytest.raises(ValueError):
        oracle.ldu(M, 0.0, 3)


# ---------------------------------------------------------------------------------------------
# Rook pivoting (reading R23; SURVEY 8(f) NEXT-4, B:5 "full/rook")
# ---------------------------------------------------------------------------------------------
ROOK_GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "prrlu_rook_hand.json")


def test_rook_golden_hand_worked_cases():
    for case in json.load(open(ROOK_GOLDEN))["cases"]:
        M = np.array(case["M"], dtype=np.float64)
        f = oracle.ldu(M, case["tol_abs"], case["maxrank"], pivoting="rook")
        assert list(f["rows"]) == case["rows"], case["name"]
        assert list(f["cols"]) == case["cols"], case["name"]
        assert np.allclose(f["D"], case["D"], rtol=1e-15, atol=0), case["name"]
        assert f["eps"] == case["eps"], case["name"]


def _residual_closed_form(M, I, J):
    """S = M - M[:, J] M[I, J]^{-1} M[I, :] (the Schur complement after pivots I, J)."""
    if not I:
        return M.copy()
    return M - M[:, J] @ np.linalg.solve(M[np.ix_(I, J)], M[I, :])


@pytest.mark.parametrize("seed", range(8))
def test_rook_pivot_is_max_of_its_row_and_column(seed):
    """Definition of a rook pivot: every accepted (p, q) is the largest |.| of its active row and
    of its active column in the residual recomputed in closed form (independent of the oracle's
    elimination); eps is the magnitude of such an entry of the final residual (or 0)."""
    rng = np.random.default_rng(seed)
    m, n = int(rng.integers(3, 12)), int(rng.integers(3, 12))
    M = rng.standard_normal((m, n))
    f = oracle.ldu(M, 0.0, min(m, n), pivoting="rook")
    I, J = [], []
    for p, q in zip(f["rows"], f["cols"]):
        S = _residual_closed_form(M, I, J)
        ar = [i for i in range(m) if i not in I]
        ac = [j for j in range(n) if j not in J]
        v = abs(S[p, q])
        assert v >= np.abs(S[p, ac]).max() * (1 - 1e-12)
        assert v >= np.abs(S[ar, q]).max() * (1 - 1e-12)
        I.append(int(p))
        J.append(int(q))
    assert len(I) == min(m, n) and f["eps"] == 0.0


def _rook_exact(M, maxrank):
    """Textbook rook pivoting (Neal & Poole) in exact rational arithmetic: start at the smallest
    active column, alternate column / row maxima (strictly larger only, ties -> smallest index)."""
    m, n = len(M), len(M[0])
    S = [[Fraction(int(x)) for x in row] for row in M]
    rd, cd = set(), set()
    piv, D = [], []
    for _ in range(min(m, n, maxrank)):
        ar = [i for i in range(m) if i not in rd]
        ac = [j for j in range(n) if j not in cd]
        c = ac[0]
        r = max(ar, key=lambda i: (abs(S[i][c]), -i))
        while True:
            c2 = max(ac, key=lambda j: (abs(S[r][j]), -j))
            if abs(S[r][c2]) <= abs(S[r][c]):
                break
            c = c2
            r2 = max(ar, key=lambda i: (abs(S[i][c]), -i))
            if abs(S[r2][c]) <= abs(S[r][c]):
                break
            r = r2
        if S[r][c] == 0:
            break
        piv.append((r, c))
        D.append(S[r][c])
        for i in ar:
            if i == r:
                continue
            li = S[i][c] / S[r][c]
            for j in ac:
                if j != c:
                    S[i][j] -= li * S[r][j]
        rd.add(r)
        cd.add(c)
    return piv, D


@pytest.mark.parametrize("seed", range(12))
def test_rook_matches_exact_rational_rook_elimination(seed):
    """Integer matrices with distinct magnitudes (no near-ties): the oracle's rook pivots equal
    exact rational rook pivoting, and its pivot values match to roundoff."""
    rng = np.random.default_rng(100 + seed)
    m, n = int(rng.integers(3, 8)), int(rng.integers(3, 8))
    vals = rng.permutation(np.arange(1, m * n + 1)) * rng.choice([-1, 1], size=m * n)
    M = vals.reshape(m, n).astype(np.float64)
    piv, D = _rook_exact(M.astype(int).tolist(), min(m, n))
    f = oracle.ldu(M, 0.0, min(m, n), pivoting="rook")
    k = len(piv)
    assert f["r"] == k
    assert [tuple(x) for x in zip(f["rows"][:k], f["cols"][:k])] == piv[:k]
    assert np.allclose(f["D"][:k], [float(x) for x in D[:k]], rtol=1e-13)


def test_rook_full_rank_reconstruction_and_interpolation():
    """Rook LDU reproduces M at full rank (L D U = M), and the cross interpolation of its pivots
    is exact on the pivot rows and columns — the identities hold for any pivot order."""
    rng = np.random.default_rng(7)
    M = rng.standard_normal((9, 7))
    f = oracle.ldu(M, 0.0, 7, pivoting="rook")
    assert f["r"] == 7
    R = f["L"] @ np.diag(f["D"]) @ f["U"]
    assert np.abs(R - M).max() <= 1e-12 * np.abs(M).max()
    I, J = list(f["rows"]), list(f["cols"])
    A = M[:, J] @ np.linalg.inv(M[np.ix_(I, J)]) @ M[I, :]
    assert np.abs(A[I, :] - M[I, :]).max() <= 1e-12 and np.abs(A[:, J] - M[:, J]).max() <= 1e-12
