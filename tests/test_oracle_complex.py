"""Pins for the complex oracle (f: C^N -> C; aci_oracle_z.c, readings RZ1-RZ6).

Independent of the oracle's arithmetic: hand-worked golden cases
(tests/golden/prrlu_complex_hand.json), exact rational complete pivoting on Gaussian
integers (fractions.Fraction), the closed-form Schur complement of a skeleton, the closed-form
product of two Fourier series, and the reduction to the real oracle when every
imaginary part is zero.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from workloads import make_config, random_tt, random_init
from workloads.generators import _rng

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "prrlu_complex_hand.json")


def test_golden_complex_hand_cases():
    for case in json.load(open(GOLDEN))["cases"]:
        M = np.array(case["M_re"], dtype=float) + 1j * np.array(case["M_im"], dtype=float)
        f = oracle.ldu_z(M, case["tol_abs"], case["maxrank"])
        assert list(f["rows"]) == case["rows"], case["name"]
        assert list(f["cols"]) == case["cols"], case["name"]
        D = np.array(case["D_re"]) + 1j * np.array(case["D_im"])
        assert np.allclose(f["D"], D, rtol=1e-15, atol=0), case["name"]
        if "eps" in case:
            assert f["eps"] == case["eps"], case["name"]
        else:
            assert f["eps"] <= case["eps_max"], case["name"]


def _gecp_exact_complex(Mre, Mim):
    """Complete pivoting in exact Gaussian-rational arithmetic: argmax |z|^2 (exact), ties to the
    smallest (row, col); returns pivots, pivot values and whether any step had an exact tie
    between distinct entries (where floating point may legitimately order them differently)."""
    m, n = Mre.shape
    S = [[(Fraction(int(Mre[i, j])), Fraction(int(Mim[i, j]))) for j in range(n)] for i in range(m)]
    rows_done, cols_done = set(), set()
    piv, D, tie = [], [], False
    for _ in range(min(m, n)):
        cand = [(S[i][j][0] ** 2 + S[i][j][1] ** 2, i, j) for i in range(m) if i not in rows_done
                for j in range(n) if j not in cols_done]
        best = max(c[0] for c in cand)
        if best == 0:
            break
        at = sorted((i, j) for w, i, j in cand if w == best)
        tie |= len(at) > 1 and len(piv) > 0
        p, q = at[0]
        cr, ci = S[p][q]
        w = cr * cr + ci * ci
        ir, ii = cr / w, -ci / w
        for i in range(m):
            if i in rows_done or i == p:
                continue
            sr, si = S[i][q]
            lr, li = sr * ir - si * ii, sr * ii + si * ir
            for j in range(n):
                if j in cols_done or j == q:
                    continue
                ur, ui = S[p][j]
                S[i][j] = (S[i][j][0] - (lr * ur - li * ui), S[i][j][1] - (lr * ui + li * ur))
        piv.append((p, q))
        D.append(complex(float(cr), float(ci)))
        rows_done.add(p)
        cols_done.add(q)
    return piv, D, tie


def test_exact_complex_gecp_on_gaussian_integers():
    rng = np.random.default_rng(11)
    checked = 0
    for trial in range(40):
        m, n = rng.integers(2, 7, size=2)
        Mre = rng.integers(-30, 31, size=(m, n))
        Mim = rng.integers(-30, 31, size=(m, n))
        piv, D, tie = _gecp_exact_complex(Mre, Mim)
        if tie:
            continue
        f = oracle.ldu_z(Mre + 1j * Mim, 0.0, min(m, n))
        assert list(zip(f["rows"], f["cols"])) == piv
        assert np.allclose(f["D"], D, rtol=1e-12, atol=0)
        checked += 1
    assert checked >= 25


def _schur_after(M, rows, cols):
    """Closed-form Schur complement of the skeleton M[I, J]: M - M[:, J] M[I, J]^{-1} M[I, :]."""
    if len(rows) == 0:
        return M.copy()
    return M - M[:, cols] @ np.linalg.solve(M[np.ix_(rows, cols)], M[rows, :])


def test_pivots_are_argmax_of_the_closed_form_residual():
    rng = np.random.default_rng(5)
    for m, n in [(12, 9), (7, 7), (5, 11)]:
        M = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
        f = oracle.ldu_z(M, 0.0, min(m, n))
        for k in range(f["r"]):
            S = _schur_after(M, list(f["rows"][:k]), list(f["cols"][:k]))
            a = np.abs(S)
            assert a[f["rows"][k], f["cols"][k]] >= a.max() * (1 - 1e-10)
            assert np.isclose(S[f["rows"][k], f["cols"][k]], f["D"][k], rtol=1e-9)
        # truncated at rank 4: eps = max |residual| of the rank-4 skeleton (R2)
        g = oracle.ldu_z(M, 0.0, 4)
        S = _schur_after(M, list(g["rows"]), list(g["cols"]))
        assert np.isclose(g["eps"], np.abs(S).max(), rtol=1e-10)


def test_rank_one_complex_matrix_stops_after_one_pivot():
    rng = np.random.default_rng(2)
    u = rng.standard_normal(9) + 1j * rng.standard_normal(9)
    v = rng.standard_normal(6) + 1j * rng.standard_normal(6)
    f = oracle.ldu_z(np.outer(u, v), 1e-12, 6, relative_to_own_max=True)
    assert f["r"] == 1


def test_unit_rows_and_interpolation_identity():
    rng = np.random.default_rng(3)
    M = rng.standard_normal((8, 10)) + 1j * rng.standard_normal((8, 10))
    f = oracle.ldu_z(M, 0.0, 5)
    U = f["U"]
    for k in range(f["r"]):
        assert U[k, f["cols"][k]] == 1.0
        for t in range(k):
            assert U[k, f["cols"][t]] == 0.0  # eliminated columns are exact zeros
        # U_k = S_k[p, :] / S_k[p, q] with S_k the closed-form residual
        S = _schur_after(M, list(f["rows"][:k]), list(f["cols"][:k]))
        assert np.allclose(U[k], S[f["rows"][k]] / S[f["rows"][k], f["cols"][k]], rtol=1e-9, atol=1e-12)


def _fourier_values(tt, samples):
    x = (samples * (2.0 ** -np.arange(1, samples.shape[1] + 1))).sum(axis=1)
    c = tt.meta["coefs"]
    return np.exp(1j * np.outer(x, np.arange(len(c)))) @ c


def test_fourier_inputs_match_their_closed_form():
    cf = make_config(5, 100, npts=2000)
    for t in cf["inputs"]:
        g = _fourier_values(t, cf["samples"])
        assert np.abs(oracle.tt_evaluate(t.cores, cf["samples"]) - g).max() <= 1e-10 * np.abs(g).max()


def test_aci_z_fourier_product_within_tolerance():
    """The paper's random Fourier series product: g1 * g2 on 2000 random points."""
    cf = make_config(5, 100, npts=2000)
    res = oracle.aci_z(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"])
    exact = _fourier_values(cf["inputs"][0], cf["samples"]) * _fourier_values(cf["inputs"][1], cf["samples"])
    y = oracle.tt_evaluate(res.cores, cf["samples"])
    assert np.abs(y - exact).max() <= 10 * cf["tol"] * np.abs(exact).max()
    assert res.ranks[15] <= 2 * max(cf["inputs"][0].ranks)


def test_aci_z_on_real_inputs_agrees_with_real_oracle():
    """Zero imaginary parts: the complex run must give the real run's values (RZ1 reduces to
    |x| argmax; the two runs differ only at roundoff)."""
    cf = make_config(0, npts=2000)
    xr = [t.cores for t in cf["inputs"]]
    xz = [[c.astype(np.complex128) for c in t.cores] for t in cf["inputs"]]
    yz = [c.astype(np.complex128) for c in cf["y_init"].cores]
    rr = oracle.aci(xr, cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"])
    rz = oracle.aci_z(xz, cf["op"], yz, cf["tol"], cf["maxrank"], cf["max_sweeps"])
    a = oracle.tt_evaluate(rr.cores, cf["samples"])
    b = oracle.tt_evaluate(rz.cores, cf["samples"])
    assert np.abs(b.imag).max() == 0.0
    assert np.abs(a - b.real).max() <= 10 * cf["tol"] * np.abs(a).max()
    same = sum(1 for u, v in zip(rr.log, rz.log) if u["r"] == v["r"] and np.array_equal(u["rows"], v["rows"]))
    assert same >= 0.9 * len(rr.log)


def test_aci_z_identity_reproduces_input():
    """N = 1, f = x on a random complex TT."""
    L = 10
    r = _rng(99, 0)
    base = random_tt(L, 2, 4, r)
    imag = random_tt(L, 2, 4, _rng(99, 1))
    x = [a + 1j * b for a, b in zip(base.cores, imag.cores)]
    from workloads import TT
    y0 = random_init([TT(x)], 8, _rng(99, 2))
    res = oracle.aci_z([x], {"coef": [1.0], "expo": [[1]]}, y0, 1e-12, 8, 4)
    assert res.report["iterations"] <= 2
    assert np.allclose(oracle.tt_dense(res.cores), oracle.tt_dense(x), rtol=0, atol=1e-12 * np.abs(oracle.tt_dense(x)).max())
