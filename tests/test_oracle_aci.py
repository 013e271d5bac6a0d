"""Pins for the oracle's TT evaluation, exact product and full ACI run (Alg. 1).

Independent references used here: closed-form functions the inputs were
built from (cosine sums, plane waves, separable Gaussians), dense products of
dense vectors, per-index brute-force TT evaluation with Python loops, rank
bounds rank(A*B) <= rank(A) rank(B), the TT-SVD error bound, and special cases
(N=1 identity, rank-1 inputs).
"""
import math

import numpy as np
import pytest

import oracle
from workloads import generators as G
from workloads import make_config


def _brute_eval(cores, idx):
    """One point, pure Python loops over the chain (the definition)."""
    v = [1.0]
    for s, c in enumerate(cores):
        sg = int(idx[s])
        nv = [0.0] * c.shape[2]
        for b in range(c.shape[2]):
            acc = 0.0
            for a in range(c.shape[0]):
                acc += v[a] * c[a, sg, b]
            nv[b] = acc
        v = nv
    return v[0]


def _closed_cosine(meta, x):
    return sum(a * np.cos(2 * np.pi * k * x + p) for k, p, a in zip(meta["ks"], meta["phis"], meta["amps"]))


def test_cosine_inputs_match_closed_form():
    cf = make_config(0, npts=0)
    x = np.arange(4096) / 4096.0
    for t in cf["inputs"]:
        assert max(t.ranks) == 8
        assert np.abs(oracle.tt_dense(t) - _closed_cosine(t.meta, x)).max() < 1e-13


def test_evaluate_matches_bruteforce_loops():
    rng = np.random.default_rng(5)
    t = G.random_tt(7, 3, 4, rng)
    idx = G.sample_indices(t.d, 40, rng)
    fast = oracle.tt_evaluate(t, idx)
    for p in range(40):
        assert abs(fast[p] - _brute_eval(t.cores, idx[p])) < 1e-13
    dense = oracle.tt_dense(t).reshape([3] * 7)
    for p in range(40):
        assert abs(dense[tuple(idx[p])] - fast[p]) < 1e-13


def test_plane_wave_inputs_match_closed_form():
    cf = make_config(4, npts=2000)
    s = cf["samples"]
    L = 20
    w = 2.0 ** -np.arange(1, L + 1)
    x = (s >> 1).astype(float) @ w
    y = (s & 1).astype(float) @ w
    for t in cf["inputs"]:
        m = t.meta
        ref = sum(a * np.cos(2 * np.pi * (kx * x + ky * y) + p)
                  for kx, ky, p, a in zip(m["kxs"], m["kys"], m["phis"], m["amps"]))
        assert max(t.ranks) == 128
        assert np.abs(oracle.tt_evaluate(t, s) - ref).max() < 1e-12


def test_gaussian3d_input_matches_closed_form():
    cf = make_config(2, npts=3000)
    psi = cf["inputs"][0]
    m = psi.meta
    s = cf["samples"].astype(np.int64)
    w = 2 ** np.arange(9, -1, -1)
    xs = [(s[:, 10 * a:10 * a + 10] @ w) / 1024.0 for a in range(3)]
    ref = 0
    for c, sg, a in zip(m["cs"], m["sigmas"], m["amps"]):
        g = [np.exp(-(t - c) ** 2 / (2 * sg ** 2)) for t in xs]
        ref = ref + a * g[0] * g[1] * g[2]
    assert np.abs(oracle.tt_evaluate(psi, cf["samples"]) - ref).max() < 1e-10 * np.abs(ref).max()


def test_exact_product_dense_and_rank_bound():
    cf = make_config(0, npts=0)
    A, B = cf["inputs"]
    x = np.arange(4096) / 4096.0
    ref = _closed_cosine(A.meta, x) * _closed_cosine(B.meta, x)
    ex = oracle.exact_product(cf["inputs"], cf["op"])
    assert all(c.shape[2] <= 64 for c in ex[:-1])  # rank(A*B) <= rank(A) rank(B)
    assert np.abs(oracle.tt_dense(ex) - ref).max() < 1e-13
    rd = oracle.tt_round(ex, 1e-12)
    err = np.linalg.norm(oracle.tt_dense(rd) - ref) / np.linalg.norm(ref)
    assert err <= 1e-12
    # the product of 4+4 cosines is a sum of <= 32 cosines: rank <= 64 (here well below)
    assert max(c.shape[2] for c in rd) <= 64


def test_exact_product_polynomial_op():
    rng = np.random.default_rng(1)
    a, b = G.random_tt(6, 2, 3, rng), G.random_tt(6, 2, 2, rng)
    op = {"coef": [1.0, 0.5], "expo": [[1, 1], [2, 0]]}
    da, db = oracle.tt_dense(a), oracle.tt_dense(b)
    ex = oracle.exact_product([a, b], op)
    assert np.abs(oracle.tt_dense(ex) - (da * db + 0.5 * da * da)).max() < 1e-13


def test_tt_norm_and_axpby_vs_dense():
    rng = np.random.default_rng(8)
    a, b = G.random_tt(8, 2, 5, rng), G.random_tt(8, 2, 3, rng)
    da, db = oracle.tt_dense(a), oracle.tt_dense(b)
    assert abs(oracle.tt_norm(a) - np.linalg.norm(da)) <= 1e-13 * np.linalg.norm(da)
    diff = oracle.tt_axpby(2.0, a, -0.5, b)
    assert np.abs(oracle.tt_dense(diff) - (2 * da - 0.5 * db)).max() <= 1e-13 * np.abs(da).max()
    # no cancellation floor: a difference of 1e-9 relative is measured to ~1e-6 relative accuracy
    c = G.TT([x.copy() for x in a.cores])
    c.cores[3] = c.cores[3] * (1 + 1e-9)
    nd = oracle.tt_norm(oracle.tt_axpby(1.0, c, -1.0, a))
    assert abs(nd - 1e-9 * np.linalg.norm(da)) <= 1e-6 * 1e-9 * np.linalg.norm(da)


def test_tt_round_error_bound():
    rng = np.random.default_rng(2)
    a = G.random_tt(8, 2, 6, rng)
    b = G.random_tt(8, 2, 5, rng)
    ex = oracle.exact_product([a, b], {"coef": [1.0], "expo": [[1, 1]]})
    full = oracle.tt_dense(ex)
    for tol in (1e-1, 1e-3, 1e-8):
        rd = oracle.tt_round(ex, tol)
        assert np.linalg.norm(oracle.tt_dense(rd) - full) <= tol * np.linalg.norm(full) * (1 + 1e-9)


# ---------------------------------------------------------------- full ACI runs
def _rel_max(y, r):
    return np.abs(y - r).max() / np.abs(r).max()


def test_aci_cfg0_matches_dense_product():
    """configs[0]: the ACI output equals the dense 4096-vector product within 10*tol (B:7)."""
    cf = make_config(0, npts=0)
    res = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"])
    x = np.arange(4096) / 4096.0
    ref = _closed_cosine(cf["inputs"][0].meta, x) * _closed_cosine(cf["inputs"][1].meta, x)
    assert _rel_max(oracle.tt_dense(res.cores), ref) <= 10 * cf["tol"]
    assert res.report["converged"]
    assert max(res.ranks) <= 64


def test_aci_cfg1_matches_exact_product():
    """configs[1]: output rank <= 64 and <= 10*tol vs Kronecker + SVD (B:8)."""
    cf = make_config(1, npts=20000)
    res = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"])
    assert max(res.ranks) <= 64
    s = cf["samples"]
    ref = oracle.tt_evaluate(cf["inputs"][0], s) * oracle.tt_evaluate(cf["inputs"][1], s)
    assert _rel_max(oracle.tt_evaluate(res.cores, s), ref) <= 10 * cf["tol"]
    ex = oracle.exact_product(cf["inputs"], cf["op"])
    frob = oracle.tt_norm(oracle.tt_axpby(1.0, res.cores, -1.0, ex)) / oracle.tt_norm(ex)
    assert frob <= 10 * cf["tol"]
    assert res.report["converged"]


def test_aci_identity_op_reproduces_input():
    """N=1, f(v)=v converges within 2 iterations and reproduces x."""
    rng = np.random.default_rng(21)
    x = G.random_tt(10, 2, 8, rng)
    y0 = G.random_init([x], 8, rng)
    res = oracle.aci([x], {"coef": [1.0], "expo": [[1]]}, y0, 1e-12, 64, 20)
    assert res.report["converged"] and res.report["iterations"] <= 2
    assert all(r <= 8 for r in res.ranks)
    assert _rel_max(oracle.tt_dense(res.cores), oracle.tt_dense(x)) <= 1e-10


def test_aci_rank_one_inputs_give_rank_one_output():
    rng = np.random.default_rng(22)
    a = G.random_tt(9, 2, 1, rng)
    b = G.random_tt(9, 2, 1, rng)
    y0 = G.random_init([a, b], 4, rng)
    res = oracle.aci([a, b], {"coef": [1.0], "expo": [[1, 1]]}, y0, 1e-12, 16, 10)
    assert max(res.ranks) == 1
    assert _rel_max(oracle.tt_dense(res.cores), oracle.tt_dense(a) * oracle.tt_dense(b)) <= 1e-13


def test_aci_random_small_suite_vs_dense():
    """SPEC acceptance, reduced: random L in 4..8, chi in 2..5,
    f in {x1*x2, x1+x2, x1*x2+x3}, tol 1e-10 -> dense max error <= 1e-8 relative."""
    rng = np.random.default_rng(2024)
    ops = [({"coef": [1.0], "expo": [[1, 1]]}, 2), ({"coef": [1.0, 1.0], "expo": [[1, 0], [0, 1]]}, 2),
           ({"coef": [1.0, 1.0], "expo": [[1, 1, 0], [0, 0, 1]]}, 3)]
    for trial in range(24):
        L = int(rng.integers(4, 9))
        op, N = ops[trial % 3]
        xs = [G.random_tt(L, 2, int(rng.integers(2, 6)), rng) for _ in range(N)]
        y0 = G.random_init(xs, 64, rng)
        res = oracle.aci(xs, op, y0, 1e-10, 64, 20)
        dense = [oracle.tt_dense(x) for x in xs]
        ref = np.zeros_like(dense[0])
        for c, e in zip(op["coef"], op["expo"]):
            term = c * np.ones_like(ref)
            for n, k in enumerate(e):
                term = term * dense[n] ** k
            ref += term
        assert _rel_max(oracle.tt_dense(res.cores), ref) <= 1e-8, trial


def test_aci_interpolation_nesting_and_frames():
    """After the final right-to-left half-sweep:
    (i) J sets are nested J_{s} > J_{s+1};
    (ii) every column of R^n_s is the partial contraction of cores s..L-1 at J_s[k] (brute force);
    (iii) every row of L^n_b is the partial contraction of cores 0..b at I_b[a];
    (iv) the output interpolates f exactly on the last-updated cross (I_0 x J_1)."""
    rng = np.random.default_rng(31)
    L = 8
    a, b = G.random_tt(L, 2, 3, rng), G.random_tt(L, 2, 2, rng)
    y0 = G.random_init([a, b], 16, rng)
    res = oracle.aci([a, b], {"coef": [1.0], "expo": [[1, 1]]}, y0, 1e-12, 64, 6)
    for s in range(1, L - 1):
        Js, Jn = res.Jset(s), res.Jset(s + 1)
        tails = {tuple(r[1:]) for r in Js}
        assert tails <= {tuple(r) for r in Jn}
    for n, x in enumerate([a, b]):
        for s in range(1, L):
            R = res.Rframe(n, s)
            for k, j in enumerate(res.Jset(s)):
                v = np.eye(x.cores[s].shape[0])
                for t, sg in zip(range(s, L), j):
                    v = v @ x.cores[t][:, sg, :]
                assert np.abs(R[:, k] - v[:, 0]).max() < 1e-13
        for bnd in range(L - 1):
            Lf = res.Lframe(n, bnd)
            for k, i in enumerate(res.Iset(bnd)):
                v = np.ones((1, 1))
                for t, sg in enumerate(i):
                    v = v @ x.cores[t][:, sg, :]
                assert np.abs(Lf[k] - v[0]).max() < 1e-13
    I0, J1 = res.Iset(0), res.Jset(1)
    pts = np.array([np.concatenate([i, j]) for i in I0 for j in J1], dtype=np.uint8)
    y = oracle.tt_evaluate(res.cores, pts)
    ref = oracle.tt_evaluate(a, pts) * oracle.tt_evaluate(b, pts)
    assert np.abs(y - ref).max() <= 1e-13 * np.abs(ref).max()


def test_assemble_pi_matches_direct_evaluation():
    """Eq. pifromframes: Pi[a,s,s',j] = f(x^n(I[a] s s' J[j])) with frames built by brute force."""
    rng = np.random.default_rng(41)
    L, b = 7, 3
    xs = [G.random_tt(L, 2, 3, rng), G.random_tt(L, 2, 4, rng)]
    I = [tuple(rng.integers(0, 2, size=b)) for _ in range(3)]
    J = [tuple(rng.integers(0, 2, size=L - b - 2)) for _ in range(4)]
    op = {"coef": [2.0, -1.0], "expo": [[1, 1], [0, 2]]}
    Ls, Rs = [], []
    for x in xs:
        Lf = np.zeros((len(I), x.cores[b].shape[0]))
        for k, i in enumerate(I):
            v = np.ones((1, 1))
            for t, sg in enumerate(i):
                v = v @ x.cores[t][:, sg, :]
            Lf[k] = v[0]
        Rf = np.zeros((x.cores[b + 2].shape[0], len(J)))
        for k, j in enumerate(J):
            v = np.eye(x.cores[b + 2].shape[0])
            for t, sg in zip(range(b + 2, L), j):
                v = v @ x.cores[t][:, sg, :]
            Rf[:, k] = v[:, 0]
        Ls.append(Lf)
        Rs.append(Rf)
    Pi = oracle.assemble_pi(Ls, [x.cores[b] for x in xs], [x.cores[b + 1] for x in xs], Rs, op)
    for ai, i in enumerate(I):
        for s in range(2):
            for sp in range(2):
                for ji, j in enumerate(J):
                    full = np.array([i + (s, sp) + j], dtype=np.uint8)
                    v = [_brute_eval(x.cores, full[0]) for x in xs]
                    ref = 2.0 * v[0] * v[1] - v[1] ** 2
                    assert abs(Pi[ai * 2 + s, sp * len(J) + ji] - ref) < 1e-13


def test_aci_deterministic():
    cf = make_config(0, npts=0)
    r1 = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"])
    r2 = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"])
    assert all(np.array_equal(x, y) for x, y in zip(r1.cores, r2.cores))
    assert all(np.array_equal(x["rows"], y["rows"]) for x, y in zip(r1.log, r2.log))


@pytest.mark.slow
def test_aci_cfg3_chi64_saturates_to_exact_product():
    """configs[3] chi=64: ranks reach 2*chi and the output matches the exact product (CI exactness)."""
    cf = make_config(3, 64, npts=5000)
    res = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"])
    assert max(res.ranks) == 128
    s = cf["samples"]
    ref = oracle.tt_evaluate(cf["inputs"][0], s) * oracle.tt_evaluate(cf["inputs"][1], s)
    assert _rel_max(oracle.tt_evaluate(res.cores, s), ref) <= 10 * cf["tol"]


def _generic_rank_model(d, true_ranks, yr, maxrank, maxiter):
    """Closed-form rank recursion of Alg. 1 on GENERIC data (exact arithmetic), independent of the
    oracle's code. Canonicalisation: |J_s| = min(r^y_s, d_s |J_{s+1}|, chi-hat,
    full bound). An update at bond b sees the block Pi of size (d_b |I_{b-1}|) x (d_{b+1} |J_{b+2}|)
    (Alg. 4) whose rank is generically min(m, n, true rank of the bond); prrLU with a tolerance
    above roundoff takes exactly that many pivots (capped at chi-hat) and its error eps is ~0 unless
    the cap binds. So rank at most multiplies by d per half-sweep from the J sets ("rank doubling"
    for d = 2), and eps alone would stop the loop after iteration 1 — only P:497's clause "the
    chi_l have not increased" keeps it running. Returns (iterations, converged, final ranks)."""
    L = len(d)

    def full(b):
        return min(int(np.prod([float(x) for x in d[:b + 1]])), int(np.prod([float(x) for x in d[b + 1:]])))

    Jn = [0] * (L + 1)
    Jn[L] = 1
    for s in range(L - 1, 0, -1):
        Jn[s] = min(yr[s], d[s] * Jn[s + 1], maxrank, full(s - 1))
    chi = [Jn[b + 1] for b in range(L - 1)]
    prev = list(chi)
    for it in range(1, maxiter + 1):
        eps_ok = True
        for bonds in (range(L - 1), range(L - 2, -1, -1)):
            for b in bonds:
                rl = 1 if b == 0 else chi[b - 1]
                rr = 1 if b + 2 == L else Jn[b + 2]
                rank_pi = min(rl * d[b], d[b + 1] * rr, true_ranks[b])
                chi[b] = Jn[b + 1] = min(rank_pi, maxrank)
                eps_ok &= chi[b] == rank_pi
        grew = any(c > p for c, p in zip(chi, prev))
        prev = list(chi)
        if not grew and eps_ok:
            return it, True, chi
    return maxiter, False, chi


def _product_true_ranks(inputs):
    """rank(A (.) B) = rank(A) rank(B) for generic inputs (B:5), capped by the full bound."""
    d = inputs[0].d
    L = len(d)
    out = []
    for b in range(L - 1):
        full = min(int(np.prod([float(x) for x in d[:b + 1]])), int(np.prod([float(x) for x in d[b + 1:]])))
        p = 1
        for t in inputs:
            p *= min(t.ranks[b + 1], full)
        out.append(min(p, full))
    return out


@pytest.mark.parametrize("cfg,chi", [(1, 0), (3, 64), (3, 128)])
def test_aci_convergence_rank_clause_matches_rank_doubling_model(cfg, chi):
    """P:497 (R10): an iteration converges only if no chi_l grew AND max eps <= tau s. On these
    generic random-TT products every block is exactly interpolated (eps ~ 1e-16 s) from the first
    iteration on, so the rank clause alone decides: the oracle's iteration count, flag and final
    ranks must equal the closed-form rank-doubling model (configs[3]
    at chi = 64 saturates in half-sweep 6 and converges at iteration 4; at chi = 128 the rank 2 chi
    is first reached in half-sweep 7, so iteration 4 still grows and the run ends unconverged).
    Dropping the clause would report convergence at iteration 1."""
    cf = make_config(cfg, chi, npts=0)
    d = cf["inputs"][0].d
    it, conv, ranks = _generic_rank_model(d, _product_true_ranks(cf["inputs"]), cf["y_init"].ranks, cf["maxrank"],
                                          cf["max_sweeps"])
    res = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"])
    assert (res.report["iterations"], bool(res.report["converged"])) == (it, conv)
    assert [res.chi(b) for b in range(len(d) - 1)] == ranks
    L = len(d)
    first = res.log[:2 * (L - 1)]
    assert max(e["eps"] for e in first) <= cf["tol"] * first[-1]["scale"]  # eps alone would stop here
    if cfg == 3:
        assert (it, conv) == ((4, True) if chi == 64 else (4, False))


def test_aci_convergence_model_small_random_cases():
    """The same model on small random products (d in {2, 3}, rank caps that bind or not): equal
    iteration counts, flags and ranks. A binding cap (chi-hat < true rank) leaves eps > tau s, so
    those runs never converge."""
    rng = np.random.default_rng(497)
    for trial in range(12):
        L = int(rng.integers(4, 9))
        d = 3 if trial % 3 == 2 else 2
        xs = [G.random_tt(L, d, int(rng.integers(1, 5)), rng) for _ in range(2)]
        maxrank = int(rng.integers(3, 10)) if trial % 4 == 1 else 64
        y0 = G.random_init(xs, maxrank, rng)
        it, conv, ranks = _generic_rank_model(xs[0].d, _product_true_ranks(xs), y0.ranks, maxrank, 12)
        res = oracle.aci(xs, {"coef": [1.0], "expo": [[1, 1]]}, y0, 1e-10, maxrank, 12)
        assert (res.report["iterations"], bool(res.report["converged"])) == (it, conv), trial
        assert [res.chi(b) for b in range(L - 1)] == ranks, trial


def test_aci_rook_pivoting_reaches_the_exact_products():
    """ACI with rook pivoting in every prrLU (R23, NEXT-4): different pivots than full pivoting,
    the same accuracy bar — configs[0] against the dense 4096-vector product, configs[1] against
    the exact Kronecker product (Frobenius and samples)."""
    cf = make_config(0, npts=0)
    r = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"], pivoting="rook")
    f = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"])
    dense = oracle.tt_dense(cf["inputs"][0]) * oracle.tt_dense(cf["inputs"][1])
    assert _rel_max(oracle.tt_dense(r.cores), dense) <= 10 * cf["tol"]
    assert any(not np.array_equal(a["rows"], b["rows"]) for a, b in zip(r.log, f.log))
    cf = make_config(1, npts=20_000)
    r = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"], pivoting="rook")
    ex = oracle.exact_product(cf["inputs"], cf["op"])
    assert oracle.tt_norm(oracle.tt_axpby(1.0, r.cores, -1.0, ex)) / oracle.tt_norm(ex) <= 10 * cf["tol"]
    s = cf["samples"]
    assert _rel_max(oracle.tt_evaluate(r.cores, s), oracle.tt_evaluate(ex, s)) <= 10 * cf["tol"]


def test_aci_cfg4_rank_capped_last_update_matches_definition():
    """configs[4] is rank-capped (chi-hat = 256 < the true rank), so no exact product pins its
    output. Its last update (bond 0, right-to-left) is pinned against the definition instead: the
    block Pi[sigma, sigma', b] = f(x(sigma, sigma', J_2[b])) built by DIRECT evaluation of the input
    TTs at the final J_2 multi-indices (P:210-214 without frames), factorised by the (separately
    pinned) full-pivoting prrLU at the logged scale, gives exactly the logged ordered pivots and the
    final J_1 set; and the output interpolates f on that cross."""
    cf = make_config(4, npts=0)
    res = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], 1)
    last = res.log[-1]
    assert last["bond"] == 0 and last["dir"] == 1
    d = cf["inputs"][0].d
    J2 = res.Jset(2)
    pts = np.array([[s0, s1] + list(j) for s0 in range(d[0]) for s1 in range(d[1]) for j in J2], dtype=np.uint8)
    vals = [oracle.tt_evaluate(x, pts) for x in cf["inputs"]]
    f = sum(c * np.prod([vals[n] ** e for n, e in enumerate(ex)], axis=0)
            for c, ex in zip(cf["op"]["coef"], cf["op"]["expo"]))
    Pi = f.reshape(d[0], d[1] * len(J2))  # row sigma, column sigma' * |J_2| + b (Alg. 4)
    lu = oracle.ldu(Pi, cf["tol"] * last["scale"], cf["maxrank"])
    assert list(lu["rows"]) == list(last["rows"]) and list(lu["cols"]) == list(last["cols"])
    J1 = res.Jset(1)
    assert [tuple(r) for r in J1] == [tuple([c // len(J2)] + list(J2[c % len(J2)])) for c in lu["cols"]]
    I0 = res.Iset(0)
    cross = np.array([np.concatenate([i, j]) for i in I0 for j in J1], dtype=np.uint8)
    y = oracle.tt_evaluate(res.cores, cross)
    vals = [oracle.tt_evaluate(x, cross) for x in cf["inputs"]]
    ref = sum(c * np.prod([vals[n] ** e for n, e in enumerate(ex)], axis=0)
              for c, ex in zip(cf["op"]["coef"], cf["op"]["expo"]))
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()
