"""GPU parity for complex values (f: C^N -> C; §8(f) NEXT-1): the CUDA path through the
C-ABI (tt_create_z, aci_elementwise on complex handles, tt_evaluate) against the complex oracle
(oracle/aci_oracle_z.c, readings RZ1-RZ6) on the same seeded inputs.

Bars: identical ordered pivot lists (the prrLU arithmetic RZ1-RZ4 is the oracle's, so equal Pi
gives equal pivots barring near-ties of roundoff size), and <= 10*tol relative error against the
closed-form product of the paper's random Fourier series on seeded random points.
"""
import numpy as np
import pytest

import oracle
from workloads import TT, make_config, random_init, random_tt
from workloads.generators import _rng

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aci():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2604_00037_b200 as aci
    aci.load()
    return aci


def _fourier_values(tt, samples):
    x = (samples * (2.0 ** -np.arange(1, samples.shape[1] + 1))).sum(axis=1)
    c = tt.meta["coefs"]
    return np.exp(1j * np.outer(x, np.arange(len(c)))) @ c


def _complex_tt(L, d, chi, seed):
    a = random_tt(L, d, chi, _rng(seed, 0))
    b = random_tt(L, d, chi, _rng(seed, 1))
    return TT([x + 1j * y for x, y in zip(a.cores, b.cores)])


def _identical(ex, ref):
    same = 0
    for g, o in zip(ex["log"], ref.log):
        if g["r"] == o["r"] and np.array_equal(g["rows"], o["rows"]) and np.array_equal(g["cols"], o["cols"]):
            same += 1
    return same


NEAR_TIE = 1e-9  # relative |z|^2 gap below which Pi's roundoff (~1e-16 s) may reorder candidates


def _pivots_identical_or_tie(ex, ref):
    """Ordered pivot lists identical for every update, up to the first update whose decision the
    oracle took between candidates tied within roundoff (gap < NEAR_TIE at or before the first
    differing step); after such a tie the index sets legitimately differ. Returns the number of
    updates compared identical."""
    for u, (g, o) in enumerate(zip(ex["log"], ref.log)):
        assert g["bond"] == o["bond"] and g["dir"] == o["dir"]
        if g["r"] == o["r"] and np.array_equal(g["rows"], o["rows"]) and np.array_equal(g["cols"], o["cols"]):
            continue
        k = next((i for i in range(min(g["r"], o["r"])) if g["rows"][i] != o["rows"][i] or g["cols"][i] != o["cols"][i]),
                 min(g["r"], o["r"]))
        assert o["gap"][:k + 1].min() < NEAR_TIE, f"update {u}: pivots differ at step {k} without a near-tie"
        return u
    return len(ref.log)


def test_complex_tt_roundtrip_and_evaluate(aci):
    x = _complex_tt(9, 3, 5, 71)
    t = aci.TensorTrain.from_cores(x.cores)
    assert t.is_complex
    for a, b in zip(t.cores(), x.cores):
        assert np.array_equal(a, b)
    idx = np.random.default_rng(0).integers(0, 3, size=(3000, 9)).astype(np.uint8)
    ref = oracle.tt_evaluate(x.cores, idx)
    got = t.evaluate(idx)
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("K", [100, 1000])
def test_fourier_product_identical_pivots_and_tolerance(aci, K):
    cf = make_config(5, K, npts=20000)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                                           log=True)
    ref = oracle.aci_z(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"])
    assert out.is_complex
    for s in range(1, 30):
        assert np.array_equal(ex["canon_cols"][s], ref.canon_cols(s))
    agree = _pivots_identical_or_tie(ex, ref)
    assert agree >= 20, agree
    exact = _fourier_values(cf["inputs"][0], cf["samples"]) * _fourier_values(cf["inputs"][1], cf["samples"])
    y = out.evaluate(cf["samples"])
    assert np.abs(y - exact).max() <= 10 * cf["tol"] * np.abs(exact).max()
    yo = oracle.tt_evaluate(ref.cores, cf["samples"])
    assert np.abs(y - yo).max() <= 10 * cf["tol"] * np.abs(yo).max()
    frob = oracle.tt_norm(oracle.tt_axpby(1.0, out.cores(), -1.0, ref.cores)) / oracle.tt_norm(ref.cores)
    assert frob <= 10 * cf["tol"]
    if agree == len(ref.log):
        assert rep["iterations"] == ref.report["iterations"]
        assert abs(rep["flops_contraction"] - ref.report["flops_contraction"]) <= 1e-9 * ref.report["flops_contraction"]


def test_complex_polynomial_three_inputs_d3(aci):
    """x1 x2 + x3^2 - 0.5 x1 on random complex TTs with d = 3 (SPEC-shaped): identical
    pivots and agreement with the dense product."""
    L = 7
    ins = [_complex_tt(L, 3, 3, 80 + i) for i in range(3)]
    op = {"coef": [1.0, 1.0, -0.5], "expo": [[1, 1, 0], [0, 0, 2], [1, 0, 0]]}
    y0 = random_init(ins, 32, _rng(83, 2))
    xs = [aci.TensorTrain.from_cores(t.cores) for t in ins]
    out, st, rep, ex = aci.aci_elementwise(op, xs, 1e-12, 32, 6, y_init=aci.TensorTrain.from_cores(y0.cores),
                                           log=True)
    ref = oracle.aci_z(ins, op, y0, 1e-12, 32, 6)
    assert _pivots_identical_or_tie(ex, ref) == len(ref.log)
    D = [oracle.tt_dense(t.cores) for t in ins]
    exact = D[0] * D[1] + D[2] ** 2 - 0.5 * D[0]
    got = oracle.tt_dense(out.cores())
    assert np.abs(got - exact).max() <= 1e-10 * np.abs(exact).max()


def test_complex_run_on_real_data_matches_real_run(aci):
    """configs[0] cast to complex: the complex kernels must reproduce the real path's values."""
    cf = make_config(0, npts=4000)
    xr = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    xz = [aci.TensorTrain.from_cores([c.astype(np.complex128) for c in t.cores]) for t in cf["inputs"]]
    yr = aci.TensorTrain.from_cores(cf["y_init"])
    yz = aci.TensorTrain.from_cores([c.astype(np.complex128) for c in cf["y_init"].cores])
    a, *_ = aci.aci_elementwise(cf["op"], xr, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=yr)
    b, *_ = aci.aci_elementwise(cf["op"], xz, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=yz)
    va, vb = a.evaluate(cf["samples"]), b.evaluate(cf["samples"])
    assert np.abs(vb.imag).max() == 0.0
    assert np.abs(va - vb.real).max() <= 10 * cf["tol"] * np.abs(va).max()


def test_complex_identity_and_mixed_dtype_error(aci):
    x = _complex_tt(10, 2, 4, 91)
    xs = [aci.TensorTrain.from_cores(x.cores)]
    out, st, rep, _ = aci.aci_elementwise({"coef": [1.0], "expo": [[1]]}, xs, 1e-12, 8, 4)
    assert rep["iterations"] <= 2
    D = oracle.tt_dense(x.cores)
    assert np.abs(oracle.tt_dense(out.cores()) - D).max() <= 1e-12 * np.abs(D).max()
    r = aci.TensorTrain.from_cores(random_tt(10, 2, 4, _rng(92, 0)).cores)
    with pytest.raises(aci.AciError):
        aci.aci_elementwise({"coef": [1.0], "expo": [[1, 1]]}, [xs[0], r], 1e-12, 8, 4)


def test_complex_concurrent_mode_and_zero_op(aci):
    """Single-cluster mode (aci_options.concurrent) on complex data gives the default path's
    pivots and cores; f == 0 gives the R17 rank-1 zero output."""
    cf = make_config(5, 1000, npts=0)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    cap = 128  # complex single-cluster blocks are limited to 256 x 512 (aci.h)
    a, _, _, ea = aci.aci_elementwise(cf["op"], xs, cf["tol"], cap, cf["max_sweeps"], y_init=y0, log=True)
    b, _, _, eb = aci.aci_elementwise(cf["op"], xs, cf["tol"], cap, cf["max_sweeps"], y_init=y0, log=True,
                                      concurrent=True)
    for g, o in zip(ea["log"], eb["log"]):
        assert np.array_equal(g["rows"], o["rows"]) and np.array_equal(g["cols"], o["cols"])
    assert all(np.array_equal(x, y) for x, y in zip(a.cores(), b.cores()))
    z, st, rep, _ = aci.aci_elementwise({"coef": [0.0], "expo": [[1, 1]]}, xs, 1e-10, 16, 2, y_init=y0)
    _, ranks = z.shape()
    assert max(ranks) == 1
    assert np.abs(z.cores()[0]).max() == 0.0  # Y_0 = Pi[:, J] = 0; the other cores are U rows e_q (R17)
    idx = np.random.default_rng(1).integers(0, 2, size=(1000, 30)).astype(np.uint8)
    assert np.abs(z.evaluate(idx)).max() == 0.0


def test_complex_absolute_tolerance_mode(aci):
    """Paper-literal absolute tau (tol_mode = ACI_TOL_ABSOLUTE) on complex data: identical
    pivots to the oracle's absolute mode and max-norm error within 10 tau on samples."""
    cf = make_config(5, 100, npts=5000)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    tau = 1e-6
    out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, tau, cf["maxrank"], cf["max_sweeps"], y_init=y0, log=True,
                                           tol_mode=aci.TOL_ABSOLUTE)
    ref = oracle.aci_z(cf["inputs"], cf["op"], cf["y_init"], tau, cf["maxrank"], cf["max_sweeps"], relative=False)
    assert _pivots_identical_or_tie(ex, ref) >= 20
    exact = _fourier_values(cf["inputs"][0], cf["samples"]) * _fourier_values(cf["inputs"][1], cf["samples"])
    assert np.abs(out.evaluate(cf["samples"]) - exact).max() <= 10 * tau


def test_complex_cluster_tiers_vs_oracle(aci):
    """Complex blocks large enough for the multi-CTA complex prrLU tiers (up to 384 live rows in
    512-row static blocks): pivots identical to the complex oracle (or diverging only at a
    roundoff-level tie), and the output equal to the exact product within 10 tol."""
    L, tol = 16, 1e-10
    a = _complex_tt(L, 2, 48, 301)
    b = _complex_tt(L, 2, 4, 302)
    y0 = random_init([a, b], 256, _rng(303, 2))
    op = {"coef": [1.0], "expo": [[1, 1]]}
    out, st, rep, ex = aci.aci_elementwise(op, [aci.TensorTrain.from_cores(a), aci.TensorTrain.from_cores(b)], tol,
                                           256, 4, y_init=aci.TensorTrain.from_cores(y0), log=True)
    assert max(out.shape()[1]) > 128  # the grid tiers were used
    ref = oracle.aci_z([a, b], op, y0, tol, 256, 4)
    _pivots_identical_or_tie(ex, ref)  # any divergence only at a roundoff-level tie
    exact = oracle.tt_dense(a) * oracle.tt_dense(b)
    assert np.abs(oracle.tt_dense(out.cores()) - exact).max() <= 10 * tol * np.abs(exact).max()
