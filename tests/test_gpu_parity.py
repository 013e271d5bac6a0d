"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star):
  * configs[0]: identical ordered pivot lists for every update and the canonicalisation, and
    <= 10*tol against the dense 4096-vector product;
  * elsewhere: relative max error <= 10*tol on seeded random multi-indices and in the
    Frobenius norm where computable; pivot lists compared and reported (identical expected
    wherever no near-tie exists).
"""
import math

import numpy as np
import pytest

import oracle
from workloads import generators as G
from workloads import make_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aci():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2604_00037_b200 as aci
    aci.load()
    return aci


def _run_both(aci, cf, log=True, sweeps=None, index_sets=False):
    sweeps = sweeps or cf["max_sweeps"]
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    handles = xs
    if cf["cfg"] == 2:  # psi^3 with three aliased handles (deduplicated by the library)
        handles = [xs[0], xs[0], xs[0]]
        op = {"coef": [1.0], "expo": [[1, 1, 1]]}
    else:
        op = cf["op"]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    out, st, rep, ex = aci.aci_elementwise(op, handles, cf["tol"], cf["maxrank"], sweeps, y_init=y0, log=log,
                                           index_sets=index_sets)
    ref = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], sweeps)
    return out, st, rep, ex, ref


def _pivot_agreement(ex, ref):
    """Number of leading updates whose ordered pivot lists are identical."""
    k = 0
    for g, o in zip(ex["log"], ref.log):
        if g["bond"] != o["bond"] or g["dir"] != o["dir"] or g["r"] != o["r"]:
            break
        if not (np.array_equal(g["rows"], o["rows"]) and np.array_equal(g["cols"], o["cols"])):
            break
        k += 1
    return k


def _rel(y, r):
    return np.abs(y - r).max() / np.abs(r).max()


def _frob_rel(a, b):
    """||a - b||_F / ||b||_F for two TTs, by a QR sweep over the difference TT (no cancellation)."""
    return oracle.tt_norm(oracle.tt_axpby(1.0, a, -1.0, b)) / oracle.tt_norm(b)


def test_cfg0_identical_pivots_and_dense(aci):
    cf = make_config(0, npts=0)
    out, st, rep, ex, ref = _run_both(aci, cf, index_sets=True)
    assert len(ex["log"]) == len(ref.log)
    assert _pivot_agreement(ex, ref) == len(ref.log)
    for s in range(1, 12):
        assert np.array_equal(ex["canon_cols"][s], ref.canon_cols(s))
        assert np.array_equal(ex["J"][s], ref.Jset(s))
    for b in range(11):
        assert np.array_equal(ex["I"][b], ref.Iset(b))
    # eps is a residual after cancellation: compare it on the scale of s (roundoff of Pi ~ 1e-16 s)
    s_max = max(e["scale"] for e in ref.log)
    for g, o in zip(ex["log"], ref.log):
        assert abs(g["eps"] - o["eps"]) <= 1e-13 * s_max
        assert g["scale"] == pytest.approx(o["scale"], rel=1e-14)
    x = np.arange(4096) / 4096.0
    m0, m1 = cf["inputs"][0].meta, cf["inputs"][1].meta
    fa = sum(a * np.cos(2 * np.pi * k * x + p) for k, p, a in zip(m0["ks"], m0["phis"], m0["amps"]))
    fb = sum(a * np.cos(2 * np.pi * k * x + p) for k, p, a in zip(m1["ks"], m1["phis"], m1["amps"]))
    dense = oracle.tt_dense(out.cores())
    assert _rel(dense, fa * fb) <= 10 * cf["tol"]
    assert _rel(dense, oracle.tt_dense(ref.cores)) <= 10 * cf["tol"]
    assert rep["converged"] == ref.report["converged"] and rep["iterations"] == ref.report["iterations"]
    _, ranks = out.shape()
    assert ranks == ref.ranks


def test_cfg1_vs_oracle_and_exact(aci):
    cf = make_config(1, npts=100_000)
    out, st, rep, ex, ref = _run_both(aci, cf)
    s = cf["samples"]
    y = out.evaluate(s)
    yo = oracle.tt_evaluate(ref.cores, s)
    exact = oracle.tt_evaluate(cf["inputs"][0], s) * oracle.tt_evaluate(cf["inputs"][1], s)
    assert _rel(y, yo) <= 10 * cf["tol"]
    assert _rel(y, exact) <= 10 * cf["tol"]
    _, ranks = out.shape()
    assert max(ranks) <= 64
    ker = oracle.exact_product(cf["inputs"], cf["op"])
    frob = oracle.tt_norm(oracle.tt_axpby(1.0, out.cores(), -1.0, ker)) / oracle.tt_norm(ker)
    assert frob <= 10 * cf["tol"]
    assert _pivot_agreement(ex, ref) == len(ref.log)


@pytest.mark.parametrize("chi", [64, 128])
def test_cfg3_vs_oracle(aci, chi):
    """configs[3] at chi = 64 and 128 (two points of the metric's chi sweep, B:2, B:10): identical
    ordered pivots on every update, <= 10 tol on 10^5 seeded samples against the oracle and the
    exact product, Frobenius against the oracle's output."""
    cf = make_config(3, chi, npts=100_000)
    out, st, rep, ex, ref = _run_both(aci, cf)
    s = cf["samples"]
    y = out.evaluate(s)
    exact = oracle.tt_evaluate(cf["inputs"][0], s) * oracle.tt_evaluate(cf["inputs"][1], s)
    assert _rel(y, oracle.tt_evaluate(ref.cores, s)) <= 10 * cf["tol"]
    assert _rel(y, exact) <= 10 * cf["tol"]
    assert _frob_rel(out.cores(), ref.cores) <= 10 * cf["tol"]
    assert max(out.shape()[1]) == 2 * chi
    assert (rep["iterations"], rep["converged"]) == (ref.report["iterations"], ref.report["converged"])
    agree = _pivot_agreement(ex, ref)
    assert agree == len(ref.log), f"pivots identical for {agree}/{len(ref.log)} updates"


def test_evaluate_matches_oracle(aci):
    rng = np.random.default_rng(3)
    t = G.random_tt(9, 3, 37, rng)
    idx = G.sample_indices(t.d, 20000, rng)
    h = aci.TensorTrain.from_cores(t)
    assert _rel(h.evaluate(idx), oracle.tt_evaluate(t, idx)) <= 1e-13
    cores = h.cores()
    assert all(np.array_equal(a, b) for a, b in zip(cores, t.cores))


def test_identity_op_and_rank_one(aci):
    rng = np.random.default_rng(21)
    x = G.random_tt(10, 2, 8, rng)
    y0 = G.random_init([x], 8, rng)
    hx, hy = aci.TensorTrain.from_cores(x), aci.TensorTrain.from_cores(y0)
    out, st, rep, _ = aci.aci_elementwise({"coef": [1.0], "expo": [[1]]}, [hx], 1e-12, 64, 20, y_init=hy)
    assert rep["converged"] and rep["iterations"] <= 2
    assert _rel(oracle.tt_dense(out.cores()), oracle.tt_dense(x)) <= 1e-10
    a, b = G.random_tt(9, 2, 1, rng), G.random_tt(9, 2, 1, rng)
    ha, hb = aci.TensorTrain.from_cores(a), aci.TensorTrain.from_cores(b)
    out, st, rep, _ = aci.aci_elementwise({"coef": [1.0], "expo": [[1, 1]]}, [ha, hb], 1e-12, 16, 10, seed=5)
    assert max(out.shape()[1]) == 1
    assert _rel(oracle.tt_dense(out.cores()), oracle.tt_dense(a) * oracle.tt_dense(b)) <= 1e-13


def test_zero_function(aci):
    """f == 0 everywhere: every Pi is 0 -> rank 1, dummy pivots, zero output (R17)."""
    rng = np.random.default_rng(4)
    a = G.random_tt(6, 2, 3, rng)
    zero = G.TT([np.zeros_like(c) for c in a.cores])
    ha, hz = aci.TensorTrain.from_cores(a), aci.TensorTrain.from_cores(zero)
    y0 = aci.TensorTrain.from_cores(G.random_init([a], 8, rng))
    out, st, rep, ex = aci.aci_elementwise({"coef": [1.0], "expo": [[1, 1]]}, [ha, hz], 1e-10, 8, 3, y_init=y0,
                                           log=True)
    assert max(out.shape()[1]) == 1
    assert np.abs(oracle.tt_dense(out.cores())).max() == 0.0
    assert all(e["r"] == 1 and e["eps"] == 0.0 for e in ex["log"])


def test_small_random_suite_vs_oracle(aci):
    """SPEC acceptance suite shapes: identical pivots and dense agreement with the oracle,
    including d = 3 local dimensions, L = 2 and 3-input polynomials."""
    rng = np.random.default_rng(2024)
    ops = [({"coef": [1.0], "expo": [[1, 1]]}, 2), ({"coef": [1.0, 1.0], "expo": [[1, 0], [0, 1]]}, 2),
           ({"coef": [1.0, -0.5], "expo": [[1, 1, 0], [0, 0, 2]]}, 3)]
    for trial in range(18):
        L = int(rng.integers(2, 9))
        d = 3 if trial % 4 == 3 else 2
        op, N = ops[trial % 3]
        xs = [G.random_tt(L, d, int(rng.integers(1, 6)), rng) for _ in range(N)]
        y0 = G.random_init(xs, 64, rng)
        hs = [aci.TensorTrain.from_cores(x) for x in xs]
        out, st, rep, ex = aci.aci_elementwise(op, hs, 1e-10, 64, 8, y_init=aci.TensorTrain.from_cores(y0),
                                               log=True)
        ref = oracle.aci(xs, op, y0, 1e-10, 64, 8)
        assert _pivot_agreement(ex, ref) == len(ref.log), trial
        assert _rel(oracle.tt_dense(out.cores()), oracle.tt_dense(ref.cores)) <= 1e-9, trial


def test_errors(aci):
    rng = np.random.default_rng(9)
    a = aci.TensorTrain.from_cores(G.random_tt(5, 2, 2, rng))
    b = aci.TensorTrain.from_cores(G.random_tt(6, 2, 2, rng))
    with pytest.raises(aci.AciError) as e:
        aci.aci_elementwise({"coef": [1.0], "expo": [[1, 1]]}, [a, b], 1e-8, 8, 2)
    assert "SHAPE" in str(e.value)
    with pytest.raises(aci.AciError):
        aci.aci_elementwise({"coef": [1.0], "expo": [[1, 1]]}, [a, a], -1.0, 8, 2)
    bad = G.random_tt(5, 2, 2, rng)
    bad.cores[2][0, 0, 0] = np.nan
    with pytest.raises(aci.AciError) as e:
        aci.TensorTrain.from_cores(bad)
    assert "NONFINITE" in str(e.value)
    bt = G.random_tt(5, 2, 2, rng)
    bt.cores = [c * 1e3 for c in bt.cores]
    big = aci.TensorTrain.from_cores(bt)
    with pytest.raises(aci.AciError) as e:  # f overflows to inf
        aci.aci_elementwise({"coef": [1e308], "expo": [[4]]}, [big], 1e-8, 8, 2)
    assert "NONFINITE" in str(e.value)
    # L = 1 has no bond to update (oracle: ORC_ERR_INVALID as well)
    one = aci.TensorTrain.from_cores(G.random_tt(1, 4, 1, rng))
    with pytest.raises(aci.AciError) as e:
        aci.aci_elementwise({"coef": [1.0], "expo": [[2]]}, [one], 1e-8, 8, 2)
    assert "INVALID" in str(e.value)


def test_prrlu_envelope(aci):
    """Blocks beyond the register-resident prrLU envelope are refused up front (ACI_ERR_UNSUPPORTED,
    nothing launched): real 2-site blocks up to aci_limits() = 1024 rows x 1184 columns, complex
    up to 512 rows; a product at the limit runs."""
    rows, cols = aci.limits()
    assert (rows, cols) == (1024, 1184)
    rng = np.random.default_rng(12)
    # maxrank 1024 at d = 2: the middle blocks have 2048 rows
    x = aci.TensorTrain.from_cores(G.random_tt(24, 2, 600, rng))
    with pytest.raises(aci.AciError) as e:
        aci.aci_elementwise({"coef": [1.0], "expo": [[2]]}, [x], 1e-8, 1024, 1)
    assert "UNSUPPORTED" in str(e.value)
    # complex, maxrank 512 -> 1024-row blocks
    tz = G.random_tt(20, 2, 300, rng)
    z = aci.TensorTrain.from_cores([c + 0.5j * c for c in tz.cores])
    with pytest.raises(aci.AciError) as e:
        aci.aci_elementwise({"coef": [1.0], "expo": [[2]]}, [z], 1e-8, 512, 1)
    assert "UNSUPPORTED" in str(e.value)
    # complex at the limit (maxrank 256 -> 512-row blocks) runs
    zs = aci.TensorTrain.from_cores([c[:min(c.shape[0], 8), :, :min(c.shape[2], 8)] + 0.5j for c in tz.cores])
    out, st, rep, _ = aci.aci_elementwise({"coef": [1.0], "expo": [[2]]}, [zs], 1e-8, 256, 1)
    assert rep["max_rank"] <= 256


def _closed_psi(meta, s):
    w = 2 ** np.arange(9, -1, -1)
    xs = [(s[:, 10 * a:10 * a + 10].astype(np.int64) @ w) / 1024.0 for a in range(3)]
    ref = 0
    for c, sg, a in zip(meta["cs"], meta["sigmas"], meta["amps"]):
        g = [np.exp(-(t - c) ** 2 / (2 * sg ** 2)) for t in xs]
        ref = ref + a * g[0] * g[1] * g[2]
    return ref


def test_cfg2_psi_cubed(aci):
    """configs[2]: psi^3 with three aliased handles (merged into one input, exponent 3); the
    output matches the oracle and psi(x)^3 from the closed form within 10*tol on 10^5 samples."""
    cf = make_config(2, npts=100_000)
    out, st, rep, ex, ref = _run_both(aci, cf)
    s = cf["samples"]
    y = out.evaluate(s)
    assert _rel(y, oracle.tt_evaluate(ref.cores, s)) <= 10 * cf["tol"]
    assert _rel(y, _closed_psi(cf["inputs"][0].meta, s) ** 3) <= 10 * cf["tol"]
    assert _frob_rel(out.cores(), ref.cores) <= 10 * cf["tol"]
    agree = _pivot_agreement(ex, ref)
    assert agree == len(ref.log), f"pivots identical for {agree}/{len(ref.log)} updates"


@pytest.mark.slow
def test_cfg4_planewave_all_iterations(aci):
    """configs[4] (f = ab + a^2, d = 4, 1024 x 1024 blocks, rank cap 256) at all 8 iterations the
    bench runs (the oracle takes minutes): identical pivots on every update and agreement on 10^5
    samples and in the Frobenius norm. The exact-error floor of the rank-capped output is
    reported, not gated."""
    cf = make_config(4, npts=100_000)
    assert cf["max_sweeps"] == 8
    out, st, rep, ex, ref = _run_both(aci, cf)
    assert len(ex["log"]) == len(ref.log) == 8 * 2 * 19
    s = cf["samples"]
    y = out.evaluate(s)
    yo = oracle.tt_evaluate(ref.cores, s)
    agree = _pivot_agreement(ex, ref)
    assert agree == len(ref.log), f"pivots identical for {agree}/{len(ref.log)} updates"
    assert _rel(y, yo) <= 10 * cf["tol"]
    assert _frob_rel(out.cores(), ref.cores) <= 10 * cf["tol"]
    assert max(out.shape()[1]) == 256


def test_cfg3_chi256_full_size(aci):
    """configs[3] at chi = 256 in the bench's configuration (4 iterations, ranks reach 2 chi):
    GPU vs oracle on 10^5 sampled outputs and vs the exact Kronecker product (rank 512)."""
    cf = make_config(3, 256, npts=100_000)
    out, st, rep, ex, ref = _run_both(aci, cf)
    s = cf["samples"]
    y = out.evaluate(s)
    assert max(out.shape()[1]) == 512
    exact = oracle.tt_evaluate(cf["inputs"][0], s) * oracle.tt_evaluate(cf["inputs"][1], s)
    assert _rel(y, exact) <= 10 * cf["tol"]
    assert _rel(y, oracle.tt_evaluate(ref.cores, s)) <= 10 * cf["tol"]
    assert _frob_rel(out.cores(), ref.cores) <= 10 * cf["tol"]
    assert _frob_rel(out.cores(), oracle.exact_product(cf["inputs"], cf["op"])) <= 10 * cf["tol"]
    agree = _pivot_agreement(ex, ref)
    assert agree == len(ref.log), f"pivots identical for {agree}/{len(ref.log)} updates"


def test_absolute_tolerance_mode(aci):
    """ACI_TOL_ABSOLUTE (paper-literal tau) matches the oracle's absolute mode."""
    rng = np.random.default_rng(12)
    xs = [G.random_tt(8, 2, 4, rng), G.random_tt(8, 2, 3, rng)]
    y0 = G.random_init(xs, 32, rng)
    hs = [aci.TensorTrain.from_cores(x) for x in xs]
    out, st, rep, ex = aci.aci_elementwise({"coef": [1.0], "expo": [[1, 1]]}, hs, 1e-3, 32, 6,
                                           y_init=aci.TensorTrain.from_cores(y0), tol_mode=aci.TOL_ABSOLUTE,
                                           log=True)
    ref = oracle.aci(xs, {"coef": [1.0], "expo": [[1, 1]]}, y0, 1e-3, 32, 6, relative=False)
    assert _pivot_agreement(ex, ref) == len(ref.log)
    assert _rel(oracle.tt_dense(out.cores()), oracle.tt_dense(ref.cores)) <= 1e-12


def test_caller_workspace_and_stream(aci):
    """Device memory and the stream come from PyTorch (aci_workspace_query + a torch tensor as
    the workspace, a torch stream as the call's stream); results equal the default path."""
    import torch
    cf = make_config(1, npts=5000)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    nbytes = aci.workspace_query(xs, cf["maxrank"], y0)
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()
    out1, _, rep1, _ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                                           workspace=(ws.data_ptr(), nbytes), stream=st.cuda_stream)
    out2, _, rep2, _ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0)
    assert rep1["graph_iterations"] == rep1["iterations"]  # a non-default stream replays one CUDA graph
    c1, c2 = out1.cores(), out2.cores()
    assert all(np.array_equal(a, b) for a, b in zip(c1, c2))
    with pytest.raises(aci.AciError) as e:
        aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                            workspace=(ws.data_ptr(), nbytes // 2))
    assert "OOM" in str(e.value)


def test_concurrent_mode_matches_default_and_runs_in_threads(aci):
    """aci_options.concurrent: single-cluster prrLU launches give the same
    pivots and cores as the default tiers, and several products run concurrently on their own
    streams from host threads with results identical to the sequential runs."""
    import threading
    import torch
    cfgs = [make_config(3, 64, npts=0), make_config(1, npts=0), make_config(0, npts=0)]
    ref = []
    for cf in cfgs:
        xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
        y0 = aci.TensorTrain.from_cores(cf["y_init"])
        a, _, ra, ea = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0, log=True)
        b, _, rb, eb = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0, log=True,
                                           concurrent=True)
        assert len(ea["log"]) == len(eb["log"])
        for g, o in zip(ea["log"], eb["log"]):
            assert np.array_equal(g["rows"], o["rows"]) and np.array_equal(g["cols"], o["cols"])
        ca, cb = a.cores(), b.cores()
        assert all(np.array_equal(x, y) for x, y in zip(ca, cb))
        ref.append(ca)
    results = [None] * len(cfgs)

    def work(i):
        cf = cfgs[i]
        s = torch.cuda.Stream()
        xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
        y0 = aci.TensorTrain.from_cores(cf["y_init"])
        for _ in range(2):
            out, *_ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                                          stream=s.cuda_stream, concurrent=True)
        results[i] = out.cores()

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(cfgs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for r, c in zip(results, ref):
        assert all(np.array_equal(x, y) for x, y in zip(r, c))


_CONC256_SCRIPT = r"""
import sys, threading
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2604_00037_b200 as aci
from workloads import make_config
aci.load()
cf = make_config(3, 256, npts=0)
xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
y0 = aci.TensorTrain.from_cores(cf["y_init"])
ref, *_ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0)
ref = ref.cores()
out = [None] * 4
def work(i):
    s = torch.cuda.Stream()
    for _ in range(2):
        o, st, rep, _ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                                            stream=s.cuda_stream, concurrent=True)
    out[i] = o.cores()
th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
[t.start() for t in th]
[t.join() for t in th]
ok = all(r is not None and all(np.array_equal(a, b) for a, b in zip(r, ref)) for r in out)
print("OK" if ok else "MISMATCH")
"""


def test_concurrent_mode_at_chi256(aci):
    """NEXT-2 at the headline size: configs[3] chi = 256 (1024 x 1024 blocks) in concurrent mode
    from 4 host threads at once — blocks beyond one cluster use the cooperative (gang-scheduled) L2
    grid tier, so the products cannot deadlock; every output equals the sequential default run bit
    for bit. Run in a subprocess under a timeout (a hang fails the test, not the box)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _CONC256_SCRIPT], cwd=root, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), (r.stdout[-500:], r.stderr[-2000:])


_STREAM_SCRIPT = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2604_00037_b200 as aci
from workloads import make_config
aci.load()
for chi in (128, 256):
    cf = make_config(3, chi, npts=0)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                                           log=True)
    h = hashlib.sha256()
    for e in ex["log"]:
        h.update(np.asarray(e["rows"], np.int32).tobytes()); h.update(np.asarray(e["cols"], np.int32).tobytes())
    for c in out.cores():
        h.update(np.ascontiguousarray(c).tobytes())
    print(chi, rep["pivot_steps"], h.hexdigest())
"""


@pytest.mark.parametrize("minimum", ["0", "67108864"])
def test_streamed_pi_bitwise_equals_unstreamed(aci, minimum):
    """Streamed Pi: the Pi of L->R bond b+1 computed beside the prrLU of bond b from
    the pivot rows as they are published. Every pivot and every output core equals the unstreamed
    run bit for bit (configs[3] chi = 128, 256; ACI_STREAM_MIN=0 streams every eligible bond).
    Subprocesses: the switches are read once per process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ({"ACI_STREAM_PI": "0"}, {"ACI_STREAM_PI": "1", "ACI_STREAM_MIN": minimum}):
        r = subprocess.run([sys.executable, "-c", _STREAM_SCRIPT], cwd=root, capture_output=True, text=True,
                           timeout=600, env={**os.environ, **env})
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.split())
    assert outs[0] == outs[1]


def test_iteration_times_reported(aci):
    cf = make_config(3, 64, npts=0)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                                           iter_times=True)
    assert len(ex["iter_ms"]) == rep["iterations"]
    assert all(t > 0 for t in ex["iter_ms"]) and sum(ex["iter_ms"]) < rep["ms"]


def test_graph_cache_under_concurrent_eviction(aci):
    """More concurrent callers (own streams) than cached graphs: entries in use are never evicted
    (the cache holds 8); every thread's results equal the sequential run's."""
    import threading
    import torch
    cf = make_config(0, npts=0)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    ref, *_ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0)
    ref = ref.cores()
    n = 12
    # several rounds: new host threads reuse pooled stream handles (graph and workspace cache keys)
    # while others capture; outputs freed mid-run exercise tt_destroy beside running captures
    for _ in range(4):
        out = [None] * n

        def work(i):
            s = torch.cuda.Stream()
            for _ in range(3):
                o, *_ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                                            stream=s.cuda_stream, concurrent=True)
            out[i] = o.cores()

        th = [threading.Thread(target=work, args=(i,)) for i in range(n)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for r in out:
            assert r is not None and all(np.array_equal(x, y) for x, y in zip(r, ref))


def test_warm_start_from_previous_output(aci):
    """Repeated products (time stepping): passing the previous output
    as y_init warm-starts the index sets, so the second product converges in at most 2
    iterations with the same accuracy."""
    cf = make_config(1, npts=20_000)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    first, st1, r1, _ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0)
    second, st2, r2, _ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=first)
    assert r2["converged"] and r2["iterations"] <= 2 < r1["iterations"]
    s = cf["samples"]
    exact = oracle.tt_evaluate(cf["inputs"][0], s) * oracle.tt_evaluate(cf["inputs"][1], s)
    assert _rel(second.evaluate(s), exact) <= 10 * cf["tol"]


def test_c_example_runs(aci):
    """The plain-C example (no Python on the compute path) checks its own result."""
    import subprocess
    from paper_2604_00037_b200 import _build
    exe = _build.build_example()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "rel max error" in r.stdout


def test_edge_shapes_vs_oracle(aci):
    """Edge cases: maxrank 1 (every bond rank 1), mixed local dimensions including d = 1 sites,
    four distinct inputs with an eight-term polynomial (the op limits of aci.h), and the same in
    complex arithmetic; identical pivots (or roundoff ties for complex) and dense agreement."""
    rng = np.random.default_rng(77)
    # maxrank 1
    xs = [G.random_tt(7, 2, 3, rng) for _ in range(2)]
    y0 = G.random_init(xs, 1, rng)
    op = {"coef": [1.0], "expo": [[1, 1]]}
    out, st, rep, ex = aci.aci_elementwise(op, [aci.TensorTrain.from_cores(x) for x in xs], 1e-12, 1, 4,
                                           y_init=aci.TensorTrain.from_cores(y0), log=True)
    ref = oracle.aci(xs, op, y0, 1e-12, 1, 4)
    assert max(out.shape()[1]) == 1 and _pivot_agreement(ex, ref) == len(ref.log)
    assert _rel(oracle.tt_dense(out.cores()), oracle.tt_dense(ref.cores)) <= 1e-12
    # mixed d (1, 3, 2, ...) and four inputs, eight terms
    dims = [2, 1, 3, 2, 1, 2]
    def rtt(chi):
        ranks = [1] + [chi] * (len(dims) - 1) + [1]
        return [rng.standard_normal((ranks[s], dims[s], ranks[s + 1])) / np.sqrt(chi * dims[s]) for s in range(len(dims))]
    xs = [rtt(int(c)) for c in (2, 3, 2, 1)]
    op = {"coef": [1.0, -0.5, 0.25, 2.0, -1.0, 0.5, 1.5, -0.75],
          "expo": [[1, 1, 0, 0], [0, 0, 1, 1], [2, 0, 0, 0], [0, 2, 0, 0], [0, 0, 2, 0], [1, 0, 0, 1],
                   [0, 1, 1, 0], [1, 1, 1, 1]]}
    from workloads import TT
    # y_init at the full-tensor bond bounds: the rank-1 input would otherwise make the R9
    # initial guess rank 1, which the d = 1 sites keep from growing (a legitimate ACI stall)
    full = [1] + [min(int(np.prod(dims[:s])), int(np.prod(dims[s:]))) for s in range(1, len(dims))] + [1]
    y0 = TT([rng.standard_normal((full[s], dims[s], full[s + 1])) for s in range(len(dims))])
    out, st, rep, ex = aci.aci_elementwise(op, [aci.TensorTrain.from_cores(x) for x in xs], 1e-12, 64, 6,
                                           y_init=aci.TensorTrain.from_cores(y0), log=True)
    ref = oracle.aci(xs, op, y0, 1e-12, 64, 6)
    assert _pivot_agreement(ex, ref) == len(ref.log)
    D = [oracle.tt_dense(x) for x in xs]
    exact = sum(c * np.prod([D[n] ** e for n, e in enumerate(ex_)], axis=0) for c, ex_ in zip(op["coef"], op["expo"]))
    assert _rel(oracle.tt_dense(out.cores()), exact) <= 1e-10
    # the same four inputs made complex
    xz = [[c + 1j * rng.standard_normal(c.shape) / 3 for c in x] for x in xs]
    yz = [c + 1j * rng.standard_normal(c.shape) for c in y0.cores]
    outz, st, rep, exz = aci.aci_elementwise(op, [aci.TensorTrain.from_cores(x) for x in xz], 1e-12, 64, 6,
                                             y_init=aci.TensorTrain.from_cores(yz), log=True)
    Dz = [oracle.tt_dense(x) for x in xz]
    exactz = sum(c * np.prod([Dz[n] ** e for n, e in enumerate(ex_)], axis=0) for c, ex_ in zip(op["coef"], op["expo"]))
    assert _rel(oracle.tt_dense(outz.cores()), exactz) <= 1e-10


_TIER_SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2604_00037_b200 as aci
from workloads import make_config
aci.load()
cf = make_config(int(sys.argv[1]), int(sys.argv[2]), npts=0)
xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
y0 = aci.TensorTrain.from_cores(cf["y_init"])
out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0, log=True)
h = hashlib.sha256()
for e in ex["log"]:
    h.update(np.asarray(e["rows"], np.int32).tobytes()); h.update(np.asarray(e["cols"], np.int32).tobytes())
print(h.hexdigest(), len(ex["log"]))
"""


@pytest.mark.parametrize("cfg,chi", [(3, 64), (1, 32), (3, 256)])
def test_prrlu_tiers_identical_pivots(aci, cfg, chi):
    """Every prrLU tier takes the same decisions (same keys, tie-break and arithmetic, R3/R4):
    the default tiers, the L2 grid tier (no clusters), 8-CTA clusters, no push tier, and direct
    launches instead of the CUDA graph give bit-identical pivot logs (subprocesses: the switches
    are read once per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = {}
    for name, env in [("default", {}), ("l2_grid", {"ACI_PRRLU_CLUSTER": "0"}), ("cluster8", {"ACI_PRRLU_CLUSTER": "8"}),
                      ("no_push", {"ACI_PRRLU_PUSH": "0"}), ("no_graph", {"ACI_NO_GRAPH": "1"})]:
        r = subprocess.run([sys.executable, "-c", _TIER_SCRIPT, str(cfg), str(chi)], cwd=root, capture_output=True,
                           text=True, timeout=300, env={**os.environ, **env})
        assert r.returncode == 0, (name, r.stderr[-2000:])
        runs[name] = r.stdout.split()
    assert len({tuple(v) for v in runs.values()}) == 1, runs


def test_batch_api_matches_single_products(aci):
    """aci_elementwise_batch (NEXT-2): several independent products on library threads/streams give
    bitwise the outputs and reports of the same products run one by one; a failing job reports its
    own status while the others complete."""
    jobs, refs = [], []
    for cfg, chi in [(0, None), (1, None), (3, 64), (0, None), (1, None), (3, 64)]:
        cf = make_config(cfg, chi, npts=0) if chi else make_config(cfg, npts=0)
        xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
        y0 = aci.TensorTrain.from_cores(cf["y_init"])
        jobs.append({"op": cf["op"], "inputs": xs, "tol": cf["tol"], "maxrank": cf["maxrank"],
                     "max_sweeps": cf["max_sweeps"], "y_init": y0})
        refs.append(aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0))
    res = aci.aci_elementwise_batch(jobs, max_parallel=4)
    for (tt, st, rep), (rtt, rst, rrep, _) in zip(res, refs):
        assert st == rst and rep["pivot_steps"] == rrep["pivot_steps"] and rep["iterations"] == rrep["iterations"]
        assert all(np.array_equal(a, b) for a, b in zip(tt.cores(), rtt.cores()))
    bad = dict(jobs[0], tol=-1.0)
    with pytest.raises(aci.AciError):
        aci.aci_elementwise_batch([jobs[0], bad])


def test_concurrent_and_batch_paths_match_oracle_pivots(aci):
    """The concurrent path (aci_options.concurrent, single-cluster prrLU tiers) and the batch API
    compared with the ORACLE itself: identical ordered pivot lists on every update, and outputs
    within 10 tol of the oracle's, for configs[3] chi = 64 and configs[1]."""
    cfgs = [make_config(3, 64, npts=20_000), make_config(1, npts=20_000)]
    refs = [oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"]) for cf in cfgs]
    jobs = []
    for cf, ref in zip(cfgs, refs):
        xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
        y0 = aci.TensorTrain.from_cores(cf["y_init"])
        out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                                               log=True, concurrent=True)
        assert _pivot_agreement(ex, ref) == len(ref.log) == len(ex["log"])
        s = cf["samples"]
        assert _rel(out.evaluate(s), oracle.tt_evaluate(ref.cores, s)) <= 10 * cf["tol"]
        jobs.append({"op": cf["op"], "inputs": xs, "tol": cf["tol"], "maxrank": cf["maxrank"],
                     "max_sweeps": cf["max_sweeps"], "y_init": y0, "log": True})
    res = aci.aci_elementwise_batch(jobs + jobs, max_parallel=4)
    for i, (tt, st, rep, ex) in enumerate(res):
        cf, ref = cfgs[i % 2], refs[i % 2]
        assert _pivot_agreement(ex, ref) == len(ref.log) == len(ex["log"]), i
        assert _rel(tt.evaluate(cf["samples"]), oracle.tt_evaluate(ref.cores, cf["samples"])) <= 10 * cf["tol"]


def test_constant_term_op_vs_oracle(aci):
    """f = 1 - a^2 b^2 (a constant term): every real entry of Pi is < 1, while padded
    tile lanes of the Pi epilogue hold f(0) = 1, which must not enter s = max |Pi| (R1) —
    identical pivots and scale to the oracle's."""
    rng = np.random.default_rng(31)
    for L, chi in [(9, 3), (12, 6)]:
        xs = [G.random_tt(L, 2, chi, rng), G.random_tt(L, 2, 2, rng)]
        op = {"coef": [1.0, -1.0], "expo": [[0, 0], [2, 2]]}
        y0 = G.random_init(xs, 64, rng)
        hs = [aci.TensorTrain.from_cores(x) for x in xs]
        out, st, rep, ex = aci.aci_elementwise(op, hs, 1e-10, 64, 10, y_init=aci.TensorTrain.from_cores(y0), log=True)
        ref = oracle.aci(xs, op, y0, 1e-10, 64, 10)
        assert _pivot_agreement(ex, ref) == len(ref.log)
        for g, o in zip(ex["log"], ref.log):
            assert g["scale"] == pytest.approx(o["scale"], rel=1e-14)
        D = [oracle.tt_dense(x) for x in xs]
        assert _rel(oracle.tt_dense(out.cores()), 1.0 - D[0] ** 2 * D[1] ** 2) <= 1e-9


def test_workspace_alignment_and_query_sweeps(aci):
    """A caller workspace must be 256-byte aligned (ACI_ERR_INVALID otherwise); aci_workspace_query
    sizes the pivot log for the max_sweeps it is given."""
    import torch
    cf = make_config(0, npts=0)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    n20 = aci.workspace_query(xs, cf["maxrank"], y0, max_sweeps=20)
    n80 = aci.workspace_query(xs, cf["maxrank"], y0, max_sweeps=80)
    assert n80 > n20
    ws = torch.empty(n80 + 512, dtype=torch.uint8, device="cuda")
    with pytest.raises(aci.AciError) as e:
        aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], 20, y_init=y0, workspace=(ws.data_ptr() + 8, n80))
    assert "INVALID" in str(e.value)
    out, st, rep, _ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], 20, y_init=y0,
                                          workspace=(ws.data_ptr(), n20))
    ref, *_ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], 20, y_init=y0)
    assert all(np.array_equal(a, b) for a, b in zip(out.cores(), ref.cores()))


@pytest.mark.parametrize("cfg,chi", [(0, 0), (1, 0), (3, 64), (3, 128)])
def test_rook_pivoting_vs_rook_oracle(aci, cfg, chi):
    """Rook pivoting (aci_options.pivoting = ACI_PIVOT_ROOK; R23) against the
    oracle's rook mode on the same seeded inputs: identical ordered pivots on every update (and the
    canonicalisation), equal iteration counts, and <= 10 tol against the oracle and the exact
    product on seeded samples."""
    cf = make_config(cfg, chi, npts=20_000) if chi else make_config(cfg, npts=20_000)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                                           log=True, pivoting="rook")
    ref = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"], pivoting="rook")
    L = len(cf["inputs"][0].d)
    for s_ in range(1, L):
        assert np.array_equal(ex["canon_cols"][s_], ref.canon_cols(s_))
    assert len(ex["log"]) == len(ref.log)
    assert _pivot_agreement(ex, ref) == len(ref.log)
    assert (rep["iterations"], rep["converged"]) == (ref.report["iterations"], ref.report["converged"])
    s = cf["samples"]
    y = out.evaluate(s)
    assert _rel(y, oracle.tt_evaluate(ref.cores, s)) <= 10 * cf["tol"]
    exact = oracle.tt_evaluate(cf["inputs"][0], s) * oracle.tt_evaluate(cf["inputs"][1], s)
    assert _rel(y, exact) <= 10 * cf["tol"]


def test_rook_pivoting_envelope(aci):
    """Rook mode runs where the factorisation fits one CTA or one 16-CTA cluster (<= 512 rows) and
    on real values; beyond that ACI_ERR_UNSUPPORTED, nothing launched."""
    cf = make_config(3, 256, npts=0)  # 1024 x 1024 blocks
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    with pytest.raises(aci.AciError) as e:
        aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], 1, pivoting="rook")
    assert e.value.code == -6
    rng = np.random.default_rng(5)
    z = aci.TensorTrain.from_cores([c + 0.5j * c for c in G.random_tt(8, 2, 3, rng).cores])
    with pytest.raises(aci.AciError) as e:
        aci.aci_elementwise({"coef": [1.0], "expo": [[2]]}, [z], 1e-8, 16, 2, pivoting="rook")
    assert e.value.code == -6


def test_peak_and_latency_probes(aci):
    """bench.py's roofline denominators (libaci_peak.so): the FP64 DMMA / DFMA loops land within a
    plausible band of the B200's nominal ~37 TF/s, and the prrLU latency probe returns, per block
    size, the pivot count of a full factorisation and an exchange-only floor below the real kernel."""
    import ctypes
    from paper_2604_00037_b200 import _build
    lib = ctypes.CDLL(_build.build_peak())
    lib.aci_peak_fp64.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    for kind in (0, 1):
        v = ctypes.c_double(0.0)
        assert lib.aci_peak_fp64(kind, 3, ctypes.byref(v)) == 0
        assert 20.0 < v.value < 45.0, (kind, v.value)
    import bench
    lat = bench.measure_prrlu_latency((64, 256, 1024))
    for m, row in lat.items():
        assert row["pivots"] == min(m, 512)
        assert 0.0 < row["floor_us"] < row["kernel_us"] < 20.0, (m, row)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,r,static", [
    (512, 1024, 512, (1024, 1024)),   # two clusters -> one at pivot 256 (hand-off pair 1)
    (400, 1000, 400, (1024, 1024)),   # pair 1, K = 232
    (512, 256, 256, (1024, 1024)),    # one cluster, 16x2 -> 12x1 at pivot 128 (pair 2)
    (450, 250, 250, (1024, 1024)),    # pair 2, K = 122 rounded to 124 (prrlu.cu ho_round)
    (300, 130, 130, (512, 256)),      # pair 2, K = 2 rounded to 4
    (1024, 1024, 512, (1024, 1024)),  # four clusters, no hand-off
    (128, 64, 64, (1024, 1024)),      # a one-CTA shape run on the cluster (CTA_MAXE)
    (200, 250, 200, (256, 256)),
])
def test_prrlu_step_vs_oracle(aci, m, n, r, static):
    """a5 alone through the C-ABI (aci_prrlu) against the oracle's Alg. 2 on the same seeded block:
    the ordered pivots identical, U = S_k[p, :] / c equal to rounding (the same FMA sequence, R4),
    including the blocks whose factorisation hands off to one cluster mid-way and
    the U entries of columns eliminated before the hand-off."""
    rng = np.random.default_rng(1000 + m + 7 * n)
    M = rng.standard_normal((m, n))
    g = aci.prrlu(M, r, 0.0, relative=False, static=static)
    o = oracle.ldu(M, 0.0, r)
    assert g["r"] == o["r"] == min(r, m, n)
    assert np.array_equal(g["rows"], o["rows"]) and np.array_equal(g["cols"], o["cols"])
    assert np.max(np.abs(g["U"] - o["U"])) <= 1e-13 * np.max(np.abs(o["U"]))
    # eliminated columns of each U row are exact zeros, the pivot column exactly 1
    for k in range(g["r"]):
        assert g["U"][k, g["cols"][k]] == 1.0
        assert np.all(g["U"][k, g["cols"][:k]] == 0.0)


@pytest.mark.gpu
def test_prrlu_step_relative_stop_rule(aci):
    """aci_prrlu with a relative tolerance stops where the oracle does (R2: the first candidate with
    |c| <= tol * |first candidate| is rejected and reported as eps) on a numerically rank-40 block."""
    rng = np.random.default_rng(77)
    M = rng.standard_normal((300, 40)) @ rng.standard_normal((40, 500)) + 1e-12 * rng.standard_normal((300, 500))
    g = aci.prrlu(M, 300, 1e-9, relative=True, static=(512, 1024))
    o = oracle.ldu(M, 1e-9, 300, relative_to_own_max=True)
    assert g["r"] == o["r"] == 40
    assert np.array_equal(g["rows"], o["rows"]) and np.array_equal(g["cols"], o["cols"])
    assert g["eps"] == o["eps"]
