"""Quick GPU-vs-oracle diagnostic (development tool): per config, pivot agreement, errors, timing."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2604_00037_b200 as aci  # noqa: E402
from workloads import make_config  # noqa: E402


def run(cfg, chi=0, sweeps=None, with_oracle=True):
    cf = make_config(cfg, chi, npts=5000)
    sweeps = sweeps or cf["max_sweeps"]
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    t = time.time()
    out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], sweeps, y_init=y0, log=True)
    t1 = time.time() - t
    t = time.time()
    out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], sweeps, y_init=y0, log=True)
    t2 = time.time() - t
    s = cf["samples"]
    y = out.evaluate(s)
    vals = [oracle.tt_evaluate(x, s) for x in cf["inputs"]]
    exact = np.zeros(len(s))
    for c, e in zip(cf["op"]["coef"], cf["op"]["expo"]):
        term = c * np.ones(len(s))
        for n, k in enumerate(e):
            term = term * vals[n] ** k
        exact += term
    msg = (f"{cf['name']}: status {st} iters {rep['iterations']} conv {rep['converged']} maxrank {rep['max_rank']} "
           f"pivots {rep['pivot_steps']} t_first {t1*1e3:.1f} ms t {t2*1e3:.1f} ms (lib {rep['ms']:.1f}) "
           f"err_vs_exact {np.abs(y-exact).max()/np.abs(exact).max():.2e}")
    if with_oracle:
        t = time.time()
        ref = oracle.aci(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], sweeps)
        to = time.time() - t
        agree = 0
        first_bad = None
        for g, o in zip(ex["log"], ref.log):
            same = g["r"] == o["r"] and np.array_equal(g["rows"], o["rows"]) and np.array_equal(g["cols"], o["cols"])
            if same:
                agree += 1
            elif first_bad is None:
                first_bad = (g["bond"], g["dir"], g["r"], o["r"])
        yo = oracle.tt_evaluate(ref.cores, s)
        msg += (f" | oracle {to:.1f}s, pivots identical {agree}/{len(ref.log)} first_bad {first_bad} "
                f"gpu-vs-oracle {np.abs(y-yo).max()/np.abs(yo).max():.2e}")
    print(msg, flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "small"
    if which == "small":
        run(0)
        run(1)
        run(3, 64)
    elif which == "big":
        run(3, 128, with_oracle=False)
        run(3, 256, with_oracle=False)
        run(2, with_oracle=False)
        run(4, with_oracle=False, sweeps=4)
