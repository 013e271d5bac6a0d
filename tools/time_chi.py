"""Time repeated configs[3] products (development helper): per-run library ms for each chi."""
import sys
sys.path.insert(0, ".")
import paper_2604_00037_b200 as aci  # noqa: E402
from workloads import make_config  # noqa: E402

chis = [int(c) for c in sys.argv[1].split(",")] if len(sys.argv) > 1 else [64, 128, 256]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
for chi in chis:
    cf = make_config(3, chi, npts=0)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    ms = []
    for _ in range(reps):
        out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0)
        out.free()
        ms.append(rep["ms"])
    print(f"chi={chi}: " + " ".join(f"{m:.1f}" for m in ms) + f" | pivots {rep['pivot_steps']}", flush=True)
    out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                                           profile=True)
    out.free()
    print("   profile (ms, launches):", {k: (round(v["ms"], 2), v["launches"]) for k, v in ex["profile"].items()},
          flush=True)
