"""Complex path diagnostics (development tool): first differing pivot per update vs the oracle."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import oracle  # noqa: E402
import paper_2604_00037_b200 as aci  # noqa: E402
from workloads import make_config  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 100
cf = make_config(5, K, npts=0)
xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
y0 = aci.TensorTrain.from_cores(cf["y_init"])
out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0, log=True)
ref = oracle.aci_z(cf["inputs"], cf["op"], cf["y_init"], cf["tol"], cf["maxrank"], cf["max_sweeps"])
print("iters gpu/oracle", rep["iterations"], ref.report["iterations"], "scale", rep["scale"], ref.report["scale"])
for u, (g, o) in enumerate(zip(ex["log"], ref.log)):
    same = g["r"] == o["r"] and np.array_equal(g["rows"], o["rows"]) and np.array_equal(g["cols"], o["cols"])
    if not same:
        k = next((i for i in range(min(g["r"], o["r"])) if g["rows"][i] != o["rows"][i] or g["cols"][i] != o["cols"][i]),
                 min(g["r"], o["r"]))
        print(f"update {u} bond {g['bond']} dir {g['dir']} rl {g['rl']}/{o['rl']} rr {g['rr']}/{o['rr']} "
              f"r {g['r']}/{o['r']} first diff at k={k} eps {g['eps']:.3e}/{o['eps']:.3e} scale {g['scale']:.6e}/{o['scale']:.6e}")
        print("   gpu rows", g["rows"][:12], "cols", g["cols"][:12])
        print("   orc rows", o["rows"][:12], "cols", o["cols"][:12])
