"""Run one configs[3] product (development helper for ncu captures)."""
import sys
sys.path.insert(0, ".")
import paper_2604_00037_b200 as aci  # noqa: E402
from workloads import make_config  # noqa: E402

chi = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cf = make_config(3, chi, npts=0)
xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
y0 = aci.TensorTrain.from_cores(cf["y_init"])
for _ in range(reps):
    out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0)
    out.free()
print(rep)
