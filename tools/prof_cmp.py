"""Per-class profile (eager launches, CUDA events per class) of one configs[3] product."""
import sys
sys.path.insert(0, ".")
import paper_2604_00037_b200 as aci  # noqa: E402
from workloads import make_config  # noqa: E402

chi = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cf = make_config(3, chi, npts=0)
xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
y0 = aci.TensorTrain.from_cores(cf["y_init"])
for rep_i in range(2):
    out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                                           profile=True)
    out.free()
print(round(rep["ms"], 2), {k: round(v["ms"], 2) for k, v in ex["profile"].items()})
