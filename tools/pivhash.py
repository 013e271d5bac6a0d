"""Hash of the ordered pivot log of one configs[3] product (A/B correctness check of two builds)."""
import hashlib, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2604_00037_b200 as aci
from workloads import make_config
aci.load()
cf = make_config(3, int(sys.argv[1]), npts=0)
xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
y0 = aci.TensorTrain.from_cores(cf["y_init"])
out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0, log=True)
h = hashlib.sha256()
for e in ex["log"]:
    h.update(np.asarray(e["rows"], np.int32).tobytes()); h.update(np.asarray(e["cols"], np.int32).tobytes())
c = hashlib.sha256(b"".join(np.ascontiguousarray(x).tobytes() for x in out.cores())).hexdigest()[:16]
print("pivots", h.hexdigest()[:16], "cores", c, len(ex["log"]))
