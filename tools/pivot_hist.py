"""Histogram of prrLU pivots by live block size for a configs[3] product (development tool)."""
import collections
import sys
sys.path.insert(0, ".")
import paper_2604_00037_b200 as aci  # noqa: E402
from workloads import make_config  # noqa: E402

chi = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cf = make_config(3, chi, npts=0)
xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
y0 = aci.TensorTrain.from_cores(cf["y_init"])
out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0, log=True)
h = collections.Counter()
hb = collections.Counter()
for e in ex["log"]:
    m, n = 2 * e["rl"], 2 * e["rr"]
    big = max(m, n)
    cls = next(c for c in (32, 64, 128, 256, 512, 1024) if big <= c)
    h[cls] += e["r"]
    hb[cls] += 1
tot = sum(h.values())
for c in sorted(h):
    print(f"max(m,n) <= {c:5d}: bonds {hb[c]:4d} pivots {h[c]:6d} ({100*h[c]/tot:4.1f}%)")
print("total pivots", tot)
