"""Stress: many host threads, own streams, concurrent mode, small products (development tool)."""
import ctypes
import sys
import threading
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2604_00037_b200 as aci  # noqa: E402
from workloads import make_config  # noqa: E402

aci.load()
ctypes.CDLL("./tools/segv_bt.so").segv_install()
cf = make_config(0, npts=0)
xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
y0 = aci.TensorTrain.from_cores(cf["y_init"])
ref, *_ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0)
ref = ref.cores()
bad = []
for rnd in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    out = [None] * 12

    def work(i):
        s = torch.cuda.Stream()
        for _ in range(3):
            o, *_ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                                        stream=s.cuda_stream, concurrent=True)
        out[i] = o.cores()

    th = [threading.Thread(target=work, args=(i,)) for i in range(12)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    ok = all(r is not None and all(np.array_equal(x, y) for x, y in zip(r, ref)) for r in out)
    print("round", rnd, "ok" if ok else "MISMATCH", flush=True)
