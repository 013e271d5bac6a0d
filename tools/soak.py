"""Soak test (development tool): many consecutive products on one stream and in concurrent
threads; checks that outputs are bitwise identical run to run, that device memory does not grow,
and reports the time distribution."""
import hashlib
import json
import sys
import threading
import time
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2604_00037_b200 as aci  # noqa: E402
from workloads import make_config  # noqa: E402


def digest(tt):
    h = hashlib.sha256()
    for c in tt.cores():
        h.update(np.ascontiguousarray(c).tobytes())
    return h.hexdigest()


def run(chi, n):
    cf = make_config(3, chi, npts=0)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    s = torch.cuda.Stream()
    ms, digests, mem = [], set(), []
    for i in range(n):
        out, st, rep, _ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                                              stream=s.cuda_stream)
        ms.append(rep["ms"])
        if i % 10 == 0:
            digests.add(digest(out))
            mem.append(torch.cuda.mem_get_info()[0])
        out.free()
    return {"chi": chi, "products": n, "ms_median": float(np.median(ms)), "ms_p99": float(np.percentile(ms, 99)),
            "ms_max": float(np.max(ms)), "distinct_outputs": len(digests),
            "free_mem_drift_mb": (mem[0] - mem[-1]) / 2**20}


def run_concurrent(chi, threads, n):
    cf = make_config(3, chi, npts=0)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    ref, *_ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0)
    want = digest(ref)
    bad = []

    def work():
        s = torch.cuda.Stream()
        for _ in range(n):
            o, *_ = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0,
                                        stream=s.cuda_stream, concurrent=True)
            if digest(o) != want:
                bad.append(1)
            o.free()

    t0 = time.time()
    th = [threading.Thread(target=work) for _ in range(threads)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return {"chi": chi, "threads": threads, "products": threads * n, "seconds": time.time() - t0,
            "mismatches": len(bad)}


res = {"sequential": [run(256, 200), run(64, 300)], "concurrent": [run_concurrent(64, 8, 40),
                                                                   run_concurrent(256, 4, 10)]}
print(json.dumps(res, indent=1))
