import sys, time, torch
sys.path.insert(0, ".")
import paper_2604_00037_b200 as aci
from workloads import make_config
aci.load()
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); sptr = stream.cuda_stream
import os
keep = []
for chi in (256, 256):
    cf = make_config(3, chi, npts=0)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    for i in range(12):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0, stream=sptr, iter_times=True)
        e1.record(stream); torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(chi, i, round(e0.elapsed_time(e1), 2), round((t1 - t0) * 1e3, 2), [round(x, 2) for x in ex["iter_ms"]], round(rep["ms"], 2), flush=True)
        (keep.append(out) if len(keep) < 12 and chi == 256 and i < 12 and os.environ.get('KEEP') else out.free())
