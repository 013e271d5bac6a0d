import sys, time
sys.path.insert(0, ".")
import torch
import paper_2604_00037_b200 as aci
from workloads import make_config
s = torch.cuda.Stream()
for cfg, chi in [(1, 0), (3, 256)]:
    cf = make_config(cfg, chi, npts=0)
    xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
    y0 = aci.TensorTrain.from_cores(cf["y_init"])
    for rep in range(3):
        for stream in (s.cuda_stream, 0):
            t = time.time()
            out, st, r, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0, stream=stream)
            torch.cuda.synchronize()
            print(cfg, chi, "stream", stream != 0, "wall %.1f ms" % ((time.time() - t) * 1e3), "lib", round(r["ms"], 1), "graph_it", r["graph_iterations"], "setup %.1f" % r["ms_graph_setup"], flush=True)
            out.free()
