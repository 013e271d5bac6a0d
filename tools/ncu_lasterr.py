"""Does a product leave a pending CUDA runtime error behind (the next torch launch would report it)?"""
import ctypes, sys
sys.path.insert(0, ".")
import hashlib
import numpy as np
import torch
import paper_2604_00037_b200 as aci
from workloads import make_config
aci.load()
rt = ctypes.CDLL("libcudart.so.12") if len(sys.argv) < 3 else None
chi = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cf = make_config(3, chi, npts=0)
xs = [aci.TensorTrain.from_cores(t) for t in cf["inputs"]]
y0 = aci.TensorTrain.from_cores(cf["y_init"])
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
x = torch.empty(1 << 20, device="cuda")
for i in range(3):
    out, st, rep, ex = aci.aci_elementwise(cf["op"], xs, cf["tol"], cf["maxrank"], cf["max_sweeps"], y_init=y0, stream=s.cuda_stream)
    torch.cuda.synchronize()
    h = hashlib.sha256(b"".join(np.ascontiguousarray(c).tobytes() for c in out.cores())).hexdigest()[:16]
    print("product", i, "cores", h, "graph iterations", rep.get("graph_iterations"), flush=True)
    try:
        x.fill_(float(i)); torch.cuda.synchronize(); print("product", i, "ok", flush=True)
    except Exception as e:
        print("product", i, "-> torch error", str(e).splitlines()[0], flush=True)
    out.free()
