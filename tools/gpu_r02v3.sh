set -x
ACI_LIB=tools/libab/libaci_dbg.so ACI_NO_GRAPH=1 ACI_STREAM_PI=1 timeout 30 python -c "
import sys; sys.path.insert(0,'.')
import paper_2604_00037_b200 as aci
from workloads import make_config
cf = make_config(0, npts=0)
xs = [aci.TensorTrain.from_cores(t) for t in cf['inputs']]
y0 = aci.TensorTrain.from_cores(cf['y_init'])
print('L', len(cf['inputs'][0].cores), [c.shape for c in cf['inputs'][0].cores][:4], flush=True)
out, st, rep, ex = aci.aci_elementwise(cf['op'], xs, cf['tol'], cf['maxrank'], cf['max_sweeps'], y_init=y0)
print('ok', rep['ms'], rep['pivot_steps'], flush=True)
" 2>&1 | head -60
