set -x
for g in 1 0; do
  for c in 0 1; do
    ACI_NO_GRAPH=$((1-g)) ACI_STREAM_PI=1 timeout 60 python -c "
import sys; sys.path.insert(0,'.')
import paper_2604_00037_b200 as aci
from workloads import make_config
cf = make_config($c, npts=0) if $c != 3 else make_config(3, 64, npts=0)
xs = [aci.TensorTrain.from_cores(t) for t in cf['inputs']]
y0 = aci.TensorTrain.from_cores(cf['y_init'])
out, st, rep, ex = aci.aci_elementwise(cf['op'], xs, cf['tol'], cf['maxrank'], cf['max_sweeps'], y_init=y0)
print('cfg', $c, 'graph', $g, 'ok', rep['ms'], rep['pivot_steps'], flush=True)
"; echo "cfg$c graph$g rc=$?"
  done
done
