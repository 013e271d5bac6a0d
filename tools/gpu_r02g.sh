set -x
timeout 300 python -c "
import sys, json; sys.path.insert(0, '.')
import bench
print(json.dumps(bench.measure_prrlu_latency(), indent=1))
" > gpurun_out/r02g_latency.json 2> gpurun_out/r02g_latency.err
for c in 8; do ACI_PRRLU_CLUSTER=$c timeout 300 python tools/time_chi.py 256 3 > gpurun_out/r02g_cluster$c.txt 2>&1; done
