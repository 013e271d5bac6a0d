set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./tools/probe/coop_cluster > gpurun_out/r02_coop_cluster.txt 2>&1
timeout 300 ./tools/prrlu_bench > gpurun_out/r02_prrlu_bench_base.txt 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r02a_gputests.log 2>&1; echo "pytest rc=$?"
timeout 1200 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo "bench rc=$?"
lscpu | head -20 > gpurun_out/r02_lscpu.txt
