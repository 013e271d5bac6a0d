set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02t_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02t_gputests.log 2>&1; echo "pytest rc=$?"
timeout 1500 python bench.py > gpurun_out/r02t_bench.json 2> gpurun_out/r02t_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 1 --warmup 3 --no-chi-sweep --no-complex --no-cpu-baseline > gpurun_out/r02t_bench_small.json 2>&1 && timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02t_bench_launches.csv python bench.py --steps 1 --warmup 3 --no-chi-sweep --no-complex --no-cpu-baseline > gpurun_out/r02t_ncu.log 2>&1; echo "ncu rc=$?"
