# session-3 final checkpoint (hand-off + narrow tiers): smoke, GPU suite, bench line, bench launch list, ncu --set full of
# the longest prrLU launch of a chi = 256 product
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3n_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/s3n_bench.json 2> gpurun_out/s3n_bench.err; echo "bench rc=$?"
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s3n_gputests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s3n_gputests.log
timeout 600 python bench.py --steps 1 --warmup 3 --no-chi-sweep --no-complex --no-cpu-baseline > gpurun_out/s3n_bench_small.json 2>&1 && timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3n_bench_launches.csv python bench.py --steps 1 --warmup 3 --no-chi-sweep --no-complex --no-cpu-baseline > gpurun_out/s3n_ncu.log 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/s3n_bench_launches.csv > gpurun_out/s3n_bench_launches_summary.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3n_chi256_launches.csv python tools/run_chi.py 256 > gpurun_out/s3n_ncu1.log 2>&1; echo "ncu1 rc=$?"
python tools/launches.py gpurun_out/s3n_chi256_launches.csv > gpurun_out/s3n_chi256_launches_summary.txt 2>&1
SKIP=$(python tools/longest_prrlu.py gpurun_out/s3n_chi256_launches.csv); echo "longest prrlu launch $SKIP"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prrlu_kernel --launch-skip $SKIP -c 1 -o gpurun_out/s3n_prrlu python tools/run_chi.py 256 > gpurun_out/s3n_ncu2.log 2>&1; echo "ncu2 rc=$?"
ls -la gpurun_out/
