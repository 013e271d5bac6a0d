# round-2 checkpoint on the streamed-Pi build: smoke, GPU suite, bench line, launch list, ncu --set full captures
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02z_gputests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02z_gputests.log
timeout 1500 python bench.py > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 1 --warmup 3 --no-chi-sweep --no-complex --no-cpu-baseline > gpurun_out/r02z_bench_small.json 2>&1 && timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z_bench_launches.csv python bench.py --steps 1 --warmup 3 --no-chi-sweep --no-complex --no-cpu-baseline > gpurun_out/r02z_ncu.log 2>&1; echo "ncu rc=$?"
timeout 300 python tools/run_chi.py 256 > gpurun_out/r02z_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:prrlu --launch-skip 321 -c 1 -o gpurun_out/r02z_prrlu python tools/run_chi.py 256 > gpurun_out/r02z_ncu2.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pi_stream --launch-skip 40 -c 1 -o gpurun_out/r02z_stream python tools/run_chi.py 256 > gpurun_out/r02z_ncu3.log 2>&1; echo "ncu3 rc=$?"
ACI_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:Cfg<\(int\)64, \(int\)64" --launch-skip 100 -c 1 -o gpurun_out/r02z_pi python tools/run_chi.py 256 > gpurun_out/r02z_ncu4.log 2>&1; echo "ncu4 rc=$?"
ls -la gpurun_out/
