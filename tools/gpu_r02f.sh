set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/r02f_bench_ref.json 2> gpurun_out/r02f_bench_ref.err; echo "ref rc=$?"
timeout 300 python tools/run_chi.py 256 > gpurun_out/r02f_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches_chi256.csv python tools/run_chi.py 256 > gpurun_out/r02f_ncu1.log 2>&1
timeout 300 python tools/run_chi.py 256 > gpurun_out/r02f_plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:prrlu --launch-skip 321 -c 1 -o gpurun_out/r02f_prrlu python tools/run_chi.py 256 > gpurun_out/r02f_ncu2.log 2>&1
ACI_NO_GRAPH=1 timeout 300 python tools/run_chi.py 256 > gpurun_out/r02f_plain3.log 2>&1 && ACI_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:Cfg<\(int\)64, \(int\)64" --launch-skip 150 -c 1 -o gpurun_out/r02f_pi python tools/run_chi.py 256 > gpurun_out/r02f_ncu3.log 2>&1
timeout 120 ./tools/prrlu_bench_li 64 > gpurun_out/r02f_plain4.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:prrlu -s 2 -c 1 -o gpurun_out/r02f_cta64 ./tools/prrlu_bench_li 64 > gpurun_out/r02f_ncu4.log 2>&1
ls -la gpurun_out/
