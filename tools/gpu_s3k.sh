# A/B: second hand-off pair (512 x <=256 single-cluster blocks: 16x2 -> 12x1 entries at pivot K) vs the
# committed hand-off; GPU suite; quick bench line with the per-shape latency floor
set -x
O=gpurun_out/s3k_ab.txt
for b in h1 h2 h1 h2; do echo "== prrlu_bench $b" >> $O; timeout 120 ./tools/prrlu_bench_$b 2>&1 | grep -v "max active" | grep "static 1024" >> $O; done
for chi in 128 256; do for L in tools/libab/libaci_h1.so paper_2604_00037_b200/libaci.so; do echo "== pivhash $chi $L" >> $O; ACI_LIB=$L timeout 300 python tools/pivhash.py $chi >> $O 2>&1; done; done
for rep in 1 2 3; do for L in tools/libab/libaci_h1.so paper_2604_00037_b200/libaci.so; do echo "== time_chi $L rep $rep" >> $O; ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 4 2>&1 | grep -v profile >> $O; done; done
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/s3k_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s3k_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-chi-sweep --no-complex --no-cpu-baseline > gpurun_out/s3k_bench_quick.json 2> gpurun_out/s3k_bench_quick.err; echo "bench rc=$?"
