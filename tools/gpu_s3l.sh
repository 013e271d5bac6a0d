# hand-off pivot rounded to a multiple of 4 (the s3k hang: phase 2's fresh mbarriers); prrLU pivot
# hashes with and without hand-off on every bench shape; GPU suite with a per-test timeout; A/B vs
# the committed hand-off; then the full bench line
set -x
O=gpurun_out/s3l_ab.txt
for b in h0 h2; do echo "== prrlu_bench $b" >> $O; timeout 120 ./tools/prrlu_bench_$b 2>&1 | grep -v "max active" >> $O; echo "rc=$?" >> $O; done
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -x --timeout 600 > gpurun_out/s3l_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s3l_tests.log
for rep in 1 2; do for L in tools/libab/libaci_h1.so paper_2604_00037_b200/libaci.so; do echo "== time_chi $L rep $rep" >> $O; ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 4 2>&1 | grep -v profile >> $O; done; done
timeout 1500 python bench.py > gpurun_out/s3l_bench.json 2> gpurun_out/s3l_bench.err; echo "bench rc=$?"
