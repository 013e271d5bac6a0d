# A/B: 128-row blocks <= 256 columns on 16 CTAs x 16 columns (NARROW128); GPU suite; results table
set -x
O=gpurun_out/s3m_ab.txt
for b in w0 w1 w0 w1; do echo "== prrlu_bench $b" >> $O; timeout 120 ./tools/prrlu_bench_$b 2>&1 | grep -v "max active" | grep -E "128x|x 64" >> $O; done
for chi in 64 128 256; do for L in tools/libab/libaci_h2.so paper_2604_00037_b200/libaci.so; do echo "== pivhash $chi $L" >> $O; ACI_LIB=$L timeout 300 python tools/pivhash.py $chi >> $O 2>&1; done; done
for rep in 1 2 3; do for L in tools/libab/libaci_h2.so paper_2604_00037_b200/libaci.so; do echo "== time_chi $L rep $rep" >> $O; ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 4 2>&1 | grep -v profile >> $O; done; done
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -x --timeout 600 > gpurun_out/s3m_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s3m_tests.log
timeout 900 python tools/results_table.py > gpurun_out/s3m_results_table.json 2> gpurun_out/s3m_results_table.err; echo "table rc=$?"
