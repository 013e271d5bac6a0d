# A/B: hand-off of the two-cluster 512 x 1024 factorisations to one cluster after K pivots (HANDOFF)
set -x
O=gpurun_out/s3i_ab.txt
for b in h0 h1; do echo "== prrlu_bench $b" >> $O; timeout 120 ./tools/prrlu_bench_$b 2>&1 | grep -v "max active" >> $O; echo "rc=$?" >> $O; done
for chi in 256 128; do for L in tools/libab/libaci_h0.so paper_2604_00037_b200/libaci.so; do echo "== pivhash $chi $L" >> $O; ACI_LIB=$L timeout 300 python tools/pivhash.py $chi >> $O 2>&1; done; done
for rep in 1 2; do for L in tools/libab/libaci_h0.so paper_2604_00037_b200/libaci.so; do echo "== time_chi $L rep $rep" >> $O; ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 4 2>&1 | grep -v profile >> $O; done; done
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/s3i_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s3i_tests.log
