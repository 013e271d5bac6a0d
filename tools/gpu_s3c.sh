# A/B: one-barrier CTA tier (XM = 4, blocks <= 256 rows in one CTA) vs the committed two-barrier tier
set -x
O=gpurun_out/s3c_ab.txt
for b in v1 v2 v1 v2; do echo "== prrlu_bench $b" >> $O; ./tools/prrlu_bench_$b >> $O 2>&1; done
for chi in 64 128 256; do for L in tools/libaci_v1.so paper_2604_00037_b200/libaci.so; do echo "== pivhash $chi $L" >> $O; ACI_LIB=$L timeout 300 python tools/pivhash.py $chi >> $O 2>&1; done; done
for rep in 1 2; do for L in tools/libaci_v1.so paper_2604_00037_b200/libaci.so; do echo "== time_chi $L rep $rep" >> $O; ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 5 >> $O 2>&1; done; done
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "parity or prrlu or tiers" > gpurun_out/s3c_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s3c_tests.log
