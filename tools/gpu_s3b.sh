# A/B: NC power of two (shift/mask pivot decode) + reciprocal issued under the column loads, vs HEAD
set -x
O=gpurun_out/s3b_ab.txt
for b in ref v1 ref v1; do echo "== prrlu_bench $b" >> $O; ./tools/prrlu_bench_$b 2>&1 | head -7 >> $O; done
for chi in 64 256; do for L in tools/libaci_ref.so paper_2604_00037_b200/libaci.so; do echo "== pivhash $chi $L" >> $O; ACI_LIB=$L timeout 300 python tools/pivhash.py $chi >> $O 2>&1; done; done
for rep in 1 2; do for L in tools/libaci_ref.so paper_2604_00037_b200/libaci.so; do echo "== time_chi $L rep $rep" >> $O; ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 5 >> $O 2>&1; done; done
