# A/B: pivot-row shared stores issued after the grid tiers' column loads (U_LATE)
set -x
O=gpurun_out/s3f_ab.txt
for b in u0 u1 u0 u1; do echo "== prrlu_bench $b" >> $O; ./tools/prrlu_bench_$b 2>&1 | grep -v "max active" >> $O; done
for chi in 64 128 256; do for L in tools/libab/libaci_u0.so paper_2604_00037_b200/libaci.so; do echo "== pivhash $chi $L" >> $O; ACI_LIB=$L timeout 300 python tools/pivhash.py $chi >> $O 2>&1; done; done
for rep in 1 2 3; do for L in tools/libab/libaci_u0.so paper_2604_00037_b200/libaci.so; do echo "== time_chi $L rep $rep" >> $O; ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 4 2>&1 | grep -v profile >> $O; done; done
