# A/B: one-CTA variants with > 32 / > 16 register entries per thread kept out of the cluster kernel (CTA_MAXE)
set -x
O=gpurun_out/s3h_ab.txt
for b in e64 e32 e64 e32; do echo "== prrlu_bench $b" >> $O; ./tools/prrlu_bench_$b 2>&1 | grep -v "max active" >> $O; done
for chi in 64 128; do for L in tools/libab/libaci_e32.so tools/libab/libaci_e16.so; do echo "== pivhash $chi $L" >> $O; ACI_LIB=$L timeout 300 python tools/pivhash.py $chi >> $O 2>&1; done; done
for rep in 1 2 3; do for L in paper_2604_00037_b200/libaci.so tools/libab/libaci_e32.so tools/libab/libaci_e16.so; do echo "== time_chi $L rep $rep" >> $O; ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 4 2>&1 | grep -v profile >> $O; done; done
