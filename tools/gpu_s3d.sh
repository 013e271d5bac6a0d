# A/B: 16-byte shared stores for the pivot row (SU) and the l column (SL) before the per-pivot barriers
set -x
O=gpurun_out/s3d_ab.txt
for b in s00 s10 s01 s11 s00 s11; do echo "== prrlu_bench $b" >> $O; ./tools/prrlu_bench_$b 2>&1 | grep -v "max active" >> $O; done
for chi in 64 128 256; do for L in tools/libab/libaci_s00.so paper_2604_00037_b200/libaci.so; do echo "== pivhash $chi $L" >> $O; ACI_LIB=$L timeout 300 python tools/pivhash.py $chi >> $O 2>&1; done; done
for rep in 1 2; do for L in tools/libab/libaci_s00.so tools/libab/libaci_s10.so tools/libab/libaci_s01.so paper_2604_00037_b200/libaci.so; do echo "== time_chi $L rep $rep" >> $O; ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 4 2>&1 | grep -v profile >> $O; done; done
