# A/B: 512-row blocks <= 256 columns on 16 CTAs x 16 columns (NARROW512) vs 8 CTAs x 32
set -x
O=gpurun_out/s3g_ab.txt
for b in n0 n1 n0 n1; do echo "== prrlu_bench $b" >> $O; ./tools/prrlu_bench_$b 2>&1 | grep -v "max active" >> $O; done
for chi in 64 128 256; do for L in tools/libab/libaci_n0.so paper_2604_00037_b200/libaci.so; do echo "== pivhash $chi $L" >> $O; ACI_LIB=$L timeout 300 python tools/pivhash.py $chi >> $O 2>&1; done; done
for rep in 1 2 3; do for L in tools/libab/libaci_n0.so paper_2604_00037_b200/libaci.so; do echo "== time_chi $L rep $rep" >> $O; ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 4 2>&1 | grep -v profile >> $O; done; done
