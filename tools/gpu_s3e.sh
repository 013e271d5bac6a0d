# A/B: warp keys as one 16-byte store (KEY_VEC) and the ballot/shuffle warp argmax (ARGMAX_BALLOT)
set -x
O=gpurun_out/s3e_ab.txt
for b in k0a0 k1a0 k0a1 k1a1 k0a0 k1a1; do echo "== prrlu_bench $b" >> $O; ./tools/prrlu_bench_$b 2>&1 | grep -v "max active" >> $O; done
for chi in 64 128 256; do for L in tools/libab/libaci_k0a0.so paper_2604_00037_b200/libaci.so; do echo "== pivhash $chi $L" >> $O; ACI_LIB=$L timeout 300 python tools/pivhash.py $chi >> $O 2>&1; done; done
for rep in 1 2; do for L in tools/libab/libaci_k0a0.so tools/libab/libaci_k1a0.so tools/libab/libaci_k0a1.so paper_2604_00037_b200/libaci.so; do echo "== time_chi $L rep $rep" >> $O; ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 4 2>&1 | grep -v profile >> $O; done; done
