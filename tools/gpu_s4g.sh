# Pi GEMM: 64x64 tile as 4 warps of 32x32 (ACI_PI_WN=32; MINB 2 / 3) vs the in-tree 8 warps of 32x16;
# whole-product A/B interleaved, parity of the variants, ncu of one full-size Pi launch per variant
set -x
O=gpurun_out/s4g_piwn_ab.txt
for rep in 1 2; do for L in paper_2604_00037_b200/libaci.so tools/libab/libaci_w32m2.so tools/libab/libaci_w32m3.so; do echo "== time_chi $L rep $rep" >> $O; ACI_LIB=$L timeout 300 python tools/time_chi.py 128,256 4 2>&1 | grep -v profile >> $O; done; done
cat $O
for v in w32m2 w32m3; do ACI_LIB=tools/libab/libaci_$v.so timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 600 -k "cfg2 or cfg3_vs_oracle or cfg3_chi256 or cfg4 or constant_term or small_random" > gpurun_out/s4g_${v}_tests.log 2>&1; echo "$v tests rc=$?"; tail -1 gpurun_out/s4g_${v}_tests.log; done
for v in w32m2 w32m3; do ACI_LIB=tools/libab/libaci_$v.so ACI_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control none --csv --kernel-name-base demangled -k "regex:Cfg<\(int\)64, \(int\)64" --launch-skip 40 -c 30 python tools/run_chi.py 256 > gpurun_out/s4g_${v}_ncu.csv 2>&1; echo "ncu $v rc=$?"; done
ACI_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control none --csv --kernel-name-base demangled -k "regex:Cfg<\(int\)64, \(int\)64" --launch-skip 40 -c 30 python tools/run_chi.py 256 > gpurun_out/s4g_base_ncu.csv 2>&1; echo "ncu base rc=$?"
