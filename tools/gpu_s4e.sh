# fresh ncu --set full of 30 Pi GEMM launches (64x64 tiles, f fused) of the current build; the full-size ones (1024 x 1024) are picked by duration
set -x
ACI_NO_GRAPH=1 timeout 300 python tools/run_chi.py 256 > gpurun_out/s4e_plain.log 2>&1; echo "plain rc=$?"
ACI_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:Cfg<\(int\)64, \(int\)64" --launch-skip 40 -c 30 -o gpurun_out/s4e_pi python tools/run_chi.py 256 > gpurun_out/s4e_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/s4e_pi.ncu-rep --page raw --csv > gpurun_out/s4e_pi_raw.csv 2>&1
ncu -i gpurun_out/s4e_pi.ncu-rep --page details --csv > gpurun_out/s4e_pi_details.csv 2>&1
tail -3 gpurun_out/s4e_ncu.log
