# fresh ncu --set full of the full-size Pi GEMM (a3+a4, 64x64 tiles, f fused) of the current build
set -x
ACI_NO_GRAPH=1 timeout 300 python tools/run_chi.py 256 > gpurun_out/s4d_plain.log 2>&1; echo "plain rc=$?"
ACI_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:Cfg<\(int\)64, \(int\)64" --launch-skip 60 -c 1 -o gpurun_out/s4d_pi python tools/run_chi.py 256 > gpurun_out/s4d_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/s4d_pi.ncu-rep --page raw --csv > gpurun_out/s4d_pi_raw.csv 2>&1
ncu -i gpurun_out/s4d_pi.ncu-rep --page details --csv > gpurun_out/s4d_pi_details.csv 2>&1
tail -3 gpurun_out/s4d_ncu.log
