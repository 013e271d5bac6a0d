set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 120 ./tools/probe/coop_spin > gpurun_out/r02_coop_spin.txt 2>&1
for v in base lpair pd8 dmnmx ch8 spread pubwin sp_pw; do
  echo "== $v" >> gpurun_out/r02_pbv.txt
  timeout 300 ./tools/pbv/pb_$v >> gpurun_out/r02_pbv.txt 2>&1
done
timeout 2400 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r02b_gputests.log 2>&1; echo "pytest rc=$?"
timeout 600 python tools/time_chi.py 64,128,256 5 > gpurun_out/r02b_time_chi.txt 2>&1
