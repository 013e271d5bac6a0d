set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for v in notma tma tma_pw; do
  echo "== $v" >> gpurun_out/r02c_pbv.txt
  timeout 300 ./tools/pbv/pb_$v >> gpurun_out/r02c_pbv.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rook or cfg0 or cfg1 or tiers or concurrent" -p no:cacheprovider > gpurun_out/r02c_gputests.log 2>&1; echo "pytest rc=$?"
timeout 600 python tools/time_chi.py 64,128,256 5 > gpurun_out/r02c_time_chi.txt 2>&1
