# session-3 re-validation of HEAD on a fresh box: smoke, GPU suite, prrLU phase baseline
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3a_smoke.log 2>&1; echo "smoke rc=$?"
./tools/prrlu_bench > gpurun_out/s3a_prrlu_bench.txt 2>&1; echo "pb rc=$?"
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/s3a_gputests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s3a_gputests.log
