set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "concurrent or tiers or batch" -p no:cacheprovider > gpurun_out/r02i_gputests.log 2>&1; echo "pytest rc=$?"
timeout 1800 python tools/results_table.py > gpurun_out/r02i_results_table.json 2> gpurun_out/r02i_results_table.err; echo "table rc=$?"
