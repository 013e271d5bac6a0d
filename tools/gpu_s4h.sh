# session-4 final check of the rebuilt library (Pi A/B switches at their defaults): smoke, bench line, GPU suite
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4h_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/s4h_bench.json 2> gpurun_out/s4h_bench.err; echo "bench rc=$?"
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 600 > gpurun_out/s4h_gputests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s4h_gputests.log
