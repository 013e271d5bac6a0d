# streamed Pi on by default: smoke + the whole GPU suite
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02w_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02w_gputests.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02w_gputests.log
