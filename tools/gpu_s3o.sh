# aci_prrlu (a5 alone through the C-ABI) vs the oracle on hand-off shapes; full GPU suite; smoke
set -x
timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -k "prrlu_step" --timeout 300 > gpurun_out/s3o_prrlu_step.log 2>&1; echo "step rc=$?"; tail -3 gpurun_out/s3o_prrlu_step.log
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 600 > gpurun_out/s3o_gputests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s3o_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3o_smoke.log 2>&1; echo "smoke rc=$?"
