set -x
timeout 1200 python tools/soak.py > gpurun_out/r02u_soak.json 2> gpurun_out/r02u_soak.err; echo "soak rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "rook or probes" -p no:cacheprovider > gpurun_out/r02u_tests.log 2>&1; echo "tests rc=$?"
