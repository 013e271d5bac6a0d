# streamed Pi: correctness (pivot/core hashes vs ACI_STREAM_PI=0, GPU parity tests) and A/B timing
set -x
for c in 64 128 256; do
  ACI_STREAM_PI=0 timeout 120 python tools/pivhash.py $c > gpurun_out/r02v_hash0_$c.txt 2>&1
  ACI_STREAM_PI=1 timeout 120 python tools/pivhash.py $c > gpurun_out/r02v_hash1_$c.txt 2>&1
done
cat gpurun_out/r02v_hash*_*.txt
for i in 1 2; do
  ACI_STREAM_PI=0 timeout 200 python tools/time_chi.py 64,128,256 5 > gpurun_out/r02v_t0_$i.txt 2>&1
  ACI_STREAM_PI=1 timeout 200 python tools/time_chi.py 64,128,256 5 > gpurun_out/r02v_t1_$i.txt 2>&1
done
cat gpurun_out/r02v_t*.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "cfg0 or cfg1 or cfg3_vs or edge or small_random or constant or identity or zero or cfg2 or warm or errors" > gpurun_out/r02v_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02v_tests.log
