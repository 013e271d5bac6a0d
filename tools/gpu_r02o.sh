set -x
timeout 120 ./tools/prrlu_bench > gpurun_out/r02o_pb_off.txt 2>&1; echo "pb off rc=$?"
ACI_PRRLU_2D=1 timeout 120 ./tools/prrlu_bench > gpurun_out/r02o_pb_2d.txt 2>&1; echo "pb 2d rc=$?"
for c in 64 128; do
  timeout 120 python tools/pivhash.py $c >> gpurun_out/r02o_hash.txt 2>&1
  ACI_PRRLU_2D=1 timeout 120 python tools/pivhash.py $c >> gpurun_out/r02o_hash.txt 2>&1
done
for rep in 1 2; do
  echo "== off rep $rep" >> gpurun_out/r02o_ab.txt; timeout 300 python tools/time_chi.py 64,128,256 3 >> gpurun_out/r02o_ab.txt 2>&1
  echo "== 2d rep $rep" >> gpurun_out/r02o_ab.txt; ACI_PRRLU_2D=1 timeout 300 python tools/time_chi.py 64,128,256 3 >> gpurun_out/r02o_ab.txt 2>&1
done
