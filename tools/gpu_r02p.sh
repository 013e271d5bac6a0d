set -x
for c in 64 256; do
  timeout 120 python tools/pivhash.py $c >> gpurun_out/r02p_hash.txt 2>&1
  ACI_PRRLU_G8=1 timeout 120 python tools/pivhash.py $c >> gpurun_out/r02p_hash.txt 2>&1
done
for rep in 1 2 3; do
  echo "== g16 rep $rep" >> gpurun_out/r02p_ab.txt; timeout 300 python tools/time_chi.py 64,128,256 3 >> gpurun_out/r02p_ab.txt 2>&1
  echo "== g8 rep $rep" >> gpurun_out/r02p_ab.txt; ACI_PRRLU_G8=1 timeout 300 python tools/time_chi.py 64,128,256 3 >> gpurun_out/r02p_ab.txt 2>&1
done
