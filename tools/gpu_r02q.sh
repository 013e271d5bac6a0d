set -x
for c in 64 128; do
  for lv in 0 1 2; do ACI_PRRLU_SPEC=$lv timeout 120 python tools/pivhash.py $c >> gpurun_out/r02q_hash.txt 2>&1; done
done
for rep in 1 2 3; do
  for lv in 0 1 2; do
    echo "== spec$lv rep $rep" >> gpurun_out/r02q_ab.txt; ACI_PRRLU_SPEC=$lv timeout 300 python tools/time_chi.py 64,128,256 3 >> gpurun_out/r02q_ab.txt 2>&1
  done
done
