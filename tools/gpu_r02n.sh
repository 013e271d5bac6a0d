set -x
for rep in 1 2; do
for v in cur novec; do
  case $v in cur) L=paper_2604_00037_b200/libaci.so;; *) L=tools/libab/libaci_$v.so;; esac
  echo "== $v rep $rep" >> gpurun_out/r02n_ab.txt
  ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 4 >> gpurun_out/r02n_ab.txt 2>&1
done
done
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02n_gputests.log 2>&1; echo "pytest rc=$?"
