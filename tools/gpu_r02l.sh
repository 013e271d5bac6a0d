set -x
for v in e64 mc; do echo "== $v" >> gpurun_out/r02l_pbv.txt; timeout 300 ./tools/pbv/pb_$v 1024 >> gpurun_out/r02l_pbv.txt 2>&1; done
for v in cur mc; do
  case $v in cur) L=paper_2604_00037_b200/libaci.so;; *) L=tools/libab/libaci_$v.so;; esac
  echo "== $v" >> gpurun_out/r02l_hash.txt
  ACI_LIB=$L timeout 300 python tools/pivhash.py 256 >> gpurun_out/r02l_hash.txt 2>&1
done
for rep in 1 2; do
for v in cur mc; do
  case $v in cur) L=paper_2604_00037_b200/libaci.so;; *) L=tools/libab/libaci_$v.so;; esac
  echo "== $v rep $rep" >> gpurun_out/r02l_ab.txt
  ACI_LIB=$L timeout 300 python tools/time_chi.py 256 4 >> gpurun_out/r02l_ab.txt 2>&1
done
done
