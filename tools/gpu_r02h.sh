set -x
for v in e64 e32 e16; do echo "== $v" >> gpurun_out/r02h_pbv.txt; timeout 300 ./tools/pbv/pb_$v >> gpurun_out/r02h_pbv.txt 2>&1; done
for rep in 1 2; do
for v in cur e32 e16; do
  case $v in
    cur) L=paper_2604_00037_b200/libaci.so;;
    *) L=tools/libab/libaci_$v.so;;
  esac
  echo "== $v rep $rep" >> gpurun_out/r02h_ab.txt
  ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 3 >> gpurun_out/r02h_ab.txt 2>&1
done
done
