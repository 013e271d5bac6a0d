set -x
for rep in 1 2; do
for v in cur pdl; do
  case $v in
    cur) L=paper_2604_00037_b200/libaci.so;;
    *) L=tools/libab/libaci_$v.so;;
  esac
  echo "== $v rep $rep" >> gpurun_out/r02j_ab.txt
  ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 3 >> gpurun_out/r02j_ab.txt 2>&1
done
done
timeout 1500 python bench.py > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; echo "bench rc=$?"
