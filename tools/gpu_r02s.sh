set -x
timeout 120 ./tools/gemm_bench2 > gpurun_out/r02s_gemm.txt 2>&1
for c in 64 256; do
  timeout 120 python tools/pivhash.py $c >> gpurun_out/r02s_hash.txt 2>&1
  ACI_LIB=tools/libab/libaci_prev.so timeout 120 python tools/pivhash.py $c >> gpurun_out/r02s_hash.txt 2>&1
done
for rep in 1 2 3; do
  echo "== cur rep $rep" >> gpurun_out/r02s_ab.txt; timeout 300 python tools/time_chi.py 64,128,256 3 >> gpurun_out/r02s_ab.txt 2>&1
  echo "== prev rep $rep" >> gpurun_out/r02s_ab.txt; ACI_LIB=tools/libab/libaci_prev.so timeout 300 python tools/time_chi.py 64,128,256 3 >> gpurun_out/r02s_ab.txt 2>&1
done
