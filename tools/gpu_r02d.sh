set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for rep in 1 2; do
for v in cur notma nolpair nolpair_nocoop; do
  case $v in
    cur) L=paper_2604_00037_b200/libaci.so; C=1;;
    notma) L=tools/libab/libaci_notma.so; C=1;;
    nolpair) L=tools/libab/libaci_nolpair.so; C=1;;
    nolpair_nocoop) L=tools/libab/libaci_nolpair.so; C=0;;
  esac
  echo "== $v rep $rep" >> gpurun_out/r02d_ab.txt
  ACI_LIB=$L ACI_PRRLU_COOP=$C timeout 300 python tools/time_chi.py 64,128,256 4 >> gpurun_out/r02d_ab.txt 2>&1
done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "rook or concurrent or tiers or batch or cfg0" -p no:cacheprovider > gpurun_out/r02d_gputests.log 2>&1; echo "pytest rc=$?"
