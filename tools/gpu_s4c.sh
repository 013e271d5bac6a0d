# update kernel: loads-before-stores frame gathers (ACI_UPDILP=1, tools/libab/libaci_ilp.so) vs the in-tree library;
# parity of the variant against the oracle on configs[0,1,3]; whole-product A/B interleaved
set -x
O=gpurun_out/s4c_upd2d_ab.txt
ACI_LIB=tools/libab/libaci_ilp.so timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 600 -k "cfg0 or cfg1 or cfg3_vs_oracle or cfg3_chi256 or streamed or concurrent_and_batch or complex_cluster" > gpurun_out/s4c_ilp_tests.log 2>&1; echo "ilp tests rc=$?"; tail -3 gpurun_out/s4c_ilp_tests.log
for rep in 1 2 3; do for L in paper_2604_00037_b200/libaci.so tools/libab/libaci_ilp.so; do echo "== time_chi $L rep $rep" >> $O; ACI_LIB=$L timeout 300 python tools/time_chi.py 64,128,256 5 2>&1 >> $O; done; done
cat $O | grep -v "^   profile"
