# soak of the final build on a fresh box: consecutive chi = 256 / 64 products (bitwise identical,
# no memory growth) and concurrent-mode products from several threads
set -x
timeout 1200 python tools/soak.py > gpurun_out/s4f_soak.json 2> gpurun_out/s4f_soak.err; echo "soak rc=$?"
tail -c 1500 gpurun_out/s4f_soak.json
