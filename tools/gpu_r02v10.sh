# streamed Pi: pivot/core hashes off vs on, then A/B product times (time_chi: 4 products, first = capture)
for c in 64 128 256; do
  echo "chi $c off: $(ACI_STREAM_PI=0 timeout 120 python tools/pivhash.py $c 2>&1 | tail -1)"
  echo "chi $c on : $(ACI_STREAM_PI=1 timeout 120 python tools/pivhash.py $c 2>&1 | tail -1)"
done
for v in "ACI_STREAM_PI=0" "ACI_STREAM_PI=1" "ACI_STREAM_MIN=0" "ACI_STREAM_PI=0" "ACI_STREAM_PI=1" "ACI_STREAM_MIN=0"; do
  echo "== $v"; env $v timeout 200 python tools/time_chi.py 64,128,256 4 2>&1 | grep -E "chi="
done
ACI_LIB=tools/libab/libaci_ts.so timeout 200 python tools/time_chi.py 256 2 2>&1 | grep -E -A1 "ts b=(0|4|8|16|24|32|36) " | head -14
