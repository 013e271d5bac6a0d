# streamed Pi: hashes vs off, A/B timing, device timestamps
for c in 64 128 256; do
  echo "chi $c off: $(ACI_STREAM_PI=0 timeout 120 python tools/pivhash.py $c 2>&1 | tail -1)"
  echo "chi $c on : $(ACI_STREAM_PI=1 timeout 120 python tools/pivhash.py $c 2>&1 | tail -1)"
done
for v in "ACI_STREAM_PI=0" "ACI_STREAM_PI=1" "ACI_STREAM_PI=0" "ACI_STREAM_PI=1"; do
  echo "== $v"; env $v timeout 200 python tools/time_chi.py 64,128,256 4 2>&1 | grep chi=
done
ACI_LIB=tools/libab/libaci_ts.so timeout 200 python tools/time_chi.py 256 2 2>&1 | grep -E -A1 "ts b=" | head -16
ACI_LIB=tools/libab/libaci_ts.so timeout 200 python tools/time_chi.py 64 2 2>&1 | grep -E -A1 "ts b=" | head -16
