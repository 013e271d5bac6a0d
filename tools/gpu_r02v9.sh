for v in "ACI_STREAM_PI=0" "ACI_STREAM_PI=1" "ACI_STREAM_PI=0" "ACI_STREAM_PI=1"; do
  echo "== $v"; env $v timeout 200 python tools/time_chi.py 64,256 3 2>&1 | grep -E "chi=|profile"
done
