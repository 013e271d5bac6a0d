# streamed Pi A/B: poll back-off
for v in "ACI_STREAM_PI=0" "ACI_STREAM_POLL_NS=128" "ACI_STREAM_POLL_NS=1000" "ACI_STREAM_POLL_NS=4000" "ACI_STREAM_PI=0"; do
  echo "== $v"; env $v timeout 200 python tools/time_chi.py 64,256 4 2>&1 | grep chi=
done
