for env in "" "TF_CLUSTER=1"; do
  echo "== $env 64"; env $env timeout 300 python tools/stream_clock_probe.py 64 3
done
echo "== 512"; timeout 300 python tools/stream_clock_probe.py 512 2
echo "== 128"; timeout 300 python tools/stream_clock_probe.py 128 2
