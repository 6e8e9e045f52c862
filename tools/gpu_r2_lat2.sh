mkdir -p gpurun_out
for v in "" "OTF_HOST_D2H_COPY=1" "OTF_PROBE_NO_H2D=1" "OTF_PROBE_NO_H2D=1 OTF_HOST_D2H_COPY=1"; do
  echo "== $v"; env $v timeout 600 python tools/latency_probe.py c1 2>&1 | tail -4
done
