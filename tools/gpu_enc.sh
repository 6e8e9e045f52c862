# pq_encode: tensor-core form vs FFMA form (parity tests, probe, bench)
timeout 600 python -m pytest tests -m gpu -q -x -k "encode" 2>&1 | tail -1
OTF_PQ_ENCODE_FFMA=1 timeout 600 python -m pytest tests -m gpu -q -x -k "encode" 2>&1 | tail -1
for v in "OTF_X=1" "OTF_PQ_ENCODE_FFMA=1"; do
  echo "== $v"; env $v python tools/enc_probe.py
  env $v timeout 600 python bench.py --config c3e --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['ms_per_step'],2), 'ms/step', round(d['value']/1e6,1), 'M vec/s', d['clocks'])"
done
