# binary scan: parity tests, then c5a with the IMMA kernel and with the byte-table kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "binary or bin or c5a" > gpurun_out/bin_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/bin_tests.log
timeout 600 python bench.py --config c5a --steps 10 --warmup 3 --no-cpu > gpurun_out/bin_imma.log 2>&1; echo imma=$?
OTF_BIN_BYTES=1 timeout 600 python bench.py --config c5a --steps 10 --warmup 3 --no-cpu > gpurun_out/bin_bytes.log 2>&1; echo bytes=$?
for f in bin_imma bin_bytes; do tail -1 gpurun_out/$f.log | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$f', round(d['ms_per_step'],4), 'ms', r['kernel'][:40], round(r['kernel_ms'],4), 'ms frac', round(r['frac'],3), 'e2e ms', d['e2e'].get('ms_per_query'), d['clocks'])"; done
