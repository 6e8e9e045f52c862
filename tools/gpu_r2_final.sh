# Round-2 evidence run: tests, the default bench line, one line per config, A/B of the fused
# dense path, ncu launch lists + one --set full capture per config, phase traces, latency probe,
# ingest bench. Everything lands in gpurun_out/r2f_*.
mkdir -p gpurun_out
line() { tail -1 $1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; e=d['e2e']
print('$2', 'step_ms', round(d['ms_per_step'],4), 'value', '%.4g' % d['value'], 'kernel_ms', round(r.get('kernel_ms',0),4), 'frac', round(r['frac'],3) if r.get('frac') else None, 'e2e_ms', round(e.get('ms_per_query', 0),4), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'], 'launches', d['gpu_launches'])"; }
s=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2f_tests.log 2>&1; echo tests=$? $(( $(date +%s)-s ))s; tail -2 gpurun_out/r2f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2f_bench.log 2>&1; echo bench=$?; line gpurun_out/r2f_bench.log default
for c in c1 c2 c3 c3x c4 c5a c5b c3e c3k; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/r2f_$c.log 2>&1; line gpurun_out/r2f_$c.log $c
done
for c in c1 c2 c4; do
  OTF_DENSE_NO_CUT=1 timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-train > gpurun_out/r2f_${c}_nocut.log 2>&1; line gpurun_out/r2f_${c}_nocut.log "$c-nocut"
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-train > gpurun_out/r2f_${c}_cut.log 2>&1; line gpurun_out/r2f_${c}_cut.log "$c-cut"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2f_ref.log 2>&1; echo ref=$?; tail -1 gpurun_out/r2f_ref.log | cut -c1-400
for spec in "c1:dense_rank_cut:1" "c2:dense_rank_cut:1" "c4:dense_rank_cut:1" "c3:pq_rank_cut|pq_build_lut:2" "c5a:bin_score|topk:3" "c5b:multi_score|topk_seg:2"; do
  IFS=: read cfg kr cnt <<< "$spec"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2f_$cfg.csv \
      python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-train > /dev/null 2>&1; echo launches_$cfg=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kr" -s 4 -c $cnt -o gpurun_out/prof_r2f_$cfg \
      python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-train > /dev/null 2>&1; echo full_$cfg=$?
done
bash tools/gpu_cut_trace.sh > gpurun_out/r2f_cut_trace.txt 2>&1; tail -8 gpurun_out/r2f_cut_trace.txt
CFG=c2 bash tools/gpu_dcut_trace.sh > gpurun_out/r2f_dcut_trace.txt 2>&1; tail -8 gpurun_out/r2f_dcut_trace.txt
timeout 600 python tools/latency_probe.py c1 c3 c2 > gpurun_out/r2f_lat.log 2>&1; tail -12 gpurun_out/r2f_lat.log
timeout 900 python tools/ingest_bench.py 100000000 /tmp > gpurun_out/r2f_ingest.log 2>&1; tail -4 gpurun_out/r2f_ingest.log
timeout 300 python tools/pq_score_probe.py > gpurun_out/r2f_pq_score.log 2>&1; OTF_PQ_SCORE_XOR=1 timeout 300 python tools/pq_score_probe.py >> gpurun_out/r2f_pq_score.log 2>&1; cat gpurun_out/r2f_pq_score.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pq_score16 -s 3 -c 1 -o gpurun_out/prof_r2f_pq_score python tools/pq_score_probe.py > /dev/null 2>&1; echo full_pq_score=$?
timeout 900 python tools/stress_cut.py 24 > gpurun_out/r2f_stress.log 2>&1; tail -3 gpurun_out/r2f_stress.log
timeout 600 python tools/seg_probe.py 10000000 128 > gpurun_out/r2f_seg.log 2>&1; tail -1 gpurun_out/r2f_seg.log
