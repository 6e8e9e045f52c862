# Copy the evidence run's outputs (tools/gpu_r2_final.sh -> gpurun_out/) into profiles/.
set -e
mkdir -p profiles/bench_r2
for f in gpurun_out/r2f_bench.log gpurun_out/r2f_c1.log gpurun_out/r2f_c2.log gpurun_out/r2f_c3.log \
         gpurun_out/r2f_c3x.log gpurun_out/r2f_c4.log gpurun_out/r2f_c5a.log gpurun_out/r2f_c5b.log \
         gpurun_out/r2f_c3e.log gpurun_out/r2f_c3k.log gpurun_out/r2f_ref.log; do
  b=$(basename "$f" .log)
  tail -1 "$f" | python -c "import json,sys; json.dump(json.loads(sys.stdin.read()), open('profiles/bench_r2/$b.json','w'), indent=1)"
done
for c in c1 c2 c3 c4 c5a c5b; do
  cp gpurun_out/launches_r2f_$c.csv profiles/launches_r2f_$c.csv
  python tools/launches.py gpurun_out/launches_r2f_$c.csv > profiles/launches_r2f_$c.txt
  python tools/ncu_summary.py gpurun_out/prof_r2f_$c.ncu-rep profiles/ncu_r2f_${c}_summary.json
  cp profiles/ncu_r2f_${c}_summary.json profiles/ncu_${c}_summary.json
done
python tools/ncu_summary.py gpurun_out/prof_r2f_pq_score.ncu-rep profiles/ncu_r2f_pq_score_summary.json
grep -A7 "^sample" gpurun_out/r2f_cut_trace.txt > profiles/cut_trace_r2_c3_summary.txt || true
grep -A7 "^sample" gpurun_out/r2f_dcut_trace.txt > profiles/dcut_trace_r2_c2_summary.txt || true
grep -v Warning gpurun_out/r2f_lat.log | grep -v "w_dev = " > profiles/latency_r2.txt
cp gpurun_out/r2f_ingest.log profiles/ingest_r2_c3_100M.txt
cp gpurun_out/r2f_pq_score.log profiles/pq_score_r2.txt
