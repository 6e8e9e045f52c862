# compute-sanitizer over every kernel family (tools/sanitize_driver.py); summaries -> gpurun_out/san_*.log
mkdir -p gpurun_out
timeout 300 python tools/sanitize_driver.py > gpurun_out/san_plain.log 2>&1; echo plain=$?; tail -1 gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck; do
  for case in dense topk pq pqcut binary multi train encode kmeans; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_driver.py $case > gpurun_out/san_${tool}_${case}.log 2>&1
    echo $tool $case rc=$? $(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error" gpurun_out/san_${tool}_${case}.log | tail -2 | tr '\n' ' ')
  done
done
