# round 2: default bench (c4 shard + trainer) both arms as the driver runs them, diag, concurrency x3
mkdir -p gpurun_out
timeout 300 python tools/diag_wallrunner.py > gpurun_out/r2b_diag.log 2>&1; echo diag=$?; cat gpurun_out/r2b_diag.log | cut -c1-200
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_concurrency.py -q -x 2>&1 | tail -1; done
/usr/bin/time -v timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2b_ref.log 2> gpurun_out/r2b_ref.err; echo ref=$?
tail -1 gpurun_out/r2b_ref.log | cut -c1-600; grep -E "Maximum resident|Elapsed" gpurun_out/r2b_ref.err
/usr/bin/time -v timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2b_c4.log 2> gpurun_out/r2b_c4.err; echo c4=$?
tail -1 gpurun_out/r2b_c4.log; grep -E "Maximum resident|Elapsed" gpurun_out/r2b_c4.err; tail -3 gpurun_out/r2b_c4.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --config c2 > gpurun_out/r2b_c2.log 2>&1; echo c2=$?
tail -1 gpurun_out/r2b_c2.log
