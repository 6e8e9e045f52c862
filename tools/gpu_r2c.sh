mkdir -p gpurun_out
s=$(date +%s); timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2c_ref.log 2>&1; echo ref=$? $(( $(date +%s)-s ))s
tail -1 gpurun_out/r2c_ref.log | cut -c1-1500
s=$(date +%s); timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2c_c4.log 2>&1; echo c4=$? $(( $(date +%s)-s ))s
tail -1 gpurun_out/r2c_c4.log
