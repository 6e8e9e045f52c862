# Round-2 validation of HEAD: full -m gpu suite, smoke, default bench line, one line per config.
mkdir -p gpurun_out
s=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/v_tests.log 2>&1; echo tests=$? $(( $(date +%s)-s ))s; tail -3 gpurun_out/v_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/v_smoke.log
s=$(date +%s); timeout 900 python bench.py > gpurun_out/v_bench.log 2>&1; echo bench=$? $(( $(date +%s)-s ))s; tail -1 gpurun_out/v_bench.log | cut -c1-3000
bash tools/gpu_all_configs.sh
