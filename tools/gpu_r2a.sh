# round 2: baseline-size parity tests, wallrunner diagnostic, whole gpu suite (no -x)
mkdir -p gpurun_out
timeout 300 python tools/diag_wallrunner.py > gpurun_out/r2a_diag.log 2>&1; echo diag=$?
timeout 1500 python -m pytest tests/test_baseline_sizes.py -m gpu -q -s -rA > gpurun_out/r2a_base.log 2>&1; echo base=$?
grep -E "C1|C2|C5|passed|failed" gpurun_out/r2a_base.log | tail -12
timeout 1200 python -m pytest tests -m gpu -q --deselect tests/test_baseline_sizes.py > gpurun_out/r2a_tests.log 2>&1; echo tests=$?
tail -4 gpurun_out/r2a_tests.log
free -g | head -2; nproc; lscpu | grep "Model name"
