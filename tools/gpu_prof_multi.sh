# ncu --set full capture of the multi-classifier kernel at a reduced row count.
mkdir -p gpurun_out
export OTF_BENCH_ROWS=${ROWS:-1000000}
python bench.py --config c5b --steps 3 --warmup 3 --no-cpu > gpurun_out/pm_plain.log 2>&1; echo plain=$?
ncu --set full --clock-control none --import-source on -k regex:multi_score_tc -s 3 -c 1 -o gpurun_out/prof_${TAG:-m}_c5b \
    python bench.py --config c5b --steps 3 --warmup 3 --no-cpu > gpurun_out/pm_ncu.log 2>&1; echo full=$?
