# Profile one config's kernels: ncu launch list + one --set full capture matching $KREGEX.
# usage: CFG=c5a KREGEX="bin_score" TAG=x bash tools/gpu_prof_one.sh
mkdir -p gpurun_out
CFG=${CFG:-c2}; KREGEX=${KREGEX:-score}; TAG=${TAG:-x}
python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_$CFG.csv \
    python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_l_$CFG.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s 4 -c 2 -o gpurun_out/prof_${TAG}_$CFG \
    python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_f_$CFG.log 2>&1; echo full=$?
