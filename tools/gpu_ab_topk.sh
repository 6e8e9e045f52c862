# A/B of a top-k kernel change on one box: the committed file (.ab_old_topk.cu) vs the working tree
mkdir -p gpurun_out
F=paper_1407_4764_b200/csrc/otf_topk.cu
cp $F /tmp/new_topk.cu
run() {
  python -c "from paper_1407_4764_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  for c in c3 c1; do
    for rep in 1 2; do
      echo "$1 $c $(timeout 600 python bench.py --config $c --steps 200 --warmup 20 --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"]*1e3)')"
    done
  done
}
run new
timeout 1200 python -m pytest tests -m gpu -x -q -k "topk or rank or chunk or random or session or graph" 2>&1 | tail -2
cp .ab_old_topk.cu $F; run old
cp /tmp/new_topk.cu $F; run new
