# Build library variants for A/B runs on the GPU box: tools/var/<name>.so from "name:flags" args.
# usage: bash tools/build_variants.sh "acc1:-DOTF_MULTI_ACC_BUFS=1" "acc2:"
set -e
mkdir -p tools/var
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  OTF_NVCC_EXTRA="$flags" python paper_1407_4764_b200/_build.py --force > /dev/null
  cp paper_1407_4764_b200/libotf_b200.so tools/var/$name.so
done
python paper_1407_4764_b200/_build.py --force > /dev/null
