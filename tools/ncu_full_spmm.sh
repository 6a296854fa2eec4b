# ncu --set full captures of the full-graph (Reddit-shape) SpMM: one launch per case
# usage: bash tools/ncu_full_spmm.sh <tag>
tag=${1:-r01g}
for w in 512 4096; do
  for sl in default 0; do
    if [ "$sl" = default ]; then envs=""; skip=$([ $w = 512 ] && echo 4 || echo 32); else envs="GIST_FULL_SLAB=0"; skip=2; fi
    env $envs timeout 900 ncu --set full --clock-control none -k regex:k_spmm --launch-skip $skip -c 1 \
      -o gpurun_out/${tag}_full_w${w}_slab${sl} python tools/kbench_full.py $w > gpurun_out/${tag}_full_w${w}_slab${sl}.log 2>&1
    echo w=$w slab=$sl rc=$?
  done
done
