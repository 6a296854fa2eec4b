set -x
CMD="python bench.py --config C3G --steps 1 --warmup 1 --zeta 30 --no-extras --no-cpu-baseline --no-eval --profile-stride 0"
$CMD > gpurun_out/r02r_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gat_(fwd|bwd_cols)" -s 20 -c 2 -o gpurun_out/r02r_gat $CMD > gpurun_out/r02r_ncu.log 2>&1; echo ncu=$?
