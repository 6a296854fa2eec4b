set -x
CMD="python bench.py --config C3G --steps 1 --warmup 1 --zeta 30 --no-extras --no-cpu-baseline --no-eval --profile-stride 0"
$CMD > gpurun_out/r02q_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 600 -c 300 --csv --log-file gpurun_out/r02q_c3g_launches.csv $CMD > gpurun_out/r02q_ncu.log 2>&1; echo ncu=$?
