# r05j: critical-path probe (temporary GIST_SKIP build, results meaningless except for timing): drop one kernel class from the step, re-time
set -x
for sk in none spmm bd gemm dwg loss opt batch xcopy; do
  GIST_SKIP=$sk python tools/proxy_step.py 8 60 2 > gpurun_out/r05j_p8_$sk.log 2>&1
  GIST_SKIP=$sk python tools/proxy_step.py 1 30 2 > gpurun_out/r05j_p1_$sk.log 2>&1
done
