# r05m: two gathers in flight per row in the 8-slot inter-cluster pass (A/B, next to k_bd_t)
set -x
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2 3; do
  GIST_INTER_U2=1 $B > gpurun_out/r05m_ab_u2_$i.json 2>/dev/null; echo u2=$?
  $B > gpurun_out/r05m_ab_u1_$i.json 2>/dev/null; echo u1=$?
done
