# r05q: k_inter_persist row dealing sweep (rows per warp from N x 8 warps x SMs)
set -x
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2; do
for n in 2 4 8 16; do
  GIST_IP_CTAS=$n $B > gpurun_out/r05q_ab_${n}_$i.json 2>/dev/null; echo n$n=$?
done
done
