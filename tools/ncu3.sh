set -x
for k in k_softmax_ce k_batch_build k_adam; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 30 -c 1 -o gpurun_out/r01g_$k python bench.py --steps 1 --warmup 1 --zeta 50 --no-cpu-baseline --no-eval > gpurun_out/ncu_$k.log 2>&1
echo $k=$?
done
