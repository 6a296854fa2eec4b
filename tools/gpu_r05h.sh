# r05h: ncu --set full of the small critical-path kernels (loss, X copy, relayout, optimizer ranges)
set -x
mkdir -p /tmp/nc
for k in k_softmax_ce k_batch_xcopy k_adam_ranges; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 20 -c 1 -o /tmp/nc/$k python bench.py --steps 1 --warmup 1 --zeta 30 --no-cpu-baseline --no-extras --no-eval > gpurun_out/r05h_ncu_$k.log 2>&1; echo $k=$?
ncu -i /tmp/nc/$k.ncu-rep --page raw --csv > gpurun_out/r05h_${k}_raw.csv
ncu -i /tmp/nc/$k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r05h_${k}_src.csv 2>&1
done
