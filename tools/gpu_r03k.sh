mkdir -p /tmp/nc
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm -s 600 -c 20 -o /tmp/nc/g8 python bench.py --steps 1 --warmup 1 --zeta 30 --no-cpu-baseline --no-extras --no-eval > /tmp/nc/g8.log 2>&1; echo ncu=$?
ncu -i /tmp/nc/g8.ncu-rep --page raw --csv > gpurun_out/r03k_g8_raw.csv
for i in 0 1 2 3 8 9; do ncu -i /tmp/nc/g8.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 > gpurun_out/r03k_g8_sass_$i.csv 2>/dev/null; done
ls -la gpurun_out/ | tail -8
