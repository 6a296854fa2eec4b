mkdir -p /tmp/nc
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_persist -s 603 -c 1 -o /tmp/nc/bd python bench.py --steps 1 --warmup 1 --zeta 30 --no-cpu-baseline --no-extras --no-eval > /tmp/nc/bd.log 2>&1; echo ncu=$?
ncu -i /tmp/nc/bd.ncu-rep --page raw --csv > gpurun_out/r03n_bd_raw.csv
ncu -i /tmp/nc/bd.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r03n_bd_src.csv 2>&1
ncu -i /tmp/nc/bd.ncu-rep --page details --csv > gpurun_out/r03n_bd_details.csv 2>&1
