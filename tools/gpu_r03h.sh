mkdir -p /tmp/nc
timeout 600 ncu --set full --clock-control none -k regex:k_spmm_ring -s 20 -c 2 -o /tmp/nc/ring python bench.py --steps 1 --warmup 1 --zeta 30 --no-cpu-baseline --no-extras --no-eval > /tmp/nc/ring.log 2>&1; echo ring=$?
GIST_SPMM_RING=0 timeout 600 ncu --set full --clock-control none -k regex:k_spmm -s 20 -c 2 -o /tmp/nc/reg python bench.py --steps 1 --warmup 1 --zeta 30 --no-cpu-baseline --no-extras --no-eval > /tmp/nc/reg.log 2>&1; echo reg=$?
ls -la /tmp/nc
ncu -i /tmp/nc/ring.ncu-rep --page raw --csv > gpurun_out/r03h_ring_raw.csv
ncu -i /tmp/nc/reg.ncu-rep --page raw --csv > gpurun_out/r03h_reg_raw.csv
ncu -i /tmp/nc/ring.ncu-rep --page details --csv > gpurun_out/r03h_ring_details.csv
