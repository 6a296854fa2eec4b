mkdir -p /tmp/nc
PROBE_ONLY=radh1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm -s 5 -c 1 -o /tmp/nc/radh1 python tools/gemm_probe.py > /tmp/nc/l.log 2>&1; echo ncu=$?
ncu -i /tmp/nc/radh1.ncu-rep --page raw --csv > gpurun_out/r03l_radh1_raw.csv
ncu -i /tmp/nc/radh1.ncu-rep --page source --csv --print-source cuda > gpurun_out/r03l_radh1_cuda.csv 2>&1
ncu -i /tmp/nc/radh1.ncu-rep --page source --csv --print-source sass > gpurun_out/r03l_radh1_sass.csv 2>&1
ncu -i /tmp/nc/radh1.ncu-rep --page details --csv > gpurun_out/r03l_radh1_details.csv 2>&1
