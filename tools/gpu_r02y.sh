set -x
python tools/proxy_step.py 8 100 3 > gpurun_out/r02y_proxy8.json 2>&1; echo proxy=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 2000 -c 200 --csv --log-file gpurun_out/r02y_proxy8_launches.csv python tools/proxy_step.py 8 100 3 > gpurun_out/r02y_ncu.log 2>&1; echo ncu=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_spmm|k_gemm_persist|k_batch_build" -s 300 -c 24 -o gpurun_out/r02y_full python tools/proxy_step.py 8 20 1 > gpurun_out/r02y_ncufull.log 2>&1; echo ncufull=$?
