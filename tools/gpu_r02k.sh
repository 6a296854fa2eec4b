set -x
python tools/proxy_step.py 8 100 3 > gpurun_out/r02k_proxy8.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 2000 -c 200 --csv --log-file gpurun_out/r02k_proxy8_launches.csv python tools/proxy_step.py 8 100 3 > gpurun_out/r02k_ncu.log 2>&1; echo ncu=$?
GIST_GRAPH=0 python tools/proxy_step.py 8 100 3 >> gpurun_out/r02k_proxy8.json 2>&1
GIST_DW_STREAM=0 python tools/proxy_step.py 8 100 3 >> gpurun_out/r02k_proxy8.json 2>&1
GIST_PDL=0 python tools/proxy_step.py 8 100 3 >> gpurun_out/r02k_proxy8.json 2>&1
GIST_BD=0 python tools/proxy_step.py 8 100 3 >> gpurun_out/r02k_proxy8.json 2>&1
GIST_REASSOC=0 python tools/proxy_step.py 8 100 3 >> gpurun_out/r02k_proxy8.json 2>&1
