# r04p: single-sub-GCN (W = 8 proxy) profile: per-class us per step and the ncu launch list
set -x
PROXY_PROF=1 python tools/proxy_step.py > gpurun_out/r04p_proxy_prof.log 2>&1; echo prof=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 2000 -c 300 --csv --log-file gpurun_out/r04p_launches.csv python tools/proxy_step.py 8 60 1 > gpurun_out/r04p_ncu.log 2>&1; echo ncu=$?
