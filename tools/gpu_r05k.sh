# r05k: inter-cluster pass with TMA bulk gathers (k_inter_bulk): tests, A/B, proxy
set -x
timeout 1200 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_heavy_rows.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py -q -x --timeout 600 > gpurun_out/r05k_pytest.log 2>&1; echo pytest=$?
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2; do
  $B > gpurun_out/r05k_ab_new_$i.json 2>/dev/null; echo new=$?
  GIST_INTER_BULK=0 $B > gpurun_out/r05k_ab_old_$i.json 2>/dev/null; echo old=$?
done
python tools/proxy_step.py > gpurun_out/r05k_proxy.log 2>&1
GIST_INTER_BULK=0 python tools/proxy_step.py > gpurun_out/r05k_proxy_old.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 3000 -c 400 --csv --log-file gpurun_out/r05k_launches.csv python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r05k_ncu.log 2>&1; echo ncu=$?
