# r04d: transposed block-diagonal aggregation (k_bd_t): GPU tests, A/B vs the row-tile kernel, proxy
set -x
timeout 600 python -m pytest tests/test_gpu_bf16.py -q -x --timeout 300 > gpurun_out/r04d_pytest_bf16.log 2>&1; echo bf16=$?
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r04d_pytest.log 2>&1; echo pytest=$?
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2; do
  $B > gpurun_out/r04d_ab_new_$i.json 2>/dev/null; echo new=$?
  GIST_BD_T=0 $B > gpurun_out/r04d_ab_old_$i.json 2>/dev/null; echo old=$?
done
python tools/proxy_step.py > gpurun_out/r04d_proxy.log 2>&1; echo proxy=$?
GIST_BD_T=0 python tools/proxy_step.py > gpurun_out/r04d_proxy_old.log 2>&1; echo proxyold=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 3000 -c 400 --csv --log-file gpurun_out/r04d_launches.csv python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r04d_ncu.log 2>&1; echo ncu=$?
