# r05i: batch build takes the batch's high-degree rows first (heavy list from the setup)
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_bf16.py tests/test_gpu_gat.py tests/test_gpu_fullsize.py -q -x --timeout 600 > gpurun_out/r05i_pytest.log 2>&1; echo pytest=$?
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2; do
  $B > gpurun_out/r05i_ab_new_$i.json 2>/dev/null; echo new=$?
done
python tools/proxy_step.py > gpurun_out/r05i_proxy.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_batch -s 30 -c 20 --csv --log-file gpurun_out/r05i_launches.csv python bench.py --steps 1 --warmup 1 --zeta 30 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r05i_ncu.log 2>&1; echo ncu=$?
