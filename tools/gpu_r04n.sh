# r04n: k_bd_t ADD residuals one chunk ahead in distinct registers; k_batch_xcopy one row per warp
set -x
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_fullsize.py tests/test_gpu_heavy_rows.py tests/test_gpu_multirank.py -q -x --timeout 300 > gpurun_out/r04n_pytest.log 2>&1; echo pytest=$?
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2; do
  $B > gpurun_out/r04n_ab_new_$i.json 2>/dev/null; echo new=$?
done
python tools/proxy_step.py > gpurun_out/r04n_proxy.log 2>&1; echo proxy=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 3000 -c 400 --csv --log-file gpurun_out/r04n_launches.csv python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r04n_ncu.log 2>&1; echo ncu=$?
