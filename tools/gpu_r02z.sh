set -x
timeout 900 python -m pytest tests/test_gpu_heavy_rows.py -x -q > gpurun_out/r02z_heavy.log 2>&1; echo heavy=$?
tail -30 gpurun_out/r02z_heavy.log
python tools/proxy_step.py 8 100 3 > gpurun_out/r02z_proxy8.json 2>&1; echo proxy=$?; cat gpurun_out/r02z_proxy8.json
timeout 1500 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py tests/test_gpu_eval.py -x -q > gpurun_out/r02z_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r02z_pytest.log
python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r02z_bench.json 2>&1; echo bench=$?
