python tools/proxy_step.py 8 100 3 2>&1 | grep -v Warn
timeout 900 python -m pytest tests/test_gpu_heavy_rows.py tests/test_gpu_bf16.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r03e_bench.json 2>&1; echo bench=$?
