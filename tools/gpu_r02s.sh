set -x
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_tf32.py -q --timeout 600 -x > gpurun_out/r02s_tests.log 2>&1; echo tests=$?
for i in 1 2; do python bench.py --steps 3 --warmup 2 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r02s_bench$i.json 2>&1; done
python tools/proxy_step.py 8 100 3 > gpurun_out/r02s_proxy.json 2>&1
