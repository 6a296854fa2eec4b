set -x
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py -q --timeout 600 > gpurun_out/r02l_tests.log 2>&1; echo tests=$?
python tools/proxy_step.py 8 100 3 > gpurun_out/r02l_proxy.json 2>&1
GIST_BD_FUSE=0 python tools/proxy_step.py 8 100 3 >> gpurun_out/r02l_proxy.json 2>&1
python tools/proxy_step.py 1 100 3 >> gpurun_out/r02l_proxy.json 2>&1
GIST_BD_FUSE=0 python tools/proxy_step.py 1 100 3 >> gpurun_out/r02l_proxy.json 2>&1
python bench.py --steps 3 --warmup 2 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r02l_bench.json 2>&1; echo bench=$?
