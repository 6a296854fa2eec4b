set -x
timeout 1200 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_errors.py -q --timeout 600 > gpurun_out/r02h_tests.log 2>&1; echo tests=$?
python bench.py --steps 2 --warmup 1 --zeta 100 --precision tf32 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r02h_tf32.json 2>&1; echo tf32=$?
