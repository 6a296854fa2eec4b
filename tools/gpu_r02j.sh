set -x
timeout 1200 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_errors.py -q --timeout 600 > gpurun_out/r02j_tests.log 2>&1; echo tests=$?
python bench.py --steps 2 --warmup 1 --zeta 100 --precision tf32 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r02j_tf32.json 2>&1; echo tf32=$?
python tools/proxy_step.py 8 100 3 > gpurun_out/r02j_proxy8.json 2>&1; echo proxy=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 2000 -c 200 --csv --log-file gpurun_out/r02j_proxy8_launches.csv python tools/proxy_step.py 8 100 3 > gpurun_out/r02j_ncu.log 2>&1; echo ncu=$?
