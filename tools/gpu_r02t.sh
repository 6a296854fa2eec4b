set -x
timeout 900 python -m pytest tests/test_gpu_gat.py tests/test_gpu_multirank.py tests/test_gpu_eval.py -q --timeout 600 -k "gat or GAT" > gpurun_out/r02t_tests.log 2>&1; echo tests=$?
python bench.py --config C3G --steps 3 --warmup 2 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r02t_c3g.json 2>&1; echo c3g=$?
