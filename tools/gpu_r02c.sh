set -x
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_gat.py -q --timeout 300 > gpurun_out/r02c_tests.log 2>&1; echo tests=$?
GIST_GROUP=1 python bench.py --steps 2 --warmup 1 --zeta 100 --no-cpu-baseline --no-eval --no-extras --profile-stride 0 > gpurun_out/r02c_g1.json 2>&1; echo g1=$?
/usr/bin/time -v python bench.py --steps 5 --warmup 3 > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo bench=$?
