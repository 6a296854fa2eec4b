set -x
timeout 900 python -m pytest tests/test_gpu_multirank.py -q --timeout 300 > gpurun_out/r02b_multirank.log 2>&1; echo multirank=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; echo smoke=$?
python bench.py --steps 3 --warmup 3 --no-eval --no-cpu-baseline > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo bench=$?
GIST_GROUP=1 python bench.py --steps 2 --warmup 1 --zeta 100 --no-cpu-baseline --no-eval --profile-stride 0 > gpurun_out/r02b_g1.json 2>&1; echo g1=$?
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r02b_pytest.log 2>&1; echo pytest=$?
