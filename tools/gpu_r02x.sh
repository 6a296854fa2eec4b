set -x
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02x_pytest.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02x_smoke.log 2>&1; echo smoke=$?
python bench.py --steps 3 --warmup 2 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r02x_bench.json 2>&1; echo bench=$?
