# r05p: validation of HEAD with the persistent-warp inter-cluster pass: GPU tests, smoke, bench (default + reference + C3G), launch list
set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r05p_pytest.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r05p_smoke.log 2>&1; echo smoke=$?
python bench.py --steps 5 --warmup 3 > gpurun_out/r05p_bench.json 2> gpurun_out/r05p_bench.err; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r05p_ref.json 2>&1; echo ref=$?
python bench.py --config C3G --steps 3 --warmup 3 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r05p_c3g.json 2>&1; echo c3g=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 3000 -c 400 --csv --log-file gpurun_out/r05p_launches.csv python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r05p_ncu.log 2>&1; echo ncu=$?
