# r05r: HEAD with k_inter_persist rows dealt over 8x the resident warps: GPU tests, smoke, bench, launch list
set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r05r_pytest.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r05r_smoke.log 2>&1; echo smoke=$?
python bench.py --steps 5 --warmup 3 > gpurun_out/r05r_bench.json 2> gpurun_out/r05r_bench.err; echo bench=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 3000 -c 400 --csv --log-file gpurun_out/r05r_launches.csv python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r05r_ncu.log 2>&1; echo ncu=$?
