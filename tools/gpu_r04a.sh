set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r04a_pytest.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r04a_smoke.log 2>&1; echo smoke=$?
python bench.py --steps 5 --warmup 3 > gpurun_out/r04a_bench.json 2> gpurun_out/r04a_bench.err; echo bench=$?
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r04a_memcheck.log 2>&1; echo memcheck=$?
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r04a_racecheck.log 2>&1; echo racecheck=$?
timeout 900 compute-sanitizer --tool synccheck --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r04a_synccheck.log 2>&1; echo synccheck=$?
