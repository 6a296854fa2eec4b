# r05t: persistent inter-cluster pass from 8,192 rows (4-slot launches): GPU tests + proxies
set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r05t_pytest.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r05t_smoke.log 2>&1; echo smoke=$?
python tools/proxy_step.py 2 > gpurun_out/r05t_p2.log 2>&1
python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r05t_ab.json 2>/dev/null; echo b=$?
