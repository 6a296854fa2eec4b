# r05e: validation of HEAD: GPU tests, smoke, bench (default + reference arm + C3G), launch list, ncu full of one step's GEMMs / block aggregations
set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r05e_pytest.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r05e_smoke.log 2>&1; echo smoke=$?
python bench.py --steps 5 --warmup 3 > gpurun_out/r05e_bench.json 2> gpurun_out/r05e_bench.err; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r05e_ref.json 2>&1; echo ref=$?
python bench.py --config C3G --steps 3 --warmup 3 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r05e_c3g.json 2>&1; echo c3g=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 3000 -c 400 --csv --log-file gpurun_out/r05e_launches.csv python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r05e_ncu.log 2>&1; echo ncu=$?
mkdir -p /tmp/nc
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_persist -s 600 -c 14 -o /tmp/nc/gemm python bench.py --steps 1 --warmup 1 --zeta 30 --no-cpu-baseline --no-extras --no-eval > gpurun_out/r05e_ncu_gemm.log 2>&1; echo ncu=$?
cp /tmp/nc/gemm.ncu-rep gpurun_out/r05e_gemm.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bd_t -s 700 -c 7 -o /tmp/nc/bdt python bench.py --steps 1 --warmup 1 --zeta 30 --no-cpu-baseline --no-extras --no-eval > gpurun_out/r05e_ncu_bdt.log 2>&1; echo ncu=$?
cp /tmp/nc/bdt.ncu-rep gpurun_out/r05e_bdt.ncu-rep
