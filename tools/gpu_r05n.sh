# r05n: ncu --set full of one step's inter-cluster passes (the largest critical-path class) at HEAD
set -x
mkdir -p /tmp/nc
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmm -s 300 -c 7 -o /tmp/nc/spmm python bench.py --steps 1 --warmup 1 --zeta 30 --no-cpu-baseline --no-extras --no-eval > gpurun_out/r05n_ncu_spmm.log 2>&1; echo ncu=$?
cp /tmp/nc/spmm.ncu-rep gpurun_out/r05n_spmm.ncu-rep
timeout 600 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r05n_pytest.log 2>&1; echo pytest=$?
