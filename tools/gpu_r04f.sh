# r04f: k_bd_t epilogue through a shared-memory transpose (row-major 16-byte residual loads and stores)
set -x
timeout 600 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_fullsize.py -q -x --timeout 300 > gpurun_out/r04f_pytest_bf16.log 2>&1; echo bf16=$?
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2; do
  $B > gpurun_out/r04f_ab_new_$i.json 2>/dev/null; echo new=$?
  GIST_BD_T=0 $B > gpurun_out/r04f_ab_old_$i.json 2>/dev/null; echo old=$?
done
python tools/proxy_step.py > gpurun_out/r04f_proxy.log 2>&1; echo proxy=$?
GIST_BD_T=0 python tools/proxy_step.py > gpurun_out/r04f_proxy_old.log 2>&1; echo proxyold=$?
mkdir -p /tmp/nc
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bd_t -s 300 -c 2 -o /tmp/nc/bdt python bench.py --steps 1 --warmup 1 --zeta 30 --no-cpu-baseline --no-extras --no-eval > gpurun_out/r04f_ncu.log 2>&1; echo ncu=$?
ncu -i /tmp/nc/bdt.ncu-rep --page raw --csv > gpurun_out/r04f_bdt_raw.csv
ncu -i /tmp/nc/bdt.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r04f_bdt_src.csv 2>&1
