# r04o: k_bd_t with one cluster-block buffer (room for the early-gather inter-cluster pass beside it) vs two
set -x
timeout 900 python -m pytest tests/test_gpu_bf16.py -q -x --timeout 300 > gpurun_out/r04o_pytest.log 2>&1; echo pytest=$?
GIST_BDT_BUFS=1 timeout 900 python -m pytest tests/test_gpu_bf16.py -q -x --timeout 300 > gpurun_out/r04o_pytest1.log 2>&1; echo pytest1=$?
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2; do
  $B > gpurun_out/r04o_ab_two_$i.json 2>/dev/null; echo two=$?
  GIST_BDT_BUFS=1 $B > gpurun_out/r04o_ab_one_$i.json 2>/dev/null; echo one=$?
done
python tools/proxy_step.py > gpurun_out/r04o_proxy_two.log 2>&1; echo proxy=$?
GIST_BDT_BUFS=1 python tools/proxy_step.py > gpurun_out/r04o_proxy_one.log 2>&1; echo proxy=$?
