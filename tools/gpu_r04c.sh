# r04c: early next-batch build inside the backward + H W_top on the side stream: GPU tests, A/B
set -x
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r04c_pytest.log 2>&1; echo pytest=$?
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2; do
  $B > gpurun_out/r04c_ab_new_$i.json 2>/dev/null; echo new=$?
  GIST_BATCH_PREFETCH=1 $B > gpurun_out/r04c_ab_late_$i.json 2>/dev/null; echo late=$?
done
python tools/proxy_step.py > gpurun_out/r04c_proxy.log 2>&1; echo proxy=$?
GIST_BATCH_PREFETCH=1 python tools/proxy_step.py > gpurun_out/r04c_proxy_late.log 2>&1; echo proxylate=$?
python tools/proxy_step.py > gpurun_out/r04c_proxy2.log 2>&1; echo proxy=$?
