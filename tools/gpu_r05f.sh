# r05f: L2 prefetch of the next batch's X rows by the early build (A/B: GIST_XPF=0)
set -x
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2 3; do
  $B > gpurun_out/r05f_ab_new_$i.json 2>/dev/null; echo new=$?
  GIST_XPF=0 $B > gpurun_out/r05f_ab_old_$i.json 2>/dev/null; echo old=$?
done
python tools/proxy_step.py > gpurun_out/r05f_proxy.log 2>&1
GIST_XPF=0 python tools/proxy_step.py > gpurun_out/r05f_proxy_old.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_bf16.py -q -x --timeout 300 > gpurun_out/r05f_pytest.log 2>&1; echo pytest=$?
