# r04q: one-pass optimizer after dW_0 on the dW stream (one group) beside the next batch's build
set -x
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py tests/test_gpu_bf16.py tests/test_gpu_shard.py -q -x --timeout 600 > gpurun_out/r04q_pytest.log 2>&1; echo pytest=$?
python tools/proxy_step.py > gpurun_out/r04q_proxy.log 2>&1; echo proxy=$?
python tools/proxy_step.py 4 > gpurun_out/r04q_proxy4.log 2>&1; echo proxy=$?
python tools/proxy_step.py 8 > gpurun_out/r04q_proxy_b.log 2>&1; echo proxy=$?
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
$B > gpurun_out/r04q_ab_new_1.json 2>/dev/null; echo new=$?
