set -x
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_tf32.py tests/test_gpu_multirank.py -q --timeout 600 > gpurun_out/r02m_tests.log 2>&1; echo tests=$?
python tools/proxy_step.py 8 100 3 > gpurun_out/r02m_proxy.json 2>&1
python tools/proxy_step.py 4 100 3 >> gpurun_out/r02m_proxy.json 2>&1
python tools/proxy_step.py 1 100 3 >> gpurun_out/r02m_proxy.json 2>&1
python tools/gemm_probe.py bn64 > gpurun_out/r02m_probe.jsonl 2>&1
