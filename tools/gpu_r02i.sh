set -x
timeout 600 python -m pytest tests/test_gpu_tf32.py -q --timeout 300 -k "gemm_layouts" > gpurun_out/r02i_tests.log 2>&1; echo tests=$?
