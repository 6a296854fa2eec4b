set -x
timeout 600 python -m pytest tests/test_gpu_p2p_agg.py -q --timeout 300 > gpurun_out/r02o_tests.log 2>&1; echo tests=$?
