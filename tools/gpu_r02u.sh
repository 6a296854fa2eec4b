set -x
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_gat.py -q -x -k "one_step and bf16 and ragged" > gpurun_out/r02u_san.log 2>&1; echo san=$?
