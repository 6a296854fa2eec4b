cp tools/ab/T.so paper_2102_10424_b200/libgist.so; python tools/gemm_trace.py radh1 fwd1 dX1 2>&1 | grep -v Warn
bash tools/ab/run.sh "bash tools/ab/cmd3.sh" P S
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_tf32.py tests/test_gpu_heavy_rows.py -x -q 2>&1 | tail -2
