set -x
CMD="python bench.py --steps 1 --warmup 1 --zeta 20 --no-extras --no-cpu-baseline --no-eval --profile-stride 0"
$CMD > gpurun_out/r02e_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm_persist -s 300 -c 4 -o gpurun_out/r02e_gemm $CMD > gpurun_out/r02e_ncu.log 2>&1
echo ncu=$?
timeout 1200 python -m pytest tests/test_gpu_gat.py tests/test_gpu_eval.py tests/test_gpu_bf16.py -q --timeout 600 > gpurun_out/r02e_tests.log 2>&1; echo tests=$?
