# r05b: 128-wide tiles for grouped GEMMs whose 256-wide tiles spill a short last wave (8-slot dW_0); large-cluster block aggregation test
set -x
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_errors.py tests/test_gpu_multirank.py -q -x --timeout 300 > gpurun_out/r05b_pytest.log 2>&1; echo pytest=$?
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2; do
  $B > gpurun_out/r05b_ab_new_$i.json 2>/dev/null; echo new=$?
  GIST_WAVE_BN=0 $B > gpurun_out/r05b_ab_old_$i.json 2>/dev/null; echo old=$?
done
