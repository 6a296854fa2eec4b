# r05o: persistent-warp inter-cluster pass for grouped launches (k_inter_persist): tests, A/B
set -x
timeout 1200 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_heavy_rows.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py -q -x --timeout 600 > gpurun_out/r05o_pytest.log 2>&1; echo pytest=$?
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2 3; do
  $B > gpurun_out/r05o_ab_new_$i.json 2>/dev/null; echo new=$?
  GIST_INTER_PERSIST=0 $B > gpurun_out/r05o_ab_old_$i.json 2>/dev/null; echo old=$?
done
