# r05l: layer 0's dW + update in two row halves, the first half's update on a third stream
set -x
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_layer_opt.py tests/test_gpu_parity.py tests/test_gpu_bf16.py tests/test_gpu_fullsize.py tests/test_gpu_shard.py -q -x --timeout 600 > gpurun_out/r05l_pytest.log 2>&1; echo pytest=$?
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2 3; do
  $B > gpurun_out/r05l_ab_new_$i.json 2>/dev/null; echo new=$?
  GIST_DW0_SPLIT=0 $B > gpurun_out/r05l_ab_old_$i.json 2>/dev/null; echo old=$?
done
