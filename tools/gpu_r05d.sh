# r05d: k_bd_t fix for clusters > 192 rows (four 32-row chunks per epilogue warp); checks + C3 bench
set -x
python tools/large_cluster_check.py > gpurun_out/r05d_lc.jsonl 2>&1
GIST_BD_T=0 python tools/large_cluster_check.py >> gpurun_out/r05d_lc.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_errors.py tests/test_gpu_fullsize.py -q --timeout 300 > gpurun_out/r05d_pytest.log 2>&1; echo pytest=$?
python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r05d_ab.json 2>/dev/null; echo b=$?
