for sk in none spmm bd; do
GIST_SKIP=$sk python tools/proxy_step.py 8 100 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sk', round(d['us_per_step'],1))"
done
timeout 900 python -m pytest tests/test_gpu_heavy_rows.py tests/test_gpu_bf16.py tests/test_gpu_multirank.py -x -q 2>&1 | tail -3
