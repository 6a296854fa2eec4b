for sk in none spmm bd gemm dwg loss optim spmm,bd gemm,dwg spmm,bd,gemm,dwg spmm,bd,gemm,dwg,loss,optim; do
GIST_SKIP=$sk python tools/proxy_step.py 8 100 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sk', round(d['us_per_step'],1))"
done
