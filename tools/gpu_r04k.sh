# r04k: k_bd_t with coalesced 8-row passes + pipelined TMEM loads: tests, A/B, proxy, trace
set -x
timeout 600 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_fullsize.py tests/test_gpu_heavy_rows.py -q -x --timeout 300 > gpurun_out/r04k_pytest_bf16.log 2>&1; echo bf16=$?
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2; do
  $B > gpurun_out/r04k_ab_new_$i.json 2>/dev/null; echo new=$?
  GIST_BD_T=0 $B > gpurun_out/r04k_ab_old_$i.json 2>/dev/null; echo old=$?
done
python tools/proxy_step.py > gpurun_out/r04k_proxy.log 2>&1; echo proxy=$?
GIST_BD_T=0 python tools/proxy_step.py > gpurun_out/r04k_proxy_old.log 2>&1; echo proxyold=$?
rm -rf build && GIST_EXTRA_NVCC_FLAGS=-DGIST_GEMM_TRACE python -m paper_2102_10424_b200.build > gpurun_out/r04k_build.log 2>&1; echo build=$?
GIST_GRAPH=0 python tools/bdt_trace.py > gpurun_out/r04k_trace.json 2> gpurun_out/r04k_trace.err; echo trace=$?
