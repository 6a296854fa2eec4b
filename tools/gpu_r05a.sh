# r05a: short-K GEMMs (K <= 128) on a 2-stage ring with double-buffered epilogue staging; ncu full of one step's GEMMs
set -x
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_multirank.py -q -x --timeout 300 > gpurun_out/r05a_pytest.log 2>&1; echo pytest=$?
PROBE_ONLY=radh8,radh1 python tools/gemm_probe.py shortk > gpurun_out/r05a_probe.jsonl 2>&1
GIST_SHORTK_EPI=0 PROBE_ONLY=radh8,radh1 python tools/gemm_probe.py default >> gpurun_out/r05a_probe.jsonl 2>&1
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2; do
  $B > gpurun_out/r05a_ab_new_$i.json 2>/dev/null; echo new=$?
  GIST_SHORTK_EPI=0 $B > gpurun_out/r05a_ab_old_$i.json 2>/dev/null; echo old=$?
done
python tools/proxy_step.py > gpurun_out/r05a_proxy.log 2>&1; echo proxy=$?
GIST_SHORTK_EPI=0 python tools/proxy_step.py > gpurun_out/r05a_proxy_old.log 2>&1; echo proxy=$?
mkdir -p /tmp/nc
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_persist -s 600 -c 14 -o /tmp/nc/gemm python bench.py --steps 1 --warmup 1 --zeta 30 --no-cpu-baseline --no-extras --no-eval > gpurun_out/r05a_ncu_gemm.log 2>&1; echo ncu=$?
cp /tmp/nc/gemm.ncu-rep gpurun_out/r05a_gemm.ncu-rep
