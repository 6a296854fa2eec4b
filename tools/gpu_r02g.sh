set -x
python tools/gemm_probe.py default > gpurun_out/r02g_probe.jsonl 2>&1; echo probe=$?
GIST_PAIR_KMIN=0 GIST_PAIR_TILES=0 python tools/gemm_probe.py pairs >> gpurun_out/r02g_probe.jsonl 2>&1; echo probe=$?
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r02g_pytest.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; echo smoke=$?
