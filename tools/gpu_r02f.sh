set -x
python tools/gemm_probe.py default > gpurun_out/r02f_probe.jsonl 2>&1; echo probe=$?
GIST_PAIR_KMIN=0 GIST_PAIR_TILES=0 python tools/gemm_probe.py pairs >> gpurun_out/r02f_probe.jsonl 2>&1; echo probe=$?
GIST_PAIR_KMIN=0 GIST_PAIR_TILES=0 GIST_BN_FEW=0 python tools/gemm_probe.py pairs_bn256 >> gpurun_out/r02f_probe.jsonl 2>&1; echo probe=$?
GIST_BN_FEW=0 python tools/gemm_probe.py bn256 >> gpurun_out/r02f_probe.jsonl 2>&1; echo probe=$?
timeout 1200 python -m pytest tests/test_gpu_gat.py tests/test_gpu_eval.py -q --timeout 600 -x > gpurun_out/r02f_tests.log 2>&1; echo tests=$?
