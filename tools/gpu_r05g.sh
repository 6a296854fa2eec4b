# r05g: bench line with per-class rooflines
set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/r05g_bench.json 2> gpurun_out/r05g_bench.err; echo bench=$?
python bench.py --precision fp32 --steps 2 --warmup 3 --zeta 100 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r05g_fp32.json 2>> gpurun_out/r05g_bench.err; echo fp32=$?
