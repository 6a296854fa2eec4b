set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02n_ref.json 2>&1; echo ref=$?
python bench.py --config C3G --steps 3 --warmup 2 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r02n_c3g.json 2>&1; echo c3g=$?
