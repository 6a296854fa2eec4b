# r05u: final full bench line at HEAD (+ reference arm)
set -x
python bench.py > gpurun_out/r05u_bench.json 2> gpurun_out/r05u_bench.err; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r05u_ref.json 2>&1; echo ref=$?
