set -x
start=$(date +%s)
python bench.py --steps 5 --warmup 3 > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo bench=$? secs=$(( $(date +%s) - start ))
for i in 1 2; do
GIST_PAIR_KMIN=0 GIST_PAIR_TILES=0 python bench.py --steps 3 --warmup 2 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r02d_pair$i.json 2>&1; echo pair=$?
python bench.py --steps 3 --warmup 2 --no-extras --no-cpu-baseline --no-eval > gpurun_out/r02d_base$i.json 2>&1; echo base=$?
done
