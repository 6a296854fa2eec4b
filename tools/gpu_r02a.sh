set -x
export GIST_GROUP=1
python bench.py --steps 2 --warmup 1 --zeta 100 --no-cpu-baseline --no-eval --profile-stride 0 > gpurun_out/r02a_g1.json 2> gpurun_out/r02a_g1.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 3000 -c 400 --csv --log-file gpurun_out/r02a_g1_launches.csv python bench.py --steps 2 --warmup 1 --zeta 100 --no-cpu-baseline --no-eval --profile-stride 0 > gpurun_out/r02a_ncu.log 2>&1
echo ncu=$?
ITERS=200 timeout 300 python tools/host_bound.py > gpurun_out/r02a_hostbound_g1.txt 2>&1
unset GIST_GROUP
ITERS=200 timeout 300 python tools/host_bound.py > gpurun_out/r02a_hostbound_g8.txt 2>&1
