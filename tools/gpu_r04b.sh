# r04b: A/B of CTA pairs on the C3 step GEMMs (env thresholds) + ncu --set full of one step's
# block-diagonal aggregations and plain GEMMs (8-slot C3)
set -x
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
for i in 1 2; do
  $B > gpurun_out/r04b_ab_default_$i.json 2>/dev/null; echo def=$?
  GIST_PAIR_KMIN=1024 GIST_PAIR_TILES=2 $B > gpurun_out/r04b_ab_pair1024_$i.json 2>/dev/null; echo pair=$?
  GIST_PAIR_KMIN=3000 GIST_PAIR_TILES=0 $B > gpurun_out/r04b_ab_pairdw_$i.json 2>/dev/null; echo pairdw=$?
done
mkdir -p /tmp/nc
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_persist -s 1900 -c 19 -o /tmp/nc/step python bench.py --steps 1 --warmup 1 --zeta 30 --no-cpu-baseline --no-extras --no-eval > gpurun_out/r04b_ncu.log 2>&1; echo ncu=$?
ncu -i /tmp/nc/step.ncu-rep --page raw --csv > gpurun_out/r04b_step_raw.csv
ncu -i /tmp/nc/step.ncu-rep --page details --csv > gpurun_out/r04b_step_details.csv 2>&1
cp /tmp/nc/step.ncu-rep gpurun_out/r04b_step.ncu-rep
