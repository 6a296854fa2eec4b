# r04s: isolated GEMM probe, single-CTA tiles vs CTA pairs at the 8-slot step shapes
set -x
PROBE_ONLY=fwd8,dX8,dW8,radh8 python tools/gemm_probe.py single > gpurun_out/r04s_probe.jsonl 2>&1; echo a=$?
GIST_PAIR_KMIN=64 GIST_PAIR_TILES=1 PROBE_ONLY=fwd8,dX8,dW8,radh8 python tools/gemm_probe.py pair >> gpurun_out/r04s_probe.jsonl 2>&1; echo b=$?
B="python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-eval"
$B > gpurun_out/r04s_ab_def.json 2>/dev/null; echo def=$?
GIST_PAIR_KMIN=64 GIST_PAIR_TILES=2 $B > gpurun_out/r04s_ab_pairall.json 2>/dev/null; echo pair=$?
