# r04r: per-layer optimizer in the single-sub-GCN regime (GIST_LAYER_OPT=1) vs the one pass after dW_0
set -x
for i in 1 2; do
python tools/proxy_step.py > gpurun_out/r04r_proxy_one_$i.log 2>&1; echo proxy=$?
GIST_LAYER_OPT=1 python tools/proxy_step.py > gpurun_out/r04r_proxy_layer_$i.log 2>&1; echo proxy=$?
done
GIST_LAYER_OPT=1 python tools/proxy_step.py 4 > gpurun_out/r04r_proxy4_layer.log 2>&1; echo proxy=$?
python tools/proxy_step.py 4 > gpurun_out/r04r_proxy4_one.log 2>&1; echo proxy=$?
python tools/proxy_step.py 2 > gpurun_out/r04r_proxy2.log 2>&1; echo proxy=$?
GIST_LAYER_OPT=0 python tools/proxy_step.py 2 > gpurun_out/r04r_proxy2_one.log 2>&1; echo proxy=$?
