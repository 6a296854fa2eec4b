# r05s: persistent inter-cluster pass forced in the 1/2/4-slot regimes (W = 8/4/2 proxies)
set -x
for W in 8 4 2; do
  python tools/proxy_step.py $W > gpurun_out/r05s_p${W}_auto.log 2>&1
  GIST_INTER_PERSIST=1 python tools/proxy_step.py $W > gpurun_out/r05s_p${W}_persist.log 2>&1
done
