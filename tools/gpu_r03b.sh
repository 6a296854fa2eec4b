./tools/micro/chain
PROXY_PROF=1 python tools/proxy_step.py 8 100 3
