#!/usr/bin/env python
"""Per-GPU subTrain step at world size W, on one GPU: the rank-0 context of a W-rank loopback group
owns exactly rank 0's slots (slot i on rank i mod W) and runs the same step launches (partition and
subTrain have no collective).  Prints steps/s of this GPU; used for launch lists / ncu at W = 8.

  python tools/proxy_step.py [W] [zeta] [rounds]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2102_10424_b200 import gist as G  # noqa: E402
from synth.planted import GRAPHS, MODELS, generate  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
zeta = int(sys.argv[2]) if len(sys.argv) > 2 else 100
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
spec = MODELS[os.environ.get("PROXY_CONFIG", "C3")]
g = generate(GRAPHS[spec.graph], seed=0, device="cuda")
lb = G.Loopback(W)
c = G.Gist(spec.arch, spec.dims, optimizer="adam", precision=os.environ.get("PROXY_PREC", "bf16"),
           clusters_per_batch=spec.q, batch_seed=1, rank=0, world_size=W, loopback=lb)
c.load_graph(g)
c.init_params(0)
st = torch.cuda.ExternalStream(c.stream())
ts = []
c.partition(seed=1, m=spec.m)   # one partition (subAgg is a collective: the other ranks are absent)
for t in range(rounds + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    c.subtrain(zeta, 0.01, want_loss=False)
    e1.record(st)
    torch.cuda.synchronize()
    if t:
        ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
prof = None
if os.environ.get("PROXY_PROF"):  # one more call with every step serialised and event-timed
    c.profile(1)
    c.subtrain(zeta, 0.01, want_loss=False)
    torch.cuda.synchronize()
    prof = {k: {"us_per_step": round(1e3 * v["ms"] / zeta, 2), "launches_per_step": v["launches"] / zeta}
            for k, v in c.profile_get().items() if v["launches"]}
    c.profile(0)
slots = len([i for i in range(spec.m) if i % W == 0])
print(json.dumps({"W": W, "slots": slots, "zeta": zeta, "us_per_step": 1e3 * ms / zeta,
                  "per_gpu_steps_s": slots * zeta / (ms / 1e3), "profile": prof, "env": {k: v for k, v in os.environ.items()
                                                                        if k.startswith("GIST_")}}), flush=True)
c.close()
lb.close()
