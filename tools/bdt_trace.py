#!/usr/bin/env python
"""Phase timeline of the transposed block aggregation (k_bd_t) in the C3 step (debug builds with
-DGIST_GEMM_TRACE): the last k_bd_t launch of a few eager steps (the backward pass of layer 1).
Per unit slot u of a CTA: producer start (p0), block wait done (blk), A stages issued (p1),
MMA accumulator free (m0), MMA issued (m1), epilogue accumulator ready (e0), epilogue done
(half 0: e1, half 1: e2); CTA: entry, set-up done, epilogue loop done, exit.  Prints [median, max]
over CTAs in ns relative to the first CTA entry.
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2102_10424_b200 import gist as G  # noqa: E402
from synth.planted import GRAPHS, MODELS, generate  # noqa: E402

spec = MODELS[os.environ.get("PROXY_CONFIG", "C3")]
g = generate(GRAPHS[spec.graph], seed=0, device="cuda")
c = G.Gist(spec.arch, spec.dims, optimizer="adam", precision="bf16", clusters_per_batch=spec.q, batch_seed=1)
c.load_graph(g)
c.init_params(0)
c.partition(seed=1, m=spec.m)
c.subtrain(4, 0.01, want_loss=False)
torch.cuda.synchronize()
lib = G.lib()
lib.gist_debug_bdt_trace.argtypes = [C.c_void_p]
buf = np.zeros((160, 10, 8), dtype=np.uint64)
assert lib.gist_debug_bdt_trace(buf.ctypes.data) == 0
live = buf[:, 9, 0] > 0
t = buf[live].astype(np.int64)
t0 = t[:, 9, 0].min()
names = ["p0", "p1", "m0", "m1", "e0", "e1", "e2", "blk"]
out = {"ctas": int(live.sum()), "cta": {}}
for k, nm in enumerate(["entry", "setup", "epi_loop_done", "exit"]):
    col = t[:, 9, k] - t0
    out["cta"][nm] = [int(np.median(col)), int(col.max())]
for u in range(6):
    d = {}
    for k, nm in enumerate(names):
        col = t[:, u, k]
        ok = col > t0
        if ok.sum():
            d[nm] = [int(np.median(col[ok] - t0)), int((col[ok] - t0).max()), int(ok.sum())]
    out[f"u{u}"] = d
# unit 0 of epilogue warp 0: chunk k: before tcgen05.ld, after its wait, after the transpose
col = t[:, 8, :] - t0
out["u0_chunks"] = [int(np.median(col[:, k])) for k in range(8)]
print(json.dumps(out))
c.close()
