#!/usr/bin/env python
"""Device time of the tcgen05 GEMM at the C3 step shapes, host overhead removed (REPS launches of
one plan through gist_gemm_reps), for A/B comparisons of GEMM variants via environment switches.

The step's grouped launches over 8 slots are reproduced as one launch whose M (or, for dW, whose
output rows) stacks the 8 slots: the same tile count and shapes.
  python tools/gemm_probe.py [label]   -> one JSON line per shape: us per launch, TFLOP/s
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2102_10424_b200 import gist  # noqa: E402

REPS = 20
label = sys.argv[1] if len(sys.argv) > 1 else "default"
NB = 3106
ONLY = os.environ.get("PROBE_ONLY")
SHAPES = {  # name: (transA, transB, M, N, K) -- single slot and 8-slot stacks
    "fwd1": (0, 0, NB, 512, 1024), "dX1": (0, 1, NB, 1024, 512), "dW1": (1, 0, 1024, 512, NB),
    "fwd8": (0, 0, 8 * NB, 512, 1024), "dX8": (0, 1, 8 * NB, 1024, 512), "dW8": (1, 0, 8 * 1024, 512, NB),
    "w4096": (0, 0, NB, 4096, 8192),
    "radh8": (0, 1, 8 * NB, 512, 96), "radh1": (0, 1, NB, 512, 96), "out8": (0, 0, 8 * NB, 512, 64),
}
dev = "cuda"
for name, (ta, tb, M, N, K) in SHAPES.items():
    if ONLY and name not in ONLY.split(","):
        continue
    A = torch.randn((K, M) if ta else (M, K), device=dev).to(torch.bfloat16)
    B = torch.randn((N, K) if tb else (K, N), device=dev).to(torch.bfloat16)
    C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    st = torch.cuda.Stream()

    def call(reps):
        gist.gemm(bool(ta), bool(tb), M, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], C.data_ptr(), N,
                  1, out_f32=False, stream=st.cuda_stream, reps=reps)
    call(3)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        call(REPS)
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / REPS)
    us = sorted(ts)[len(ts) // 2] * 1e3
    print(json.dumps({"label": label, "shape": name, "M": M, "N": N, "K": K, "us": round(us, 2),
                      "tflops": round(2.0 * M * N * K / (us * 1e-6) / 1e12, 1)}), flush=True)
