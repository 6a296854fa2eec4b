#!/usr/bin/env python
"""Phase timeline of the tcgen05 GEMM's first tile per CTA (debug builds with -DGIST_GEMM_TRACE:
GIST_EXTRA_NVCC_FLAGS=-DGIST_GEMM_TRACE).  One launch of a probe shape after warm-up; prints the
median / max over CTAs of each phase (ns, relative to the earliest CTA entry).
  python tools/gemm_trace.py fwd1|dX1|dW1|radh1|fwd8|...
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2102_10424_b200 import gist  # noqa: E402

NB = 3106
SHAPES = {"fwd1": (0, 0, NB, 512, 1024), "dX1": (0, 1, NB, 1024, 512), "dW1": (1, 0, 1024, 512, NB),
          "radh1": (0, 1, NB, 512, 96), "fwd8": (0, 0, 8 * NB, 512, 1024), "out8": (0, 0, 8 * NB, 512, 64)}
PH = ["entry", "pdl_wait", "tma_issue", "stage0_landed", "mma_done", "acc_ready", "epi_done", "exit", "epi_tmem_ld0", "epi_box_staged", "epi_store_issued", "", "before_wait"]
for name in sys.argv[1:]:
    ta, tb, M, N, K = SHAPES[name]
    A = torch.randn((K, M) if ta else (M, K), device="cuda").to(torch.bfloat16)
    B = torch.randn((N, K) if tb else (K, N), device="cuda").to(torch.bfloat16)
    Cm = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    call = lambda r: gist.gemm(bool(ta), bool(tb), M, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1],
                               Cm.data_ptr(), N, 1, out_f32=False, reps=r)
    call(5)
    torch.cuda.synchronize()
    buf = np.zeros((1024, 16), dtype=np.uint64)
    lib = gist.lib()
    lib.gist_debug_gemm_trace.argtypes = [C.c_void_p, C.c_int]
    lib.gist_debug_gemm_trace(buf.ctypes.data, 1024)   # clear view of the last warm-up launch
    buf[:] = 0
    lib.gist_debug_gemm_trace  # noqa
    call(1)
    torch.cuda.synchronize()
    lib.gist_debug_gemm_trace(buf.ctypes.data, 1024)
    live = buf[:, 0] > 0
    t = buf[live].astype(np.int64)
    t0 = t[:, 0].min()
    rel = t - t0
    out = {"shape": name, "ctas": int(live.sum())}
    for k, p in enumerate(PH):
        if not p:
            continue
        col = rel[:, k]
        out[p] = [int(np.median(col)), int(col.max())]
    out["kernel_span_ns"] = int(rel.max())
    print(json.dumps(out), flush=True)
