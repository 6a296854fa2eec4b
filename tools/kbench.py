#!/usr/bin/env python
"""Isolated kernel timings through the C-ABI kernel entry points (gist_spmm, gist_gemm).

  python tools/kbench.py spmm      # batch-shaped (C3 n_b=3106, ~58 nnz/row, cluster locality) and
                                   # full Reddit-shaped graph (HBM-bound) SpMMs, bf16
  python tools/kbench.py gemm      # the C3 sub-GCN step GEMMs and the m=1 width-4096 GEMMs, bf16 tcgen05
Prints one JSON line per case: time (CUDA events, median of reps), compulsory bytes / FLOPs and rates.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2102_10424_b200 import gist  # noqa: E402

PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def timeit(fn, reps=20, warm=3, flush=None):
    """Device time per call.  Without flush: `reps` back-to-back launches between two events
    (host work of the next call overlaps the GPU), averaged.  With flush: L2 flushed before
    every call, each timed alone, median."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    if flush is None:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def batch_csr(nb=3106, csize=155, deg_in=53, deg_out=5, seed=0):
    rng = np.random.default_rng(seed)
    rows = []
    for v in range(nb):
        c0 = (v // csize) * csize
        a = rng.integers(c0, min(c0 + csize, nb), deg_in)
        b = rng.integers(0, nb, deg_out)
        r = np.unique(np.concatenate([a, b]))
        rows.append(r[r != v])
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    return rp, np.concatenate(rows).astype(np.int32)


def spmm_case(name, rp, ci, w, dtype, scales, flush=None, reps=50):
    dev = "cuda"
    n = len(rp) - 1
    ld = (w + 7) // 8 * 8
    tdt = torch.bfloat16 if dtype == 1 else torch.float32
    e = 2 if dtype == 1 else 4
    H = torch.randn(n, ld, device=dev).to(tdt)
    out = torch.empty_like(H)
    rpd = torch.from_numpy(rp).to(dev)
    cid = torch.from_numpy(ci).to(dev)
    deg = torch.from_numpy(np.diff(rp)).to(dev).float()
    sc = (1.0 / torch.sqrt(deg + 1)).contiguous()
    rs = sc.data_ptr() if scales else None
    ms = timeit(lambda: gist.spmm(rpd.data_ptr(), cid.data_ptr(), n, rs, rs, scales, H.data_ptr(), out.data_ptr(),
                                  w, ld, dtype), reps=reps, flush=flush)
    nnz = int(rp[-1])
    comp = 8 * (n + 1) + 4 * nnz + 2 * n * ld * e + (8 * n if scales else 0)
    gather = nnz * ld * e
    print(json.dumps({"case": name, "n": n, "nnz": nnz, "w": w, "dtype": "bf16" if dtype else "f32", "ms": ms,
                      "compulsory_GBps": comp / ms / 1e6, "hbm_frac": comp / ms / 1e6 / PEAKS["hbm_gbs"],
                      "gather_GBps": gather / ms / 1e6}), flush=True)


def spmm_main():
    rp, ci = batch_csr()
    for w in (48, 512, 608, 1024):
        spmm_case("batch", rp, ci, w, 1, False)
    spmm_case("batch-scaled", rp, ci, 512, 1, True)
    spmm_case("batch-f32", rp, ci, 512, 0, True)
    from synth.planted import GRAPHS, generate
    g = generate(GRAPHS["reddit"], seed=0, device="cuda")
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for w in (512, 4096):
        spmm_case("reddit-full", g["row_ptr"], g["col_idx"], w, 1, True, flush=flush, reps=5)


def gemm_case(name, ta, tb, M, N, K, out_f32=False, relu=False, reps=50):
    dev = "cuda"
    pad = lambda x: (x + 7) // 8 * 8
    a = torch.randn((K, pad(M)) if ta else (M, pad(K)), device=dev).to(torch.bfloat16)
    b = torch.randn((N, pad(K)) if tb else (K, pad(N)), device=dev).to(torch.bfloat16)
    c = torch.empty((M, pad(N)), device=dev, dtype=torch.float32 if out_f32 else torch.bfloat16)
    ms = timeit(lambda: gist.gemm(bool(ta), bool(tb), M, N, K, a.data_ptr(), a.shape[1], b.data_ptr(), b.shape[1],
                                  c.data_ptr(), pad(N), 1, out_f32=out_f32, relu=relu), reps=reps)
    tf = 2.0 * M * N * K / ms / 1e9
    print(json.dumps({"case": name, "M": M, "N": N, "K": K, "ta": ta, "tb": tb, "ms": ms, "TFLOPs": tf,
                      "frac_burst": tf / PEAKS["bf16_tflops"]}), flush=True)


def gemm_main():
    nb = 3106
    # C3 m=8 sub-GCN step (SAGE, Kp = 1216 / 1024, Np = 512 / 48)
    gemm_case("fwd-L0", 0, 0, nb, 512, 1216, relu=True)
    gemm_case("fwd-L1", 0, 0, nb, 512, 1024, relu=True)
    gemm_case("fwd-L3", 0, 0, nb, 48, 1024, out_f32=True)
    gemm_case("dX-L1", 0, 1, nb, 1024, 512)
    gemm_case("dX-L3", 0, 1, nb, 1024, 48)
    gemm_case("dW-L0", 1, 0, 1216, 512, nb, out_f32=True)
    gemm_case("dW-L1", 1, 0, 1024, 512, nb, out_f32=True)
    gemm_case("dW-L3", 1, 0, 1024, 48, nb, out_f32=True)
    # m = 1 width-4096 (north_star GEMM target shapes)
    gemm_case("w4096-fwd", 0, 0, nb, 4096, 8192, relu=True, reps=10)
    gemm_case("w4096-dX", 0, 1, nb, 8192, 4096, reps=10)
    gemm_case("w4096-dW", 1, 0, 8192, 4096, nb, out_f32=True, reps=10)
    gemm_case("square-8192", 0, 1, 8192, 8192, 8192, reps=5)


if __name__ == "__main__":
    torch.cuda.init()
    {"spmm": spmm_main, "gemm": gemm_main}[sys.argv[1]]()
