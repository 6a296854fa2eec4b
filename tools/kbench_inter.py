#!/usr/bin/env python
"""Microbenchmark of the few-neighbour sparse pass shape (the inter-cluster edges of a C3
batch group: 8 x 3,120 rows, 512 bf16 columns, ~5.5 neighbours per row) through gist_spmm,
with and without a heavy tail of long rows.  Prints one line per case: us per launch."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_10424_b200 import gist  # noqa: E402


def run(deg, w=512, ld=1024, reps=50, block=0, rowscale=False, cold=False):
    """block > 0: neighbours drawn inside the row's own block of `block` rows (the 8 slots of a
    grouped launch each gather inside their own 3,120-row batch)."""
    rows = len(deg)
    rng = np.random.default_rng(0)
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    if block:
        owner = np.repeat(np.arange(rows) // block * block, deg)
        col = (owner + rng.integers(0, block, rp[-1])).astype(np.int32)
    else:
        col = rng.integers(0, rows, rp[-1]).astype(np.int32)
    dev = torch.device("cuda")
    rpd, cd = torch.from_numpy(rp).to(dev), torch.from_numpy(col).to(dev)
    H = torch.randn(rows, ld, device=dev).to(torch.bfloat16)
    out = torch.zeros_like(H)
    sc = torch.rand(rows, device=dev) if rowscale else None
    f = lambda: gist.spmm(rpd.data_ptr(), cd.data_ptr(), rows, sc.data_ptr() if rowscale else None, None, False,
                          H.data_ptr(), out.data_ptr(), w, ld, 1)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    if cold:  # L2 flushed before every call (256 MiB write), each call timed alone
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        return float(np.median(ts))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


if __name__ == "__main__":
    rows = 8 * 3120
    rng = np.random.default_rng(1)
    base = rng.poisson(5.4, rows).astype(np.int64)
    print("uniform-ish poisson(5.4):", round(run(base), 1), "us")
    t = base.copy(); t[rng.choice(rows, 8, replace=False)] = 60
    print("+ 8 rows of 60:", round(run(t), 1), "us")
    t = base.copy(); t[rng.choice(rows, 250, replace=False)] = 22
    print("+ 250 rows of 22 (p99):", round(run(t), 1), "us")
    print("all zero:", round(run(np.zeros(rows, np.int64)), 1), "us")
    print("all 6:", round(run(np.full(rows, 6, np.int64)), 1), "us")
    print("poisson(5.4), neighbours inside 3,120-row blocks:", round(run(base, block=3120), 1), "us")
    print("poisson(5.4), inside 390-row blocks (one cluster-pair):", round(run(base, block=390), 1), "us")
    print("poisson(5.4) + rowscale:", round(run(base, rowscale=True), 1), "us")
    print("poisson(5.4) + rowscale, COLD (L2 flushed, timed alone):", round(run(base, rowscale=True, cold=True), 1), "us")
    print("all zero, COLD:", round(run(np.zeros(rows, np.int64), cold=True), 1), "us")
