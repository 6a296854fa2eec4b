"""Full-graph (Reddit-shape) SpMM through gist_spmm at widths 512 / 4096 (bf16), for ncu DRAM-throughput capture."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_10424_b200 import gist
from synth.planted import GRAPHS, generate
g = generate(GRAPHS["reddit"], seed=0, device="cuda")
n = g["n"]
rp = torch.from_numpy(g["row_ptr"]).cuda(); ci = torch.from_numpy(g["col_idx"]).cuda()
deg = torch.from_numpy(np.diff(g["row_ptr"])).cuda().float()
sc = (1.0 / torch.sqrt(deg + 1)).contiguous()
for w in [int(x) for x in (sys.argv[1:] or ["512", "4096"])]:
    H = torch.randn(n, w, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(H)
    for _ in range(2):
        gist.spmm(rp.data_ptr(), ci.data_ptr(), n, sc.data_ptr(), sc.data_ptr(), True, H.data_ptr(), out.data_ptr(), w, w, 1)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); gist.spmm(rp.data_ptr(), ci.data_ptr(), n, sc.data_ptr(), sc.data_ptr(), True, H.data_ptr(), out.data_ptr(), w, w, 1); b.record()
    torch.cuda.synchronize()
    print(f"w={w} ms={a.elapsed_time(b):.3f}", flush=True)
    del H, out
