"""Is a subTrain loop host-bound?  Host enqueue time of gist_subtrain (no loss readback, so no
sync inside) vs the device time of the same call (CUDA events), for lockstep group sizes set by
GIST_GROUP (1 slot per group ~ the per-GPU work at W = 8)."""
import os, sys, time, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_10424_b200 import gist as G
from synth.planted import GRAPHS, MODELS, generate
spec = MODELS["C3"]
ITERS = int(os.environ.get("ITERS", "200"))  # few iterations: the launch queue never fills
g = generate(GRAPHS[spec.graph], seed=0, device="cuda")
gx = G.Gist(spec.arch, spec.dims, optimizer="adam", precision="bf16", clusters_per_batch=spec.q, batch_seed=1)
gx.load_graph(g)
gx.init_params(0)
stream = torch.cuda.ExternalStream(gx.stream())
for t in range(3):
    gx.partition(seed=t, m=spec.m)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h0 = time.perf_counter()
    gx.subtrain(ITERS, 0.01, want_loss=False)
    host = time.perf_counter() - h0
    e1.record(stream)
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / 1e3
    gx.aggregate()
    print(json.dumps({"group": os.environ.get("GIST_GROUP", "8"), "host_ms_per_step": 1e3 * host / ITERS,
                      "device_ms_per_step": 1e3 * dev / ITERS}), flush=True)
