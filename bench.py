#!/usr/bin/env python
"""GIST hot-path benchmark (BASELINE.json metric: sub-GCN epoch time & train steps/s,
Reddit-shape GraphSAGE; workload = configs[2] = C3 by default).

A bench "step" is one GIST round of Algorithm 1, i.e. one pass
of every SURVEY 8(a) row: subGCNs (partition + extract), zeta subTrain steps of
every sub-GCN (batch build, SpMM, GEMMs, CE, backward, Adam), subAgg.
`value` = sub-GCN train steps per second of the whole job (all ranks), device-timed
with CUDA events on the library stream, inputs resident in HBM, L2 flushed
between timed rounds.  `e2e` = the same metric through the public API from host
buffers: gist_load_graph of the host graph + the rounds + per-round loss readback.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--precision fp32|bf16]
  python bench.py --impl reference ...   # the FP64 oracle on host cores (rank 0 only)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from synth.planted import GRAPHS, MODELS, generate  # noqa: E402

METRIC = "sub-GCN train steps/s (box-level), Reddit-shape GraphSAGE"  # BASELINE.json metric (C3)


def metric_for(spec):
    """BASELINE's metric string for C3; the same quantity named after the graph / model
    family for the other configs."""
    if spec.graph == "reddit" and spec.arch == "sage":
        return METRIC
    shape = {"cora": "Cora", "arxiv": "arxiv", "reddit": "Reddit", "amazon2m": "Amazon2M"}.get(spec.graph, spec.graph)
    fam = {"sage": "GraphSAGE", "gat": "GAT"}.get(spec.arch, "GCN")
    return f"sub-GCN train steps/s (box-level), {shape}-shape {fam}"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16": d["bf16_tflops"], "bf16_sustained": d.get("bf16_tflops_sustained"),
                "sm_max_mhz": d.get("sm_max_mhz", 1965.0), "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "sm_max_mhz": 1965.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                s, mx = float(r[1]), float(r[2])
            except (ValueError, IndexError):
                continue
            smax = mx
            sm.append(s)
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower() in ("active", "1", "yes"):
                    reasons.add(nm)
        load = [s for s in sm if s > 0.5 * (smax or 1)] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# --------------------------------------------------------------------------- oracle
def oracle_steps_per_s(spec, g, seconds: float, max_steps: int, min_steps: int = 2, seed: int = 0):
    """Times the FP64 oracle (as it stands) on a bounded sample of the workload:
    consecutive subTrain steps of the sub-GCNs (batch build + fwd/bwd + Adam)."""
    from oracle import gist_oracle as O
    o = O.OracleGIST(arch=spec.arch, dims=list(spec.dims), optimizer="adam", clusters_per_batch=spec.q, batch_seed=1)
    o.load_graph(g["row_ptr"], g["col_idx"], g["X"], g["labels"], g["num_classes"], g["split"],
                 g["cluster_ids"], g["num_clusters"])
    rng = np.random.default_rng(seed)   # timing only: random weights instead of the (slow) Philox init
    th = []
    for l in range(len(spec.dims) - 1):
        rows = O.weight_rows(spec.arch, spec.dims[l])
        th.append(rng.uniform(-0.05, 0.05, size=(rows, spec.dims[l + 1])))
    o.set_params(th)
    o.partition(seed=1, m=spec.m)
    t0 = time.perf_counter()
    n = 0
    while n < max_steps and (n < min_steps or time.perf_counter() - t0 < seconds):
        o.train_step(n % spec.m, n // spec.m, 0.01)
        n += 1
    dt = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    return n / dt, n, dt, cores


def run_reference(args, spec, rank, world):
    if rank != 0:
        return 0
    g = generate(GRAPHS[spec.graph], seed=args.seed)
    # warm-up W steps, then K timed steps; each step = one oracle subTrain step (bounded sample)
    oracle_steps_per_s(spec, g, seconds=0.0, max_steps=args.warmup, min_steps=args.warmup)
    v, n, dt, cores = oracle_steps_per_s(spec, g, seconds=0.0, max_steps=args.steps, min_steps=args.steps)
    line = {
        "impl": "reference", "metric": metric_for(spec), "value": v, "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(n, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": spec.name, "m": spec.m, "q": spec.q, "dims": list(spec.dims), "arch": spec.arch},
        "cpu_baseline": {"value": v, "unit": "steps/s", "cores": cores, "kind": "oracle",
                         "sample": f"{n} consecutive sub-GCN subTrain steps of {spec.name} (FP64 numpy/scipy)"},
        "e2e": {"value": v, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- launcher
def maybe_spawn(args):
    """`bench.py --gpus N` without a torchrun environment: re-exec under torch.distributed.run
    with N ranks (one per GPU, rendezvous on 127.0.0.1).  Returns an exit code or None."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    # NCCL communicator-init lines on stderr (rank / nranks / NVLS), so a run's rank layout is auditable
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


# --------------------------------------------------------------------------- extras (rank 0, N = 1)
def scaling_proxy(G, spec, g, zeta, lr, worlds=(2, 4, 8)):
    """Per-GPU sub-GCN step rate at world size W, measured on this one GPU: the rank-0 context of
    a W-rank loopback group (include/gist.h) owns exactly the slots rank 0 owns in a W-GPU run
    (slot i on rank i mod W) and runs the same subTrain launches; partition and subTrain have no
    collective, so no other rank is needed.  Predicted box rate = W x per-GPU rate (before the
    once-per-round all-gather; measured subAgg time is reported separately)."""
    import torch
    out = {}
    for W in worlds:
        if spec.m % W:
            continue
        lb = G.Loopback(W)
        c = G.Gist(spec.arch, spec.dims, optimizer="adam", precision="bf16", clusters_per_batch=spec.q, batch_seed=1,
                   rank=0, world_size=W, loopback=lb)
        c.load_graph(g)
        c.init_params(0)
        st = torch.cuda.ExternalStream(c.stream())
        c.partition(seed=1, m=spec.m)
        c.subtrain(min(zeta, 50), 0.01, want_loss=False)       # warm-up (graph capture, clocks)
        torch.cuda.synchronize()
        ts = []
        for t in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            c.subtrain(zeta, lr, want_loss=False)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        per_gpu = (spec.m // W) * zeta / (ms / 1e3)
        out[str(W)] = {"slots_per_gpu": spec.m // W, "per_gpu_steps_s": per_gpu, "predicted_box_steps_s": W * per_gpu,
                       "ms_per_local_step": ms / zeta}
        c.close()
        lb.close()
    return out


def kernel_targets(G, g, pk):
    """north_star kernel targets, timed in this run through the C-ABI kernel entry points:
    the full-graph SpMM (HBM roofline; Reddit-shape graph, bf16, widths 512 / 4096 = the eval
    operator) and the m = 1 width-4096 GEMMs (tensor roofline)."""
    import torch
    dev = "cuda"
    res = {}
    rp = torch.from_numpy(np.ascontiguousarray(g["row_ptr"], dtype=np.int64)).to(dev)
    ci = torch.from_numpy(np.ascontiguousarray(g["col_idx"], dtype=np.int32)).to(dev)
    n, nnz = int(g["n"]), int(g["row_ptr"][-1])
    deg = torch.diff(rp).float()
    rs = torch.where(deg > 0, 1.0 / deg.clamp(min=1), torch.zeros_like(deg)).contiguous()  # SAGE mean (R2)

    def tm(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)
    for w in (512, 4096):
        H = torch.randn(n, w, device=dev).to(torch.bfloat16)
        out = torch.empty_like(H)
        ms = tm(lambda: G.spmm(rp.data_ptr(), ci.data_ptr(), n, rs.data_ptr(), None, False, H.data_ptr(),
                               out.data_ptr(), w, w, 1))
        comp = 8 * (n + 1) + 4 * nnz + 2 * n * w * 2 + 4 * n   # CSR + H and out once + row scale
        res[f"full_spmm_w{w}"] = {"ms": ms, "compulsory_gb": comp / 1e9, "compulsory_gbs": comp / (ms / 1e3) / 1e9,
                                  "frac_hbm_compulsory": comp / (ms / 1e3) / 1e9 / pk["hbm_gbs"],
                                  "gather_model_gb": (2 * nnz * w) / 1e9,
                                  "gather_model_gbs": (2 * nnz * w) / (ms / 1e3) / 1e9}
        del H, out
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp))
        for w in (512, 4096):
            k = f"full_spmm_w{w}"
            if k in tj and tj[k]:
                res[k]["ncu_dram_gb"] = tj[k] / 1e9
                res[k]["ncu_dram_gbs"] = tj[k] / (res[k]["ms"] / 1e3) / 1e9
                res[k]["frac_hbm_dram"] = res[k]["ncu_dram_gbs"] / pk["hbm_gbs"]
    M = 3106
    for name, (ta, tb, Mm, N, K) in {"fwd": (0, 0, M, 4096, 8192), "dX": (0, 1, M, 8192, 4096),
                                     "dW": (1, 0, 8192, 4096, M)}.items():
        A = torch.randn((K, Mm) if ta else (Mm, K), device=dev).to(torch.bfloat16)
        B = torch.randn((N, K) if tb else (K, N), device=dev).to(torch.bfloat16)
        C = torch.empty(Mm, N, device=dev, dtype=torch.float32)
        ms = tm(lambda: G.gemm(bool(ta), bool(tb), Mm, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1],
                               C.data_ptr(), N, 1, out_f32=True), reps=10)
        tf = 2.0 * Mm * N * K / (ms / 1e3) / 1e12
        res[f"gemm_w4096_{name}"] = {"M": Mm, "N": N, "K": K, "ms": ms, "tflops": tf, "frac_bf16_burst": tf / pk["bf16"]}
        del A, B, C
    torch.cuda.empty_cache()
    return res


def oracle_extras(spec, g):
    """BASELINE.md §4 / SURVEY §8(d): the oracle's 1-thread step time and its partition + aggregate
    time for one round of the workload (FP64 numpy/scipy as it stands)."""
    from oracle import gist_oracle as O
    from threadpoolctl import threadpool_limits
    o = O.OracleGIST(arch=spec.arch, dims=list(spec.dims), optimizer="adam", clusters_per_batch=spec.q, batch_seed=1)
    o.load_graph(g["row_ptr"], g["col_idx"], g["X"], g["labels"], g["num_classes"], g["split"],
                 g["cluster_ids"], g["num_clusters"])
    rng = np.random.default_rng(0)
    o.set_params([rng.uniform(-0.05, 0.05, size=(O.weight_rows(spec.arch, spec.dims[l]), spec.dims[l + 1]))
                  for l in range(len(spec.dims) - 1)])
    t0 = time.perf_counter()
    o.partition(seed=1, m=spec.m)
    t_part = time.perf_counter() - t0
    with threadpool_limits(limits=1):
        o.train_step(0, 0, 0.01)
        t0 = time.perf_counter()
        o.train_step(0, 1, 0.01)
        t1 = time.perf_counter() - t0
    t0 = time.perf_counter()
    o.aggregate()
    t_agg = time.perf_counter() - t0
    return {"one_thread_step_s": t1, "partition_s": t_part, "aggregate_s": t_agg,
            "note": "FP64 oracle; partition = subGCNs + extract of all m slots, aggregate = subAgg of all m slots"}


def c1_side_by_side(G, seed=0):
    """C1 (Cora-shaped GCN, m = 2, 5 rounds x 10 local iterations) completely on both
    the oracle and the CUDA path (FP32 parity mode), with their per-round losses and wall times.
    SGD (lr 0.1): under Adam the two trajectories separate by design after the first round (its
    first step after every re-partition is -lr sign(g))."""
    import torch
    from oracle import gist_oracle as O
    spec = MODELS["C1"]
    g = generate(GRAPHS[spec.graph], seed=seed)
    o = O.OracleGIST(arch=spec.arch, dims=list(spec.dims), optimizer="sgd", clusters_per_batch=spec.q, batch_seed=1)
    o.load_graph(g["row_ptr"], g["col_idx"], g["X"], g["labels"], g["num_classes"], g["split"],
                 g["cluster_ids"], g["num_clusters"])
    o.init_params(seed)
    c = G.Gist(spec.arch, spec.dims, optimizer="sgd", precision="fp32", clusters_per_batch=spec.q, batch_seed=1)
    t0 = time.perf_counter()
    c.load_graph(g)
    c.init_params(seed)
    lg = []
    for t in range(spec.rounds):
        c.partition(seed=1000 + t, m=spec.m)
        lg.append(c.subtrain(spec.zeta, 0.1))
        c.aggregate()
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    lo = []
    for t in range(spec.rounds):
        o.partition(seed=1000 + t, m=spec.m)
        lo.append(o.subtrain(spec.zeta, 0.1))
        o.aggregate()
    t_or = time.perf_counter() - t0
    c.close()
    lg, lo = np.array(lg, dtype=np.float64), np.array(lo)
    return {"rounds": spec.rounds, "zeta": spec.zeta, "m": spec.m, "optimizer": "sgd", "lr": 0.1,
            "gpu_s": t_gpu, "oracle_s": t_or,
            "max_rel_loss_diff": float(np.max(np.abs(lg - lo) / np.maximum(np.abs(lo), 1e-12))),
            "gpu_losses": lg.round(6).tolist(), "oracle_losses": lo.round(6).tolist()}


# --------------------------------------------------------------------------- GIST
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gist", choices=["gist", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(MODELS))
    ap.add_argument("--precision", default="bf16", choices=["fp32", "bf16", "tf32"])
    ap.add_argument("--zeta", type=int, default=0, help="local iterations per round (0 = paper's zeta, capped)")
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--agg", default="allgather", choices=["allgather", "p2p", "symm"],
                    help="subAgg transport (gist_config.agg_mode; p2p / symm = SURVEY §8 f2 peer stores over CUDA IPC /"
                         " the NCCL device API)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--profile-stride", type=int, default=32,
                    help="every N-th step of the extra profiled round is timed per kernel class (0: no profile)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-eval", action="store_true", help="skip the (untimed-for-value) evaluation timings")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the N=1 extras (scaling proxy, kernel targets, FP32 line, oracle extras, C1 run)")
    ap.add_argument("--eval-parts", type=int, default=5000, help="partitions of the partition-wise eval (P:697)")
    args = ap.parse_args()
    rc = maybe_spawn(args)
    if rc is not None:
        return rc
    spec = MODELS[args.config]
    rank, world, local = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args, spec, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2102_10424_b200 import gist as G

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    zeta = args.zeta or spec.zeta
    t_gen = time.perf_counter()
    g = generate(GRAPHS[spec.graph], seed=args.seed, device=f"cuda:{local}")
    t_gen = time.perf_counter() - t_gen

    def make(precision=args.precision):
        # every context builds its own NCCL communicator, so every one needs a fresh unique id
        # (an ncclUniqueId's bootstrap root serves exactly one communicator init)
        uid = None
        if world > 1:
            obj = [G.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        return G.Gist(spec.arch, spec.dims, optimizer="adam", precision=precision, clusters_per_batch=spec.q,
                      batch_seed=1, rank=rank, world_size=world, device=local, nccl_unique_id=uid,
                      agg_mode=args.agg)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ------------------------------------------------ device-resident timing (value): profiler off
    gx = make()
    gx.load_graph(g)
    gx.init_params(args.seed)
    stream = torch.cuda.ExternalStream(gx.stream())
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")  # > 126 MB L2

    def one_round(c, t, want_loss=False, z=zeta):
        c.partition(seed=1000 + t, m=spec.m)
        loss = c.subtrain(z, args.lr, want_loss=want_loss)
        c.aggregate()
        return loss

    for t in range(args.warmup):
        one_round(gx, t)
    torch.cuda.synchronize()
    k0 = gx.stat(G.STAT_KERNELS)
    times = []
    with ClockSampler(local) as clk:
        for t in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            one_round(gx, args.warmup + t)
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            times.append(e0.elapsed_time(e1))
    launches = gx.stat(G.STAT_KERNELS) - k0
    total_ms = max_over_ranks(float(sum(times)))
    steps_total = args.steps * zeta * spec.m          # sub-GCN steps of all ranks
    value = steps_total / (total_ms / 1e3)
    B = -(-g["num_clusters"] // spec.q)
    # ------------------------------------------------ one extra profiled round (not part of `value`):
    # every stride-th step runs serialised with CUDA events around every launch
    prof = None
    if args.profile_stride > 0:
        gx.profile(args.profile_stride)
        one_round(gx, args.warmup + args.steps)
        prof = gx.profile_get()
        gx.profile(0)
    nb_last = gx.stat(G.STAT_LAST_NB)
    block_agg = gx.stat(G.STAT_BLOCK_AGG)
    block_density = gx.stat(G.STAT_BLOCK_DENSITY_PPM) / 1e6
    nnzb_last = gx.stat(G.STAT_LAST_NNZ_B)
    gx.close()
    del gx

    # ------------------------------------------------ end-to-end through the public API (e2e)
    # the host inputs live in pinned memory (untimed staging, as a data loader would hold them)
    def pinned(a):
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()
    gp = dict(g)
    for key, dt in (("row_ptr", np.int64), ("col_idx", np.int32), ("X", np.float32), ("labels", np.int32),
                    ("split", np.uint8), ("cluster_ids", np.int32)):   # the binding's dtypes: no re-copy
        gp[key] = pinned(np.ascontiguousarray(g[key], dtype=dt))
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    ge = make()
    ge.load_graph(gp)                                  # pinned host arrays -> device (timed)
    ge.init_params(args.seed)
    torch.cuda.synchronize()
    t_load = time.perf_counter() - t0
    for t in range(args.steps):
        one_round(ge, t, want_loss=True)               # per-round loss read back to host
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    h2d = ge.stat(G.STAT_H2D_BYTES)
    d2h = ge.stat(G.STAT_D2H_BYTES)
    # ------------------------------------------------ evaluation (not part of `value`): after the
    # timed e2e region (its large temporary buffers would otherwise perturb the e2e allocations)
    ev = None
    if not args.no_eval:
        n = g["n"]
        order = np.argsort(g["cluster_ids"], kind="stable")
        part = np.empty(n, np.int32)
        part[order] = (np.arange(n) * args.eval_parts) // n     # METIS stand-in: cluster-sorted order cut
        torch.cuda.synchronize()
        barrier()
        lf = af = t_full = None
        if max(spec.dims[1:-1]) <= 4096:   # wider models are evaluated on partitions only
            t0 = time.perf_counter()
            lf, af = ge.eval(2)
            t_full = max_over_ranks(time.perf_counter() - t0)
        barrier()
        t0 = time.perf_counter()
        lp, apc, _, _ = ge.eval_parts(2, part, args.eval_parts)
        t_parts = max_over_ranks(time.perf_counter() - t0)
        ev = {"split": "test", "full_graph_s": t_full, "full_graph_loss": lf, "full_graph_acc": af,
              "parts": args.eval_parts, "parts_s": t_parts, "parts_loss": lp, "parts_acc": apc,
              "note": "after the timed rounds; wall clock around each ABI call (host setup included); "
                      "world > 1: rows (full graph) / partitions split across ranks"}
    ge.close()

    # ------------------------------------------------ roofline of the dominant kernel class
    pk = peaks()
    roof = None
    subagg = None
    if prof and max(v["ms"] for v in prof.values()) > 0:
        step_classes = {k: v for k, v in prof.items() if k not in ("partition", "aggregate", "comm")}
        dom = max(step_classes, key=lambda k: step_classes[k]["ms"])
        pd = prof[dom]
        avg_ms = pd["ms"] / max(pd["launches"], 1)
        work_per = pd["work"] / max(pd["launches"], 1)
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(f"{args.precision}:{dom}")
        if dom in ("gemm", "agg_tc"):
            if args.precision == "bf16":
                roof = {"bound": "tensor", "peak": pk["bf16_sustained"] or pk["bf16"], "unit": "TFLOP/s",
                        "peak_src": f"{pk['src']} bf16 sustained"}
            elif args.precision == "tf32":   # a contraction takes its own dtype's peak: bf16 x 1/2 (nominal ratio)
                roof = {"bound": "tensor", "peak": 0.5 * (pk["bf16_sustained"] or pk["bf16"]), "unit": "TFLOP/s",
                        "peak_src": f"{pk['src']} bf16 sustained x nominal tf32/bf16 ratio 1.13/2.25"}
            else:
                # FP32 SIMT: 148 SMs x 128 FP32 lanes x 2 flop x max SM clock
                roof = {"bound": "alu", "peak": 148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12, "unit": "TFLOP/s",
                        "peak_src": "derived: 148 SM x 128 FFMA lanes x 2 x sm_max_mhz"}
            achieved = work_per / (avg_ms / 1e3) / 1e12
        else:
            roof = {"bound": "hbm", "peak": pk["hbm_gbs"], "unit": "GB/s", "peak_src": f"{pk['src']} hbm copy"}
            achieved = work_per / (avg_ms / 1e3) / 1e9
        roof.update({"kernel": dom, "achieved": achieved, "frac": achieved / roof["peak"], "traffic": traffic,
                     "avg_launch_ms": avg_ms, "work_per_launch": work_per,
                     "share_of_profiled_ms": pd["ms"] / max(sum(v["ms"] for v in step_classes.values()), 1e-9)})
        # every step class against its own bound (same profiled round): tensor classes by algorithmic
        # FLOP (agg_tc: 2 BS^2 w per batch cluster -- a dense contraction of a 34%-dense block, so its
        # tensor fraction is low by construction), the others by compulsory bytes against HBM
        class_roof = {}
        for k, v in step_classes.items():
            if v["launches"] <= 0 or v["ms"] <= 0:
                continue
            rate = v["work"] / (v["ms"] / 1e3)
            if k in ("gemm", "agg_tc"):
                pk_t = roof["peak"] if dom in ("gemm", "agg_tc") else (pk["bf16_sustained"] or pk["bf16"])
                class_roof[k] = {"bound": roof["bound"] if dom in ("gemm", "agg_tc") else "tensor",
                                 "achieved": rate / 1e12, "unit": "TFLOP/s", "frac": rate / 1e12 / pk_t}
            else:
                class_roof[k] = {"bound": "hbm", "achieved": rate / 1e9, "unit": "GB/s", "frac": rate / 1e9 / pk["hbm_gbs"]}
            class_roof[k].update({"avg_launch_ms": v["ms"] / v["launches"], "launches": v["launches"]})
        roof["classes"] = class_roof
        # subAgg (a9): the per-round collective and local scatter of the profiled round
        cm = prof.get("comm", {"ms": 0.0, "launches": 0, "work": 0.0})
        ag = prof["aggregate"]
        subagg = {"scatter_ms": ag["ms"], "collective_ms": cm["ms"], "bytes_received_per_rank": cm["work"]}
        if world > 1 and cm["ms"] > 0:
            busbw = cm["work"] / (cm["ms"] / 1e3) / 1e9        # (W-1)/W of the gathered bytes per rank
            subagg.update({"busbw_gbs": busbw, "frac_nvlink_measured_770": busbw / 770.0})

    line = {
        "metric": metric_for(spec), "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": {"fp32": "f32", "tf32": "tf32", "bf16": "bf16"}[args.precision],
        "data": "synthetic",
        "config": {"workload": spec.name, "graph": f"{spec.graph}-shaped planted-cluster synthetic "
                   f"(n={g['n']}, nnz={int(g['row_ptr'][-1])})", "arch": spec.arch, "dims": list(spec.dims),
                   "m": spec.m, "q": spec.q, "zeta": zeta, "step": "one GIST round (partition + zeta subTrain "
                   "steps of all m sub-GCNs + aggregate)", "parallelism": f"gist-m{spec.m}-over-{world}gpu",
                   "slots_per_gpu": -(-spec.m // world), "agg": args.agg,
                   "precision": args.precision, "l2": "256 MiB buffer written between timed rounds",
                   "epoch_s": spec.m * B / value, "batches_per_epoch": B, "last_n_b": nb_last,
                   "last_nnz_b": nnzb_last, "gen_s": t_gen, "profile": f"one extra round, every "
                   f"{args.profile_stride}-th step serialised and event-timed (not in value)",
                   "block_agg": bool(block_agg), "block_density": block_density},
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "roofline": roof,
        "kernel_profile": {k: {"ms": v["ms"], "launches": v["launches"]} for k, v in prof.items()} if prof else None,
        "subagg": subagg,
        "eval": ev,
        "e2e": {"value": steps_total / e2e_s, "unit": "steps/s", "h2d_bytes_per_step": h2d / args.steps,
                "d2h_bytes_per_step": d2h / args.steps,
                "includes": "gist_load_graph from pinned host arrays + init + K rounds with per-round loss readback",
                "load_and_init_s": t_load},
    }
    if rank == 0 and world == 1 and not args.no_extras:
        line["scaling_proxy"] = scaling_proxy(G, spec, g, zeta, args.lr)
        for W, d in line["scaling_proxy"].items():
            d["predicted_speedup_vs_1gpu"] = d["predicted_box_steps_s"] / value
        if spec.graph == "reddit":
            line["kernel_targets"] = kernel_targets(G, g, pk)
        if args.precision == "bf16":
            # the paper's precision (PyTorch's FP32 default, R13): FP32 parity mode (SIMT GEMMs) and
            # TF32 mode (FP32 storage, tcgen05 kind::tf32 GEMMs), same workload, zeta capped at 100
            notes = {"fp32": "FP32 parity mode (FP32 storage, SIMT FFMA GEMMs)",
                     "tf32": "TF32 mode (FP32 storage, tcgen05 kind::tf32 GEMMs, fp32 accumulation)"}
            for prec, note in notes.items():
                z32 = min(zeta, 100)
                c32 = make(prec)
                c32.load_graph(g)
                c32.init_params(args.seed)
                st32 = torch.cuda.ExternalStream(c32.stream())
                one_round(c32, 0, z=z32)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st32)
                for t in range(2):
                    one_round(c32, 1 + t, z=z32)
                e1.record(st32)
                torch.cuda.synchronize()
                line[prec] = {"value": 2 * z32 * spec.m / (e0.elapsed_time(e1) / 1e3), "unit": "steps/s",
                              "zeta": z32, "rounds": 2, "note": note}
                c32.close()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, n, dt, cores = oracle_steps_per_s(spec, g, seconds=args.cpu_seconds, max_steps=64)
        line["cpu_baseline"] = {"value": v, "unit": "steps/s", "cores": cores, "kind": "oracle",
                                "sample": f"{n} consecutive sub-GCN subTrain steps of {spec.name} "
                                          f"(FP64 numpy/scipy, {dt:.1f} s)"}
        if not args.no_extras:
            line["cpu_baseline"]["extras"] = oracle_extras(spec, g)
            line["c1_side_by_side"] = c1_side_by_side(G)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
