"""Seeded planted-cluster graph generator (inputs only; holds none of GIST's arithmetic).

Shared by the oracle tests, the GPU parity tests and bench.py.  It produces the
graph that `gist_load_graph` consumes: a symmetric CSR without self loops,
fp32 features, int32 labels, uint8 split (0 train / 1 val / 2 test) and int32
cluster ids (the stand-in for METIS, which is out of scope).

Recipe (after SURVEY.md 8(d)):
  * communities: a seeded permutation of the nodes is cut into `communities`
    near-equal groups (so groups are not contiguous in input ids);
  * clusters: the batching partition; equal to the communities when
    clusters > 1 (METIS on a planted graph recovers them), 1 cluster otherwise;
  * degrees: per-node lognormal(sigma) weights; each node draws that many edge
    endpoints, a fraction f_in inside its community and the rest uniform over the
    graph; symmetrise, drop self loops and duplicates, then thin the unique
    undirected edges by a Bernoulli draw to ~nnz/2 (realised nnz is reported);
  * labels: each community gets a class; a node keeps it with prob 0.9, else a
    uniform class;
  * features: x_v = mu_{label} + 0.5 eps, mu, eps ~ N(0, I) (fp32);
  * split: seeded random assignment with the configured fractions / counts.

Determinism: all random draws come from numpy PCG64(seed); the heavy
sort/unique step may run on a torch device, whose result (sorted unique keys)
does not depend on the device.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class GraphSpec:
    name: str
    n: int
    nnz: int                 # stored nonzeros of symmetric A, no self loops (R15)
    d0: int
    classes: int
    communities: int
    clusters: int
    f_in: float
    split: tuple             # (train, val, test): fractions (sum 1) or absolute counts
    sigma: float = 1.0


# Shapes from BASELINE.json configs and PAPER.md Table 5.
GRAPHS = {
    "cora": GraphSpec("cora", 2708, 10556, 1433, 7, 7, 1, 0.8, (140, 500, 1000)),
    "arxiv": GraphSpec("arxiv", 169343, 1166243, 128, 40, 20, 20, 0.8, (0.54, 0.18, 0.28)),
    "reddit": GraphSpec("reddit", 232965, 114615892, 602, 41, 1500, 1500, 0.156, (0.66, 0.10, 0.24)),
    "amazon2m": GraphSpec("amazon2m", 2449029, 61859140, 100, 47, 15000, 15000, 0.7, (0.70, 0.0, 0.30)),
}


@dataclass(frozen=True)
class ModelSpec:
    name: str
    graph: str
    arch: str                # "gcn" | "sage" | "gat"
    dims: tuple
    m: int
    q: int                   # clusters per mini-batch
    zeta: int                # local iterations per round
    rounds: int = 1


# BASELINE.json configs[0..4]; zeta per PAPER.md:641, 681, 689 (R17).
MODELS = {
    "C1": ModelSpec("C1-cora-gcn2-256", "cora", "gcn", (1433, 256, 7), 2, 1, 10, 5),
    "C2": ModelSpec("C2-arxiv-gcn3-1024", "arxiv", "gcn", (128, 1024, 1024, 40), 4, 1, 100),
    "C3": ModelSpec("C3-reddit-sage4-4096", "reddit", "sage", (602, 4096, 4096, 4096, 41), 8, 20, 500),
    "C4": ModelSpec("C4-amazon2m-sage3-8192", "amazon2m", "sage", (100, 8192, 8192, 47), 8, 10, 5000),
    "C5": ModelSpec("C5-amazon2m-sage3-32768", "amazon2m", "sage", (100, 32768, 32768, 47), 8, 10, 5000),
    # the paper's Reddit GAT (256-dimensional, two to four layers;
    # m = 2 gives its best F1), on the C3 graph and batching (R21)
    "C3G": ModelSpec("C3G-reddit-gat2-256", "reddit", "gat", (602, 256, 41), 2, 20, 500),
}


def _split_counts(n: int, split) -> tuple:
    if all(isinstance(s, int) for s in split):
        return tuple(split)
    a = int(round(split[0] * n))
    b = int(round(split[1] * n))
    return (a, b, n - a - b)


def _unique_sorted(keys: np.ndarray, device: str | None) -> np.ndarray:
    if device is not None:
        import torch
        t = torch.from_numpy(keys).to(device)
        return torch.unique(t, sorted=True).cpu().numpy()
    s = np.sort(keys)
    return s[np.concatenate([[True], s[1:] != s[:-1]])] if len(s) else s


def _sorted(keys: np.ndarray, device: str | None) -> np.ndarray:
    if device is not None:
        import torch
        return torch.sort(torch.from_numpy(keys).to(device))[0].cpu().numpy()
    return np.sort(keys)


def generate(spec: GraphSpec, seed: int = 0, device: str | None = None, oversample: float = 1.25) -> dict:
    rng = np.random.Generator(np.random.PCG64(seed))
    n = spec.n
    # communities: permutation cut into near-equal groups
    perm = rng.permutation(n)
    comm = np.empty(n, dtype=np.int64)
    bounds = np.linspace(0, n, spec.communities + 1).round().astype(np.int64)
    for j in range(spec.communities):
        comm[perm[bounds[j]:bounds[j + 1]]] = j
    comm_members = perm                       # members of j = perm[bounds[j]:bounds[j+1]]
    comm_start = bounds[comm]
    comm_size = (bounds[1:] - bounds[:-1])[comm]

    # degrees (half-edges drawn per node)
    target_und = spec.nnz // 2
    w = np.exp(spec.sigma * rng.standard_normal(n))
    w *= (target_und * oversample) / w.sum()
    cnt = np.floor(w).astype(np.int64)
    cnt += (rng.random(n) < (w - cnt)).astype(np.int64)
    src = np.repeat(np.arange(n, dtype=np.int64), cnt)
    E = len(src)
    inside = rng.random(E) < spec.f_in
    dst = rng.integers(0, n, size=E, dtype=np.int64)
    pick = (rng.random(E) * comm_size[src]).astype(np.int64)
    dst_in = comm_members[comm_start[src] + pick]
    dst = np.where(inside, dst_in, dst)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    lo, hi = np.minimum(src, dst), np.maximum(src, dst)
    und = _unique_sorted(lo * n + hi, device)
    if len(und) > target_und:                  # thin to ~nnz/2 undirected edges (Bernoulli)
        und = und[rng.random(len(und)) < (target_und / len(und))]
    a, b = und // n, und % n
    both = _sorted(np.concatenate([a * n + b, b * n + a]), device)   # CSR order, cols ascending
    rows, cols = both // n, both % n
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])

    # labels
    comm_class = rng.integers(0, spec.classes, size=spec.communities)
    if spec.communities == spec.classes:
        comm_class = rng.permutation(spec.classes)
    labels = comm_class[comm]
    flip = rng.random(n) >= 0.9
    labels = np.where(flip, rng.integers(0, spec.classes, size=n), labels).astype(np.int32)

    # features
    mu = rng.standard_normal((spec.classes, spec.d0)).astype(np.float32)
    X = mu[labels]
    X += np.float32(0.5) * rng.standard_normal((n, spec.d0), dtype=np.float32)

    # split
    ntr, nva, nte = _split_counts(n, spec.split)
    order = rng.permutation(n)
    split = np.full(n, 3, dtype=np.uint8)      # 3 = unused (only for count-based splits)
    split[order[:ntr]] = 0
    split[order[ntr:ntr + nva]] = 1
    split[order[ntr + nva:ntr + nva + nte]] = 2

    clusters = comm.astype(np.int32) if spec.clusters > 1 else np.zeros(n, dtype=np.int32)
    return {
        "n": n, "row_ptr": row_ptr, "col_idx": cols.astype(np.int32), "X": X,
        "labels": labels, "num_classes": spec.classes, "split": split,
        "cluster_ids": clusters, "num_clusters": max(spec.clusters, 1),
    }


def tiny_spec(n=600, nnz=4000, d0=37, classes=5, clusters=12, f_in=0.7, name="tiny") -> GraphSpec:
    """Small ragged graphs for parity tests (several tiles + ragged tails)."""
    return GraphSpec(name, n, nnz, d0, classes, clusters, clusters, f_in, (0.6, 0.2, 0.2))


def graph_by_name(name: str, seed: int = 0, device: str | None = None) -> dict:
    return generate(GRAPHS[name], seed=seed, device=device)
