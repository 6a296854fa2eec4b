"""Pins for the oracle's partition-wise evaluation (reading R20 in
DESIGN.md): hand-computed values on a path graph, the closed form for singleton
partitions, the invariant that partitions equal to connected components reproduce the
full-graph forward, and the reduction of one all-covering partition to full-graph eval."""
import math

import numpy as np
import pytest

from oracle import gist_oracle as O
from synth.planted import generate, tiny_spec


def csr_from_edges(n, edges):
    adj = [set() for _ in range(n)]
    for a, b in edges:
        adj[a].add(b)
        adj[b].add(a)
    rp = np.zeros(n + 1, dtype=np.int64)
    cols = []
    for v in range(n):
        c = sorted(adj[v])
        cols.extend(c)
        rp[v + 1] = len(cols)
    return rp, np.asarray(cols, dtype=np.int64)


def oracle_on(arch, dims, rp, ci, X, labels, split):
    n = len(rp) - 1
    o = O.OracleGIST(arch=arch, dims=list(dims))
    o.load_graph(rp, ci, X, labels, dims[-1], split, np.zeros(n, np.int64), 1)
    return o


def test_path_graph_by_hand_gcn():
    """Path 0-1-2-3 cut into {0,1} and {2,3} (+ node 4 alone, holding no evaluated node).
    Inside a 2-node partition D~ = 2, so A_hat = [[.5,.5],[.5,.5]] (the full graph would
    give node 1 the factor 1/3): A_hat X = 1.5 (part 0) and 3.5 (part 1); W = [1, -1]
    gives logits [z, -z]."""
    rp, ci = csr_from_edges(5, [(0, 1), (1, 2), (2, 3), (3, 4)])
    X = np.array([[1.0], [2.0], [3.0], [4.0], [9.0]])
    labels = np.array([0, 1, 0, 0, 1])
    split = np.array([1, 1, 1, 1, 0])
    o = oracle_on("gcn", (1, 2), rp, ci, X, labels, split)
    o.set_params([np.array([[1.0, -1.0]])])
    part = np.array([0, 0, 1, 1, 2])
    loss, acc, lp, ap = o.eval_partitions(1, part, 3)
    l0 = (math.log1p(math.exp(-3.0)) + math.log1p(math.exp(3.0))) / 2   # labels 0, 1 at z = 1.5
    l1 = math.log1p(math.exp(-7.0))                                      # labels 0, 0 at z = 3.5
    assert lp[0] == pytest.approx(l0, rel=1e-12) and lp[1] == pytest.approx(l1, rel=1e-12)
    assert ap[0] == 0.5 and ap[1] == 1.0
    assert math.isnan(lp[2]) and math.isnan(ap[2])
    assert loss == pytest.approx((l0 + l1) / 2, rel=1e-12) and acc == 0.75


def test_path_graph_by_hand_sage():
    """Same cut, GraphSAGE-mean: inside {0,1} N = [[0,1],[1,0]], so [X || N X] =
    [[1,2],[2,1]]; inside {2,3} [[3,4],[4,3]]; node 4 alone: [9, 0]."""
    rp, ci = csr_from_edges(5, [(0, 1), (1, 2), (2, 3), (3, 4)])
    X = np.array([[1.0], [2.0], [3.0], [4.0], [9.0]])
    labels = np.array([1, 1, 0, 1, 0])
    split = np.array([2, 2, 2, 2, 2])
    o = oracle_on("sage", (1, 2), rp, ci, X, labels, split)
    o.set_params([np.eye(2)])        # logits = [x_v, (N X)_v]
    loss, acc, lp, ap = o.eval_partitions(2, np.array([0, 0, 1, 1, 2]), 3)
    ce = lambda z, y: math.log(math.exp(z[0]) + math.exp(z[1])) - z[y]
    want_l = [(ce([1, 2], 1) + ce([2, 1], 1)) / 2, (ce([3, 4], 0) + ce([4, 3], 1)) / 2, ce([9, 0], 0)]
    want_a = [0.5, 0.0, 1.0]
    assert np.allclose(lp, want_l, rtol=1e-12) and np.array_equal(ap, want_a)
    assert loss == pytest.approx(np.mean(want_l), rel=1e-12) and acc == pytest.approx(0.5)


@pytest.mark.parametrize("arch", ["gcn", "sage"])
def test_singleton_partitions_closed_form(arch):
    """Every node alone: the GCN operator is I (D~ = 1) and the GraphSAGE neighbour mean
    is 0, so the model collapses to a per-node MLP (SAGE: only the self rows W[:d]).
    Catches global degrees or cut edges leaking into the partition operator."""
    g = generate(tiny_spec(n=120, nnz=900, d0=6, classes=4, clusters=5), seed=3)
    dims = (6, 9, 7, 4)
    o = O.OracleGIST(arch=arch, dims=list(dims))
    o.load_graph(g["row_ptr"], g["col_idx"], g["X"], g["labels"], 4, g["split"], g["cluster_ids"], 5)
    o.init_params(2)
    n = len(g["labels"])
    _, _, lp, ap = o.eval_partitions(0, np.arange(n), n)
    H = np.asarray(g["X"], np.float64)
    for l, W in enumerate(o.theta):
        Z = H @ (W if arch == "gcn" else W[:dims[l]])
        H = np.maximum(Z, 0.0) if l + 1 < len(o.theta) else Z
    for v in range(n):
        if g["split"][v] != 0:
            assert math.isnan(ap[v])
            continue
        z = H[v]
        want = np.log(np.sum(np.exp(z - z.max()))) + z.max() - z[g["labels"][v]]
        assert lp[v] == pytest.approx(want, rel=1e-10, abs=1e-12)
        assert ap[v] == float(np.argmax(z) == g["labels"][v])


@pytest.mark.parametrize("arch", ["gcn", "sage"])
def test_component_partitions_reproduce_full_graph(arch):
    """Disjoint union of three random graphs, partitions = components: no edge is cut, so
    the per-node logits equal the full-graph forward's, and each partition's accuracy is
    the brute-force count over its nodes."""
    rng = np.random.default_rng(4)
    sizes = [17, 30, 9]
    edges, base = [], 0
    for s in sizes:
        for a in range(s):
            for b in range(a + 1, s):
                if rng.random() < 0.25:
                    edges.append((base + a, base + b))
        base += s
    n = sum(sizes)
    perm = rng.permutation(n)                      # interleave the components' ids
    edges = [(perm[a], perm[b]) for a, b in edges]
    comp = np.empty(n, np.int64)
    comp[perm] = np.repeat(np.arange(3), sizes)
    rp, ci = csr_from_edges(n, edges)
    dims = (5, 8, 3)
    X = rng.normal(size=(n, 5))
    labels = rng.integers(0, 3, n)
    split = rng.integers(0, 2, n)
    o = oracle_on(arch, dims, rp, ci, X, labels, split)
    o.init_params(9)
    _, _, logits = o.eval(1)
    loss, acc, lp, ap = o.eval_partitions(1, comp, 3)
    pred = np.argmax(logits, axis=1)
    for p in range(3):
        rows = (comp == p) & (split == 1)
        z = logits[rows]
        ce = np.log(np.exp(z - z.max(1, keepdims=True)).sum(1)) + z.max(1) - z[np.arange(len(z)), labels[rows]]
        assert lp[p] == pytest.approx(ce.mean(), rel=1e-10)
        assert ap[p] == pytest.approx(np.mean(pred[rows] == labels[rows]), abs=0)
    assert acc == pytest.approx(np.mean(ap)) and loss == pytest.approx(np.mean(lp))


def test_one_partition_is_full_graph_eval():
    g = generate(tiny_spec(n=200, nnz=1500, d0=7, classes=3, clusters=4), seed=1)
    o = O.OracleGIST(arch="sage", dims=[7, 10, 3])
    o.load_graph(g["row_ptr"], g["col_idx"], g["X"], g["labels"], 3, g["split"], g["cluster_ids"], 4)
    o.init_params(5)
    l_full, a_full, _ = o.eval(0)
    l, a, lp, ap = o.eval_partitions(0, np.zeros(200, np.int64), 1)
    assert l == pytest.approx(l_full, rel=1e-12) and a == a_full and lp[0] == l and ap[0] == a


@pytest.mark.parametrize("arch", ["gcn", "sage"])
@pytest.mark.parametrize("L", [2, 3])
def test_eval_scale_mean_closed_form(arch, L):
    """R10 "mean" (the theory's 1/m output scaling): every contraction over a
    partitioned (hidden) input dimension is scaled by 1/m.  ReLU is positively homogeneous, so
    for GCN / GraphSAGE the scaled logits are the unscaled ones times m^-(L-1) exactly (each of
    the L-1 layers after the first contributes one factor); m = 1 and "none" change nothing."""
    g = generate(tiny_spec(n=150, nnz=900, d0=6, classes=3, clusters=3), seed=2)
    dims = [6] + [8] * (L - 1) + [3]
    o = O.OracleGIST(arch=arch, dims=dims)
    o.load_graph(g["row_ptr"], g["col_idx"], g["X"], g["labels"], 3, g["split"], g["cluster_ids"], 3)
    o.init_params(4)
    _, _, base = o.eval(0)
    o.partition(seed=1, m=4)
    o.aggregate()                        # no training: Theta unchanged, m = 4 recorded
    _, _, none = o.eval(0, eval_scale="none")
    _, _, mean = o.eval(0, eval_scale="mean")
    assert np.array_equal(none, base)
    np.testing.assert_allclose(mean, base / 4.0 ** (L - 1), rtol=1e-12, atol=1e-14)
    ref = np.zeros_like(base)
    o.eval_partitions(0, np.zeros(150, np.int64), 1, logits_out=ref, eval_scale="mean")
    np.testing.assert_allclose(ref, mean, rtol=1e-12, atol=1e-14)
    o.partition(seed=2, m=1)
    o.aggregate()
    assert np.array_equal(o.eval(0, eval_scale="mean")[2], base)
