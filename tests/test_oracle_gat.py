"""Pins for the oracle's GAT sub-GCNs (reading R21): the
attention layer against a dense masked-softmax brute force, the uniform-attention closed
form (zero attention vectors give the mean over N(i) and i), finite differences of every
parameter including the attention vectors, the extract/aggregate layout of the attention
rows, and GIST(m=1) = plain training."""
import numpy as np
import pytest

from oracle import gist_oracle as O
from synth.planted import generate, tiny_spec
from tests.test_oracle_model import loss_of, rand_graph


def dense_gat_logits(theta, A, X):
    """Dense restatement: E = LeakyReLU(t 1^T + 1 s^T) masked to A + I, row softmax, out = P Z."""
    n = A.shape[0]
    mask = (A + np.eye(n)) > 0
    H = X
    for l, T in enumerate(theta):
        d = H.shape[1]
        Z = H @ T[:d]
        E = (Z @ T[d + 1])[:, None] + (Z @ T[d])[None, :]
        E = np.where(E > 0, E, 0.2 * E)
        E = np.where(mask, E, -np.inf)
        P = np.exp(E - E.max(axis=1, keepdims=True))
        P /= P.sum(axis=1, keepdims=True)
        out = P @ Z
        H = np.maximum(out, 0.0) if l + 1 < len(theta) else out
    return H


def test_attention_equals_dense_bruteforce():
    rng = np.random.default_rng(0)
    for n, dims in [(1, [3, 2]), (9, [4, 6, 3]), (20, [5, 8, 7, 4])]:
        rp, ci, A = rand_graph(n, 0.3, rng)
        theta = [rng.standard_normal((O.weight_rows("gat", dims[l]), dims[l + 1])) for l in range(len(dims) - 1)]
        X = rng.standard_normal((n, dims[0]))
        got = O.forward("gat", theta, O.gat_structure(rp, ci, n), X)["logits"]
        assert np.allclose(got, dense_gat_logits(theta, A, X), rtol=1e-12, atol=1e-12)


def test_zero_attention_is_mean_over_closed_neighbourhood():
    """a_src = a_dst = 0: every e_ij = 0, alpha_ij = 1 / (deg_i + 1), so one layer is
    D~^{-1} (A + I) X W (a closed form with no softmax in it)."""
    rng = np.random.default_rng(1)
    n = 15
    rp, ci, A = rand_graph(n, 0.25, rng)
    W = rng.standard_normal((6, 4))
    theta = [np.vstack([W, np.zeros((2, 4))])]
    X = rng.standard_normal((n, 6))
    got = O.forward("gat", theta, O.gat_structure(rp, ci, n), X)["logits"]
    Dt = A.sum(axis=1) + 1.0
    assert np.allclose(got, ((A + np.eye(n)) / Dt[:, None]) @ X @ W, rtol=1e-12, atol=1e-12)


def test_isolated_node_attends_to_itself():
    theta = [np.array([[1.0, -2.0], [0.5, 0.25], [3.0, -1.0]])]      # d_0 = 1: W, a_src, a_dst
    rp = np.array([0, 0], dtype=np.int64)
    got = O.forward("gat", theta, O.gat_structure(rp, np.zeros(0, np.int64), 1), np.array([[2.0]]))["logits"]
    assert np.array_equal(got, np.array([[2.0, -4.0]]))


@pytest.mark.parametrize("dims", [[5, 3], [5, 7, 3], [4, 6, 5, 3]])
def test_backward_matches_finite_differences(dims):
    rng = np.random.default_rng(4)
    n = 10
    rp, ci, _ = rand_graph(n, 0.3, rng)
    op = O.gat_structure(rp, ci, n)
    theta = [rng.standard_normal(w.shape) for w in O.glorot_init("gat", dims, 1)]
    X = rng.standard_normal((n, dims[0]))
    labels = rng.integers(0, dims[-1], size=n)
    mask = rng.random(n) < 0.7
    tape = O.forward("gat", theta, op, X)
    _, dlog = O.softmax_ce(tape["logits"], labels, mask)
    grads = O.backward("gat", theta, op, tape, dlog)
    h = 1e-5
    for l, W in enumerate(theta):
        assert grads[l].shape == W.shape
        fd = np.zeros_like(W)
        for idx in np.ndindex(W.shape):
            wp = [w.copy() for w in theta]; wp[l][idx] += h
            wm = [w.copy() for w in theta]; wm[l][idx] -= h
            fd[idx] = (loss_of("gat", wp, op, X, labels, mask) - loss_of("gat", wm, op, X, labels, mask)) / (2 * h)
        err = np.max(np.abs(fd - grads[l])) / max(np.max(np.abs(fd)), 1e-12)
        assert err < 1e-4, (l, err)
        # the attention rows get a gradient of their own (they are trained)
        assert np.max(np.abs(fd[dims[l]:])) > 0


def test_extract_aggregate_attention_rows():
    dims, m = [6, 12, 10, 3], 3
    theta = O.glorot_init("gat", dims, 4)
    assert [w.shape for w in theta] == [(8, 12), (14, 10), (12, 3)]
    blocks = O.sample_partition(dims, m, seed=1, t=0)
    sets = [O.sub_index_sets("gat", dims, blocks, i) for i in range(m)]
    subs = [O.extract(theta, s) for s in sets]
    for i in range(m):
        r, c = sets[i][1]
        assert list(r[-2:]) == [12, 13] and np.array_equal(c, blocks[2][i])
        assert np.array_equal(subs[i][1][-2:], theta[1][[12, 13]][:, blocks[2][i]])
    counts = [np.zeros_like(w, dtype=int) for w in theta]
    for s in sets:
        for l, (r, c) in enumerate(s):
            counts[l][np.ix_(r, c)] += 1
    # disjoint everywhere except the output layer's attention rows: the class dimension is not
    # partitioned, so every sub-GCN holds all of them (R21: subAgg averages those)
    assert all(c[:-2].max() <= 1 for c in counts) and counts[0].max() == 1 and counts[1].max() == 1
    assert np.all(counts[1][12:] == 1) and np.all(counts[0][6:] == 1) and np.all(counts[2][10:] == m)
    before = [w.copy() for w in theta]
    O.aggregate(theta, subs, sets)
    assert all(np.array_equal(a, b) for a, b in zip(theta, before))
    assert O.sub_param_count("gat", dims, m, 0) == sum(s.size for s in subs[0])
    # OracleGIST.aggregate: replacement, then the shared rows = mean of the m copies
    o = O.OracleGIST(arch="gat", dims=dims)
    o.theta = [w.copy() for w in before]
    o.index_sets, o.m = sets, m
    o.sub = [[w.copy() for w in sub] for sub in subs]
    for i in range(m):
        o.sub[i][2][-2:] += float(i + 1)          # copy i moved by i + 1
        o.sub[i][1][:3] -= 7.0                    # a disjoint entry: replaced, not averaged
    o.aggregate()
    assert np.allclose(o.theta[2][10:], before[2][10:] + (m + 1) / 2.0, rtol=0, atol=1e-12)
    for i in range(m):
        r, c = sets[i][1]
        assert np.array_equal(o.theta[1][np.ix_(r[:3], c)], subs[i][1][:3] - 7.0)


def test_glorot_gat_scale_and_rows():
    th = O.glorot_init("gat", [10, 6, 3], 7)
    assert th[0].shape == (12, 6) and th[1].shape == (8, 3)
    assert np.max(np.abs(th[0])) <= np.sqrt(6.0 / 16.0) and np.max(np.abs(th[1])) <= np.sqrt(6.0 / 9.0)
    r, c = np.array([0, 11]), np.array([1, 5])
    assert np.array_equal(O.glorot_block("gat", [10, 6, 3], 7, 0, r, c), th[0][np.ix_(r, c)])


def test_gat_m1_reduces_to_plain_training():
    dims, zeta = (8, 10, 4), 3
    g = generate(tiny_spec(n=200, nnz=1200, d0=8, classes=4, clusters=6), seed=0)
    o = O.OracleGIST(arch="gat", dims=list(dims), optimizer="adam", clusters_per_batch=2, batch_seed=5)
    o.load_graph(g["row_ptr"], g["col_idx"], g["X"], g["labels"], 4, g["split"], g["cluster_ids"], 6)
    o.init_params(17)
    theta = [w.copy() for w in o.theta]
    o.partition(seed=1, m=1)
    o.subtrain(zeta, lr=0.05)
    o.aggregate()
    state = [{} for _ in theta]
    for z in range(zeta):
        nodes, rp, ci = o.make_batch(0, z)
        op = O.gat_structure(rp, ci, len(nodes))
        tape = O.forward("gat", theta, op, o.X[nodes])
        _, dlog = O.softmax_ce(tape["logits"], o.labels[nodes], o.split[nodes] == 0)
        grads = O.backward("gat", theta, op, tape, dlog)
        theta = [O.adam_step(w, gr, st, 0.05) for w, gr, st in zip(theta, grads, state)]
    assert all(np.array_equal(a, b) for a, b in zip(theta, o.theta))
