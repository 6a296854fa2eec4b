"""Pins for the oracle's model arithmetic (SpMM, operators, forward, backward, loss,
optimizers, init).  Each test checks the oracle against something other than
itself: the paper's worked values, dense brute force, finite differences, the
closed-form gradient of PAPER.md Appendix C.1, or an algebraic identity."""
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import gist_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def rand_graph(n, p, rng):
    """Symmetric 0/1 adjacency without self loops as CSR arrays (+ dense)."""
    A = (rng.random((n, n)) < p).astype(np.float64)
    A = np.triu(A, 1)
    A = A + A.T
    rp = np.zeros(n + 1, dtype=np.int64)
    cols = []
    for i in range(n):
        c = np.nonzero(A[i])[0]
        cols.append(c)
        rp[i + 1] = rp[i] + len(c)
    ci = np.concatenate(cols) if cols else np.zeros(0, np.int64)
    return rp, ci, A


# ----------------------------------------------------------------- SpMM -----
def test_spmm_equals_dense_bruteforce_integer_exact():
    rng = np.random.default_rng(0)
    for n, w in [(1, 1), (7, 3), (33, 17), (64, 5)]:
        rp, ci, A = rand_graph(n, 0.2, rng)
        H = rng.integers(-5, 6, size=(n, w)).astype(np.float64)
        got = O.spmm(O._adjacency(rp, ci, n), H)
        want = np.zeros((n, w))
        for i in range(n):                          # brute force dense loops
            for j in range(n):
                want[i] += A[i, j] * H[j]
        assert np.array_equal(got, want)


def test_spmm_zero_and_identity():
    n = 9
    H = np.arange(n * 4, dtype=np.float64).reshape(n, 4)
    Z = sp.csr_matrix((n, n))
    assert np.array_equal(O.spmm(Z, H), np.zeros_like(H))
    assert np.array_equal(O.spmm(sp.identity(n, format="csr"), H), H)


# ------------------------------------------------------------ operators -----
def p2():
    return np.array([0, 1, 2]), np.array([1, 0])


def test_p2_renorm_and_chebyshev_paper_values():
    rp, ci = p2()
    assert np.allclose(O.gcn_operator(rp, ci, 2).toarray(), GOLD["p2_renorm"]["A_hat"], atol=0, rtol=1e-15)
    assert np.array_equal(O.chebyshev_operator(rp, ci, 2).toarray(), np.array(GOLD["p2_chebyshev"]["A_bar"]))


def test_edgeless_renorm_is_identity_and_sage_is_zero():
    rp, ci = np.zeros(5, dtype=np.int64), np.zeros(0, dtype=np.int64)
    assert np.array_equal(O.gcn_operator(rp, ci, 4).toarray(), np.eye(4))
    assert np.array_equal(O.sage_operator(rp, ci, 4).toarray(), np.zeros((4, 4)))


def test_operators_structure():
    rng = np.random.default_rng(1)
    rp, ci, A = rand_graph(40, 0.15, rng)
    G = O.gcn_operator(rp, ci, 40).toarray()
    assert np.array_equal(G, G.T) or np.max(np.abs(G - G.T)) < 1e-16
    deg = A.sum(1)
    # entry-wise definition D~^-1/2 (A+I) D~^-1/2
    dt = deg + 1
    for i in range(40):
        for j in range(40):
            want = (A[i, j] + (i == j)) / math.sqrt(dt[i] * dt[j])
            assert abs(G[i, j] - want) < 1e-15
    N = O.sage_operator(rp, ci, 40).toarray()
    rs = N.sum(1)
    assert np.allclose(rs[deg > 0], 1.0, atol=1e-14) and np.all(rs[deg == 0] == 0)
    # N^T = A diag(1/deg): the backward SpMM uses a column scale
    inv = np.where(deg > 0, 1 / np.maximum(deg, 1), 0)
    assert np.allclose(N.T, A * inv[None, :], atol=1e-15)


def test_chebyshev_eigen_range():
    """2 = lambda_max >= lambda_min >= 0 for Eq. (3) (graphs without isolated nodes)."""
    rng = np.random.default_rng(2)
    rp, ci, A = rand_graph(30, 0.3, rng)
    assert A.sum(1).min() > 0
    ev = np.linalg.eigvalsh(O.chebyshev_operator(rp, ci, 30).toarray())
    assert ev.max() <= 2 + 1e-9 and ev.min() >= -1e-9


# --------------------------------------------------------------- forward ----
def test_chebyshev_forward_paper_example():
    g = GOLD["p2_chebyshev_forward"]
    rp, ci = p2()
    op = O.chebyshev_operator(rp, ci, 2)
    out = O.forward("gcn", [np.array(g["theta0"])], op, np.array(g["X"]))
    assert np.array_equal(out["logits"], np.array(g["logits"]))


@pytest.mark.parametrize("arch", ["gcn", "sage"])
def test_two_layer_sum_identity(arch):
    """For L=2, the sub-GCN logits sum to the global logits on a common graph:
    Z1 = sum_r relu(C0 W0)[:, r] W1[r, :] and the blocks D_1^(i) partition r."""
    rng = np.random.default_rng(3)
    n, dims, m = 25, [6, 12, 4], 3
    rp, ci, _ = rand_graph(n, 0.2, rng)
    op = O.gcn_operator(rp, ci, n) if arch == "gcn" else O.sage_operator(rp, ci, n)
    theta = O.glorot_init(arch, dims, seed=11)
    X = rng.standard_normal((n, dims[0]))
    glob = O.forward(arch, theta, op, X)["logits"]
    blocks = O.sample_partition(dims, m, seed=5, t=0)
    tot = np.zeros_like(glob)
    for i in range(m):
        sub = O.extract(theta, O.sub_index_sets(arch, dims, blocks, i))
        tot += O.forward(arch, sub, op, X)["logits"]
    assert np.max(np.abs(tot - glob)) <= 1e-12 * np.max(np.abs(glob))


def test_relu_zeroes_negative_preactivation():
    rp, ci = p2()
    op = O.gcn_operator(rp, ci, 2)
    X = np.array([[1.0], [1.0]])
    out = O.forward("gcn", [np.array([[-1.0, 2.0]]), np.array([[1.0], [1.0]])], op, X)
    assert np.all(out["H"][1][:, 0] == 0) and np.all(out["H"][1][:, 1] > 0)


# -------------------------------------------------------------- backward ----
def loss_of(arch, theta, op, X, labels, mask):
    return O.softmax_ce(O.forward(arch, theta, op, X)["logits"], labels, mask)[0]


@pytest.mark.parametrize("arch", ["gcn", "sage"])
@pytest.mark.parametrize("dims", [[5, 3], [5, 7, 3], [4, 6, 5, 3]])
def test_backward_matches_finite_differences(arch, dims):
    rng = np.random.default_rng(4)
    n = 10
    rp, ci, _ = rand_graph(n, 0.3, rng)
    op = O.gcn_operator(rp, ci, n) if arch == "gcn" else O.sage_operator(rp, ci, n)
    theta = [rng.standard_normal(w.shape) for w in O.glorot_init(arch, dims, 1)]
    X = rng.standard_normal((n, dims[0]))
    labels = rng.integers(0, dims[-1], size=n)
    mask = rng.random(n) < 0.7
    tape = O.forward(arch, theta, op, X)
    _, dlog = O.softmax_ce(tape["logits"], labels, mask)
    grads = O.backward(arch, theta, op, tape, dlog)
    h = 1e-5
    for l, W in enumerate(theta):
        fd = np.zeros_like(W)
        for idx in np.ndindex(W.shape):
            wp = [w.copy() for w in theta]; wp[l][idx] += h
            wm = [w.copy() for w in theta]; wm[l][idx] -= h
            fd[idx] = (loss_of(arch, wp, op, X, labels, mask) - loss_of(arch, wm, op, X, labels, mask)) / (2 * h)
        err = np.max(np.abs(fd - grads[l])) / max(np.max(np.abs(fd)), 1e-12)
        assert err < 1e-4, (l, err)


def test_backward_closed_form_one_hidden_layer():
    """PAPER.md:823-826 (App. C.1): dL/dtheta_r = 1/sqrt(d1) sum_i sum_i' (yhat_i - y_i) A_ii' a_r
    xhat_i' 1{<theta_r, xhat_i'> >= 0}, with xhat = A_bar X.  The printed formula
    omits the factor 2 of d||y - yhat||^2, i.e. it is the gradient of (1/2)||.||^2 (reading G13),
    so dlogits = yhat - y here."""
    rng = np.random.default_rng(5)
    n, d, d1 = 12, 4, 9
    rp, ci, _ = rand_graph(n, 0.3, rng)
    Abar = O.chebyshev_operator(rp, ci, n)
    X = rng.standard_normal((n, d))
    Theta = rng.standard_normal((d, d1))
    a = rng.choice([-1.0, 1.0], size=d1)
    W1 = (a / math.sqrt(d1))[:, None]
    y = rng.standard_normal((n, 1))
    tape = O.forward("gcn", [Theta, W1], Abar, X)
    yhat = tape["logits"]
    grads = O.backward("gcn", [Theta, W1], Abar, tape, yhat - y)
    Ad = Abar.toarray()
    xhat = Ad @ X
    closed = np.zeros((d, d1))
    for r in range(d1):
        for i in range(n):
            for ip in range(n):
                ind = 1.0 if xhat[ip] @ Theta[:, r] >= 0 else 0.0
                closed[:, r] += (yhat[i, 0] - y[i, 0]) * Ad[i, ip] * a[r] * xhat[ip] * ind / math.sqrt(d1)
    assert np.max(np.abs(closed - grads[0])) < 1e-12 * max(1.0, np.max(np.abs(closed)))


def test_zero_dlogits_give_zero_grads():
    rng = np.random.default_rng(6)
    rp, ci, _ = rand_graph(8, 0.4, rng)
    op = O.sage_operator(rp, ci, 8)
    theta = O.glorot_init("sage", [3, 4, 2], 0)
    tape = O.forward("sage", theta, op, rng.standard_normal((8, 3)))
    for g in O.backward("sage", theta, op, tape, np.zeros((8, 2))):
        assert np.all(g == 0)


# ------------------------------------------------------------------ loss ----
def test_ce_uniform_logits_is_ln_k():
    for k in (2, 7, 41):
        loss, d = O.softmax_ce(np.zeros((5, k)), np.arange(5) % k, np.ones(5, bool))
        assert abs(loss - math.log(k)) < 1e-12
        assert np.allclose(d.sum(1), 0, atol=1e-15)


def test_ce_fd_and_masking():
    rng = np.random.default_rng(7)
    z = rng.standard_normal((6, 4)) * 3
    y = rng.integers(0, 4, 6)
    mask = np.array([1, 0, 1, 1, 0, 1], bool)
    loss, d = O.softmax_ce(z, y, mask)
    assert np.all(d[~mask] == 0)
    # direct definition: mean over masked rows of -log softmax
    direct = np.mean([-(z[i, y[i]] - math.log(np.sum(np.exp(z[i])))) for i in np.nonzero(mask)[0]])
    assert abs(loss - direct) < 1e-12
    h = 1e-6
    for idx in np.ndindex(z.shape):
        zp = z.copy(); zp[idx] += h
        zm = z.copy(); zm[idx] -= h
        fd = (O.softmax_ce(zp, y, mask)[0] - O.softmax_ce(zm, y, mask)[0]) / (2 * h)
        assert abs(fd - d[idx]) < 1e-8
    l0, d0 = O.softmax_ce(z, y, np.zeros(6, bool))
    assert l0 == 0.0 and np.all(d0 == 0)


# ------------------------------------------------------------ optimizers ----
def test_adam_first_step_closed_form():
    """Adam step 1: mhat = g, vhat = g^2 => delta = -lr g / (|g| + eps)."""
    g = np.array([[0.3, -2.0, 1e-9, 0.0]])
    w = np.array([[1.0, 1.0, 1.0, 1.0]])
    st = {}
    w1 = O.adam_step(w, g, st, lr=0.01)
    assert np.allclose(w1 - w, -0.01 * g / (np.abs(g) + 1e-8), rtol=1e-12, atol=0)
    w2 = O.adam_step(w1, np.zeros_like(g), st, lr=0.01)   # second step, zero grad
    m = 0.9 * 0.1 * g; v = 0.999 * 0.001 * g * g
    want = w1 - 0.01 * (m / (1 - 0.81)) / (np.sqrt(v / (1 - 0.999 ** 2)) + 1e-8)
    assert np.allclose(w2, want, rtol=1e-12, atol=1e-15)


def test_sgd_linearity():
    w = np.array([1.0, 2.0]); g = np.array([0.5, -1.0])
    assert np.array_equal(O.sgd_step(O.sgd_step(w, g, 0.25), g, 0.25), O.sgd_step(w, 2 * g, 0.25))  # exact binary values
    assert np.array_equal(O.sgd_step(w, np.zeros(2), 0.1), w)


def test_lr_schedule_paper_values():
    for base, ep, tot, want in GOLD["lr_schedule"]["cases"]:
        assert abs(O.lr_step_schedule(base, ep, tot) - want) < 1e-15


# ------------------------------------------------------------------ init ----
def test_glorot_init_bounds_determinism_and_fp32():
    th = O.glorot_init("gcn", [4, 3], 7)
    assert th[0].shape == (4, 3) and np.all(np.abs(th[0]) <= math.sqrt(6 / 7))
    assert all(np.array_equal(a, b) for a, b in zip(th, O.glorot_init("gcn", [4, 3], 7)))
    assert not np.array_equal(th[0], O.glorot_init("gcn", [4, 3], 8)[0])
    ts = O.glorot_init("sage", [5, 6, 2], 1)
    assert ts[0].shape == (10, 6) and ts[1].shape == (12, 2)
    big = O.glorot_init("gcn", [300, 200], 3)[0]
    assert np.array_equal(big, big.astype(np.float32).astype(np.float64))   # exact fp32 values
    s = math.sqrt(6 / 500)
    assert abs(big.mean()) < 0.01 * s and abs(big.std() - s / math.sqrt(3)) < 0.01 * s


def test_glorot_block_equals_full_init_slices():
    rng = np.random.default_rng(0)
    for arch, dims in [("gcn", [30, 40, 7]), ("sage", [25, 33, 9])]:
        full = O.glorot_init(arch, dims, 13)
        for l in range(len(dims) - 1):
            rows = np.sort(rng.choice(full[l].shape[0], 6, replace=False))
            cols = np.sort(rng.choice(full[l].shape[1], 5, replace=False))
            assert np.array_equal(O.glorot_block(arch, dims, 13, l, rows, cols), full[l][np.ix_(rows, cols)])
