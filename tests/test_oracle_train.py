"""End-to-end pins of the oracle's Algorithm 1 driver."""
import numpy as np
import pytest

from oracle import gist_oracle as O
from synth.planted import generate, tiny_spec


def make(arch, dims, optimizer="sgd", q=3, seed=0, spec=None):
    g = generate(spec or tiny_spec(n=300, nnz=2000, d0=dims[0], classes=dims[-1], clusters=9), seed=seed)
    o = O.OracleGIST(arch=arch, dims=list(dims), optimizer=optimizer, clusters_per_batch=q, batch_seed=5)
    o.load_graph(g["row_ptr"], g["col_idx"], g["X"], g["labels"], g["num_classes"], g["split"],
                 g["cluster_ids"], g["num_clusters"])
    o.init_params(17)
    return o, g


@pytest.mark.parametrize("arch", ["gcn", "sage"])
@pytest.mark.parametrize("optimizer", ["sgd", "adam"])
def test_m1_reduces_to_plain_training(arch, optimizer):
    """GIST with m=1 is plain training: partition = identity, extract /
    aggregate = identity.  The plain loop below uses only forward/backward/optimizer
    on the full Theta; Adam restarts every zeta steps (R8)."""
    dims, zeta, rounds = (8, 10, 6, 4), 3, 2
    o, _ = make(arch, dims, optimizer)
    theta = [w.copy() for w in o.theta]
    for t in range(rounds):
        o.partition(seed=1, m=1)
        o.subtrain(zeta, lr=0.05)
        o.aggregate()
    # plain training
    p, _ = make(arch, dims, optimizer)
    assert all(np.array_equal(a, b) for a, b in zip(theta, p.theta))
    step = 0
    for t in range(rounds):
        state = [{} for _ in theta]
        for z in range(zeta):
            nodes, rp, ci = p.make_batch(0, step)
            op = p.operator(rp, ci, len(nodes))
            tape = O.forward(arch, theta, op, p.X[nodes])
            _, dl = O.softmax_ce(tape["logits"], p.labels[nodes], p.split[nodes] == 0)
            gr = O.backward(arch, theta, op, tape, dl)
            for l in range(len(theta)):
                theta[l] = (O.adam_step(theta[l], gr[l], state[l], 0.05) if optimizer == "adam"
                            else O.sgd_step(theta[l], gr[l], 0.05))
            step += 1
    assert all(np.array_equal(a, b) for a, b in zip(theta, o.theta))


@pytest.mark.parametrize("arch", ["gcn", "sage"])
def test_m1_persistent_adam_reduces_to_plain_adam(arch):
    """SURVEY §8 f3 (persistent sliced optimizer state): with m = 1 every slice is the whole
    model, so GIST with persistent Adam state is plain Adam training WITHOUT restarts: the
    plain loop below keeps one Adam state for the whole run (bit-exact)."""
    dims, zeta, rounds = (8, 10, 6, 4), 3, 3
    o, _ = make(arch, dims, "adam")
    o.opt_state = "persistent"
    theta = [w.copy() for w in o.theta]
    for t in range(rounds):
        o.partition(seed=1, m=1)
        o.subtrain(zeta, lr=0.05)
        o.aggregate()
    p, _ = make(arch, dims, "adam")
    state = [{} for _ in theta]
    step = 0
    for t in range(rounds * zeta):
        nodes, rp, ci = p.make_batch(0, step)
        op = p.operator(rp, ci, len(nodes))
        tape = O.forward(arch, theta, op, p.X[nodes])
        _, dl = O.softmax_ce(tape["logits"], p.labels[nodes], p.split[nodes] == 0)
        gr = O.backward(arch, theta, op, tape, dl)
        for l in range(len(theta)):
            theta[l] = O.adam_step(theta[l], gr[l], state[l], 0.05)
        step += 1
    assert all(np.array_equal(a, b) for a, b in zip(theta, o.theta))
    assert o.t_global == rounds * zeta


def test_persistent_moments_slice_like_the_weights():
    """f3: after a round with m = 2 the global moments are nonzero exactly on the entries the
    sub-GCNs own (write-back by replacement), zero elsewhere; the step counter advanced by zeta;
    and with opt_state = "reset" (default) the second round restarts from t = 0."""
    dims = (8, 12, 10, 4)
    o, _ = make("sage", dims, "adam")
    o.opt_state = "persistent"
    o.partition(seed=3, m=2)
    sets = o.index_sets
    o.subtrain(4, lr=0.01)
    o.aggregate()
    assert o.t_global == 4
    for l in range(3):
        cov = np.zeros_like(o.theta[l], dtype=bool)
        for s in sets:
            cov[np.ix_(*s[l])] = True
        assert np.all(o.vel[l][~cov] == 0) and np.all(o.mom[l][~cov] == 0)
        assert np.mean(o.vel[l][cov] > 0) > 0.5      # second moments of trained entries
    o.partition(seed=4, m=2)
    assert all(st["t"] == 4 for so in o.opt for st in so)   # counter carried into the new round
    r, _ = make("sage", dims, "adam")
    r.partition(seed=3, m=2)
    assert all(st == {} for so in r.opt for st in so)        # default: reset per round (R8)


def test_only_covered_entries_change_after_a_round():
    dims = (8, 12, 10, 4)
    o, _ = make("gcn", dims, "adam")
    before = [w.copy() for w in o.theta]
    o.partition(seed=3, m=2)
    sets = o.index_sets
    o.subtrain(4, lr=0.01)
    o.aggregate()
    for l in range(3):
        cov = np.zeros_like(before[l], dtype=bool)
        for s in sets:
            cov[np.ix_(*s[l])] = True
        changed = o.theta[l] != before[l]
        assert not np.any(changed & ~cov)       # untouched entries keep their bits
        assert changed[cov].mean() > 0.5        # trained entries moved (dead ReLU units stay)


def test_gist_loss_decreases_and_is_deterministic():
    dims = (16, 32, 6)
    spec = tiny_spec(n=400, nnz=3000, d0=16, classes=6, clusters=8)
    o, g = make("gcn", dims, "adam", q=2, spec=spec)
    first = None
    for t in range(8):
        o.partition(seed=11, m=2)
        loss = o.subtrain(5, lr=0.01)
        o.aggregate()
        first = loss.mean() if first is None else first
    last = loss.mean()
    assert last < 0.7 * first
    _, acc, _ = o.eval(0)
    assert acc > 2.0 / 6
    o2, _ = make("gcn", dims, "adam", q=2, spec=spec)
    for t in range(8):
        o2.partition(seed=11, m=2)
        o2.subtrain(5, lr=0.01)
        o2.aggregate()
    assert all(np.array_equal(a, b) for a, b in zip(o.theta, o2.theta))
