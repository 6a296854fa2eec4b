"""Pins for subGCNs / subAgg in the oracle: Philox KATs, partition invariants
(PAPER.md:147-161, 801-806), extract/aggregate, batch
schedule and induced subgraphs."""
import json
import os

import numpy as np
import pytest

from oracle import gist_oracle as O

HERE = os.path.dirname(__file__)
GOLD = json.load(open(os.path.join(HERE, "golden", "paper_examples.json")))


def kat_rows():
    for line in open(os.path.join(HERE, "golden", "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        yield v[:4], v[4:6], v[6:10]


def test_philox_known_answers():
    for ctr, key, out in kat_rows():
        got = O.philox4x32_10(np.array([ctr], dtype=np.uint64), tuple(key))[0]
        assert [int(x) for x in got] == out


@pytest.mark.parametrize("dims,m", [([11, 40, 33, 5], 4), ([7, 9, 3], 2), ([3, 8, 8, 8, 2], 8), ([5, 6, 2], 1)])
def test_partition_disjoint_cover_balance(dims, m):
    blocks = O.sample_partition(dims, m, seed=123, t=3)
    L = len(dims) - 1
    for l, d in enumerate(dims):
        if l in (0, L):      # d_0 and d_L never partitioned
            for b in blocks[l]:
                assert np.array_equal(b, np.arange(d))
            continue
        allu = np.concatenate(blocks[l])
        assert np.array_equal(np.sort(allu), np.arange(d))      # disjoint cover
        sizes = [len(b) for b in blocks[l]]
        assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
        for b in blocks[l]:
            assert np.all(np.diff(b) > 0)                      # ascending (R5)
        if m == 1:
            assert np.array_equal(blocks[l][0], np.arange(d))


def test_partition_footnote_format():
    g = GOLD["footnote_partition"]
    blocks = O.sample_partition([3, g["d"], 2], g["m"], seed=0, t=0)[1]
    assert sorted(len(b) for b in blocks) == [2, 2]
    assert sorted(int(x) for b in blocks for x in b) == [0, 1, 2, 3]
    # the paper's example itself is a valid output of the same format
    ex = [np.array(b) - 1 for b in g["blocks_1based"]]
    assert sorted(np.concatenate(ex).tolist()) == [0, 1, 2, 3]


def test_partition_deterministic_and_fresh_per_round():
    a = O.sample_partition([4, 64, 4], 4, seed=9, t=0)
    b = O.sample_partition([4, 64, 4], 4, seed=9, t=0)
    c = O.sample_partition([4, 64, 4], 4, seed=9, t=1)
    assert all(np.array_equal(x, y) for x, y in zip(a[1], b[1]))
    assert not all(np.array_equal(x, y) for x, y in zip(a[1], c[1]))


def test_partition_marginal_is_one_over_m():
    g = GOLD["mask_marginal"]
    d, m, trials = g["d"], g["m"], 4000
    hits = np.zeros(d)
    for t in range(trials):
        hits[O.sample_partition([2, d, 2], m, seed=77, t=t)[1][0]] += 1
    freq = hits / trials
    assert np.all(np.abs(freq - g["p"]) < 0.04), freq


def test_partition_rejects_m_above_hidden_dim():
    with pytest.raises(ValueError):
        O.sample_partition([5, 3, 2], 4, 0, 0)


@pytest.mark.parametrize("arch", ["gcn", "sage"])
def test_extract_aggregate_roundtrip_write_once_coverage(arch):
    dims, m = [6, 12, 10, 3], 3
    theta = O.glorot_init(arch, dims, 4)
    before = [w.copy() for w in theta]
    blocks = O.sample_partition(dims, m, seed=1, t=0)
    sets = [O.sub_index_sets(arch, dims, blocks, i) for i in range(m)]
    subs = [O.extract(theta, s) for s in sets]
    for i in range(m):                         # shapes (SAGE rows doubled)
        f = 2 if arch == "sage" else 1
        assert subs[i][0].shape == (f * 6, len(blocks[1][i]))
        assert subs[i][2].shape == (f * len(blocks[2][i]), 3)
    O.aggregate(theta, subs, sets)             # aggregate(extract) = identity
    assert all(np.array_equal(a, b) for a, b in zip(theta, before))
    # write-once: count writes per entry
    counts = [np.zeros_like(w, dtype=int) for w in theta]
    for s in sets:
        for l, (r, c) in enumerate(s):
            counts[l][np.ix_(r, c)] += 1
    assert all(c.max() <= 1 for c in counts)
    # mark-and-aggregate: uncovered entries keep their bits, covered ones change
    marked = [[w + 1000.0 for w in sub] for sub in subs]
    O.aggregate(theta, marked, sets)
    for l in range(3):
        changed = theta[l] != before[l]
        assert np.array_equal(changed, counts[l] == 1)
    # hidden layer coverage exactly 1/m when m divides the dims
    assert O.coverage_fraction([6, 12, 9, 3], O.sample_partition([6, 12, 9, 3], 3, 2, 0), 1, 3, arch) == pytest.approx(1 / 3, abs=0)


def test_delta_sum_equals_replacement_within_ulp():
    dims, m = [5, 8, 8, 2], 2
    theta = O.glorot_init("gcn", dims, 4)
    blocks = O.sample_partition(dims, m, seed=1, t=0)
    sets = [O.sub_index_sets("gcn", dims, blocks, i) for i in range(m)]
    s0 = [O.extract(theta, s) for s in sets]
    rng = np.random.default_rng(0)
    s1 = [[w + 0.01 * rng.standard_normal(w.shape) for w in sub] for sub in s0]
    delta = O.aggregate_delta_sum(theta, s0, s1, sets)
    repl = [w.copy() for w in theta]
    O.aggregate(repl, s1, sets)
    for a, b in zip(delta, repl):
        assert np.all(np.abs(a - b) <= np.spacing(np.maximum(np.abs(a), np.abs(b))))


def test_comm_accounting_paper_dims():
    g = GOLD["comm_scalars"]
    assert O.sub_param_count("gcn", g["dims"], g["m"]) == g["gist_per_worker"]
    assert O.sub_param_count("gcn", g["dims"], 1) == g["full_model"]


# ----------------------------------------------------------------- batches --
def test_batch_schedule_each_cluster_once_per_epoch():
    c, q = 23, 5
    B = -(-c // q)
    for slot in (0, 3):
        for e in range(3):
            seen = np.concatenate([O.batch_schedule(c, q, 99, slot, e * B + p) for p in range(B)])
            assert np.array_equal(np.sort(seen), np.arange(c))
    a = np.concatenate([O.batch_schedule(c, q, 99, 0, p) for p in range(B)])
    b = np.concatenate([O.batch_schedule(c, q, 99, 1, p) for p in range(B)])
    assert not np.array_equal(a, b)           # slots draw independent sequences (R7)


def test_induced_subgraph_bruteforce():
    rng = np.random.default_rng(3)
    n = 30
    A = np.triu((rng.random((n, n)) < 0.2).astype(int), 1); A = A + A.T
    rp = np.concatenate([[0], np.cumsum(A.sum(1))])
    ci = np.concatenate([np.nonzero(A[i])[0] for i in range(n)])
    nodes = np.sort(rng.choice(n, 12, replace=False))
    brp, bci = O.induced_subgraph(rp, ci, nodes)
    sub = A[np.ix_(nodes, nodes)]
    for i in range(len(nodes)):
        assert np.array_equal(bci[brp[i]:brp[i + 1]], np.nonzero(sub[i])[0])
    # triangle K3, nodes {0,1} -> P2
    rp3, ci3 = np.array([0, 2, 4, 6]), np.array([1, 2, 0, 2, 0, 1])
    r, c = O.induced_subgraph(rp3, ci3, np.array([0, 1]))
    assert r.tolist() == [0, 1, 2] and c.tolist() == [1, 0]
