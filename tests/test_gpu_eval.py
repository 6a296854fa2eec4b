"""Parity of partition-wise evaluation (gist_eval_parts, reading R20)
against the FP64 oracle: small ragged graphs with random partitions (an empty partition,
partitions without evaluated nodes, chunking forced down to a few rows), the training
clusters as partitions, one all-covering partition against the full-graph eval, and the
Reddit-shaped C3 graph at the bench's global width 4096 on sampled partitions."""
import math

import numpy as np
import pytest

from oracle import gist_oracle as O
from synth.planted import GRAPHS, MODELS, generate, tiny_spec
from tests.gpu_helpers import make_pair

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "bf16": 2e-2}


def check(lg, ag, lpg, apg, lo, ao, lpo, apo, precision):
    ok = ~np.isnan(apo)
    assert np.array_equal(ok, ~np.isnan(apg))        # the same partitions are evaluated
    t = TOL[precision]
    assert np.max(np.abs(lpg[ok] - lpo[ok])) <= t * max(1.0, np.max(np.abs(lpo[ok])))
    assert abs(lg - lo) <= t * max(1.0, abs(lo))
    if precision == "fp32":
        assert np.array_equal(apg[ok], apo[ok].astype(np.float32))
        assert ag == pytest.approx(ao, abs=1e-6)
    else:   # bf16: an argmax may flip on a near tie
        assert abs(ag - ao) <= 0.02


@pytest.mark.parametrize("arch", ["gcn", "sage"])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("max_rows", [0, 37])
def test_eval_parts_random_partitions(arch, precision, max_rows):
    g = generate(tiny_spec(n=700, nnz=6000, d0=29, classes=6, clusters=11), seed=2)
    dims = (29, 40, 24, 6)
    gpu, ora = make_pair(g, arch, dims, precision=precision)
    rng = np.random.default_rng(1)
    n = len(g["labels"])
    # 23 partitions: a few large, one empty (id 5), one without split-0 nodes (id 7)
    part = (rng.integers(0, 22, n) + (rng.random(n) < 0.3) * (np.arange(n) % 3)) % 22
    part[part >= 5] += 1
    part[(part == 7) & (g["split"] == 0)] = 8
    lg, ag, lpg, apg = gpu.eval_parts(0, part, 23, max_rows=max_rows)
    lo, ao, lpo, apo = ora.eval_partitions(0, part, 23)
    assert math.isnan(apo[5]) and math.isnan(apo[7])
    check(lg, ag, lpg, apg, lo, ao, lpo, apo, precision)


@pytest.mark.parametrize("arch", ["gcn", "sage"])
def test_eval_parts_training_clusters_and_full_graph(arch):
    g = generate(tiny_spec(n=500, nnz=4000, d0=17, classes=5, clusters=9), seed=4)
    dims = (17, 32, 5)
    gpu, ora = make_pair(g, arch, dims, q=2)
    gpu.partition(seed=3, m=2)      # one trained round so the weights are not the init
    ora.partition(seed=3, m=2)
    gpu.subtrain(3, lr=0.02)
    ora.subtrain(3, lr=0.02)
    gpu.aggregate()
    ora.aggregate()
    for code in (0, 2):
        lg, ag, lpg, apg = gpu.eval_parts(code)            # NULL = the training clusters
        lo, ao, lpo, apo = ora.eval_partitions(code, g["cluster_ids"], g["num_clusters"])
        check(lg, ag, lpg, apg, lo, ao, lpo, apo, "fp32")
    n = len(g["labels"])
    lg, ag, _, _ = gpu.eval_parts(1, np.zeros(n, np.int32), 1)
    lf, af = gpu.eval(1)
    lo, ao, _ = ora.eval(1)
    assert abs(lg - lo) <= 1e-4 * max(1.0, lo) and abs(lf - lg) <= 1e-5 * max(1.0, lf)
    assert ag == pytest.approx(ao, abs=1e-6)


def test_eval_parts_bad_ids():
    from paper_2102_10424_b200.gist import GistError
    g = generate(tiny_spec(n=100, nnz=600, d0=5, classes=3, clusters=4), seed=0)
    gpu, _ = make_pair(g, "gcn", (5, 8, 3))
    part = np.zeros(100, np.int32)
    part[3] = 4
    with pytest.raises(GistError):
        gpu.eval_parts(0, part, 4)
    with pytest.raises(GistError):
        gpu.eval_parts(7, part, 5)


@pytest.fixture(scope="module")
def c3():
    spec = MODELS["C3"]
    g = generate(GRAPHS["reddit"], seed=0, device="cuda")
    dims = list(spec.dims)
    n = len(g["labels"])
    order = np.argsort(g["cluster_ids"], kind="stable")
    part = np.empty(n, np.int32)
    part[order] = (np.arange(n) * 5000) // n
    ora = O.OracleGIST(arch=spec.arch, dims=dims)
    ora.load_graph(g["row_ptr"], g["col_idx"], g["X"], g["labels"], g["num_classes"], g["split"],
                   g["cluster_ids"], g["num_clusters"])
    ora.init_params(11)     # the same counter-based Glorot init (R11), computed on the host
    return spec, g, part, ora


@pytest.mark.slow
@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_eval_parts_c3_full_size_sampled(c3, precision):
    """C3 graph (232,965 nodes, 114.6M nnz), global 4-layer GraphSAGE at width 4096 — the
    regime where the paper evaluates on 5,000 partitions.  Partitions: the cluster-sorted
    node order cut into 5,000 contiguous pieces (≈ 47 nodes, mostly inside one cluster).
    The oracle recomputes 12 sampled partitions in FP64."""
    from paper_2102_10424_b200.gist import Gist
    spec, g, part, ora = c3
    gpu = Gist(spec.arch, list(spec.dims), precision=precision, clusters_per_batch=spec.q)
    gpu.load_graph(g)
    gpu.init_params(11)
    from tests.gpu_helpers import rel_err
    lg, ag, lpg, apg = gpu.eval_parts(2, part, 5000)
    sample = np.random.default_rng(0).choice(5000, 12, replace=False)
    lref = np.zeros((len(g["labels"]), g["num_classes"]))
    _, _, lpo, apo = ora.eval_partitions(2, part, 5000, parts=sample, logits_out=lref)
    ok = ~np.isnan(apo[sample])
    assert ok.sum() >= 8
    s = sample[ok]
    t = TOL[precision]
    # per node: the logits of every node of the sampled partitions
    lgot = gpu.eval_logits(1, part, 5000)
    nodes = np.nonzero(np.isin(part, sample))[0]
    assert rel_err(lgot[nodes], lref[nodes]) <= t
    assert np.max(np.abs(lpg[s] - lpo[s])) <= t * max(1.0, np.max(np.abs(lpo[s])))
    if precision == "fp32":
        assert np.array_equal(apg[s], apo[s].astype(np.float32))
    # the means cover every evaluated partition
    okg = ~np.isnan(apg)
    assert lg == pytest.approx(float(np.mean(lpg[okg].astype(np.float64))), rel=1e-5)
    assert ag == pytest.approx(float(np.mean(apg[okg].astype(np.float64))), rel=1e-5)


@pytest.mark.slow
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_full_graph_eval_c2_full_size(precision):
    """C2 (ogbn-arxiv-shaped, 169,343 nodes, 1.17 M edges), 3-layer GCN hidden 1024: the
    full-graph eval operator runs in L2-sized column slabs (n >= 65,536), GCN scalings and the
    self term included; the FP64 oracle computes the whole forward."""
    spec = MODELS["C2"]
    g = generate(GRAPHS["arxiv"], seed=0, device="cuda")
    dims = list(spec.dims)
    gpu, ora = make_pair(g, spec.arch, dims, precision=precision, q=spec.q)
    t = TOL[precision]
    from tests.gpu_helpers import rel_err
    for code in (1, 2):
        lg, ag = gpu.eval(code)
        lo, ao, lref = ora.eval(code)
        assert abs(lg - lo) <= t * max(1.0, abs(lo)), (code, lg, lo)
        if code == 1:   # per node, every one of the 169,343 rows
            assert rel_err(gpu.eval_logits(0), lref) <= t
        assert abs(ag - ao) <= (1e-5 if precision == "fp32" else 5e-3), (code, ag, ao)
    # partition-wise over the training clusters, checked on every partition
    lg, ag, lpg, apg = gpu.eval_parts(2)
    lo, ao, lpo, apo = ora.eval_partitions(2, g["cluster_ids"], g["num_clusters"])
    ok = ~np.isnan(apo)
    assert np.max(np.abs(lpg[ok] - lpo[ok])) <= t * max(1.0, np.max(np.abs(lpo[ok])))


# ---------------------------------------------------------------- per-node eval logits
# gist_eval_logits returns the logits of exactly the forward gist_eval (mode 0) / gist_eval_parts
# (mode 1) run, so the evaluation is checked element by element, not only through its means.
def _trained_pair(arch, precision, dims=(29, 40, 24, 6), optimizer="adam"):
    g = generate(tiny_spec(n=700, nnz=6000, d0=dims[0], classes=dims[-1], clusters=11), seed=2)
    gpu, ora = make_pair(g, arch, dims, precision=precision, q=3, optimizer=optimizer)
    gpu.partition(seed=3, m=2)
    ora.partition(seed=3, m=2)
    gpu.subtrain(2, lr=0.01)
    ora.subtrain(2, lr=0.01)
    gpu.aggregate()
    ora.aggregate()
    # the trained weights may differ slightly between the two (Adam sign steps):
    # evaluate both at the GPU's global weights, so the eval forward alone is compared
    ora.set_params([gpu.get_params(l).astype(np.float64) for l in range(len(dims) - 1)])
    return g, gpu, ora


@pytest.mark.parametrize("arch", ["gcn", "sage", "gat"])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_eval_logits_full_graph_per_node(arch, precision):
    from tests.gpu_helpers import rel_err
    g, gpu, ora = _trained_pair(arch, precision)
    got = gpu.eval_logits(0)
    _, _, ref = ora.eval(2)
    assert got.shape == ref.shape
    assert rel_err(got, ref) <= TOL[precision], rel_err(got, ref)
    # the loss / accuracy of gist_eval are those of these logits
    lg, ag = gpu.eval(2)
    rows = g["split"] == 2
    z = got[rows].astype(np.float64)
    ce = np.log(np.exp(z - z.max(1, keepdims=True)).sum(1)) + z.max(1) - z[np.arange(len(z)), g["labels"][rows]]
    assert lg == pytest.approx(ce.mean(), rel=1e-5)
    assert ag == pytest.approx(np.mean(np.argmax(got[rows], 1) == g["labels"][rows]), abs=1e-6)


@pytest.mark.parametrize("arch", ["gcn", "sage", "gat"])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_eval_logits_partitions_per_node(arch, precision):
    from tests.gpu_helpers import rel_err
    g, gpu, ora = _trained_pair(arch, precision)
    n = len(g["labels"])
    rng = np.random.default_rng(1)
    part = (rng.integers(0, 22, n) + (rng.random(n) < 0.3) * (np.arange(n) % 3)) % 22
    part[part >= 5] += 1                        # partition 5 empty
    got = gpu.eval_logits(1, part, 23, max_rows=37)
    ref = np.zeros((n, g["num_classes"]))
    ora.eval_partitions(0, part, 23, logits_out=ref)
    assert rel_err(got, ref) <= TOL[precision], rel_err(got, ref)
    # per partition too: a wrong row inside one small partition cannot hide in the max
    for p in range(23):
        idx = np.nonzero(part == p)[0]
        if len(idx):
            assert rel_err(got[idx], ref[idx]) <= TOL[precision], p


@pytest.mark.parametrize("arch", ["gcn", "sage", "gat"])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_eval_scale_mean(arch, precision):
    """R10 "mean": contractions over the partitioned hidden input dims scaled by
    1/m in the evaluation forward -- per-node logits of the full-graph and the partition-wise
    evaluation against the oracle's scaled forward (m = 3 of the last partition)."""
    from paper_2102_10424_b200.gist import Gist
    from tests.gpu_helpers import rel_err
    g = generate(tiny_spec(n=600, nnz=5000, d0=21, classes=5, clusters=9), seed=3)
    dims = (21, 36, 30, 5)
    gpu = Gist(arch, dims, optimizer="sgd", precision=precision, clusters_per_batch=3, batch_seed=2,
               eval_scale="mean")
    gpu.load_graph(g)
    gpu.init_params(5)
    ora = O.OracleGIST(arch=arch, dims=list(dims), optimizer="sgd", clusters_per_batch=3, batch_seed=2)
    ora.load_graph(g["row_ptr"], g["col_idx"], g["X"], g["labels"], g["num_classes"], g["split"],
                   g["cluster_ids"], g["num_clusters"])
    gpu.partition(seed=4, m=3)
    gpu.subtrain(2, lr=0.05)
    gpu.aggregate()
    ora.set_params([gpu.get_params(l).astype(np.float64) for l in range(len(dims) - 1)])
    ora.m = 3
    _, _, ref = ora.eval(2, eval_scale="mean")
    _, _, unscaled = ora.eval(2)
    assert rel_err(ref, unscaled) > 0.5                 # the scaling is visible
    assert rel_err(gpu.eval_logits(0), ref) <= TOL[precision]
    part = (np.arange(len(g["labels"])) * 5) % 7
    pref = np.zeros_like(ref)
    ora.eval_partitions(2, part, 7, logits_out=pref, eval_scale="mean")
    assert rel_err(gpu.eval_logits(1, part, 7), pref) <= TOL[precision]
