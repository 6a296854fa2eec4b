"""The library's world > 1 code paths, executed on ONE GPU through the loopback transport.

The method shards its sub-GCNs across GPUs ("each sub-GCN is trained on
a separate GPU"; slot i on rank i mod W) and exchanges parameters once per round
(subAgg).  Only one GPU is available to this build, so W contexts of this
process, each driven by its own host thread, stand in for W ranks (gist_loopback_create,
include/gist.h): every collective (the subAgg all-gather, the eval all-gathers / all-reduces,
the P2P barriers and replica pointers) is carried out by the host with device-to-device copies,
while everything else -- slot ownership, the packed buffers, the unpack offsets of the gathered
buffer (gist_aggregate), the peer stores into every replica (agg_mode P2P), the row-split
full-graph eval and the partition-wise eval ownership -- is the code a multi-GPU run executes.
No kernel waits on another rank.

Property (SURVEY §8(c) determinism pin, "world size 1/2/4/8 -> same bits"): after several
rounds the global Theta of every rank is bit-identical to the single-context run, the per-slot
losses are identical, and the evaluation (loss, accuracy, per-node logits) matches.
"""
import threading

import numpy as np
import pytest

from synth.planted import generate, tiny_spec
from tests.test_gpu_parity import CASES

pytestmark = pytest.mark.gpu

ZETA, ROUNDS = 3, 3


def _world(W, arch, dims, m, q, g, precision="fp32", agg_mode="allgather", opt_state="reset",
           optimizer="adam", lr=0.003, parts=None, timeout=600, theta="replicated", extra=None):
    from paper_2102_10424_b200.gist import Gist, Loopback
    lb = Loopback(W) if W > 1 else None
    ctxs = [Gist(arch, dims, optimizer=optimizer, precision=precision, clusters_per_batch=q, batch_seed=5,
                 opt_state=opt_state, agg_mode=agg_mode, rank=r, world_size=W, loopback=lb, theta=theta)
            for r in range(W)]
    out = [None] * W
    errs = []

    def body(r):
        try:
            c = ctxs[r]
            c.load_graph(g)
            c.init_params(11)
            hist, losses = [], []
            for t in range(ROUNDS):
                c.partition(seed=31 + t, m=m)
                losses.append(c.subtrain(ZETA, lr=lr))
                c.aggregate()
                hist.append([c.get_params(l).copy() for l in range(len(dims) - 1)])
            res = {"hist": hist, "losses": losses, "eval": c.eval(2), "logits": c.eval_logits(0)}
            if extra is not None:
                res["extra"] = extra(c, r)
            if parts is not None:
                res["parts"] = c.eval_parts(2, parts, int(parts.max()) + 1, max_rows=97)
                res["plogits"] = c.eval_logits(1, parts, int(parts.max()) + 1, max_rows=97)
            out[r] = res
        except Exception as e:  # noqa: BLE001 -- re-raised in the main thread
            errs.append((r, e))

    threads = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(W)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout)
    assert not errs, errs
    assert all(not t.is_alive() for t in threads), "a rank did not finish (collective mismatch?)"
    for c in ctxs:
        c.close()
    if lb is not None:
        lb.close()
    return out


def _check(ref, got, W, parts=False, eval_tol=0.0):
    for r in range(W):
        for t in range(ROUNDS):
            for l in range(len(ref["hist"][t])):
                np.testing.assert_array_equal(got[r]["hist"][t][l], ref["hist"][t][l],
                                              err_msg=f"rank {r} round {t} layer {l}")
        # each rank fills its own slots' losses; together they are the single-context losses
    for t in range(ROUNDS):
        tot = np.sum([got[r]["losses"][t] for r in range(W)], axis=0)
        np.testing.assert_array_equal(tot, ref["losses"][t], err_msg=f"round {t} losses")
    for r in range(W):
        np.testing.assert_array_equal(got[r]["logits"], ref["logits"], err_msg=f"rank {r} eval logits")
        assert abs(got[r]["eval"][0] - ref["eval"][0]) <= eval_tol * max(1.0, abs(ref["eval"][0])), \
            (got[r]["eval"], ref["eval"])
        assert got[r]["eval"][1] == ref["eval"][1]
        if parts:
            assert got[r]["parts"][0] == ref["parts"][0] and got[r]["parts"][1] == ref["parts"][1]
            np.testing.assert_array_equal(got[r]["parts"][2], ref["parts"][2])
            np.testing.assert_array_equal(got[r]["plogits"], ref["plogits"], err_msg=f"rank {r} partition logits")


@pytest.mark.parametrize("case,m,W,precision", [
    (1, 8, 2, "fp32"),   # GraphSAGE, 4 slots per rank
    (1, 8, 4, "bf16"),   # block-diagonal tensor-core aggregation + re-association off (narrow)
    (1, 8, 8, "fp32"),   # one slot per rank (the paper's layout at m = 8)
    (0, 3, 2, "fp32"),   # GCN, ragged ownership (rank 0: slots 0, 2; rank 1: slot 1)
    (0, 2, 4, "bf16"),   # ranks 2, 3 own no slot (empty packed buffers)
    (3, 4, 2, "bf16"),   # GCN tiles: the re-associated last layer in BF16
])
def test_allgather_world_matches_single(case, m, W, precision):
    _, kw, arch, dims, q = CASES[case]
    g = generate(tiny_spec(**kw), seed=4)
    parts = (np.arange(g["n"]) * 7 // g["n"]).astype(np.int32)[np.random.default_rng(0).permutation(g["n"])]
    ref = _world(1, arch, dims, m, q, g, precision=precision, parts=parts)[0]
    got = _world(W, arch, dims, m, q, g, precision=precision, parts=parts)
    # the full-graph loss is a sum over W row blocks (different grouping of the same doubles)
    _check(ref, got, W, parts=True, eval_tol=1e-12)


@pytest.mark.parametrize("case,m,W,precision,opt_state", [
    (1, 4, 2, "fp32", "reset"),
    (1, 3, 4, "bf16", "persistent"),
    (0, 8, 8, "fp32", "persistent"),
])
def test_p2p_world_matches_single_allgather(case, m, W, precision, opt_state):
    """agg_mode P2P at W > 1: the owner of each slot stores its block into every rank's replica
    (k_scatter_peers with W destinations) between two barriers."""
    _, kw, arch, dims, q = CASES[case]
    g = generate(tiny_spec(**kw), seed=4)
    ref = _world(1, arch, dims, m, q, g, precision=precision, opt_state=opt_state)[0]
    got = _world(W, arch, dims, m, q, g, precision=precision, opt_state=opt_state, agg_mode="p2p")
    _check(ref, got, W, eval_tol=1e-12)


def test_gat_world_matches_single():
    """GAT (R21): the gathered buffers also feed the mean of the shared last-layer attention rows."""
    g = generate(tiny_spec(n=500, nnz=4000, d0=33, classes=5, clusters=10), seed=0)
    dims = (33, 40, 24, 5)
    ref = _world(1, "gat", dims, 3, 3, g, optimizer="sgd", lr=0.05)[0]
    got = _world(2, "gat", dims, 3, 3, g, optimizer="sgd", lr=0.05)
    _check(ref, got, 2, eval_tol=0.0)


def test_loopback_rejects_mismatch():
    """A loopback group serves exactly world_size ranks, one context per rank."""
    from paper_2102_10424_b200.gist import Gist, GistError, Loopback
    lb = Loopback(2)
    with pytest.raises(GistError):
        Gist("gcn", (8, 8, 3), rank=0, world_size=3, loopback=lb)
    a = Gist("gcn", (8, 8, 3), rank=0, world_size=2, loopback=lb)
    with pytest.raises(GistError):
        Gist("gcn", (8, 8, 3), rank=0, world_size=2, loopback=lb)
    a.close()
    lb.close()


@pytest.mark.parametrize("case", [0, 1])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_step_schedules_bit_identical(monkeypatch, precision, case):
    """The step is captured once per (own batch build, next-batch prefetch) variant as a CUDA graph
    and replayed; profiled steps run eagerly; the slots may run as several lockstep groups.  Every
    schedule enqueues the same kernels on the same data: Theta and the losses are bit-identical
    to the eager, unprefetched, single-group run -- including the early next-batch build inside
    the backward (default) and the late one during the optimizer (GIST_BATCH_PREFETCH=1)."""
    _, kw, arch, dims, q = CASES[case]
    g = generate(tiny_spec(**kw), seed=4)

    def run(env, prof=0):
        for k in ("GIST_GRAPH", "GIST_BATCH_PREFETCH", "GIST_GROUP"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        from paper_2102_10424_b200.gist import Gist
        c = Gist(arch, dims, optimizer="adam", precision=precision, clusters_per_batch=q, batch_seed=5)
        c.load_graph(g)
        c.init_params(11)
        c.profile(prof)
        out = []
        for t in range(3):
            c.partition(seed=31 + t, m=8)
            out.append(c.subtrain(7, lr=0.003))
            c.aggregate()
        out += [c.get_params(l) for l in range(len(dims) - 1)]
        c.close()
        return out

    ref = run({"GIST_GRAPH": "0", "GIST_BATCH_PREFETCH": "0"})
    for env, prof in (({}, 0), ({}, 3), ({"GIST_GROUP": "3"}, 0), ({"GIST_GROUP": "1", "GIST_GRAPH": "0"}, 2),
                      ({"GIST_BATCH_PREFETCH": "1"}, 0), ({"GIST_GROUP": "1"}, 0)):
        got = run(env, prof)
        for a, b in zip(got, ref):
            np.testing.assert_array_equal(a, b, err_msg=f"{env} profile {prof}")
