"""Owner-sharded global model (GIST_THETA_SHARDED, the C5 variant of the subAgg:
"owner-sharded Theta, with all-to-all re-partition and aggregate", in place of the paper's
parameter server), on one GPU through the loopback transport (W ranks = W
contexts of this process; see tests/test_gpu_multirank.py).

Rank r keeps physical rows [K r / W, K (r+1) / W) of each Theta_l.  subGCNs (R6)
sends every owned row of every sub-model to the sub-model's rank; subAgg (R9)
sends the updated rows back.  Property: the same floats land in the same places as with the
replicated model -- Theta after every round, the per-slot losses, the evaluation and the
per-node logits are bit-identical to the replicated run at the same world size (which
tests/test_gpu_multirank.py pins to the single-context run), while each rank stores ~1/W of
the model."""
import numpy as np
import pytest

from synth.planted import generate, tiny_spec
from tests.test_gpu_multirank import _check, _world
from tests.test_gpu_parity import CASES

pytestmark = pytest.mark.gpu


def _same(ref, got, W, parts=False):
    """Sharded vs replicated at the same world size (the same row split in eval): every
    observable bit-identical (_check with eval_tol 0); ref = the replicated run's ranks."""
    merged = dict(ref[0])
    merged["losses"] = [np.sum([ref[r]["losses"][t] for r in range(W)], axis=0) for t in range(len(ref[0]["losses"]))]
    _check(merged, got, W, parts=parts, eval_tol=0.0)


@pytest.mark.parametrize("W", [1, 2, 4])
@pytest.mark.parametrize("case", [0, 1])
def test_sharded_bit_identical_fp32(W, case):
    name, kw, arch, dims, q = CASES[case]
    g = generate(tiny_spec(**kw), seed=0)
    ref = _world(W, arch, dims, 4, q, g)
    got = _world(W, arch, dims, 4, q, g, theta="sharded")
    _same(ref, got, W)


@pytest.mark.parametrize("W", [2, 3])
def test_sharded_bit_identical_bf16_sage(W):
    name, kw, arch, dims, q = CASES[2]
    g = generate(tiny_spec(**kw), seed=0)
    ref = _world(W, arch, dims, 3, q, g, precision="bf16")
    got = _world(W, arch, dims, 3, q, g, precision="bf16", theta="sharded")
    _same(ref, got, W)


def test_sharded_persistent_adam_moments():
    """f3 (persistent moments) travel with the weights: the moments are sharded too."""
    name, kw, arch, dims, q = CASES[1]
    g = generate(tiny_spec(**kw), seed=0)
    ref = _world(2, arch, dims, 4, q, g, opt_state="persistent")
    got = _world(2, arch, dims, 4, q, g, opt_state="persistent", theta="sharded")
    _same(ref, got, 2)


def test_sharded_gat():
    """GAT (R21): the last layer's attention rows are the mean of the m copies, taken by the rank
    holding them."""
    g = generate(tiny_spec(n=700, nnz=6000, d0=29, classes=6, clusters=11), seed=0)
    dims = (29, 40, 24, 6)
    ref = _world(2, "gat", dims, 2, 3, g)
    got = _world(2, "gat", dims, 2, 3, g, theta="sharded")
    _same(ref, got, 2)


def test_sharded_memory_and_partition_eval():
    """Each rank stores its share of the rows (GIST_STAT_THETA_BYTES); partition-wise eval works."""
    from paper_2102_10424_b200 import gist as G
    name, kw, arch, dims, q = CASES[3]
    g = generate(tiny_spec(**kw), seed=0)
    parts = np.arange(g["n"], dtype=np.int32) % 5
    stat = lambda c, r: c.stat(G.STAT_THETA_BYTES)
    W = 4
    ref = _world(W, arch, dims, 2, q, g, parts=parts, extra=stat)
    got = _world(W, arch, dims, 2, q, g, theta="sharded", parts=parts, extra=stat)
    _same(ref, got, W, parts=True)
    full = ref[0]["extra"]
    assert sum(got[r]["extra"] for r in range(W)) == full
    assert max(got[r]["extra"] for r in range(W)) <= full / W * 1.25


def test_sharded_checkpoint_round_trip(tmp_path):
    """gist_save_checkpoint is a collective under sharding (the rows are gathered): every rank
    writes the replicated model's bytes; loading writes the local rows only."""
    from paper_2102_10424_b200.gist import Gist, Loopback
    import threading
    name, kw, arch, dims, q = CASES[0]
    g = generate(tiny_spec(**kw), seed=0)
    rep = Gist(arch, dims, clusters_per_batch=q)
    rep.load_graph(g)
    rep.init_params(4)
    rep.save_checkpoint(str(tmp_path / "rep.gist"))
    W = 2
    lb = Loopback(W)
    ctxs = [Gist(arch, dims, clusters_per_batch=q, rank=r, world_size=W, loopback=lb, theta="sharded")
            for r in range(W)]
    errs = []

    def body(r):
        try:
            c = ctxs[r]
            c.load_graph(g)
            c.init_params(4)
            c.save_checkpoint(str(tmp_path / f"sh{r}.gist"))
            c.init_params(99)
            c.load_checkpoint(str(tmp_path / "rep.gist"))
            c.save_checkpoint(str(tmp_path / f"re{r}.gist"))
        except Exception as e:  # noqa: BLE001
            errs.append((r, e))
    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not errs, errs
    want = (tmp_path / "rep.gist").read_bytes()
    for r in range(W):
        assert (tmp_path / f"sh{r}.gist").read_bytes() == want
        assert (tmp_path / f"re{r}.gist").read_bytes() == want
    for c in ctxs:
        c.close()
    lb.close()
    rep.close()


def test_sharded_refusals():
    from paper_2102_10424_b200.gist import Gist, GistError
    for mode in ("p2p", "symm"):
        with pytest.raises(GistError, match="UNSUPPORTED"):
            Gist("gcn", (6, 8, 3), agg_mode=mode, theta="sharded")
