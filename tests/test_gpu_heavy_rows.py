"""Mini-batch aggregation with a heavy degree tail (the split of heavy rows across a CTA in
k_spmm, csrc/spmm.cu).  The planted graphs here draw node weights lognormal(sigma = 2) so that
a few hubs carry 50-100x the mean degree -- inside a batch, rows with several hundred neighbours
(above the 128-neighbour split threshold of the full-batch passes) and, with a low in-community
fraction, well over 32 inter-cluster neighbours (the threshold of the block-diagonal path's
inter-cluster pass).  Gates as in test_gpu_parity / test_gpu_bf16 (Eq. 1-2, PAPER.md:129-133,
151-155), plus bit-identity of the split across lockstep group sizes and world sizes (the split
depends only on the row's degree)."""
import numpy as np
import pytest

from synth.planted import GraphSpec, generate
from tests.gpu_helpers import align, make_pair, rel_err
from tests.test_gpu_multirank import _world

pytestmark = pytest.mark.gpu


def hub_graph(seed=0, f_in=0.5):
    return generate(GraphSpec("hubs", 1500, 60000, 24, 5, 6, 6, f_in, (0.6, 0.2, 0.2), sigma=2.0), seed=seed)


def test_hub_graph_has_heavy_batch_rows():
    """The fixture does what the docstring says: batch degrees above both thresholds."""
    g = hub_graph()
    deg = np.diff(g["row_ptr"])
    cl = g["cluster_ids"]
    assert deg.max() > 8 * deg.mean()
    # a q = 2 batch of clusters {0, 1}: within-batch neighbours of its rows
    rows = np.nonzero(np.isin(cl, [0, 1]))[0]
    inb = [np.isin(cl[g["col_idx"][g["row_ptr"][v]:g["row_ptr"][v + 1]]], [0, 1]) for v in rows]
    bdeg = np.array([x.sum() for x in inb])
    inter = np.array([np.sum(x & (cl[g["col_idx"][g["row_ptr"][v]:g["row_ptr"][v + 1]]] != cl[v]))
                      for x, v in zip(inb, rows)])
    assert bdeg.max() > 128 and inter.max() > 32


def _one_step(arch, dims, precision):
    """One step of both slots; returns the GPU's per-slot logits, activations and gradients
    (in the oracle's row order) and the oracle's."""
    g = hub_graph()
    gpu, ora = make_pair(g, arch, dims, optimizer="adam", q=2, precision=precision)
    gpu.partition(seed=7, m=2)
    ora.partition(seed=7, m=2)
    gpu.subtrain(1, lr=0.01)
    got, ref = [], []
    for i in range(2):
        ora.train_step(i, 0, 0.01)
        tr = ora.last_trace[i]
        nodes = gpu.trace(i, 0)
        p = align(nodes, tr["nodes"])
        q = np.argsort(p)                     # GPU rows -> oracle row order
        nb = len(nodes)
        got.append([gpu.trace(i, 2).reshape(nb, -1)[q]]
                   + [gpu.trace(i, 1, l).reshape(nb, -1)[q] for l in range(1, len(dims) - 1)]
                   + [gpu.trace(i, 3, l).reshape(ora.sub[i][l].shape) for l in range(len(dims) - 1)])
        ref.append([tr["tape"]["logits"]] + [tr["tape"]["H"][l] for l in range(1, len(dims) - 1)]
                   + [tr["grads"][l] for l in range(len(dims) - 1)])
    gpu.close()
    return got, ref


@pytest.mark.parametrize("arch,dims", [("gcn", (24, 300, 40, 5)), ("sage", (24, 300, 40, 5))])
def test_heavy_rows_fp32(arch, dims):
    got, ref = _one_step(arch, dims, "fp32")
    na = len(dims) - 1                        # logits + hidden activations
    for gs, rs in zip(got, ref):
        for k, (a, b) in enumerate(zip(gs, rs)):
            assert rel_err(a, b) <= (1e-4 if k < na else 1e-3), k


@pytest.mark.parametrize("bd", ["1", "0"])
@pytest.mark.parametrize("arch,dims", [("sage", (24, 600, 40, 5)), ("gcn", (24, 300, 40, 5))])
def test_heavy_rows_bf16(arch, dims, bd, monkeypatch):
    """Activations and logits within the BF16 gate of the oracle.  The gradients of this hub
    fixture sit at 2.9e-2 (SAGE, layer 0) / 4.0e-2 (GCN, layer 1) of the FP64 oracle with and
    without the split alike (bf16 rounding of the hubs' operands, profiles/r03a_heavy_rows_bf16.txt),
    so the split itself is pinned against the unsplit row sums of the same kernels
    (GIST_SPMM_SPLIT=0): only the fp32 summation order differs."""
    monkeypatch.setenv("GIST_BD", bd)
    got, ref = _one_step(arch, dims, "bf16")
    monkeypatch.setenv("GIST_SPMM_SPLIT", "0")
    base, _ = _one_step(arch, dims, "bf16")
    na = len(dims) - 1
    for gs, rs, bs in zip(got, ref, base):
        for k in range(len(gs)):
            if k < na:
                assert rel_err(gs[k], rs[k]) <= 2e-2, k
            assert rel_err(gs[k], bs[k]) <= 2e-3, k


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_heavy_rows_bit_identical_across_world_sizes(precision):
    """m = 4 sub-GCNs: one context running 4 lockstep slots vs 4 loopback ranks of one slot
    each (the single-slot launches take the small-launch kernel variants)."""
    g = hub_graph(seed=1)
    dims = (24, 256, 64, 5)
    ref = _world(1, "sage", dims, 4, 2, g, precision=precision)[0]
    got = _world(4, "sage", dims, 4, 2, g, precision=precision)
    for r in range(4):
        for t in range(len(ref["hist"])):
            for l in range(len(dims) - 1):
                np.testing.assert_array_equal(got[r]["hist"][t][l], ref["hist"][t][l])



@pytest.mark.parametrize("arch,dims", [("sage", (24, 600, 40, 5)), ("sage", (24, 256, 64, 5))])
def test_heavy_rows_persistent_pass_bit_identical(arch, dims, monkeypatch):
    """The persistent-warp inter-cluster pass (k_inter_persist: grouped launches of > 16,384 rows,
    forced here with GIST_INTER_PERSIST=1) sums light rows and the CTA-split heavy rows in exactly
    the order of k_spmm: the same bits as k_spmm (GIST_INTER_PERSIST=0) on the hub graph, BF16
    block-diagonal path, m = 4 lockstep slots over 2 rounds."""
    g = hub_graph(seed=3)
    out = {}
    for force in ("1", "0"):
        monkeypatch.setenv("GIST_INTER_PERSIST", force)
        out[force] = _world(1, arch, dims, 4, 2, g, precision="bf16")[0]
    for t in range(len(out["0"]["hist"])):
        for l in range(len(dims) - 1):
            np.testing.assert_array_equal(out["1"]["hist"][t][l], out["0"]["hist"][t][l])
