"""Parity at BASELINE.json's full size, in the launch configuration bench.py times:
C3 (Reddit-shaped graph, 232,965 nodes / 114.6M nnz, 4-layer GraphSAGE hidden 4096,
m = 8 sub-GCNs on one GPU, 20 clusters per batch).  One subTrain step of all 8 slots runs
on the GPU; the FP64 oracle recomputes slot 0's step (its sub-weights evaluated entry by
entry from the init counter, R11) and every activation / logit / gradient of that slot is
compared (R18 metric).  FP32 mode: 1e-4 / 1e-3; BF16 mode: 2e-2."""
import numpy as np
import pytest

from oracle import gist_oracle as O
from synth.planted import GRAPHS, MODELS, generate
from tests.gpu_helpers import align, rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def reddit():
    return generate(GRAPHS["reddit"], seed=0, device="cuda")


@pytest.mark.parametrize("precision,act_tol,grad_tol", [("bf16", 2e-2, 2e-2), ("fp32", 1e-4, 1e-3)])
def test_c3_full_size_one_step(reddit, precision, act_tol, grad_tol):
    from paper_2102_10424_b200.gist import STAT_BLOCK_AGG, Gist
    spec = MODELS["C3"]
    dims = list(spec.dims)
    g = reddit
    gpu = Gist(spec.arch, dims, optimizer="adam", precision=precision, clusters_per_batch=spec.q, batch_seed=3)
    gpu.load_graph(g)
    gpu.init_params(7)
    if precision == "bf16":
        assert gpu.stat(STAT_BLOCK_AGG) == 1   # the block-diagonal tensor-core path is exercised
    gpu.partition(seed=5, m=spec.m)
    gpu.subtrain(1, lr=0.01)

    ora = O.OracleGIST(arch=spec.arch, dims=dims, optimizer="adam", clusters_per_batch=spec.q, batch_seed=3)
    ora.load_graph(g["row_ptr"], g["col_idx"], g["X"], g["labels"], g["num_classes"], g["split"],
                   g["cluster_ids"], g["num_clusters"])
    blocks = O.sample_partition(dims, spec.m, seed=5, t=0)
    sets = O.sub_index_sets(spec.arch, dims, blocks, 0)
    ora.m = spec.m
    ora.sub = [[O.glorot_block(spec.arch, dims, 7, l, r, c) for l, (r, c) in enumerate(sets)]] + [None] * (spec.m - 1)
    ora.opt = [[{} for _ in dims[:-1]] for _ in range(spec.m)]
    for l in range(len(dims)):  # partition indices: bit-exact at full size
        assert np.array_equal(gpu.get_partition(l)[0], blocks[l][0])
    ora.train_step(0, 0, 0.01)
    tr = ora.last_trace[0]
    nodes = gpu.trace(0, 0)
    p = align(nodes, tr["nodes"])
    nb = len(nodes)
    errs = {"logits": rel_err(gpu.trace(0, 2).reshape(nb, -1), tr["tape"]["logits"][p])}
    for l in range(1, len(dims) - 1):
        errs[f"H{l}"] = rel_err(gpu.trace(0, 1, l).reshape(nb, -1), tr["tape"]["H"][l][p])
    for l in range(len(dims) - 1):
        errs[f"dW{l}"] = rel_err(gpu.trace(0, 3, l).reshape(ora.sub[0][l].shape), tr["grads"][l])
    print(precision, "full-size C3 slot-0 errors", errs)
    for k, v in errs.items():
        assert v <= (act_tol if k[0] in "Hl" else grad_tol), (k, v)
    assert abs(gpu.trace(0, 4)[0] - tr["loss"]) <= act_tol * max(1.0, tr["loss"])
