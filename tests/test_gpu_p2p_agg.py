"""subAgg over peer memory (gist_config.agg_mode = GIST_AGG_P2P).

One GPU is available to this build, so the P2P path runs at world 1 here: Theta (and the f3
moments) live in the single cudaMalloc region the IPC handles export, and gist_aggregate
writes every slot through k_scatter_peers with the local region as the only destination.
The contract checked: bit-identical Theta to the ALLGATHER path (the paper's subAgg,
PAPER.md:118, 185-190, a bitwise block copy, R9) after several rounds, so the region layout,
the per-layer offsets into it and the one-read / W-store kernel place every element where
k_scatter does.  Moments are covered through the weights: a wrong moment slice changes the
next round's Adam step.  The world > 1 protocol (who writes which slot into which replica,
the two barriers) is covered by tests/test_dist_gloo.py on CPU.
"""
import numpy as np
import pytest

from synth.planted import generate, tiny_spec
from tests.test_gpu_parity import CASES

pytestmark = pytest.mark.gpu


def _run(arch, dims, m, q, g, agg_mode, precision, opt_state, rounds=3):
    from paper_2102_10424_b200.gist import Gist
    gpu = Gist(arch, dims, optimizer="adam", precision=precision, clusters_per_batch=q, batch_seed=5,
               opt_state=opt_state, agg_mode=agg_mode)
    gpu.load_graph(g)
    gpu.init_params(11)
    hist, losses = [], []
    for t in range(rounds):
        gpu.partition(seed=31 + t, m=m)
        losses.append(gpu.subtrain(3, lr=0.003))
        gpu.aggregate()
        hist.append([gpu.get_params(l).copy() for l in range(len(dims) - 1)])
    gpu.close()
    return hist, losses


@pytest.mark.parametrize("case,m,precision,opt_state", [
    (1, 2, "fp32", "reset"),
    (1, 3, "fp32", "persistent"),
    (0, 3, "fp32", "reset"),
    (2, 2, "bf16", "persistent"),
    (3, 4, "bf16", "reset"),
])
def test_p2p_aggregate_bit_identical_to_allgather(case, m, precision, opt_state):
    _, kw, arch, dims, q = CASES[case]
    g = generate(tiny_spec(**kw), seed=4)
    ref, lref = _run(arch, dims, m, q, g, "allgather", precision, opt_state)
    got, lgot = _run(arch, dims, m, q, g, "p2p", precision, opt_state)
    for t in range(len(ref)):
        np.testing.assert_array_equal(np.asarray(lgot[t]), np.asarray(lref[t]), err_msg=f"round {t} losses")
        for l in range(len(ref[t])):
            np.testing.assert_array_equal(got[t][l], ref[t][l], err_msg=f"round {t} layer {l}")


def test_p2p_rejects_gat():
    """R21 averages the m copies of the GAT attention rows: P2P is refused at create."""
    from paper_2102_10424_b200.gist import Gist, GistError
    with pytest.raises(GistError, match="UNSUPPORTED"):
        Gist("gat", (16, 8, 4), agg_mode="p2p")


@pytest.mark.parametrize("case,m,precision,opt_state", [
    (1, 2, "fp32", "reset"),
    (0, 3, "fp32", "persistent"),
    (3, 4, "bf16", "reset"),
])
def test_symm_window_aggregate_bit_identical_to_allgather(case, m, precision, opt_state):
    """agg_mode SYMM (SURVEY §8 f2 with the NCCL device API): Theta in an ncclMemAlloc region
    registered as a symmetric window, a device communicator, and the owners' stores through
    ncclGetLsaPointer.  World 1 (one-rank communicator): bit-identical Theta to the all-gather."""
    _, kw, arch, dims, q = CASES[case]
    g = generate(tiny_spec(**kw), seed=4)
    ref, lref = _run(arch, dims, m, q, g, "allgather", precision, opt_state)
    got, lgot = _run(arch, dims, m, q, g, "symm", precision, opt_state)
    for t in range(len(ref)):
        np.testing.assert_array_equal(np.asarray(lgot[t]), np.asarray(lref[t]), err_msg=f"round {t} losses")
        for l in range(len(ref[t])):
            np.testing.assert_array_equal(got[t][l], ref[t][l], err_msg=f"round {t} layer {l}")


def test_symm_refusals():
    from paper_2102_10424_b200.gist import Gist, GistError, Loopback
    with pytest.raises(GistError, match="UNSUPPORTED"):
        Gist("gat", (16, 8, 4), agg_mode="symm")
    lb = Loopback(2)
    with pytest.raises(GistError, match="UNSUPPORTED"):
        Gist("gcn", (16, 8, 4), agg_mode="symm", rank=0, world_size=2, loopback=lb)
    lb.close()
