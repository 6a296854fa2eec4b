"""Per-layer optimizer (GCN / GraphSAGE; csrc/step.cu layer_optimizer, csrc/train.cu
k_adam_ranges): each layer's Adam / SGD update (R8) runs on the dW stream
right after that layer's dW GEMM, overlapping the rest of the backward chain, and the step ends
with a one-thread step-state advance instead of one optimizer pass after the backward.  The
element arithmetic is k_adam's / k_sgd's, and a layer's dW and update are ordered after the
step's last reader of that layer's weights (dX, or GCN's re-associated dH), so per-layer and
one-pass give the same bits -- pinned here against GIST_LAYER_OPT=0 over several steps and
rounds (weights, gradients, losses, all precisions), on top of the oracle gates of
test_gpu_parity / test_gpu_bf16 / test_gpu_tf32."""
import numpy as np
import pytest

from synth.planted import generate, tiny_spec
from tests.test_gpu_parity import CASES

pytestmark = pytest.mark.gpu


def _run(g, arch, dims, precision, optimizer, opt_state, m, q, rounds=3, zeta=4):
    from paper_2102_10424_b200.gist import Gist
    c = Gist(arch, dims, optimizer=optimizer, precision=precision, clusters_per_batch=q, batch_seed=2,
             opt_state=opt_state)
    c.load_graph(g)
    c.init_params(3)
    out = []
    for t in range(rounds):
        c.partition(seed=10 + t, m=m)
        out.append(np.asarray(c.subtrain(zeta, lr=0.01 if optimizer == "adam" else 0.05)))
        for i in range(m):
            for l in range(len(dims) - 1):
                out.append(c.trace(i, 3, l).copy())      # last step's gradient
                out.append(c.get_sub_params(i, l).copy())
        c.aggregate()
        out += [c.get_params(l).copy() for l in range(len(dims) - 1)]
    c.close()
    return out


@pytest.mark.parametrize("case,precision,optimizer,opt_state,reassoc", [
    (2, "bf16", "adam", "reset", None),        # GraphSAGE: block-diagonal + re-associated last layer
    (1, "bf16", "sgd", "reset", None),
    (1, "bf16", "adam", "persistent", None),   # f3 moments carried across rounds
    (0, "bf16", "adam", "reset", "1"),         # GCN with the re-associated last layer (dH reads W)
    (3, "bf16", "sgd", "reset", None),
    (1, "tf32", "adam", "reset", None),        # TF32: fp32 weights read by the GEMMs directly
    (0, "fp32", "adam", "reset", None),        # FP32 parity mode (SIMT GEMMs)
    (1, "fp32", "sgd", "persistent", None),
])
def test_layer_optimizer_bit_identical(case, precision, optimizer, opt_state, reassoc, monkeypatch):
    name, kw, arch, dims, q = CASES[case]
    g = generate(tiny_spec(**kw), seed=1)
    if reassoc is not None:
        monkeypatch.setenv("GIST_REASSOC", reassoc)
    monkeypatch.setenv("GIST_LAYER_OPT", "1")
    fused = _run(g, arch, dims, precision, optimizer, opt_state, 3, q)
    monkeypatch.setenv("GIST_LAYER_OPT", "0")
    sep = _run(g, arch, dims, precision, optimizer, opt_state, 3, q)
    assert len(fused) == len(sep)
    for k, (a, b) in enumerate(zip(fused, sep)):
        np.testing.assert_array_equal(a, b, err_msg=str(k))


def test_layer_optimizer_dw_side_stream_off(monkeypatch):
    """The same with the dW GEMMs on the main stream (GIST_DW_STREAM=0) and eager launches."""
    name, kw, arch, dims, q = CASES[1]
    g = generate(tiny_spec(**kw), seed=2)
    monkeypatch.setenv("GIST_LAYER_OPT", "1")
    ref = _run(g, arch, dims, "bf16", "adam", "reset", 2, q)
    monkeypatch.setenv("GIST_DW_STREAM", "0")
    monkeypatch.setenv("GIST_GRAPH", "0")
    got = _run(g, arch, dims, "bf16", "adam", "reset", 2, q)
    for k, (a, b) in enumerate(zip(ref, got)):
        np.testing.assert_array_equal(a, b, err_msg=str(k))
