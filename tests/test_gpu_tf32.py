"""TF32 tensor-core mode (R13: FP32 storage everywhere; the step GEMMs on tcgen05 kind::tf32 --
the tensor core reads the fp32 operands at tf32 precision, 10 explicit mantissa bits -- with fp32
accumulation).  Gates (north_star, "bf16/TF32 mode"): relative error <= 2e-2 against the FP64
oracle and the loss curve within 1% over 10 rounds.  The GEMM kernel itself is checked against
the FP64 product of the fp32 operands: a tf32 operand carries a relative error <= 2^-10 (rounding
or truncation of the 13 dropped bits), so a dot product of K random terms is off by ~2^-10 of its
magnitude -- gated at 3e-3, while a wrong K advance, swizzle or box (the layout bugs this catches)
gives O(1) errors."""
import numpy as np
import pytest

from synth.planted import GRAPHS, generate, tiny_spec
from tests.gpu_helpers import align, make_pair, rel_err

pytestmark = pytest.mark.gpu
TF32_TOL = 2e-2


@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (517, 131, 263), (3106, 512, 1216), (300, 48, 1024),
                                   (1216, 512, 3106), (70, 8, 40)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("relu", [False, True])
def test_tf32_gemm_layouts(M, N, K, ta, tb, relu):
    import torch
    from paper_2102_10424_b200 import gist
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    pad = lambda x: (x + 7) // 8 * 8
    a_shape = (K, pad(M)) if ta else (M, pad(K))
    b_shape = (N, pad(K)) if tb else (K, pad(N))
    a = rng.standard_normal(a_shape).astype(np.float32)
    b = rng.standard_normal(b_shape).astype(np.float32)
    dev = torch.device("cuda")
    ad = torch.from_numpy(a).to(dev)
    bd = torch.from_numpy(b).to(dev)
    ldc = pad(N)
    c = torch.zeros((M, ldc), dtype=torch.float32, device=dev)
    gist.gemm(bool(ta), bool(tb), M, N, K, ad.data_ptr(), a_shape[1], bd.data_ptr(), b_shape[1],
              c.data_ptr(), ldc, 2, out_f32=True, relu=relu)
    torch.cuda.synchronize()
    A = (a[:, :M].T if ta else a[:, :K]).astype(np.float64)
    B = (b[:, :K].T if tb else b[:, :N]).astype(np.float64)
    ref = A @ B
    if relu:
        ref = np.maximum(ref, 0)
    got = c.cpu().numpy()
    assert rel_err(got[:, :N], ref) <= 3e-3, rel_err(got[:, :N], ref)
    assert np.all(got[:, N:] == 0)           # never writes past N
    # not the FP32 SIMT path in disguise: tf32 operands leave an error far above fp32 rounding
    assert rel_err(got[:, :N], ref) > 1e-6 or K < 8


CASES = [
    ("gcn-ragged", dict(n=700, nnz=6000, d0=37, classes=5, clusters=14), "gcn", (37, 45, 29, 5), 3),
    ("sage-ragged", dict(n=650, nnz=5000, d0=23, classes=7, clusters=13), "sage", (23, 40, 33, 7), 4),
    ("sage-wide", dict(n=900, nnz=20000, d0=130, classes=11, clusters=9), "sage", (130, 300, 11), 2),
    ("gat", dict(n=700, nnz=6000, d0=29, classes=6, clusters=11), "gat", (29, 40, 24, 6), 3),
]


@pytest.mark.parametrize("name,kw,arch,dims,q", CASES)
def test_tf32_one_step(name, kw, arch, dims, q):
    g = generate(tiny_spec(**kw), seed=0)
    gpu, ora = make_pair(g, arch, dims, optimizer="adam", q=q, precision="tf32")
    gpu.partition(seed=99, m=2)
    ora.partition(seed=99, m=2)
    gpu.subtrain(1, lr=0.01)
    for i in range(2):
        ora.train_step(i, 0, 0.01)
        tr = ora.last_trace[i]
        nodes = gpu.trace(i, 0)
        p = align(nodes, tr["nodes"])
        nb = len(nodes)
        assert rel_err(gpu.trace(i, 2).reshape(nb, -1), tr["tape"]["logits"][p]) <= TF32_TOL
        for l in range(1, len(dims) - 1):
            assert rel_err(gpu.trace(i, 1, l).reshape(nb, -1), tr["tape"]["H"][l][p]) <= TF32_TOL
        for l in range(len(dims) - 1):
            assert rel_err(gpu.trace(i, 3, l).reshape(ora.sub[i][l].shape), tr["grads"][l]) <= TF32_TOL, l


@pytest.mark.parametrize("arch,dims", [("gcn", (1433, 256, 7)), ("sage", (1433, 256, 7))])
def test_tf32_loss_curve_C1_10_rounds(arch, dims):
    """Loss curve within 1% of the FP64 oracle's over 10 rounds (C1 = Cora-shaped, m = 2,
    10 local iterations, SGD)."""
    g = generate(GRAPHS["cora"], seed=0)
    gpu, ora = make_pair(g, arch, dims, optimizer="sgd", q=1, precision="tf32")
    lg, lo = [], []
    for t in range(10):
        gpu.partition(seed=11 + t, m=2)
        ora.partition(seed=11 + t, m=2)
        lg.append(float(np.mean(gpu.subtrain(10, lr=0.1))))
        lo.append(float(np.mean(ora.subtrain(10, lr=0.1))))
        gpu.aggregate()
        ora.aggregate()
    err = max(abs(a - b) for a, b in zip(lg, lo)) / max(lo)
    print(f"tf32 C1 {arch} loss curve gpu={lg} oracle={lo} err={err:.3e}")
    assert err <= 1e-2, (err, lg, lo)


def test_tf32_eval_and_rounds():
    """Three rounds (weights within 2e-2) and the evaluation forward of the trained global model."""
    _, kw, arch, dims, q = CASES[1]
    g = generate(tiny_spec(**kw), seed=1)
    gpu, ora = make_pair(g, arch, dims, optimizer="sgd", q=q, precision="tf32")
    for t in range(3):
        gpu.partition(seed=5 + t, m=3)
        ora.partition(seed=5 + t, m=3)
        gpu.subtrain(3, lr=0.1)
        ora.subtrain(3, lr=0.1)
        gpu.aggregate()
        ora.aggregate()
        for l in range(len(dims) - 1):
            assert rel_err(gpu.get_params(l), ora.theta[l]) <= TF32_TOL, (t, l)
    _, _, ref = ora.eval(2)
    assert rel_err(gpu.eval_logits(0), ref) <= TF32_TOL
