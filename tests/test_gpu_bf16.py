"""BF16 tensor-core mode (tcgen05 GEMMs, bf16 activations, fp32 accumulation/master
weights/optimizer).  Gates (north_star): relative error <= 2e-2 against the FP64
oracle; loss curve within 1% of the oracle's over 10 rounds.  The GEMM kernel itself
is checked against an FP64 product of the same bf16-rounded operands (only fp32
accumulation-order error remains)."""
import numpy as np
import pytest

from synth.planted import generate, tiny_spec, GRAPHS
from tests.gpu_helpers import align, make_pair, rel_err

pytestmark = pytest.mark.gpu
BF16_TOL = 2e-2


def bf16_round(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).float().numpy()


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (517, 131, 263), (3106, 512, 1216), (300, 48, 1024),
                                   (1216, 512, 3106), (3106, 4096, 1024), (70, 8, 40),
                                   (3106, 512, 96), (777, 300, 128)])  # K <= 128: 2-stage ring, double staging
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0)])
@pytest.mark.parametrize("out_f32,relu", [(True, False), (False, True)])
def test_tc_gemm_layouts(M, N, K, ta, tb, out_f32, relu):
    import torch
    from paper_2102_10424_b200 import gist
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    pad = lambda x: (x + 7) // 8 * 8
    a_shape = (K, pad(M)) if ta else (M, pad(K))
    b_shape = (N, pad(K)) if tb else (K, pad(N))
    a = bf16_round(rng.standard_normal(a_shape))
    b = bf16_round(rng.standard_normal(b_shape))
    dev = torch.device("cuda")
    ad = torch.from_numpy(a).to(dev).to(torch.bfloat16)
    bd = torch.from_numpy(b).to(dev).to(torch.bfloat16)
    ldc = pad(N)
    c = torch.zeros((M, ldc), dtype=torch.float32 if out_f32 else torch.bfloat16, device=dev)
    gist.gemm(bool(ta), bool(tb), M, N, K, ad.data_ptr(), a_shape[1], bd.data_ptr(), b_shape[1],
              c.data_ptr(), ldc, 1, out_f32=out_f32, relu=relu)
    torch.cuda.synchronize()
    A = (a[:, :M].T if ta else a[:, :K]).astype(np.float64)
    B = (b[:, :K].T if tb else b[:, :N]).astype(np.float64)
    ref = A @ B
    if relu:
        ref = np.maximum(ref, 0)
    got = c.float().cpu().numpy()[:, :N]
    tol = 1e-5 if out_f32 else 8e-3          # bf16 output rounding: 2^-8 relative
    assert rel_err(got, ref) <= tol, rel_err(got, ref)
    assert np.all(c.float().cpu().numpy()[:, N:] == 0)   # never writes past N


CASES = [
    ("gcn-ragged", dict(n=700, nnz=6000, d0=37, classes=5, clusters=14), "gcn", (37, 45, 29, 5), 3),
    ("sage-ragged", dict(n=650, nnz=5000, d0=23, classes=7, clusters=13), "sage", (23, 40, 33, 7), 4),
    ("sage-wide", dict(n=900, nnz=20000, d0=130, classes=11, clusters=9), "sage", (130, 300, 11), 2),
]


@pytest.mark.parametrize("name,kw,arch,dims,q", CASES)
def test_bf16_one_step(name, kw, arch, dims, q):
    g = generate(tiny_spec(**kw), seed=0)
    gpu, ora = make_pair(g, arch, dims, optimizer="adam", q=q, precision="bf16")
    gpu.partition(seed=99, m=2)
    ora.partition(seed=99, m=2)
    gpu.subtrain(1, lr=0.01)
    for i in range(2):
        ora.train_step(i, 0, 0.01)
        tr = ora.last_trace[i]
        nodes = gpu.trace(i, 0)
        p = align(nodes, tr["nodes"])
        nb = len(nodes)
        assert rel_err(gpu.trace(i, 2).reshape(nb, -1), tr["tape"]["logits"][p]) <= BF16_TOL
        for l in range(1, len(dims) - 1):
            assert rel_err(gpu.trace(i, 1, l).reshape(nb, -1), tr["tape"]["H"][l][p]) <= BF16_TOL
        for l in range(len(dims) - 1):
            assert rel_err(gpu.trace(i, 3, l).reshape(ora.sub[i][l].shape), tr["grads"][l]) <= BF16_TOL, l


@pytest.mark.parametrize("bd,reassoc", [("1", "1"), ("0", "1"), ("1", "0"), ("0", "0")])
@pytest.mark.parametrize("name,kw,arch,dims,q", [c for c in CASES if c[2] == "sage"])
def test_bf16_one_step_sage_aggregation_variants(name, kw, arch, dims, q, bd, reassoc, monkeypatch):
    """GraphSAGE BF16 with and without the block-diagonal tensor-core aggregation (GIST_BD) and
    with the re-associated last layer forced on / off (GIST_REASSOC: Z = H W_top + N (H W_bot),
    Q = N^T dZ at the class width, R19; by default only for slices >= 256 wide)."""
    monkeypatch.setenv("GIST_BD", bd)
    monkeypatch.setenv("GIST_REASSOC", reassoc)
    test_bf16_one_step(name, kw, arch, dims, q)


def test_bf16_one_step_gcn_reassociated(monkeypatch):
    """GCN BF16 with the re-associated last layer forced on (GIST_REASSOC=1; by default it
    is used only when the layer's input slice is >= 256 wide): logits = A_hat (H W),
    Q = A_hat dZ, dW = H^T Q, dH = Q W^T."""
    monkeypatch.setenv("GIST_REASSOC", "1")
    name, kw, arch, dims, q = CASES[0]
    test_bf16_one_step(name, kw, arch, dims, q)


@pytest.mark.parametrize("optimizer,lr", [("sgd", 0.1), ("adam", 0.001)])  # well-conditioned trajectories
def test_bf16_loss_curve_C1_10_rounds(optimizer, lr):
    """north_star: BF16 mode loss curve within 1% after 10 rounds (C1 = Cora-shaped, m=2,
    10 local iterations).  Metric: max_t |l_gpu(t) - l_oracle(t)| / max_t l_oracle(t)."""
    g = generate(GRAPHS["cora"], seed=0)
    gpu, ora = make_pair(g, "gcn", (1433, 256, 7), optimizer=optimizer, q=1, precision="bf16")
    lg, lo = [], []
    for t in range(10):
        gpu.partition(seed=11, m=2)
        ora.partition(seed=11, m=2)
        lg.append(float(np.mean(gpu.subtrain(10, lr=lr))))
        lo.append(float(np.mean(ora.subtrain(10, lr=lr))))
        gpu.aggregate()
        ora.aggregate()
    err = max(abs(a - b) for a, b in zip(lg, lo)) / max(lo)
    print(f"bf16 C1 {optimizer} loss curve gpu={lg} oracle={lo} err={err:.3e}")
    assert err <= 1e-2, (err, lg, lo)


@pytest.mark.parametrize("optimizer,lr", [("sgd", 0.05), ("adam", 0.001)])
def test_bf16_loss_curve_sage_benchmark_path_10_rounds(optimizer, lr):
    """north_star's BF16 loss-curve gate (within 1% after 10 rounds) on the path the benchmark
    runs: GraphSAGE in BF16 with the block-diagonal tensor-core aggregation (small dense
    clusters), the sparse inter-cluster pass, the re-associated last layer (its input slice is
    256 wide at m = 2), the dW side stream, the batch prefetch and the CUDA-graph step replay."""
    from paper_2102_10424_b200.gist import STAT_BLOCK_AGG
    g = generate(tiny_spec(n=2000, nnz=60000, d0=64, classes=8, clusters=20, f_in=0.8), seed=5)
    gpu, ora = make_pair(g, "sage", (64, 512, 512, 8), optimizer=optimizer, q=4, precision="bf16")
    assert gpu.stat(STAT_BLOCK_AGG) == 1
    lg, lo = [], []
    for t in range(10):
        gpu.partition(seed=100 + t, m=2)
        ora.partition(seed=100 + t, m=2)
        lg.append(float(np.mean(gpu.subtrain(10, lr=lr))))
        lo.append(float(np.mean(ora.subtrain(10, lr=lr))))
        gpu.aggregate()
        ora.aggregate()
    err = max(abs(a - b) for a, b in zip(lg, lo)) / max(lo)
    print(f"bf16 SAGE {optimizer} loss curve gpu={lg} oracle={lo} err={err:.3e}")
    assert lo[-1] < lo[0]            # it trains
    assert err <= 1e-2, (err, lg, lo)


def test_bf16_block_diagonal_aggregation_rounds():
    """SAGE in BF16 mode on small dense clusters uses the block-diagonal tensor-core
    aggregation (intra-cluster blocks) + the sparse inter-cluster pass; q does not divide c,
    so every epoch ends with a short batch (inert dummy rows).  Per-round mean losses and the
    global weights after each round stay within the BF16 tolerance of the FP64 oracle."""
    from paper_2102_10424_b200.gist import STAT_BLOCK_AGG
    g = generate(tiny_spec(n=780, nnz=16000, d0=40, classes=6, clusters=13, f_in=0.8), seed=2)
    gpu, ora = make_pair(g, "sage", (40, 96, 64, 6), optimizer="sgd", q=4, precision="bf16")
    assert gpu.stat(STAT_BLOCK_AGG) == 1
    for t in range(3):
        gpu.partition(seed=3, m=2)
        ora.partition(seed=3, m=2)
        lg = gpu.subtrain(5, lr=0.1)
        lo = ora.subtrain(5, lr=0.1)
        assert np.max(np.abs(lg - lo)) <= BF16_TOL * max(1.0, np.max(np.abs(lo))), (t, lg, lo)
        gpu.aggregate()
        ora.aggregate()
        for l in range(3):
            assert rel_err(gpu.get_params(l), ora.theta[l]) <= BF16_TOL, (t, l)


@pytest.mark.parametrize("bdt,bufs", [("1", "2"), ("1", "1"), ("0", "2")])
def test_bf16_block_diagonal_kernels(bdt, bufs, monkeypatch):
    """Both block-diagonal aggregation kernels against the FP64 oracle: the transposed one (k_bd_t:
    D^T = H^T Blk with Blk symmetric, one unit per cluster and 128-feature tile) with two cluster
    blocks in shared memory (clusters of <= 160 rows) or one (GIST_BDT_BUFS=1: the mode of clusters
    of 161-256 rows), and the row-tile one (GIST_BD_T=0)."""
    monkeypatch.setenv("GIST_BD_T", bdt)
    monkeypatch.setenv("GIST_BDT_BUFS", bufs)
    test_bf16_block_diagonal_aggregation_rounds()
    monkeypatch.setenv("GIST_BD", "1")
    name, kw, arch, dims, q = CASES[1]
    test_bf16_one_step(name, kw, arch, dims, q)


def test_bf16_block_diagonal_large_clusters():
    """Clusters of ~200 rows (> 160): the transposed block aggregation keeps one cluster block in
    shared memory (a block load waits for the previous cluster's MMAs) -- the path taken without
    any switch.  Rounds against the FP64 oracle at the BF16 tolerance."""
    from paper_2102_10424_b200.gist import STAT_BLOCK_AGG
    g = generate(tiny_spec(n=1000, nnz=24000, d0=36, classes=5, clusters=5, f_in=0.8), seed=6)
    gpu, ora = make_pair(g, "sage", (36, 80, 5), optimizer="sgd", q=2, precision="bf16")
    assert gpu.stat(STAT_BLOCK_AGG) == 1
    for t in range(2):
        gpu.partition(seed=9 + t, m=2)
        ora.partition(seed=9 + t, m=2)
        lg = gpu.subtrain(4, lr=0.1)
        lo = ora.subtrain(4, lr=0.1)
        assert np.max(np.abs(lg - lo)) <= BF16_TOL * max(1.0, np.max(np.abs(lo))), (t, lg, lo)
        gpu.aggregate()
        ora.aggregate()
        for l in range(2):
            assert rel_err(gpu.get_params(l), ora.theta[l]) <= BF16_TOL, (t, l)
