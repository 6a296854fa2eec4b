"""GPU parity: the CUDA path (through the C ABI) against the FP64 oracle on the same
seeded inputs.  Gates (BASELINE.json north_star, metric R18):
  * partition indices, slice layouts, init: bit-exact;
  * FP32 mode: activations and logits <= 1e-4, gradients and one-round weights <= 1e-3.
"""
import numpy as np
import pytest

from oracle import gist_oracle as O
from synth.planted import generate, tiny_spec, GRAPHS
from tests.gpu_helpers import align, make_pair, rel_err

pytestmark = pytest.mark.gpu

ACT_TOL, GRAD_TOL = 1e-4, 1e-3

CASES = [
    # (name, graph spec kwargs, arch, dims, q)
    ("gcn-ragged", dict(n=700, nnz=6000, d0=37, classes=5, clusters=14), "gcn", (37, 45, 29, 5), 3),
    ("sage-ragged", dict(n=650, nnz=5000, d0=23, classes=7, clusters=13), "sage", (23, 40, 33, 7), 4),
    ("sage-wide", dict(n=900, nnz=20000, d0=130, classes=11, clusters=9), "sage", (130, 300, 11), 2),
    ("gcn-tiles", dict(n=1200, nnz=15000, d0=150, classes=9, clusters=6), "gcn", (150, 260, 140, 9), 2),
]


def graph(kw, seed=0):
    return generate(tiny_spec(**kw), seed=seed)


@pytest.mark.parametrize("arch,dims", [("gcn", (37, 45, 29, 5)), ("sage", (23, 40, 33, 7)), ("sage", (602, 4096, 41))])
def test_init_bitexact(arch, dims):
    g = graph(dict(n=200, nnz=800, d0=dims[0], classes=dims[-1], clusters=4))
    gpu, ora = make_pair(g, arch, dims)
    for l in range(len(dims) - 1):
        assert np.array_equal(gpu.get_params(l).astype(np.float64), ora.theta[l])


@pytest.mark.parametrize("m", [1, 2, 3, 8])
def test_partition_and_extract_bitexact(m):
    dims = (19, 64, 45, 24, 6)
    g = graph(dict(n=300, nnz=1500, d0=19, classes=6, clusters=5))
    for arch in ("gcn", "sage"):
        gpu, ora = make_pair(g, arch, dims)
        for t in range(3):
            gpu.partition(seed=1234, m=m)
            ora.partition(seed=1234, m=m)
            for l in range(len(dims)):
                got = gpu.get_partition(l)
                for i in range(m):
                    assert np.array_equal(got[i], ora.blocks[l][i]), (arch, t, l, i)
            for i in range(m):
                for l in range(len(dims) - 1):
                    assert np.array_equal(gpu.get_sub_params(i, l).astype(np.float64), ora.sub[i][l])
            gpu.aggregate()
            ora.aggregate()
            for l in range(len(dims) - 1):   # aggregate(extract) = identity, bit-exact
                assert np.array_equal(gpu.get_params(l).astype(np.float64), ora.theta[l])


@pytest.mark.parametrize("name,kw,arch,dims,q", CASES)
@pytest.mark.parametrize("optimizer", ["sgd", "adam"])
def test_one_step_parity(name, kw, arch, dims, q, optimizer):
    g = graph(kw)
    gpu, ora = make_pair(g, arch, dims, optimizer=optimizer, q=q)
    m = 2
    gpu.partition(seed=99, m=m)
    ora.partition(seed=99, m=m)
    gpu.subtrain(1, lr=0.01)
    for i in range(m):
        ora.train_step(i, 0, 0.01)
        tr = ora.last_trace[i]
        nodes = gpu.trace(i, 0)
        p = align(nodes, tr["nodes"])
        nb = len(nodes)
        logits = gpu.trace(i, 2).reshape(nb, -1)
        assert rel_err(logits, tr["tape"]["logits"][p]) <= ACT_TOL
        for l in range(1, len(dims) - 1):
            act = gpu.trace(i, 1, l).reshape(nb, -1)
            assert rel_err(act, tr["tape"]["H"][l][p]) <= ACT_TOL, (l,)
        for l in range(len(dims) - 1):
            grad = gpu.trace(i, 3, l).reshape(ora.sub[i][l].shape)
            assert rel_err(grad, tr["grads"][l]) <= GRAD_TOL, (l,)
            w = gpu.get_sub_params(i, l)
            assert rel_err(w, ora.sub[i][l]) <= GRAD_TOL, (l,)
        loss = gpu.trace(i, 4)[0]
        assert abs(loss - tr["loss"]) <= ACT_TOL * max(1.0, abs(tr["loss"]))


@pytest.mark.parametrize("case", [0, 1])
def test_one_step_parity_global_cluster_map(case, monkeypatch):
    """The batch build's global (tagged map64) membership path, taken when the cluster ->
    offset map does not fit shared memory (> 16k clusters), forced here by env."""
    monkeypatch.setenv("GIST_BATCH_GLOBAL_MAP", "1")
    name, kw, arch, dims, q = CASES[case]
    test_one_step_parity(name, kw, arch, dims, q, "sgd")


@pytest.mark.parametrize("name,kw,arch,dims,q", CASES[:2])
def test_rounds_parity(name, kw, arch, dims, q):
    """Several rounds (partition -> zeta steps -> aggregate): global weights <= 1e-3."""
    g = graph(kw, seed=1)
    gpu, ora = make_pair(g, arch, dims, optimizer="adam", q=q)
    for t in range(3):
        gpu.partition(seed=5, m=3)
        ora.partition(seed=5, m=3)
        lg = gpu.subtrain(4, lr=0.005)
        lo = ora.subtrain(4, lr=0.005)
        assert np.max(np.abs(lg - lo)) <= 1e-4 * max(1.0, np.max(np.abs(lo)))
        gpu.aggregate()
        ora.aggregate()
        for l in range(len(dims) - 1):
            assert rel_err(gpu.get_params(l), ora.theta[l]) <= GRAD_TOL, (t, l)
    for code in (0, 1, 2):
        lg, ag = gpu.eval(code)
        lo, ao, _ = ora.eval(code)
        assert abs(lg - lo) <= 1e-4 * max(1.0, abs(lo))
        assert abs(ag - ao) <= 2.0 / (g["split"] == code).sum()


@pytest.mark.parametrize("optimizer", ["adam", "sgd"])
def test_cora_config_C1_end_to_end(optimizer):
    """BASELINE configs[0]: Cora-shaped graph, 2-layer GCN hidden 256, m=2, 5 rounds x 10 iters.
    Adam: the north_star gate is one round (weights <= 1e-3, losses <= 1e-4).  Over later
    rounds Adam's sign-like normalised step turns FP32 rounding into O(lr) weight differences;
    a plain float32 numpy twin of the same algorithm diverges from the FP64 oracle exactly as
    much as the GPU does ("Adam multi-round conditioning"), so multi-round weight
    parity is gated with SGD, which is well-conditioned: every round <= 1e-3."""
    g = generate(GRAPHS["cora"], seed=0)
    gpu, ora = make_pair(g, "gcn", (1433, 256, 7), optimizer=optimizer, q=1)
    lr = 0.01 if optimizer == "adam" else 0.5
    loss_err, w_err = [], []
    for t in range(5):
        gpu.partition(seed=11, m=2)
        ora.partition(seed=11, m=2)
        lg = gpu.subtrain(10, lr=lr)
        lo = ora.subtrain(10, lr=lr)
        loss_err.append(float(np.max(np.abs(lg - lo) / np.maximum(1.0, np.abs(lo)))))
        gpu.aggregate()
        ora.aggregate()
        w_err.append(max(rel_err(gpu.get_params(l), ora.theta[l]) for l in range(2)))
    print(f"C1 {optimizer} per-round loss rel err", loss_err, "weight rel err", w_err)
    assert loss_err[0] <= 1e-4 and w_err[0] <= GRAD_TOL, (loss_err, w_err)
    if optimizer == "sgd":
        assert max(loss_err) <= 1e-4 and max(w_err) <= GRAD_TOL, (loss_err, w_err)
        lg, ag = gpu.eval(2)
        lo, ao, _ = ora.eval(2)
        assert abs(lg - lo) <= 1e-4 * max(1.0, lo) and abs(ag - ao) <= 2e-3, (lg, lo, ag, ao)


def test_edge_cases_m1_tail_batch_isolated_nodes():
    # m=1 (GIST == plain training), q not dividing c (short last batch), isolated nodes (SAGE deg 0),
    # tiny clusters, batches with no train rows
    spec = tiny_spec(n=90, nnz=60, d0=9, classes=3, clusters=30)
    g = generate(spec, seed=4)
    for arch in ("gcn", "sage"):
        gpu, ora = make_pair(g, arch, (9, 12, 3), optimizer="adam", q=7)
        gpu.partition(seed=2, m=1)
        ora.partition(seed=2, m=1)
        lg = gpu.subtrain(6, lr=0.01)      # 30 clusters / 7 = 5 batches per epoch: crosses an epoch
        lo = ora.subtrain(6, lr=0.01)
        assert abs(lg[0] - lo[0]) <= 1e-4 * max(1.0, abs(lo[0]))
        for l in range(2):
            assert rel_err(gpu.get_sub_params(0, l), ora.sub[0][l]) <= GRAD_TOL


def test_kernel_spmm_and_gemm_entry_points():
    import torch
    from paper_2102_10424_b200 import gist
    rng = np.random.default_rng(0)
    n, w, ld = 333, 300, 304
    A = np.triu(rng.random((n, n)) < 0.05, 1)
    A = (A | A.T)
    rp = np.concatenate([[0], np.cumsum(A.sum(1))]).astype(np.int64)
    ci = np.concatenate([np.nonzero(A[i])[0] for i in range(n)]).astype(np.int32)
    deg = A.sum(1).astype(np.float64)
    H = np.zeros((n, ld), np.float32)
    H[:, :w] = rng.integers(-3, 4, size=(n, w))
    dev = torch.device("cuda")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    rpd, cid, Hd = t(rp), t(ci), t(H)
    out = torch.zeros_like(Hd)
    gist.spmm(rpd.data_ptr(), cid.data_ptr(), n, None, None, False, Hd.data_ptr(), out.data_ptr(), w, ld, 0)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy()[:, :w], (A.astype(np.float64) @ H[:, :w].astype(np.float64)))
    sc = (1.0 / np.sqrt(deg + 1)).astype(np.float32)
    scd = t(sc)
    gist.spmm(rpd.data_ptr(), cid.data_ptr(), n, scd.data_ptr(), scd.data_ptr(), True, Hd.data_ptr(),
              out.data_ptr(), w, ld, 0)
    torch.cuda.synchronize()
    ref = O.spmm(O.gcn_operator(rp, ci, n), H[:, :w].astype(np.float64))
    assert rel_err(out.cpu().numpy()[:, :w], ref) <= 1e-6
    for ta, tb in [(0, 0), (0, 1), (1, 0)]:
        M, N, K = 517, 131, 263
        a = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
        b = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
        ad, bd = t(a), t(b)
        c = torch.zeros((M, N), dtype=torch.float32, device=dev)
        gist.gemm(bool(ta), bool(tb), M, N, K, ad.data_ptr(), a.shape[1], bd.data_ptr(), b.shape[1],
                  c.data_ptr(), N, 0)
        torch.cuda.synchronize()
        ref = (a.T if ta else a).astype(np.float64) @ (b.T if tb else b).astype(np.float64)
        assert rel_err(c.cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("ta,tb,M,N,K,out_f32", [
    (0, 0, 3120, 512, 1216, False),   # forward a3 (several tiles per persistent CTA, ragged last M tile)
    (0, 1, 3120, 1024, 512, False),   # dX
    (1, 0, 1216, 512, 3120, True),    # dW, fp32 out
    (0, 0, 3120, 48, 1024, True),     # last layer, fp32 logits (N < one 128-byte box)
    (0, 0, 777, 136, 200, False),     # N not a multiple of the tile, small
    (0, 1, 300, 131, 64, True),       # ldc*4 not 16-byte aligned: direct-store epilogue
    (0, 0, 12480, 512, 1024, False),  # ~3 tiles per persistent CTA (the grouped step's regime)
    (0, 1, 12480, 1024, 512, False),
    (1, 0, 4864, 512, 3120, True),
    (0, 0, 24960, 48, 1024, True),    # narrow N, many tiles per CTA (logits of a grouped step)
])
def test_kernel_gemm_bf16_tcgen05_shapes(ta, tb, M, N, K, out_f32):
    """tcgen05 GEMM entry point (gist_gemm dtype 1) at the subTrain step's shapes against an
    fp64 product of the same bf16-rounded operands (fp32 out: 1e-5; bf16 out: one bf16
    rounding of the result, 2^-8 relative)."""
    import torch
    from paper_2102_10424_b200 import gist
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(M * 7 + N)
    a = torch.randn((K, M) if ta else (M, K), generator=g).to(torch.bfloat16)
    b = torch.randn((N, K) if tb else (K, N), generator=g).to(torch.bfloat16)
    ad, bd = a.to(dev), b.to(dev)
    c = torch.zeros((M, N), dtype=torch.float32 if out_f32 else torch.bfloat16, device=dev)
    gist.gemm(bool(ta), bool(tb), M, N, K, ad.data_ptr(), a.shape[1], bd.data_ptr(), b.shape[1], c.data_ptr(), N, 1,
              out_f32=out_f32)
    torch.cuda.synchronize()
    A = (a.T if ta else a).double().numpy()
    B = (b.T if tb else b).double().numpy()
    ref = A @ B
    got = c.float().cpu().numpy().astype(np.float64)
    err = np.abs(got - ref) / (np.abs(ref) + np.sqrt(K))  # |ref| ~ sqrt(K) for unit normal operands
    assert err.max() <= (1e-5 if out_f32 else 2.0 ** -8), err.max()


@pytest.mark.parametrize("arch,dims,m", [("sage", (23, 40, 33, 7), 2), ("gcn", (37, 45, 29, 5), 3),
                                         ("sage", (23, 40, 33, 7), 1)])
def test_persistent_adam_state_rounds(arch, dims, m):
    """persistent sliced Adam state (GIST_OPT_STATE_PERSISTENT) against the
    oracle's persistent mode over 3 rounds (FP32).  After the first step the moments are no
    longer sign-like, so the weights stay within 1e-3 across rounds; m = 1
    is plain Adam without restarts."""
    kw = CASES[1][1] if arch == "sage" else CASES[0][1]
    q = CASES[1][4] if arch == "sage" else CASES[0][4]
    g = graph(kw, seed=2)
    from paper_2102_10424_b200.gist import Gist
    gpu = Gist(arch, dims, optimizer="adam", precision="fp32", clusters_per_batch=q, batch_seed=3,
               opt_state="persistent")
    gpu.load_graph(g)
    gpu.init_params(7)
    ora = O.OracleGIST(arch=arch, dims=list(dims), optimizer="adam", clusters_per_batch=q, batch_seed=3,
                       opt_state="persistent")
    ora.load_graph(g["row_ptr"], g["col_idx"], g["X"], g["labels"], g["num_classes"], g["split"],
                   g["cluster_ids"], g["num_clusters"])
    ora.init_params(7)
    for t in range(3):
        gpu.partition(seed=21, m=m)
        ora.partition(seed=21, m=m)
        lg = gpu.subtrain(4, lr=0.002)
        lo = ora.subtrain(4, lr=0.002)
        assert np.max(np.abs(lg - lo)) <= 1e-4 * max(1.0, np.max(np.abs(lo))), (t, lg, lo)
        gpu.aggregate()
        ora.aggregate()
        for l in range(len(dims) - 1):
            assert rel_err(gpu.get_params(l), ora.theta[l]) <= GRAD_TOL, (t, l)
