"""GIST oracle (FP64, numpy/scipy) -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU implementation of the GIST training loop
(Algorithm 1) restricted to the hot path named by
BASELINE.json's north_star: subGCNs (partition + extract), subTrain (Cluster
mini-batch, GCN / GraphSAGE forward + backward, softmax-CE, Adam/SGD) and
subAgg (replacement write-back), plus full-graph and partition-wise (R20) evaluation.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
`--impl reference`) may import this module.  It shares no code with the CUDA
path.  Every step is written in the paper's order and notation; library
primitives used as single steps: numpy matmul, scipy CSR @ dense, argsort.

Readings R1..R18 (where the paper is silent) are listed in DESIGN.md; they
follow SURVEY.md section 8(c).  Parity unpinned: accuracy on real datasets
(no data here); everything else is pinned in tests/test_oracle_*.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

__all__ = [
    "philox4x32_10", "philox_keys64", "split_seed",
    "PURPOSE_PARTITION", "PURPOSE_BATCH", "PURPOSE_INIT",
    "sample_partition", "sub_index_sets", "extract", "aggregate",
    "aggregate_delta_sum", "coverage_fraction", "sub_param_count",
    "glorot_init", "glorot_block", "batch_schedule", "batch_nodes", "induced_subgraph",
    "gcn_operator", "sage_operator", "chebyshev_operator", "spmm", "gat_structure", "gat_attention",
    "weight_rows",
    "forward", "backward", "softmax_ce", "adam_step", "sgd_step",
    "OracleGIST", "lr_step_schedule",
]

MASK32 = np.uint64(0xFFFFFFFF)

# ---------------------------------------------------------------------------
# Philox4x32-10 (Random123).  Counter-based generator used by
# R5 (partition), R7 (batch schedule) and R11 (init).  The CUDA path carries
# its own implementation; both are pinned to the Random123 known-answer tests.
# ---------------------------------------------------------------------------
PHILOX_M0 = np.uint64(0xD2511F53)
PHILOX_M1 = np.uint64(0xCD9E8D57)
PHILOX_W0 = np.uint64(0x9E3779B9)
PHILOX_W1 = np.uint64(0xBB67AE85)

PURPOSE_PARTITION = 1
PURPOSE_BATCH = 2
PURPOSE_INIT = 3


def split_seed(seed: int) -> tuple[int, int]:
    """64-bit seed -> Philox key (lo32, hi32)."""
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & 0xFFFFFFFF, seed >> 32


def philox4x32_10(ctr: np.ndarray, key: tuple[int, int]) -> np.ndarray:
    """Philox4x32 with 10 rounds.  ctr: (N, 4) uint32-valued; returns (N, 4) uint32."""
    c = np.asarray(ctr, dtype=np.uint64).reshape(-1, 4)
    c0, c1, c2, c3 = (c[:, j].copy() for j in range(4))
    k0 = np.uint64(key[0] & 0xFFFFFFFF)
    k1 = np.uint64(key[1] & 0xFFFFFFFF)
    for _ in range(10):
        p0 = PHILOX_M0 * c0                       # < 2^64: exact in uint64
        p1 = PHILOX_M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        k0 = (k0 + PHILOX_W0) & MASK32
        k1 = (k1 + PHILOX_W1) & MASK32
    return np.stack([c0, c1, c2, c3], axis=1).astype(np.uint32)


def philox_keys64(idx: np.ndarray, c1: int, c2: int, purpose: int, seed: int) -> np.ndarray:
    """64-bit sort keys (w1 << 32) | w0 for counters (idx, c1, c2, purpose)."""
    idx = np.asarray(idx, dtype=np.uint64)
    ctr = np.stack([idx, np.full_like(idx, c1 & 0xFFFFFFFF),
                    np.full_like(idx, c2 & 0xFFFFFFFF),
                    np.full_like(idx, purpose)], axis=1)
    w = philox4x32_10(ctr, split_seed(seed)).astype(np.uint64)
    return (w[:, 1] << np.uint64(32)) | w[:, 0]


def _philox_permutation(count: int, c1: int, c2: int, purpose: int, seed: int) -> np.ndarray:
    """Units 0..count-1 ordered by (64-bit Philox key, unit index) ascending."""
    units = np.arange(count, dtype=np.int64)
    keys = philox_keys64(units, c1, c2, purpose, seed)
    return units[np.lexsort((units, keys))]


# ---------------------------------------------------------------------------
# subGCNs: random disjoint equal-size partition of every hidden dimension.
# PAPER.md:147-161 (Sec. 2.1): "a random, disjoint partition of the feature set
# [d_l] into m equally-sized blocks"; d_0 and d_L are not partitioned
# (Fig. 2 caption).  Reading R5 fixes the sampler.
# ---------------------------------------------------------------------------
def sample_partition(dims: list[int], m: int, seed: int, t: int) -> list[list[np.ndarray]]:
    """Returns blocks[l][i] = D_l^(i) as an ascending int64 array, l = 0..L.

    Hidden dims l = 1..L-1: pi = Philox permutation with counter (r, t, l, 1);
    block i = pi[b_i : b_{i+1}] re-sorted ascending, where the first d mod m
    blocks get ceil(d/m) units and the rest floor(d/m) (R5).
    d_0 and d_L: every sub-GCN gets the full index set.
    """
    L = len(dims) - 1
    if m < 1:
        raise ValueError("m must be >= 1")
    for l in range(1, L):
        if m > dims[l]:
            raise ValueError(f"m={m} exceeds hidden dim d_{l}={dims[l]}")
    blocks: list[list[np.ndarray]] = []
    for l, d in enumerate(dims):
        if l == 0 or l == L:
            blocks.append([np.arange(d, dtype=np.int64) for _ in range(m)])
            continue
        pi = _philox_permutation(d, t, l, PURPOSE_PARTITION, seed)
        base, extra = divmod(d, m)
        sizes = [base + (1 if i < extra else 0) for i in range(m)]
        offs = np.concatenate([[0], np.cumsum(sizes)])
        blocks.append([np.sort(pi[offs[i]:offs[i + 1]]) for i in range(m)])
    return blocks


def sub_index_sets(arch: str, dims: list[int], blocks, i: int):
    """Row/column index sets of Theta_l^(i) = [Theta_l]_{D_l^(i) x D_{l+1}^(i)}.

    GraphSAGE weights act on [H || N H] (R2), so their rows are D_l^(i) followed by
    d_l + D_l^(i) (self block, then neighbour block; R6).  GAT weights carry the two
    attention vectors as rows d_l (a_src) and d_l + 1 (a_dst) (R21); every sub-GCN keeps
    both rows, sliced to its output units.
    """
    out = []
    for l in range(len(dims) - 1):
        rows = blocks[l][i]
        if arch == "sage":
            rows = np.concatenate([rows, dims[l] + rows])
        elif arch == "gat":      # R21: the attention vectors (rows d_l, d_l + 1) follow the output units
            rows = np.concatenate([rows, [dims[l], dims[l] + 1]])
        out.append((rows, blocks[l + 1][i]))
    return out


def extract(theta: list[np.ndarray], index_sets) -> list[np.ndarray]:
    """Theta^(i)_l = Theta_l[rows, cols], logical row-major (R6)."""
    return [theta[l][np.ix_(r, c)].copy() for l, (r, c) in enumerate(index_sets)]


def aggregate(theta: list[np.ndarray], subs: list[list[np.ndarray]], all_index_sets) -> None:
    """subAgg by replacement (R9): each worker writes its block
    back into Theta; entries outside every block keep their exact value."""
    for sub, sets in zip(subs, all_index_sets):
        for l, (r, c) in enumerate(sets):
            theta[l][np.ix_(r, c)] = sub[l]


def aggregate_delta_sum(theta, subs_start, subs_end, all_index_sets):
    """The one-hidden-layer form PAPER.md:815: theta_{t+1} = theta_t + sum_j (theta^(j)_{t,zeta} - theta^(j)_{t,0}).
    Used only as a tolerance pin for `aggregate` (equal up to rounding for disjoint blocks)."""
    out = [w.copy() for w in theta]
    for s0, s1, sets in zip(subs_start, subs_end, all_index_sets):
        for l, (r, c) in enumerate(sets):
            out[l][np.ix_(r, c)] += s1[l] - s0[l]
    return out


def weight_rows(arch: str, d: int) -> int:
    """Logical rows of Theta_l for input width d: GCN d, GraphSAGE 2d (R2), GAT d + 2 (R21)."""
    return 2 * d if arch == "sage" else (d + 2 if arch == "gat" else d)


def coverage_fraction(dims, blocks, l: int, m: int, arch: str = "gcn") -> float:
    """Fraction of Theta_l entries inside the union of the m diagonal blocks."""
    rows = weight_rows(arch, dims[l])
    mask = np.zeros((rows, dims[l + 1]), dtype=bool)
    for i in range(m):
        r, c = sub_index_sets(arch, dims, blocks, i)[l]
        mask[np.ix_(r, c)] = True
    return float(mask.mean())


def sub_param_count(arch: str, dims, m: int, i: int = 0) -> int:
    """Scalars of one sub-GCN (PAPER.md:228 communication term).  Uses the balanced
    block sizes of R5 (block i gets ceil(d/m) if i < d mod m)."""
    L = len(dims) - 1
    def size(l):
        if l == 0 or l == L:
            return dims[l]
        base, extra = divmod(dims[l], m)
        return base + (1 if i < extra else 0)
    return sum(weight_rows(arch, size(l)) * size(l + 1) for l in range(L))


# ---------------------------------------------------------------------------
# Initialisation ("randomly initialize GCN"; reading R11: Glorot
# uniform from Philox, computed in fp32 so that both sides agree bit-exactly).
# ---------------------------------------------------------------------------
def glorot_init(arch: str, dims: list[int], seed: int) -> list[np.ndarray]:
    theta = []
    for l in range(len(dims) - 1):
        rows = weight_rows(arch, dims[l])
        cols = dims[l + 1]
        fan_in = dims[l] if arch == "gat" else rows       # R21: GAT fan_in = d_l
        s = np.sqrt(np.float32(6.0) / np.float32(fan_in + cols), dtype=np.float32)
        flat = np.arange(rows * cols, dtype=np.uint64)
        ctr = np.stack([flat & MASK32, np.full_like(flat, l), flat >> np.uint64(32),
                        np.full_like(flat, PURPOSE_INIT)], axis=1)
        w0 = philox4x32_10(ctr, split_seed(seed))[:, 0]
        u = (w0 >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)
        tt = np.float32(2.0) * u - np.float32(1.0)          # exact in fp32
        w = (tt * s).astype(np.float32)                      # one rounded fp32 multiply
        theta.append(w.astype(np.float64).reshape(rows, cols))
    return theta


def glorot_block(arch: str, dims: list[int], seed: int, l: int, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """Theta_l[rows, cols] of glorot_init without materialising Theta_l: every entry is a
    function of its own counter (flat index, l, 0, PURPOSE_INIT) only (R11).  Used for
    full-size parity checks; pinned against glorot_init in tests/test_oracle_model.py."""
    nrows = weight_rows(arch, dims[l])
    ncols = dims[l + 1]
    fan_in = dims[l] if arch == "gat" else nrows
    s = np.sqrt(np.float32(6.0) / np.float32(fan_in + ncols), dtype=np.float32)
    r = np.asarray(rows, dtype=np.uint64)[:, None]
    c = np.asarray(cols, dtype=np.uint64)[None, :]
    flat = (r * np.uint64(ncols) + c).ravel()
    ctr = np.stack([flat & MASK32, np.full_like(flat, l), flat >> np.uint64(32),
                    np.full_like(flat, PURPOSE_INIT)], axis=1)
    w0 = philox4x32_10(ctr, split_seed(seed))[:, 0]
    u = (w0 >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)
    tt = np.float32(2.0) * u - np.float32(1.0)
    return (tt * s).astype(np.float32).astype(np.float64).reshape(len(rows), len(cols))


# ---------------------------------------------------------------------------
# Cluster mini-batches (Sec. 2.2: "subTrain first selects one of
# the c subgraphs ... Alternatively, the union of several sub-graphs").
# Reading R7: each slot has its own Philox-permuted cluster order per epoch.
# ---------------------------------------------------------------------------
def batch_schedule(num_clusters: int, q: int, batch_seed: int, slot: int, step: int) -> np.ndarray:
    """Cluster ids of slot `slot`'s mini-batch at its step `step` (R7)."""
    B = -(-num_clusters // q)
    e, p = divmod(step, B)
    perm = _philox_permutation(num_clusters, e, slot, PURPOSE_BATCH, batch_seed)
    return perm[p * q: min((p + 1) * q, num_clusters)]


def batch_nodes(cluster_ids: np.ndarray, chosen: np.ndarray) -> np.ndarray:
    """Batch nodes = union of chosen clusters, ascending global id (R7)."""
    return np.nonzero(np.isin(cluster_ids, chosen))[0].astype(np.int64)


def induced_subgraph(row_ptr, col_idx, nodes: np.ndarray):
    """Keep exactly the edges with both endpoints in `nodes`; local ids follow the
    order of `nodes`.  Returns (row_ptr_b, col_idx_b) int64."""
    n = len(row_ptr) - 1
    local = np.full(n, -1, dtype=np.int64)
    local[nodes] = np.arange(len(nodes))
    rp = [0]
    cols = []
    for v in nodes:
        nb = col_idx[row_ptr[v]:row_ptr[v + 1]]
        keep = local[nb]
        keep = np.sort(keep[keep >= 0])
        cols.append(keep)
        rp.append(rp[-1] + len(keep))
    col = np.concatenate(cols) if cols else np.zeros(0, dtype=np.int64)
    return np.asarray(rp, dtype=np.int64), col.astype(np.int64)


# ---------------------------------------------------------------------------
# Aggregation operators.
# GCN (Eq. 1): A_bar = degree-normalised adjacency with added
#   self-loops; reading R1 = renormalisation trick
#   A_hat = D~^{-1/2} (A + I) D~^{-1/2}, D~ = deg + 1, on the batch subgraph.
# Theory form (Eq. 3): I + D^{-1/2} A D^{-1/2} (tests only).
# GraphSAGE-mean (R2): N = D^{-1} A, isolated rows -> 0.
# ---------------------------------------------------------------------------
def _adjacency(row_ptr, col_idx, n) -> sp.csr_matrix:
    vals = np.ones(len(col_idx), dtype=np.float64)
    return sp.csr_matrix((vals, np.asarray(col_idx), np.asarray(row_ptr)), shape=(n, n))


def gcn_operator(row_ptr, col_idx, n) -> sp.csr_matrix:
    A = _adjacency(row_ptr, col_idx, n)
    dt = np.asarray(A.sum(axis=1)).ravel() + 1.0
    Dm = sp.diags(1.0 / np.sqrt(dt))
    return (Dm @ (A + sp.identity(n, format="csr")) @ Dm).tocsr()


def chebyshev_operator(row_ptr, col_idx, n) -> sp.csr_matrix:
    A = _adjacency(row_ptr, col_idx, n)
    deg = np.asarray(A.sum(axis=1)).ravel()
    inv = np.where(deg > 0, 1.0 / np.sqrt(np.where(deg > 0, deg, 1.0)), 0.0)
    Dm = sp.diags(inv)
    return (sp.identity(n, format="csr") + Dm @ A @ Dm).tocsr()


def sage_operator(row_ptr, col_idx, n) -> sp.csr_matrix:
    A = _adjacency(row_ptr, col_idx, n)
    deg = np.asarray(A.sum(axis=1)).ravel()
    inv = np.where(deg > 0, 1.0 / np.where(deg > 0, deg, 1.0), 0.0)
    return (sp.diags(inv) @ A).tocsr()


def gat_structure(row_ptr, col_idx, n) -> sp.csr_matrix:
    """GAT attends over N(i) and i itself (R21): the 0/1 pattern of A + I."""
    S = (_adjacency(row_ptr, col_idx, n) + sp.identity(n, format="csr")).tocsr()
    S.data[:] = 1.0
    S.sort_indices()
    return S


def gat_attention(S: sp.csr_matrix, Z: np.ndarray, a_src: np.ndarray, a_dst: np.ndarray, slope: float = 0.2):
    """Attention of one GAT layer (Velickovic et al., R21): s = Z a_src, t = Z a_dst,
    e_ij = LeakyReLU(t_i + s_j) on the pattern S, alpha_ij = softmax_j(e_ij) per row.
    Returns (alpha as a CSR matrix with S's pattern, pre-activation e per stored entry)."""
    s = Z @ a_src
    t = Z @ a_dst
    rows = np.repeat(np.arange(S.shape[0]), np.diff(S.indptr))
    pre = t[rows] + s[S.indices]
    e = np.where(pre > 0, pre, slope * pre)
    alpha = np.empty_like(e)
    for i in range(S.shape[0]):
        a, b = S.indptr[i], S.indptr[i + 1]
        x = np.exp(e[a:b] - e[a:b].max())
        alpha[a:b] = x / x.sum()
    return sp.csr_matrix((alpha, S.indices.copy(), S.indptr.copy()), shape=S.shape), pre


def spmm(op: sp.csr_matrix, H: np.ndarray) -> np.ndarray:
    """Sparse (n x n) times dense (n x w), FP64 (library primitive)."""
    return np.asarray(op @ H)


# ---------------------------------------------------------------------------
# Forward / backward (Eq. 1 / Eq. 2).
# H_{l+1} = ReLU(A_bar H_l Theta_l) for l < L-1; logits = A_bar H_{L-1} Theta_{L-1}
# (last activation identity; R3).  GraphSAGE: A_bar H_l is replaced
# by the concatenation [H_l || N H_l] (R2).
# ---------------------------------------------------------------------------
def forward(arch: str, theta: list[np.ndarray], op: sp.csr_matrix, X: np.ndarray) -> dict:
    H = [np.asarray(X, dtype=np.float64)]
    agg, Z = [], []
    L = len(theta)
    for l in range(L):
        if arch == "gat":                               # R21: out = alpha(Z) Z, Z = H W
            d = H[l].shape[1]
            C = H[l] @ theta[l][:d]
            alpha, _ = gat_attention(op, C, theta[l][d], theta[l][d + 1])
            z = spmm(alpha, C)
        elif arch == "gcn":
            C = spmm(op, H[l])                          # A_bar H_l
            z = C @ theta[l]
        else:
            C = np.concatenate([H[l], spmm(op, H[l])], axis=1)   # [H_l || N H_l]
            z = C @ theta[l]
        agg.append(C)
        Z.append(z)
        if l < L - 1:
            H.append(np.maximum(z, 0.0))
    return {"H": H, "C": agg, "Z": Z, "logits": Z[-1]}


def backward(arch: str, theta, op: sp.csr_matrix, tape: dict, dlogits: np.ndarray) -> list[np.ndarray]:
    """Reverse-mode gradient of the loss w.r.t. every Theta_l given dL/dlogits.
    ReLU'(0) := 0 (R3)."""
    L = len(theta)
    grads = [None] * L
    G = np.asarray(dlogits, dtype=np.float64)            # dL/dZ_{L-1}
    opT = op.T.tocsr()
    for l in range(L - 1, -1, -1):
        if arch == "gat":                                  # R21, chain rule through the attention
            H_l, Zl = tape["H"][l], tape["C"][l]
            d = H_l.shape[1]
            a_src, a_dst = theta[l][d], theta[l][d + 1]
            alpha, pre = gat_attention(op, Zl, a_src, a_dst)
            rows = np.repeat(np.arange(op.shape[0]), np.diff(op.indptr))
            cols = op.indices
            dZ = spmm(alpha.T.tocsr(), G)                  # through out_i = sum_j alpha_ij Z_j
            dal = np.einsum("ek,ek->e", G[rows], Zl[cols])  # d alpha_ij = G_i . Z_j
            Srow = np.bincount(rows, weights=alpha.data * dal, minlength=op.shape[0])
            de = alpha.data * (dal - Srow[rows])           # softmax backward
            dpre = de * np.where(pre > 0, 1.0, 0.2)        # LeakyReLU backward
            dt = np.bincount(rows, weights=dpre, minlength=op.shape[0])
            ds = np.bincount(cols, weights=dpre, minlength=op.shape[0])
            dZ = dZ + np.outer(ds, a_src) + np.outer(dt, a_dst)
            grads[l] = np.vstack([H_l.T @ dZ, (Zl.T @ ds)[None, :], (Zl.T @ dt)[None, :]])
            if l == 0:
                break
            dH = dZ @ theta[l][:d].T
            G = dH * (tape["Z"][l - 1] > 0.0)
            continue
        grads[l] = tape["C"][l].T @ G                      # dTheta_l = C_l^T G
        if l == 0:
            break
        dC = G @ theta[l].T                                # dL/dC_l
        if arch == "gcn":
            dH = spmm(opT, dC)                             # A_bar^T dC
        else:
            d = tape["H"][l].shape[1]
            dH = dC[:, :d] + spmm(opT, dC[:, d:])          # self part + N^T (neigh part)
        G = dH * (tape["Z"][l - 1] > 0.0)                  # through ReLU of layer l-1
    return grads


def softmax_ce(logits: np.ndarray, labels: np.ndarray, rows_mask: np.ndarray):
    """Mean softmax cross-entropy over rows with rows_mask (R4).
    Returns (loss, dlogits); with no masked rows: (0, zeros)."""
    logits = np.asarray(logits, dtype=np.float64)
    mx = logits.max(axis=1, keepdims=True)
    lse = mx[:, 0] + np.log(np.exp(logits - mx).sum(axis=1))
    p = np.exp(logits - lse[:, None])
    idx = np.nonzero(rows_mask)[0]
    nt = len(idx)
    d = np.zeros_like(logits)
    if nt == 0:
        return 0.0, d
    y = np.asarray(labels)[idx]
    loss = float(np.sum(lse[idx] - logits[idx, y]) / nt)
    d[idx] = p[idx]
    d[idx, y] -= 1.0
    d[idx] /= nt
    return loss, d


def adam_step(w, g, state, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """Adam (Kingma & Ba; R8), bias-corrected, no weight decay."""
    state["t"] = state.get("t", 0) + 1
    t = state["t"]
    m = state.setdefault("m", np.zeros_like(w))
    v = state.setdefault("v", np.zeros_like(w))
    m *= beta1
    m += (1.0 - beta1) * g
    v *= beta2
    v += (1.0 - beta2) * g * g
    mhat = m / (1.0 - beta1 ** t)
    vhat = v / (1.0 - beta2 ** t)
    return w - lr * mhat / (np.sqrt(vhat) + eps)


def sgd_step(w, g, lr):
    """One SGD step (one application of subTrain = one SGD step)."""
    return w - lr * g


def lr_step_schedule(base_lr: float, epoch: int, total: int) -> float:
    """10x decay at 50% and 75% of training.  Driver-side only."""
    if epoch < 0.5 * total:
        return base_lr
    if epoch < 0.75 * total:
        return base_lr / 10.0
    return base_lr / 100.0


# ---------------------------------------------------------------------------
# Algorithm 1 driver mirroring the C ABI (gist_load_graph / gist_init_params /
# gist_partition / gist_subtrain / gist_aggregate / gist_eval).
# ---------------------------------------------------------------------------
@dataclass
class OracleGIST:
    arch: str                    # "gcn", "sage" or "gat" (R21)
    dims: list
    optimizer: str = "adam"      # "adam" or "sgd"
    clusters_per_batch: int = 1  # q
    batch_seed: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    # Adam state across rounds: "reset" = moments and step counter restart at every
    # partition (R8, the default); "persistent" = SURVEY §8 f3: the global first
    # and second moments are shaped like Theta, partitioned / extracted / aggregated with the
    # weights, and the step counter carries over (the paper is silent)
    opt_state: str = "reset"
    # state
    theta: list = field(default_factory=list)
    round: int = 0
    step: int = 0                # steps taken by every slot so far (R7 counter)
    m: int = 0
    blocks: list = None
    sub: list = None
    opt: list = None
    index_sets: list = None
    last_trace: dict = field(default_factory=dict)

    def load_graph(self, row_ptr, col_idx, X, labels, num_classes, split, cluster_ids, num_clusters):
        self.row_ptr = np.asarray(row_ptr, dtype=np.int64)
        self.col_idx = np.asarray(col_idx, dtype=np.int64)
        self.n = len(self.row_ptr) - 1
        self.X = np.asarray(X, dtype=np.float64)
        self.labels = np.asarray(labels, dtype=np.int64)
        self.num_classes = int(num_classes)
        self.split = np.asarray(split, dtype=np.int64)
        self.cluster_ids = np.asarray(cluster_ids, dtype=np.int64)
        self.num_clusters = int(num_clusters)
        assert self.X.shape == (self.n, self.dims[0]) and self.dims[-1] == self.num_classes

    def init_params(self, seed: int):
        self.theta = glorot_init(self.arch, self.dims, seed)
        self.reset_moments()

    def reset_moments(self):
        """Global Adam moments (zero) and step counter for opt_state == "persistent"."""
        self.mom = [np.zeros_like(w) for w in self.theta]
        self.vel = [np.zeros_like(w) for w in self.theta]
        self.t_global = 0

    def set_params(self, theta):
        self.theta = [np.asarray(w, dtype=np.float64).copy() for w in theta]
        if not hasattr(self, "mom"):
            self.reset_moments()

    # subGCNs (Alg. 1 line "subGCNs")
    def partition(self, seed: int, m: int):
        self.m = m
        self.blocks = sample_partition(self.dims, m, seed, self.round)
        self.index_sets = [sub_index_sets(self.arch, self.dims, self.blocks, i) for i in range(m)]
        self.sub = [extract(self.theta, s) for s in self.index_sets]
        if self.opt_state == "persistent":      # f3: slice the global moments like the weights
            self.opt = [[{"m": mm, "v": vv, "t": self.t_global}
                         for mm, vv in zip(extract(self.mom, s), extract(self.vel, s))] for s in self.index_sets]
        else:
            self.opt = [[{} for _ in self.theta] for _ in range(m)]   # reset per round (R8)

    def make_batch(self, slot: int, step: int):
        chosen = batch_schedule(self.num_clusters, self.clusters_per_batch, self.batch_seed, slot, step)
        nodes = batch_nodes(self.cluster_ids, chosen)
        rp, ci = induced_subgraph(self.row_ptr, self.col_idx, nodes)
        return nodes, rp, ci

    def operator(self, rp, ci, n):
        if self.arch == "gat":
            return gat_structure(rp, ci, n)
        return gcn_operator(rp, ci, n) if self.arch == "gcn" else sage_operator(rp, ci, n)

    def train_step(self, slot: int, step: int, lr: float) -> float:
        """One subTrain application."""
        nodes, rp, ci = self.make_batch(slot, step)
        op = self.operator(rp, ci, len(nodes))
        W = self.sub[slot]
        tape = forward(self.arch, W, op, self.X[nodes])
        loss, dlog = softmax_ce(tape["logits"], self.labels[nodes], self.split[nodes] == 0)
        grads = backward(self.arch, W, op, tape, dlog)
        for l in range(len(W)):
            if self.optimizer == "adam":
                W[l] = adam_step(W[l], grads[l], self.opt[slot][l], lr, self.beta1, self.beta2, self.eps)
            else:
                W[l] = sgd_step(W[l], grads[l], lr)
        self.last_trace[slot] = {"nodes": nodes, "tape": tape, "loss": loss,
                                 "dlogits": dlog, "grads": grads}
        return loss

    def subtrain(self, local_iters: int, lr: float) -> np.ndarray:
        """zeta = local_iters steps for every sub-GCN; returns mean loss per slot."""
        losses = np.zeros(self.m)
        for i in range(self.m):                   # slots are independent
            for z in range(local_iters):
                losses[i] += self.train_step(i, self.step + z, lr)
        self.step += local_iters
        return losses / max(local_iters, 1)

    # subAgg
    def aggregate(self):
        aggregate(self.theta, self.sub, self.index_sets)
        if self.arch == "gat":   # R21: the output layer's attention rows are shared by all m sub-GCNs
            self._mean_shared_rows(self.theta, self.sub)
        if self.opt_state == "persistent" and self.optimizer == "adam":  # f3: moments written back too
            aggregate(self.mom, [[st["m"] for st in o] for o in self.opt], self.index_sets)
            aggregate(self.vel, [[st["v"] for st in o] for o in self.opt], self.index_sets)
            if self.arch == "gat":
                self._mean_shared_rows(self.mom, [[st["m"] for st in o] for o in self.opt])
                self._mean_shared_rows(self.vel, [[st["v"] for st in o] for o in self.opt])
            self.t_global = self.opt[0][0].get("t", self.t_global)
        self.round += 1
        self.sub = None

    def _mean_shared_rows(self, theta, subs):
        """GAT (R21): the class dimension d_L is not partitioned, so the attention vectors of
        the last layer (its rows d_{L-1}, d_{L-1} + 1) are trained by every sub-GCN; subAgg sets
        them to the mean of the m trained copies (replacement stays for every disjoint entry)."""
        L = len(self.dims) - 1
        d = self.dims[L - 1]
        theta[L - 1][d:d + 2] = np.mean([sub[L - 1][-2:] for sub in subs], axis=0)

    def eval_theta(self, eval_scale: str = "none"):
        """The weights the evaluation forward uses.  R10 (the theory scales the
        global output by 1/m so that E[sub-GCN output] = global output): "none" (default) = Eq. (1)
        as written; "mean" = every contraction over a partitioned input dimension -- the hidden
        dims d_1..d_{L-1}, i.e. layers l >= 1 -- is scaled by 1/m (m of the last partition), done
        by scaling those layers' W rows (GAT: the W rows, not the attention vectors)."""
        if eval_scale == "none" or self.m <= 1:
            return self.theta
        out = [self.theta[0]]
        for l in range(1, len(self.theta)):
            w = self.theta[l].copy()
            rows = self.dims[l] if self.arch == "gat" else w.shape[0]
            w[:rows] /= self.m
            out.append(w)
        return out

    def eval(self, split_code: int, eval_scale: str = "none"):
        """Forward of the global model on the full graph (R10: no output scaling by default)."""
        op = self.operator(self.row_ptr, self.col_idx, self.n)
        logits = forward(self.arch, self.eval_theta(eval_scale), op, self.X)["logits"]
        rows = self.split == split_code
        loss, _ = softmax_ce(logits, self.labels, rows)
        acc = float(np.mean(np.argmax(logits[rows], axis=1) == self.labels[rows])) if rows.any() else 0.0
        return loss, acc, logits

    def eval_partitions(self, split_code: int, part_ids, num_parts: int, parts=None, logits_out=None,
                        eval_scale: str = "none"):
        """Partition-wise evaluation (Appendix "Training Ultra-Wide GCNs";
        reading R20): the graph is cut into `num_parts` partitions (part_ids[v] in
        [0, num_parts)); every partition is evaluated on its own induced subgraph with the
        training batch operator (R1/R2 on that subgraph, R10 no output scaling), and the
        score measured on each partition is averaged over the partitions that hold at least
        one node with split == split_code.  Single-label F1 (micro) = accuracy.
        `parts`: evaluate only these partition ids (the means then cover only them).
        `logits_out`: optional float array [n x d_L]; the rows of every evaluated partition's
        nodes receive their logits (also for partitions without split_code nodes).
        Returns (mean loss, mean acc, per-partition loss, per-partition acc; NaN = no
        evaluated node)."""
        part = np.asarray(part_ids, dtype=np.int64)
        assert part.shape == (self.n,) and (num_parts == 0 or (part.min() >= 0 and part.max() < num_parts))
        loss_p = np.full(num_parts, np.nan)
        acc_p = np.full(num_parts, np.nan)
        for p in (range(num_parts) if parts is None else parts):
            nodes = np.nonzero(part == p)[0]              # ascending global id
            rows = self.split[nodes] == split_code
            if not rows.any() and (logits_out is None or len(nodes) == 0):
                continue
            rp, ci = induced_subgraph(self.row_ptr, self.col_idx, nodes)
            op = self.operator(rp, ci, len(nodes))
            logits = forward(self.arch, self.eval_theta(eval_scale), op, self.X[nodes])["logits"]
            if logits_out is not None:
                logits_out[nodes] = logits
            if not rows.any():
                continue
            y = self.labels[nodes]
            loss_p[p], _ = softmax_ce(logits, y, rows)
            acc_p[p] = float(np.mean(np.argmax(logits[rows], axis=1) == y[rows]))
        ok = ~np.isnan(acc_p)
        if not ok.any():
            return 0.0, 0.0, loss_p, acc_p
        return float(np.mean(loss_p[ok])), float(np.mean(acc_p[ok])), loss_p, acc_p
