"""BF16-operand twin of the GAT sub-GCN step (test infrastructure; reading R13 / R21).

The BF16 mode of the library (include/gist.h, R13) stores what its tensor cores and gathers
read in bf16 and accumulates in fp32.  The north_star gates the BF16 mode at 2e-2 against the
FP64 oracle.  For GAT (R21) that gate is below what bf16 storage allows: the attention
gradient is a softmax-backward difference, d e_ij = alpha_ij (G_i . Z_j - S_i), whose inputs
change by O(2^-9) when the forward operands are rounded to bf16, and the gradient of the
weights picks that up with an amplification of 5-20 on small graphs (tests/test_bf16_twin.py
measures it).  This twin makes the floor checkable: it is the FP64 GAT step of the oracle
(oracle/gist_oracle.py forward / backward for arch "gat", restated here, not imported), with
the values rounded to bf16 exactly where the CUDA path stores bf16:

  X (features)            bf16 (gist_load_graph stores X in the mode's element type)
  W in Z = H W, dH = dZ W^T  bf16 shadow of the fp32 master weights (the scores use fp32 W a)
  Z = H W                 bf16 (gathered by the attention passes)
  H (hidden outputs)      bf16 after ReLU (the next layer's GEMM operand)
  dlogits, dZ, dH         bf16 (gathered / GEMM operands of the backward)
  logits, s, t, alpha, S_i, dt, ds, dW, d a   fp64 here (fp32 on the device)

With rounding off (rnd=None) it reproduces the oracle's gradients to rounding error (pinned in
tests/test_bf16_twin.py).  It shares no code with the CUDA path.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

SLOPE = 0.2


def bf16(x) -> np.ndarray:
    """Round to the nearest bf16 (ties to even), returned as float64."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def _softmax_ce(logits, labels, rows_mask):
    mx = logits.max(axis=1, keepdims=True)
    lse = mx[:, 0] + np.log(np.exp(logits - mx).sum(axis=1))
    p = np.exp(logits - lse[:, None])
    idx = np.nonzero(rows_mask)[0]
    d = np.zeros_like(logits)
    if len(idx) == 0:
        return 0.0, d
    y = np.asarray(labels)[idx]
    d[idx] = p[idx]
    d[idx, y] -= 1.0
    d[idx] /= len(idx)
    return float(np.sum(lse[idx] - logits[idx, y]) / len(idx)), d


def gat_step(theta, S: sp.csr_matrix, X, labels, train, rnd=bf16, where=None):
    """One GAT sub-GCN forward + backward on the batch pattern S (A + I, R21).
    rnd: rounding applied at the CUDA path's bf16 storage points (None: FP64 throughout);
    where: optional set restricting rounding to these points ("X", "W", "Z", "H", "G", "dZ", "dH").
    Returns (loss, logits, hidden activations H_1.., gradients per layer [W rows; a_src; a_dst])."""
    def r(k, x):
        x = np.asarray(x, dtype=np.float64)
        return rnd(x) if rnd is not None and (where is None or k in where) else x
    L = len(theta)
    n = S.shape[0]
    rows = np.repeat(np.arange(n), np.diff(S.indptr))
    cols = S.indices
    H = [r("X", X)]
    Zs, pres, alphas = [], [], []
    logits = None
    for l in range(L):
        d = H[l].shape[1]
        W = theta[l][:d]
        Z = r("Z", H[l] @ r("W", W))
        s = H[l] @ (W @ theta[l][d])          # scores from the fp32 master W (W a_src, W a_dst)
        t = H[l] @ (W @ theta[l][d + 1])
        pre = t[rows] + s[cols]
        e = np.where(pre > 0, pre, SLOPE * pre)
        alpha = np.empty_like(e)
        for i in range(n):
            a, b = S.indptr[i], S.indptr[i + 1]
            x = np.exp(e[a:b] - e[a:b].max())
            alpha[a:b] = x / x.sum()
        A = sp.csr_matrix((alpha, cols, S.indptr), shape=S.shape)
        out = np.asarray(A @ Z)
        Zs.append(Z)
        pres.append(pre)
        alphas.append(A)
        if l < L - 1:
            H.append(r("H", np.maximum(out, 0.0)))
        else:
            logits = out
    loss, dlog = _softmax_ce(logits, labels, train)
    G = r("G", dlog)
    grads = [None] * L
    for l in range(L - 1, -1, -1):
        d = H[l].shape[1]
        A, Z, pre = alphas[l], Zs[l], pres[l]
        a_src, a_dst = theta[l][d], theta[l][d + 1]
        if l < L - 1:
            G = G * (H[l + 1] > 0.0)             # ReLU'(0) = 0 (R3)
        dal = np.einsum("ek,ek->e", G[rows], Z[cols])
        Srow = np.bincount(rows, weights=A.data * dal, minlength=n)
        dpre = A.data * (dal - Srow[rows]) * np.where(pre > 0, 1.0, SLOPE)
        dt = np.bincount(rows, weights=dpre, minlength=n)
        ds = np.bincount(cols, weights=dpre, minlength=n)
        dZ = r("dZ", np.asarray(A.T.tocsr() @ G) + np.outer(ds, a_src) + np.outer(dt, a_dst))
        grads[l] = np.vstack([H[l].T @ dZ, (Z.T @ ds)[None, :], (Z.T @ dt)[None, :]])
        if l == 0:
            break
        G = r("dH", dZ @ r("W", theta[l][:d]).T)
    return loss, logits, H[1:], grads
