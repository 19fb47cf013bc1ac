"""fp64 tolerance oracle for the BASELINE's full-size configs (test infrastructure only).

The bit-exact oracle (``saga.py``) composes the reference's ``tensor.py`` primitives edge by
edge (``np.add.at``), which takes ~25 min for one Reddit layer-1 pass.  At full size the parity
bar is the tolerance one (GPU fp32 vs the **fp64** oracle, 1e-4), and in fp64
the order of a row's sum is immaterial at that bar, so this module restates the same math
 with order-free fp64 kernels:

* GCN propagation ``a[u] = sum_{e in in(u)} w_e h[src_e]`` (tensor.py:424-450 composed as
  take_rows -> mul -> segment_sum) as one fp64 sparse-matrix product with A[u, v] = sum of the
  weights of the v->u edges (multi-edges kept: their weights add), row-blocked over threads;
  backward ``dh = A^T da`` (tensor.py:431-434, :447-448);
* G-GCN gated propagation (hoisted: P = h W_H, Q = h W_C) and its two
  backward duals on destination-sorted edge blocks with
  ``np.add.reduceat``;
* ApplyVertex, ReLU, softmax-CE and their backward rules are ``primitives.py`` (tensor.py:207,
  :235-236, :306-319, :487-506) unchanged.

It is pinned against ``saga.gcn_epoch`` / ``saga.ggcn_epoch`` (themselves pinned bit-for-bit to
the real reference) on small graphs to 1e-12 in fp64 (tests/test_oracle_fullsize.py).
``tests/golden/make_fullsize.py`` runs it once to produce the full-size fixtures.
"""

from concurrent.futures import ThreadPoolExecutor
import os

import numpy as np

from . import primitives as prim

_THREADS = max(1, min(16, os.cpu_count() or 1))


# ------------------------------------------------------------------ GCN (sparse product)
def gcn_operator(src, dst, V, w, dtype=np.float64):
    """CSR matrix A (rows = destinations) with A[u, v] = sum of w_e over the edges v -> u."""
    import scipy.sparse as sp

    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    A = sp.csr_matrix((np.asarray(w, dtype), (dst, src)), shape=(V, V), dtype=dtype)
    A.sum_duplicates()
    return A


def _spmm(A, H):
    """A @ H in A's dtype, row blocks over threads (scipy's kernels release the GIL)."""
    V = A.shape[0]
    n = _THREADS
    bounds = [V * k // n for k in range(n + 1)]
    H = np.ascontiguousarray(H, A.dtype)
    out = np.empty((V, H.shape[1]), A.dtype)

    def blk(k):
        b, e = bounds[k], bounds[k + 1]
        if e > b:
            out[b:e] = A[b:e] @ H

    with ThreadPoolExecutor(n) as ex:
        list(ex.map(blk, range(n)))
    return out


def gcn_forward(src, dst, V, X, Ws, labels, A=None, dtype=np.float64):
    """Forward half of gcn_epoch: dict(A, AT, a, z, out, loss, p, labels, Ws)."""
    if A is None:
        din = np.bincount(dst, minlength=V).astype(np.float64)
        dout = np.bincount(src, minlength=V).astype(np.float64)
        w = 1.0 / np.sqrt(dout[src] * din[dst])
        A = gcn_operator(src, dst, V, w.astype(dtype), dtype)
    Ws = [np.asarray(W, dtype) for W in Ws]
    hs, As, Zs = [np.asarray(X, dtype)], [], []
    for W in Ws:
        a = _spmm(A, hs[-1])
        z = a @ W
        As.append(a)
        Zs.append(z)
        hs.append(prim.relu(z))
    loss, p = prim.softmax_cross_entropy(hs[-1], labels)
    return dict(A=A, AT=None, a=As, z=Zs, out=hs[1:], loss=loss, p=p, labels=labels, Ws=Ws)


def gcn_backward(f, masks=None):
    """Backward half: parameter gradients from gcn_forward's cache.  ``masks`` (one bool array
    per layer) replaces z_l > 0 in the ReLU backward (saga.gcn_epoch's kink routing)."""
    if f["AT"] is None:
        f["AT"] = f["A"].T.tocsr()
    dtype = f["z"][0].dtype
    g = prim.softmax_cross_entropy_bwd(np.asarray(1.0, dtype), f["p"], f["labels"])
    L = len(f["Ws"])
    grads = [None] * L
    for l in range(L - 1, -1, -1):
        gz = prim.relu_bwd(g, f["z"][l]) if masks is None else g * masks[l]
        ga, grads[l] = prim.matmul_bwd(gz, f["a"][l], f["Ws"][l])
        if l > 0:
            g = _spmm(f["AT"], ga)
    return grads


def gcn_epoch(src, dst, V, X, Ws, labels, A=None, AT=None, dtype=np.float64, masks=None):
    """L-layer GCN forward + backward in ``dtype`` (fp64: the tolerance oracle; fp32: an fp32
    run of the same math, whose distance from fp64 measures the fp32 rounding noise of each
    tensor) -- same structure as saga.gcn_epoch.

    Returns dict(loss, out=[h_1..h_L], z=[...], a=[...], grads=[dW...])."""
    f = gcn_forward(src, dst, V, X, Ws, labels, A=A, dtype=dtype)
    f["AT"] = AT
    grads = gcn_backward(f, masks)
    return dict(loss=f["loss"], p=f["p"], a=f["a"], z=f["z"], out=f["out"], grads=grads)


# ------------------------------------------------------------------ G-GCN (edge blocks)
class SortedEdges:
    """Edges sorted by a key vertex (destination for CSC, source for CSR), in blocks of
    about ``block`` edges that never split a key's run."""

    def __init__(self, key, other, V, block=1 << 20):
        key = np.asarray(key, np.int64)
        o = np.argsort(key, kind="stable")
        self.key, self.other = key[o], np.asarray(other, np.int64)[o]
        self.ptr = np.zeros(V + 1, np.int64)
        np.cumsum(np.bincount(self.key, minlength=V), out=self.ptr[1:])
        cuts = np.searchsorted(self.ptr, np.arange(0, self.ptr[-1], block), side="right") - 1
        rows = np.unique(np.concatenate([cuts, [V]]))
        self.blocks = list(zip(rows[:-1], rows[1:]))

    def each(self):
        """Yield (row_begin, row_end, key[e], other[e], seg_starts, nonempty_rows)."""
        for r0, r1 in self.blocks:
            e0, e1 = self.ptr[r0], self.ptr[r1]
            if e1 == e0:
                continue
            deg = np.diff(self.ptr[r0:r1 + 1])
            nz = np.nonzero(deg)[0]
            starts = (self.ptr[r0:r1][nz] - e0).astype(np.int64)
            yield r0, r1, self.key[e0:e1], self.other[e0:e1], starts, nz + r0


def _seg(out, t, starts, rows):
    out[rows] += np.add.reduceat(t, starts, axis=0)


def ggcn_fwd(csc, h, P_, Q_):
    """a[u] = sum_{in(u)} sigmoid(P[v] + Q[u]) * h[v]."""
    a = np.zeros_like(h)
    for _, _, u, v, st, rows in csc.each():
        eta = prim.sigmoid(P_[v] + Q_[u])
        _seg(a, eta * h[v], st, rows)
    return a


def ggcn_bwd(csc, csr, h, P_, Q_, Ga):
    """(dQ, dP, dH) exactly as saga.ggcn_propagate_bwd: t_e = (Ga[u] h[v]) eta (1 - eta);
    dQ[u] = sum_in(u) t_e, dP[v] = sum_out(v) t_e, dH[v] = sum_out(v) Ga[u] eta."""
    dQ, dP, dH = np.zeros_like(h), np.zeros_like(h), np.zeros_like(h)
    for _, _, u, v, st, rows in csc.each():
        eta = prim.sigmoid(P_[v] + Q_[u])
        _seg(dQ, prim.sigmoid_bwd(Ga[u] * h[v], eta), st, rows)
    for _, _, v, u, st, rows in csr.each():
        eta = prim.sigmoid(P_[v] + Q_[u])
        Gu = Ga[u]
        _seg(dP, prim.sigmoid_bwd(Gu * h[v], eta), st, rows)
        _seg(dH, Gu * eta, st, rows)
    return dQ, dP, dH


def ggcn_epoch(src, dst, V, X, layers, labels, block=1 << 20, dtype=np.float64):
    """L-layer hoisted G-GCN forward + backward in ``dtype`` (same structure as
    saga.ggcn_epoch); ``layers`` = [(W_H, W_C, W), ...]."""
    csc = SortedEdges(dst, src, V, block)
    csr = SortedEdges(src, dst, V, block)
    hs, cache = [np.asarray(X, dtype)], []
    for (WH, WC, W) in layers:
        h = hs[-1]
        P_ = h @ np.asarray(WH, dtype)
        Q_ = h @ np.asarray(WC, dtype)
        a = ggcn_fwd(csc, h, P_, Q_)
        z = a @ np.asarray(W, dtype)
        cache.append((h, P_, Q_, a, z))
        hs.append(prim.relu(z))
    loss, p = prim.softmax_cross_entropy(hs[-1], labels)
    g = prim.softmax_cross_entropy_bwd(np.asarray(1.0, dtype), p, labels)
    grads = [None] * len(layers)
    for l in range(len(layers) - 1, -1, -1):
        WH, WC, W = (np.asarray(x, dtype) for x in layers[l])
        h, P_, Q_, a, z = cache[l]
        gz = prim.relu_bwd(g, z)
        ga, gW = prim.matmul_bwd(gz, a, W)
        dQ, dP, dH = ggcn_bwd(csc, csr, h, P_, Q_, ga)
        gh_q, gWC = prim.matmul_bwd(dQ, h, WC)
        gh_p, gWH = prim.matmul_bwd(dP, h, WH)
        grads[l] = (gWH, gWC, gW)
        g = (dH + gh_q) + gh_p
    return dict(loss=loss, p=p, out=hs[1:], grads=grads)
