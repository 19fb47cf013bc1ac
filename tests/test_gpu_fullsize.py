"""Parity at the BASELINE's full sizes, through a size-independent property.

Every destination row of a gather is an independent reduction, so the full-size GPU pass can
be checked row by row: sample rows (always including the heaviest, split ones), rebuild their
in-edge lists from the raw edge list with numpy (the canonical CSC order: by source, then
input order), and re-add the reference's terms in that order with the split
rule of oracle/saga.py:seq_sum_rows.  The GPU rows must match bit for bit (GCN) or to the
gate's tolerance (G-GCN).  Graph, features and weights are the bench's synthetic inputs.
"""

import numpy as np
import pytest
import torch

from conftest import assert_close

pytestmark = pytest.mark.gpu

T_SPLIT = 4096


def _rows_ref(keys, order_key, sample, n_keys):
    """For each sampled key: the edge ids with that key in canonical order (by order_key,
    then edge id)."""
    lut = np.zeros(n_keys, bool)
    lut[sample] = True
    eids = np.nonzero(lut[keys])[0]
    o = np.lexsort((eids, order_key[eids], keys[eids]))
    eids = eids[o]
    k = keys[eids]
    return {int(u): eids[k == u] for u in sample}


def _seq_sum(term_fn, n, T):
    """oracle/saga.py:seq_sum_rows for ONE row of n edges, streamed: a row of <= T edges is
    added left to right from 0; a longer row is split into consecutive subgroups of T edges,
    each added left to right from 0, and the partials are added in order.  np.cumsum adds
    sequentially in the array's dtype (np.sum would not), so the last cumsum row is the
    sequential fp32 sum.  ``term_fn(a, b)`` returns the fp32 terms of edges [a, b)."""
    if n <= T:
        return np.cumsum(term_fn(0, n), axis=0, dtype=np.float32)[-1]
    parts = [np.cumsum(term_fn(a, min(a + T, n)), axis=0, dtype=np.float32)[-1] for a in range(0, n, T)]
    return np.cumsum(np.stack(parts), axis=0, dtype=np.float32)[-1]


def _sample(deg, n, seed):
    r = np.random.default_rng(seed)
    heavy = np.argsort(deg)[-4:]                     # the heaviest rows (split subgroups)
    nz = np.nonzero(deg)[0]
    return np.unique(np.concatenate([heavy, r.choice(nz, n, replace=False), np.nonzero(deg == 0)[0][:2]]))


@pytest.fixture(scope="module")
def reddit():
    import paper_1810_08403_b200 as sg

    V, E, F = 232965, 114615892, 602
    g = sg.rmat_graph(V, E, seed=0)
    grid = sg.ChunkGrid(g, V)
    X = sg.synthetic_features(V, F, seed=1, ld=604)
    dout = np.bincount(g.src, minlength=V).astype(np.float64)
    din = np.bincount(g.dst, minlength=V).astype(np.float64)
    return sg, g, grid, X, dout, din


def test_reddit_layer1_gather_rows_bitwise(reddit):
    """Full Reddit-shaped layer-1 forward gather (E = 114.6M, F = 602) == the reference's
    take_rows -> mul -> segment_sum, re-added on the host, for sampled and the heaviest rows."""
    from paper_1810_08403_b200 import _lib
    from paper_1810_08403_b200 import kernels as K

    sg, g, grid, X, dout, din = reddit
    V, F = g.V, 602
    Xd = torch.from_numpy(X).cuda()[:, :F]
    out = torch.zeros((V, 604), device="cuda")[:, :F]
    K.propagate(grid.csc[(0, 0)], _lib.PROP_GCN, Xd, out, F)
    got = out.cpu().numpy()
    sample = _sample(din, 48, 1)
    rows = _rows_ref(g.dst, g.src, sample, V)
    for u, eids in rows.items():
        s = g.src[eids]
        w = (1.0 / np.sqrt(dout[s] * din[u])).astype(np.float32)
        # mul(take_rows(h, src), w) in fp32, then segment_sum's sequential adds
        ref = _seq_sum(lambda a, b: X[s[a:b], :F] * w[a:b, None], len(s), T_SPLIT) if len(s) \
            else np.zeros(F, np.float32)
        assert np.array_equal(got[u], ref), f"row {u} (in-degree {len(eids)})"


def test_reddit_layer2_backward_rows_bitwise(reddit):
    """Full-size backward dual over the transposed (CSR) index with the ReLU mask, F = 128:
    dH[v] = relu_bwd(sum_{out(v)} w_e G[dst_e], Z[v]) in CSR order, for sampled source rows."""
    from paper_1810_08403_b200 import _lib
    from paper_1810_08403_b200 import kernels as K

    sg, g, grid, X, dout, din = reddit
    V, F = g.V, 128
    G = sg.synthetic_features(V, F, seed=7)
    Z = sg.synthetic_features(V, F, seed=8)
    Gd, Zd = torch.from_numpy(G).cuda(), torch.from_numpy(Z).cuda()
    out = torch.zeros((V, F), device="cuda")
    K.propagate(grid.csr[(0, 0)], _lib.PROP_GCN, Gd, out, F, mask=Zd)
    got = out.cpu().numpy()
    sample = _sample(dout, 48, 2)
    # CSR rows list a source's edges in CSC order: by destination, then source (fixed), then id
    rows = _rows_ref(g.src, g.dst, sample, V)
    for v, eids in rows.items():
        d = g.dst[eids]
        w = (1.0 / np.sqrt(dout[v] * din[d])).astype(np.float32)
        ref = _seq_sum(lambda a, b: G[d[a:b]] * w[a:b, None], len(d), T_SPLIT) if len(d) \
            else np.zeros(F, np.float32)
        ref = ref * (Z[v] > 0.0)                          # relu bwd: g * (x > 0) (tensor.py:236)
        assert np.array_equal(got[v], ref), f"row {v} (out-degree {len(eids)})"


def test_blogcatalog10_ggcn_gather_rows():
    """Full BlogCatalog x10 G-GCN forward gather (E = 6.68M, F = 128): sampled rows vs the
    reference's sigmoid(P[src] + Q[dst]) * h[src] summed in CSC order (gate tolerance)."""
    import paper_1810_08403_b200 as sg
    from oracle import primitives as prim
    from paper_1810_08403_b200 import _lib
    from paper_1810_08403_b200 import kernels as K

    V, E, F = 10312, 6680000, 128
    g = sg.uniform_graph(V, E, seed=0)
    grid = sg.ChunkGrid(g, V, gcn_weights=False)
    h = sg.synthetic_features(V, F, seed=1)
    P = sg.synthetic_features(V, F, seed=2)
    Q = sg.synthetic_features(V, F, seed=3)
    HP = torch.from_numpy(np.concatenate([h, P], 1)).cuda()
    Qd = torch.from_numpy(Q).cuda()
    out = torch.zeros((V, F), device="cuda")
    S = torch.zeros((V, F), device="cuda")
    K.propagate(grid.csc[(0, 0)], _lib.PROP_GGCN_FWD_S, HP, out, F, g_off=F, R=Qd, out1=S)
    got, gotS = out.cpu().numpy(), S.cpu().numpy()
    din = np.bincount(g.dst, minlength=V)
    sample = _sample(din, 24, 3)
    rows = _rows_ref(g.dst, g.src, sample, V)
    ref, refS = np.zeros((len(rows), F)), np.zeros((len(rows), F))
    ref32, refS32 = np.zeros((len(rows), F), np.float32), np.zeros((len(rows), F), np.float32)
    for k, (u, eids) in enumerate(rows.items()):
        s = g.src[eids]
        eta = prim.sigmoid(P[s].astype(np.float64) + Q[u].astype(np.float64))
        ref[k] = (eta * h[s]).sum(0)
        refS[k] = (h[s] * eta * (1.0 - eta)).sum(0)
        # the same terms in fp32, added in edge order (the reference's fp32 arithmetic)
        e32 = prim.sigmoid(P[s] + Q[u])
        ref32[k] = np.cumsum(e32 * h[s], 0, dtype=np.float32)[-1] if len(s) else 0
        refS32[k] = np.cumsum(h[s] * e32 * (np.float32(1) - e32), 0, dtype=np.float32)[-1] if len(s) else 0
    keys = list(rows)
    assert_close(got[keys], ref, 1e-5, "G-GCN aggregate", ref32=ref32)
    assert_close(gotS[keys], refS, 1e-5, "S", ref32=refS32)
