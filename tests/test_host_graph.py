"""Native graph store (libsagann sg_host_*) vs the oracle, byte for byte (CPU only)."""

import ctypes

import numpy as np
import pytest

import paper_1810_08403_b200 as sg
from paper_1810_08403_b200 import _lib
from paper_1810_08403_b200 import graph as G
from oracle import graph as og
from oracle import rng
from oracle import saga


def test_library_exports_every_header_symbol():
    syms = _lib.header_symbols()
    assert len(syms) > 20
    missing = [s for s in syms if not hasattr(_lib.lib, s)]
    assert not missing, missing
    so = ctypes.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert getattr(so, s) is not None
    assert _lib.lib.sg_version() >= 1


@pytest.mark.parametrize("V,E,seed", [(64, 600, 12), (1000, 20000, 3), (233, 5000, 0), (1, 10, 5)])
def test_rmat_generator_bitwise(V, E, seed):
    g = sg.rmat_graph(V, E, seed=seed)
    s, d = rng.rmat_edges(V, E, seed=seed)
    assert np.array_equal(g.src, s) and np.array_equal(g.dst, d)


@pytest.mark.parametrize("V,E,seed", [(40, 160, 11), (5000, 50000, 1)])
def test_uniform_generator_bitwise(V, E, seed):
    g = sg.uniform_graph(V, E, seed=seed)
    s, d = rng.uniform_edges(V, E, seed=seed)
    assert np.array_equal(g.src, s) and np.array_equal(g.dst, d)


def test_features_bitwise_and_padding():
    x = sg.synthetic_features(37, 13, seed=1, ld=16)
    ref = rng.features(37, 13, seed=1)
    assert np.array_equal(x[:, :13], ref)
    assert np.all(x[:, 13:] == 0)
    assert x.min() >= -1 and x.max() < 1


def test_rmat_is_skewed():
    g = sg.rmat_graph(4096, 200000, seed=0)
    dout, din = g.degrees()
    assert din.max() > 50 * din.mean()


@pytest.mark.parametrize("V,E,size,gen", [(50, 400, 13, "u"), (64, 600, 64, "r"), (97, 900, 10, "r"),
                                          (30, 0, 7, "u"), (6, 1, 2, "u"), (1000, 30000, 128, "r")])
def test_partition_2d_bitwise(V, E, size, gen):
    s, d = (rng.uniform_edges if gen == "u" else rng.rmat_edges)(V, E, seed=7)
    if V == 6:
        s, d = np.array([4], np.int32), np.array([1], np.int32)
    g = sg.Graph(V, s, d)
    a = sg.partition_2d(g, size)
    b = og.partition_2d(s, d, V, size)
    assert a.P == b.P
    for k in ("sizes", "edge_off", "cptr_off", "rptr_off", "csc_ptr", "csc_idx", "csc_eid",
              "csr_ptr", "csr_idx", "csr_eid"):
        x, y = getattr(a, k), getattr(b, k)
        assert x.dtype == y.dtype and np.array_equal(x, y), k


@pytest.mark.parametrize("V,E,P", [(97, 900, 1), (97, 900, 3), (200, 3000, 4), (8, 7, 2)])
def test_reencode_balance_bitwise(V, E, P):
    s, d = rng.rmat_edges(V, E, seed=P)
    if V == 8:
        s, d = np.zeros(7, np.int32), np.arange(1, 8, dtype=np.int32)
    g2, perm = sg.reencode_balance(sg.Graph(V, s, d), P)
    assert np.array_equal(perm, og.reencode_balance(s, d, V, P))
    assert np.array_equal(g2.src, perm[s]) and np.array_equal(g2.dst, perm[d])


def test_gcn_weights_bitwise():
    s, d = rng.rmat_edges(300, 4000, seed=2)
    g = sg.Graph(300, s, d)
    p = sg.partition_2d(g, 300)
    w = g.gcn_weights(p.csc_eid)
    ref = og.gcn_edge_weights(s, d, 300, np.float32)[p.csc_eid]
    assert np.array_equal(w, ref)


def test_graph_format_errors():
    with pytest.raises(sg.GraphFormatError):
        sg.Graph(2, [5], [0])  # SPEC.md:129 id out of range
    with pytest.raises(sg.GraphFormatError):
        sg.Graph(2, [0, 1], [0])


def _plan_sum(ptr, t, T):
    """Evaluate a native plan on the CPU with the kernel's rule and compare to the oracle."""
    items, splits, n_slots = G.plan(ptr, T, pack_edges=5, max_rows=3)
    out = np.zeros((len(ptr) - 1, t.shape[1]), t.dtype)
    partial = np.zeros((n_slots, t.shape[1]), t.dtype)
    seen_rows = np.zeros(len(ptr) - 1, int)
    for it in items:
        if it["split"] < 0:
            for r in range(it["row_begin"], it["row_end"]):
                seen_rows[r] += 1
                acc = np.zeros(t.shape[1], t.dtype)
                for e in range(ptr[r], ptr[r + 1]):
                    acc = acc + t[e]
                out[r] = acc
        else:
            acc = np.zeros(t.shape[1], t.dtype)
            for e in range(it["e_begin"], it["e_end"]):
                acc = acc + t[e]
            partial[splits[it["split"]]["slot0"] + it["sub"]] = acc
    for sp in splits:
        seen_rows[sp["row"]] += 1
        acc = np.zeros(t.shape[1], t.dtype)
        for k in range(sp["n_sub"]):
            acc = acc + partial[sp["slot0"] + k]
        out[sp["row"]] = acc
    assert np.all(seen_rows == 1)
    return out


@pytest.mark.parametrize("T", [1, 2, 3, 7, 1000])
def test_plan_matches_split_semantics(T):
    s, d = rng.rmat_edges(60, 700, seed=1)
    p = og.partition_2d(s, d, 60, 60)
    ptr = p.csc_ptr
    t = rng.features(700, 3, dtype=np.float32)
    assert np.array_equal(_plan_sum(ptr, t, T), saga.seq_sum_rows(ptr, t, T=T))


def test_plan_split_items_first_and_cover_all_edges():
    ptr = np.array([0, 10, 10, 11, 40, 41], np.int64)
    items, splits, n_slots = G.plan(ptr, 4, pack_edges=2, max_rows=4)
    kinds = [int(i["split"]) >= 0 for i in items]
    assert kinds == sorted(kinds, reverse=True)  # split items first
    assert n_slots == 3 + 8 and len(splits) == 2


def _stage_plan(ptr, idx, w, T, G_, S, EMAX):
    from paper_1810_08403_b200._lib import nptr

    args = (nptr(ptr), nptr(idx), nptr(w), len(ptr) - 1, T, G_, S, EMAX)
    sz = np.zeros(6, np.int64)
    _lib.check(_lib.lib.sg_host_stage_plan(*args, None, None, None, None, None, None, None, nptr(sz)))
    ng, nb, ns, ne = (int(x) for x in sz[:4])
    pst = (G_ + 1 + 7) // 8 * 8
    out = dict(pieces=np.zeros((max(ng, 1) * G_, 4), np.int32), gb=np.zeros(ng + 1, np.int32),
               bso=np.zeros(nb + 1, np.int64), bs=np.zeros(max(ns, 1), np.int32),
               beo=np.zeros(nb + 1, np.int64), ent=np.zeros(max(ne, 2), np.uint64),
               pofs=np.zeros(max(nb, 1) * pst, np.uint16))
    _lib.check(_lib.lib.sg_host_stage_plan(*args, *(nptr(out[k]) for k in
                                                    ("pieces", "gb", "bso", "bs", "beo", "ent", "pofs")),
                                           nptr(sz)))
    out.update(ng=ng, nb=nb, pst=pst, n_splits=int(sz[4]), n_slots=int(sz[5]))
    return out


def _stage_sum(ptr, idx, w, X, T, G_, S, EMAX):
    """Run a staged-gather plan on the CPU with the kernel's rule (sg_propagate_staged): per
    group, batch by batch, each piece adds its run entries' terms (x * w, count times) in order;
    split subgroups into partial slots, combined in subgroup order."""
    pl = _stage_plan(ptr, idx, w, T, G_, S, EMAX)
    n_rows, F = len(ptr) - 1, X.shape[1]
    out = np.full((n_rows, F), np.nan, np.float32)
    partial = np.zeros((max(pl["n_slots"], 1), F), np.float32)
    done = np.zeros(max(pl["n_splits"], 1), int)
    for g in range(pl["ng"]):
        acc = np.zeros((G_, F), np.float32)
        for b in range(pl["gb"][g], pl["gb"][g + 1]):
            rows = pl["bs"][pl["bso"][b]: pl["bso"][b + 1]]
            assert len(rows) <= S and np.all(np.diff(rows) > 0)
            ent = pl["ent"][pl["beo"][b]: pl["beo"][b + 1]]
            po = pl["pofs"][b * pl["pst"]: b * pl["pst"] + G_ + 1]
            assert po[G_] <= EMAX
            for q in range(G_):
                for x in ent[po[q]: po[q + 1]]:
                    x = int(x)
                    slot, cnt = x & 0xFFFF, (x >> 16) & 0xFFFF
                    wv = np.uint32(x >> 32).view(np.float32)
                    t = X[rows[slot]] * wv
                    for _ in range(cnt):
                        acc[q] = acc[q] + t
        for q in range(G_):
            row, split, slot0, sn = pl["pieces"][g * G_ + q]
            if row < 0:
                continue
            if split < 0:
                out[row] = acc[q]
            else:
                partial[slot0 + (sn >> 16)] = acc[q]
                done[split] += 1
                if done[split] == (sn & 0xFFFF):
                    s4 = np.zeros(F, np.float32)
                    for k in range(sn & 0xFFFF):
                        s4 = s4 + partial[slot0 + k]
                    out[row] = s4
    return out


@pytest.mark.parametrize("T,G_,S,EMAX", [(4096, 32, 44, 1024), (16, 8, 3, 12), (7, 4, 1, 4),
                                         (64, 128, 161, 4096)])
def test_stage_plan_matches_split_semantics(T, G_, S, EMAX):
    """sg_host_stage_plan covers every edge once, keeps each row's edge order, and its pieces
    are sg_host_plan's subgroups: simulated with the staged kernel's rule it equals the oracle's
    seq_sum_rows of the GCN terms bit for bit (tiny batches exercise the batch boundaries)."""
    V, E = 150, 3000
    s, d = rng.rmat_edges(V, E, seed=4)
    p = og.partition_2d(s, d, V, V)
    ptr = p.csc_ptr.astype(np.int64)
    idx = p.csc_idx.astype(np.int32)
    w = og.gcn_edge_weights(s, d, V, np.float32)[p.csc_eid]
    X = rng.features(V, 3, dtype=np.float32)
    got = _stage_sum(ptr, idx, w, X, T, G_, S, EMAX)
    want = saga.seq_sum_rows(ptr, X[idx] * w[:, None], T=T)
    assert np.array_equal(got, want)
    _, splits, n_slots = G.plan(ptr, T)
    pl = _stage_plan(ptr, idx, w, T, G_, S, EMAX)
    assert pl["n_splits"] == len(splits) and pl["n_slots"] == n_slots


def test_stage_plan_rejects_unsorted_rows():
    ptr = np.array([0, 3], np.int64)
    idx = np.array([2, 1, 3], np.int32)
    with pytest.raises(Exception):
        _stage_plan(ptr, idx, None, 4096, 32, 8, 64)
