"""Pin the fp64 full-size oracle (oracle/fullsize.py) to the bit-exact chunked oracle
(oracle/saga.py, itself pinned to the real reference's golden outputs) on small graphs."""

import numpy as np
import pytest

from oracle import fullsize as fs
from oracle import graph as og
from oracle import rng
from oracle import saga


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("gen,V,E", [("rmat", 300, 5000), ("uniform", 257, 3000), ("uniform", 50, 0)])
def test_fullsize_gcn_epoch_matches_chunked_oracle(gen, V, E):
    s, d = (rng.rmat_edges if gen == "rmat" else rng.uniform_edges)(V, E, seed=4)
    X = rng.features(V, 23, seed=1, dtype=np.float64)
    Ws = [w.astype(np.float64) for w in rng.glorot([(23, 16), (16, 5)], seed=2)]
    lab = rng.labels(V, 5)
    part = og.partition_2d(s, d, V, 100)
    ref = saga.gcn_epoch(part, X, Ws, lab, og.gcn_edge_weights(s, d, V, np.float64))
    got = fs.gcn_epoch(s, d, V, X, Ws, lab)
    assert abs(float(np.ravel(got["loss"])[0]) - float(np.ravel(ref["loss"])[0])) <= 1e-12
    for k in range(2):
        assert _rel(got["out"][k], ref["out"][k]) <= 1e-12
        assert _rel(got["grads"][k], ref["grads"][k]) <= 1e-12 or E == 0


@pytest.mark.parametrize("gen,V,E", [("rmat", 200, 3000), ("uniform", 120, 900)])
def test_fullsize_ggcn_epoch_matches_chunked_oracle(gen, V, E):
    s, d = (rng.rmat_edges if gen == "rmat" else rng.uniform_edges)(V, E, seed=5)
    F, H, C = 12, 8, 4
    X = rng.features(V, F, seed=1, dtype=np.float64)
    Ls = [w.astype(np.float64) for w in rng.glorot([(F, F), (F, F), (F, H), (H, H), (H, H), (H, C)], seed=2)]
    layers = [tuple(Ls[0:3]), tuple(Ls[3:6])]
    lab = rng.labels(V, C)
    part = og.partition_2d(s, d, V, 64)
    ref = saga.ggcn_epoch(part, X, layers, lab)
    got = fs.ggcn_epoch(s, d, V, X, layers, lab, block=257)   # small blocks: many cuts
    assert abs(float(np.ravel(got["loss"])[0]) - float(np.ravel(ref["loss"])[0])) <= 1e-12
    for k in range(2):
        assert _rel(got["out"][k], ref["out"][k]) <= 1e-12
        for gg, gr in zip(got["grads"][k], ref["grads"][k]):
            assert _rel(gg, gr) <= 1e-11
