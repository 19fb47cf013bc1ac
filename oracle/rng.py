"""Counter-based synthetic data generator (test infrastructure only).

Restates, in numpy uint64 arithmetic, the generator the product implements in
C++ (``paper_1810_08403_b200/csrc/host_graph.cpp``) so that synthetic graphs and
features are a pure function of (seed, index) and identical on every side.
The generator itself is a build decision: the
reference pins no generator; SURVEY.md §8(d) pins the shapes, seeds
(graph 0, features 1, weights 2, labels 3) and R-MAT parameters.

    splitmix64(x):  z = x + 0x9E3779B97F4A7C15
                    z = (z ^ z>>30) * 0xBF58476D1CE4E5B9
                    z = (z ^ z>>27) * 0x94D049BB133111EB
                    return z ^ z>>31
    stream_key(seed, stream) = splitmix64(seed * 256 + stream)
    draw(seed, stream, i)    = splitmix64(stream_key + i)
    u53(h)                   = (h >> 11) * 2^-53            (double in [0,1))
"""

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

STREAM_UNIFORM = 1
STREAM_FEATURE = 2
STREAM_RMAT = 3

RMAT_ABC = (0.57, 0.19, 0.19)  # R-MAT (0.57, 0.19, 0.19, 0.05)


def splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def stream_key(seed, stream):
    with np.errstate(over="ignore"):
        return splitmix64(np.uint64(seed) * np.uint64(256) + np.uint64(stream))


def draw(seed, stream, idx):
    key = stream_key(seed, stream)
    with np.errstate(over="ignore"):
        return splitmix64(key + np.asarray(idx, dtype=np.uint64))


def u53(h):
    return (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def rmat_thresholds(abc=RMAT_ABC):
    a, b, c = abc
    t1 = a
    t2 = a + b
    t3 = t2 + c
    return t1, t2, t3


def rmat_scale(V):
    s = 0
    while (1 << s) < V:
        s += 1
    return max(s, 1)


def rmat_edges(V, E, seed=0, abc=RMAT_ABC, edge_begin=0):
    """R-MAT edges [edge_begin, edge_begin+E): quadrant per level from one draw.

    Level l of edge k uses draw(seed, STREAM_RMAT, k*scale + l); quadrant
    a=(0,0) b=(0,1) c=(1,0) d=(1,1) as (src bit, dst bit), MSB first; ids are
    folded into [0, V) with ``% V`` ("ids truncated to V").
    """
    s = rmat_scale(V)
    t1, t2, t3 = rmat_thresholds(abc)
    k = np.arange(edge_begin, edge_begin + E, dtype=np.uint64)
    src = np.zeros(E, dtype=np.uint64)
    dst = np.zeros(E, dtype=np.uint64)
    key = stream_key(seed, STREAM_RMAT)
    for lvl in range(s):
        with np.errstate(over="ignore"):
            h = splitmix64(key + k * np.uint64(s) + np.uint64(lvl))
        u = u53(h)
        sb = (u >= t2).astype(np.uint64)
        db = ((u >= t1) & (u < t2)) | (u >= t3)
        src = (src << np.uint64(1)) | sb
        dst = (dst << np.uint64(1)) | db.astype(np.uint64)
    return (src % np.uint64(V)).astype(np.int32), (dst % np.uint64(V)).astype(np.int32)


def uniform_edges(V, E, seed=0, edge_begin=0):
    """Uniform random edges: src = draw(2k) % V, dst = draw(2k+1) % V."""
    k = np.arange(edge_begin, edge_begin + E, dtype=np.uint64)
    key = stream_key(seed, STREAM_UNIFORM)
    with np.errstate(over="ignore"):
        hs = splitmix64(key + k * np.uint64(2))
        hd = splitmix64(key + k * np.uint64(2) + np.uint64(1))
    return (hs % np.uint64(V)).astype(np.int32), (hd % np.uint64(V)).astype(np.int32)


def features(V, F, seed=1, dtype=np.float32, row_begin=0):
    """x[v, f] = (draw(seed, FEATURE, v*F + f) >> 40) * 2^-23 - 1, exact in fp32."""
    idx = (np.arange(row_begin, row_begin + V, dtype=np.uint64)[:, None] * np.uint64(F)
           + np.arange(F, dtype=np.uint64)[None, :])
    h = draw(seed, STREAM_FEATURE, idx)
    k = (h >> np.uint64(40)).astype(np.float32)
    x = k * np.float32(1.0 / 8388608.0) - np.float32(1.0)
    return x.astype(dtype)


def glorot(shapes, seed=2, dtype=np.float32):
    """Glorot-uniform weights from ``default_rng(seed)`` in list order."""
    rng = np.random.default_rng(seed)
    out = []
    for fin, fout in shapes:
        lim = np.sqrt(6.0 / (fin + fout))
        out.append(rng.uniform(-lim, lim, (fin, fout)).astype(dtype))
    return out


def labels(V, C, seed=3):
    return np.random.default_rng(seed).integers(0, C, V).astype(np.int64)
