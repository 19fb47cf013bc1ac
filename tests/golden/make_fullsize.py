"""Full-size parity fixtures from the fp64 oracle (run here, once; not on the GPU box).

    PYTHONPATH=/root/repo python tests/golden/make_fullsize.py [reddit] [blogcatalog10]

Runs ``oracle/fullsize.py`` (fp64; pinned to the bit-exact chunked oracle, which is pinned to
the real reference) on the BASELINE's full-size synthetic configs (the bench's
generators and seeds: graph 0, features 1, weights 2, labels 3) and stores what the GPU test
compares (tests/test_gpu_configs.py): the loss, every parameter gradient and a fixed sample of
activation rows.  Gradients and rows are stored as fp32 (rounding 6e-8 relative, far inside
the 1e-4 bar) to keep the fixtures small.
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import fullsize as fs  # noqa: E402
from oracle import rng  # noqa: E402

N_ROWS = 128

CONFIGS = {
    # the bench headline
    "reddit": dict(model="gcn", graph="rmat", V=232965, E=114615892, F=602, H=128, C=41),
    # config 3 -- G-GCN on BlogCatalog with the edge count scaled 10x
    "blogcatalog10": dict(model="ggcn", graph="uniform", V=10312, E=6680000, F=128, H=128, C=39),
}


def sample_rows(V, n=N_ROWS, seed=11):
    return np.sort(np.random.default_rng(seed).choice(V, n, replace=False))


def param_shapes(cfg):
    F, H, C = cfg["F"], cfg["H"], cfg["C"]
    if cfg["model"] == "gcn":
        return [(F, H), (H, C)]
    return [(F, F), (F, F), (F, H), (H, H), (H, H), (H, C)]


def needed_floor(got, ref, rel=1e-4):
    """tests/conftest.py:needed_floor -- the elementwise floor ``got`` needs against ``ref``."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = float(np.abs(ref).max())
    return float(np.max((np.abs(got - ref) - rel * np.abs(ref)) / (rel * scale), initial=0.0)) if scale else 0.0


def run(cfg, s, d, X, Ws, lab, dtype):
    V = cfg["V"]
    if cfg["model"] == "gcn":
        r = fs.gcn_epoch(s, d, V, X, Ws, lab, dtype=dtype)
        return r, list(r["grads"])
    r = fs.ggcn_epoch(s, d, V, X, [tuple(Ws[0:3]), tuple(Ws[3:6])], lab, dtype=dtype)
    return r, [g for layer in r["grads"] for g in layer]


def make(name):
    cfg = CONFIGS[name]
    V, E = cfg["V"], cfg["E"]
    t0 = time.time()
    gen = rng.rmat_edges if cfg["graph"] == "rmat" else rng.uniform_edges
    s, d = gen(V, E, seed=0)
    X = rng.features(V, cfg["F"], seed=1).astype(np.float64)
    Ws = [w.astype(np.float64) for w in rng.glorot(param_shapes(cfg), seed=2)]  # fp32 values
    lab = rng.labels(V, cfg["C"], seed=3)
    print(f"{name}: inputs {time.time() - t0:.1f} s", flush=True)
    r, grads = run(cfg, s, d, X, Ws, lab, np.float64)
    print(f"{name}: fp64 epoch {time.time() - t0:.1f} s, loss {float(np.ravel(r['loss'])[0]):.9f}",
          flush=True)
    # the same epoch in fp32: how far an fp32 computation of this math lands from fp64 on each
    # tensor (its needed elementwise floor), the noise level the GPU's fp32 run is judged against
    r32, grads32 = run(cfg, s, d, X.astype(np.float32), [w.astype(np.float32) for w in Ws], lab, np.float32)
    print(f"{name}: fp32 epoch {time.time() - t0:.1f} s, loss {float(np.ravel(r32['loss'])[0]):.9f}",
          flush=True)
    rows = sample_rows(V)
    out = {"loss": np.asarray(np.ravel(r["loss"])[0], np.float64), "rows": rows,
           "loss32": np.asarray(np.ravel(r32["loss"])[0], np.float64)}
    for k, (g, g32) in enumerate(zip(grads, grads32)):
        out[f"grad{k}"] = g.astype(np.float32)
        out[f"floor32_grad{k}"] = np.float64(needed_floor(g32, g))
    for k, (h, h32) in enumerate(zip(r["out"], r32["out"])):
        out[f"out{k}_rows"] = h[rows].astype(np.float32)
        out[f"floor32_out{k}_rows"] = np.float64(needed_floor(h32[rows], h[rows]))
    print(name, {k: float(v) for k, v in out.items() if k.startswith("floor32") or k.startswith("loss")}, flush=True)
    path = os.path.join(HERE, f"fullsize_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: wrote {path} ({os.path.getsize(path) / 1e3:.0f} KB)", flush=True)


if __name__ == "__main__":
    for n in (sys.argv[1:] or list(CONFIGS)):
        make(n)
