"""One training step of every model family on the same Reddit-sized R-MAT graph (E/4 = 28.6M
edges), CUDA events, median of 5 after 2 warm-ups.  F = 128 (GG-NN: state 64), C = 41."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_08403_b200 as sg  # noqa: E402

V, E, C = 232965, 114615892 // 4, 41
g = sg.rmat_graph(V, E, seed=0)
lab = np.random.default_rng(3).integers(0, C, V)
res = {"V": V, "E": E}
for name in ("gcn", "ggcn", "commnet", "mpgcn", "ggnn"):
    grid = sg.ChunkGrid(g, V, gcn_weights=name == "gcn")
    F = 64 if name == "ggnn" else 128
    if name == "ggnn":
        m = sg.ggnn_model(grid, F, 3, C, np.random.default_rng(5).integers(0, 3, E))
    else:
        m = getattr(sg, f"{name}_model")(grid, [F, 128, C])
    m.load_features(torch.from_numpy(sg.synthetic_features(V, F, seed=1)))
    m.load_labels(lab)
    for _ in range(2):
        m.train_step(0.01)
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        m.train_step(0.01)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    res[name] = {"step_ms": round(ms, 3), "edges_per_s": round(E / ms * 1e3 / 1e9, 2)}
    del m, grid
    torch.cuda.empty_cache()
print(json.dumps(res))
