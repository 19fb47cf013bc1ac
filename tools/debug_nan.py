"""Strict-mode check of a NaN feature row, printing where the NaN goes (f32 and bf16)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_08403_b200 as sg  # noqa: E402
from oracle import rng  # noqa: E402

V, E, F, H, C = 500, 6000, 64, 16, 4
s, d = rng.rmat_edges(V, E, seed=2)
grid = sg.ChunkGrid(sg.Graph(V, s, d), V)
for dtype in ("f32", "bf16"):
    for bad in (np.nan, -np.inf):
        m = sg.gcn_model(grid, [F, H, C], dtype=dtype)
        X = rng.features(V, F, seed=1)
        X[int(s[0])] = bad
        m.load_features(torch.from_numpy(X))
        m.load_labels(rng.labels(V, C))
        m.forward()
        m.backward()
        torch.cuda.synchronize()
        L0, L1 = m.layers
        nn = lambda t: int((~torch.isfinite(t.float())).sum()) if t is not None else -1  # noqa: E731
        print(dtype, bad, "X", nn(m.X), "a0", nn(L0.a), "z0", nn(L0.z), "h1", nn(L0.hout), "a1", nn(L1.a),
              "z1", nn(L1.z), "loss", m.loss.item(), "flag", int(m.nonfinite.item()), flush=True)
