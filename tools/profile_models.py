"""One training step of MP-GCN and GG-NN on a Reddit-sized R-MAT graph (for ncu captures).

    python tools/profile_models.py mpgcn|ggnn
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_08403_b200 as sg  # noqa: E402

which = sys.argv[1]
V, E = 232965, 114615892 // 4
g = sg.rmat_graph(V, E, seed=0)
grid = sg.ChunkGrid(g, V, gcn_weights=False)
if which == "mpgcn":
    F, C = 128, 41
    m = sg.mpgcn_model(grid, [F, 64, C])
else:
    F, C = 64, 41
    m = sg.ggnn_model(grid, F, 3, C, np.random.default_rng(5).integers(0, 3, E))
m.load_features(torch.from_numpy(sg.synthetic_features(V, F, seed=1)))
m.load_labels(np.random.default_rng(3).integers(0, C, V))
for _ in range(2):
    m.train_step(0.01)
torch.cuda.synchronize()
print(which, "loss", m.loss.item())
