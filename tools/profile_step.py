"""One Reddit-shaped GCN training step after one warm-up step (for ncu captures).

    ncu --set full --clock-control none -k regex:'prop_kernel|gemm_tma' --launch-skip 8 \
        --launch-count 8 -o gpurun_out/step python tools/profile_step.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_08403_b200 as sg  # noqa: E402

V, E, F, H, C = 232965, 114615892, 602, 128, 41
g = sg.rmat_graph(V, E, seed=0)
grid = sg.ChunkGrid(g, V)
m = sg.gcn_model(grid, [F, H, C])
m.load_features(torch.from_numpy(sg.synthetic_features(V, F, seed=1)))
m.load_labels(np.random.default_rng(3).integers(0, C, V))
for _ in range(2):
    m.train_step(0.01)
torch.cuda.synchronize()
print("loss", m.loss.item())
