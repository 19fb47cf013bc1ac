"""Bisect helper: one small GCN step with a chosen GEMM path (run under ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1810_08403_b200 as sg
from paper_1810_08403_b200 import _lib
prec = {"f32": _lib.GEMM_F32, "tc": _lib.GEMM_TF32X3}[sys.argv[1]]
V, E = 3000, 30000
g = sg.rmat_graph(V, E, seed=1)
grid = sg.ChunkGrid(g, V)
m = sg.gcn_model(grid, [64, 32, 8], gemm_prec=prec)
m.load_features(torch.from_numpy(sg.synthetic_features(V, 64)))
m.load_labels(np.random.default_rng(3).integers(0, 8, V))
for _ in range(2):
    m.train_step(0.01)
torch.cuda.synchronize()
print("ok", sys.argv[1], m.loss.item())
