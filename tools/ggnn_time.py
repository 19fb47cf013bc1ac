"""GG-NN training step on a Reddit-sized R-MAT graph (E/4), CUDA-event time per step."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1810_08403_b200 as sg
V, E = 232965, 114615892 // 4
g = sg.rmat_graph(V, E, seed=0)
grid = sg.ChunkGrid(g, V, gcn_weights=False)
F, C = 64, 41
m = sg.ggnn_model(grid, F, 3, C, np.random.default_rng(5).integers(0, 3, E))
m.load_features(torch.from_numpy(sg.synthetic_features(V, F, seed=1)))
m.load_labels(np.random.default_rng(3).integers(0, C, V))
for _ in range(2):
    m.train_step(0.01)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    m.train_step(0.01)
b.record()
torch.cuda.synchronize()
print(json.dumps({"ggnn_step_ms": round(a.elapsed_time(b) / 5, 3), "E": E, "F": F}))
