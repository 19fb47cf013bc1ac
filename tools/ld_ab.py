"""Row padding A/B: GCN gather on the Reddit graph at F = 41 with ld 44 (16-B rows) vs 64
(128-B aligned rows)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1810_08403_b200 as sg
from paper_1810_08403_b200 import _lib
from paper_1810_08403_b200 import kernels as K
V, E = 232965, 114615892
g = sg.rmat_graph(V, E, seed=0)
grid = sg.ChunkGrid(g, V)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ws = K.Workspace(torch.device("cuda"))
res = {}
for F, ld in ((41, 44), (41, 64), (41, 48), (100, 100), (100, 128)):
    X = torch.rand((V, ld), device="cuda")[:, :F]
    out = torch.empty((V, ld), device="cuda")[:, :F]
    pi = grid.csc[(0, 0)]
    for _ in range(2):
        K.propagate(pi, _lib.PROP_GCN, X, out, F, ws=ws)
    ts = []
    for _ in range(5):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        K.propagate(pi, _lib.PROP_GCN, X, out, F, ws=ws)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    res[f"F{F}_ld{ld}"] = round(float(np.median(ts)), 3)
print(json.dumps(res))
