"""One narrow-row sweep point (uniform graph) for ncu: PASS gather, F, avg degree.

    ncu --set full -k regex:prop_kernel --launch-skip 2 --launch-count 1 python tools/narrow_point.py 16 4
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1810_08403_b200 as sg  # noqa: E402
from paper_1810_08403_b200 import _lib  # noqa: E402
from paper_1810_08403_b200 import kernels as K  # noqa: E402

F, deg = int(sys.argv[1]), int(sys.argv[2])
V = min(1 << 22, (1 << 28) // deg)
g = sg.uniform_graph(V, V * deg, seed=deg)
grid = sg.ChunkGrid(g, V, gcn_weights=False)
pi = grid.csc[(0, 0)]
ld = (F + 7) // 8 * 8
X = torch.rand((V, ld), device="cuda")[:, :F]
out = torch.empty((V, ld), device="cuda")[:, :F]
for _ in range(4):
    K.propagate(pi, _lib.PROP_PASS, X, out, F)
torch.cuda.synchronize()
print("items", pi.n_items, "splits", pi.n_splits)
