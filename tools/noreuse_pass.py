"""The bench's no-reuse point alone (for ncu): the layer-1 GCN gather on a uniform graph of
Reddit's V, E, F (X = 563 MB >> L2).  Three launches; capture the third.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:prop_kernel --launch-skip 2 --launch-count 1 python tools/noreuse_pass.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1810_08403_b200 as sg  # noqa: E402
from paper_1810_08403_b200 import _lib  # noqa: E402
from paper_1810_08403_b200 import kernels as K  # noqa: E402

V, E, F = 232965, 114615892, 602
g = sg.uniform_graph(V, E, seed=0)
grid = sg.ChunkGrid(g, V)
X = torch.from_numpy(sg.synthetic_features(V, F, seed=1, ld=604)).cuda()[:, :F]
out = torch.zeros((V, 604), device="cuda")[:, :F]   # 16-B rows: the vector path
for _ in range(3):
    K.propagate(grid.csc[(0, 0)], _lib.PROP_GCN, X, out, F)
torch.cuda.synchronize()
print("ok")
