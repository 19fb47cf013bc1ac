"""A/B timing of one GCN propagation pass on the Reddit-shaped graph at several widths.

    SG_PROP_TEAM_MAXV=8 python tools/narrow_ab.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_08403_b200 as sg  # noqa: E402
from paper_1810_08403_b200 import _lib  # noqa: E402
from paper_1810_08403_b200 import kernels as K  # noqa: E402

V, E = 232965, 114615892
g = sg.rmat_graph(V, E, seed=0)
grid = sg.ChunkGrid(g, V)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ws = K.Workspace(torch.device("cuda"))
res = {"env": {k: v for k, v in os.environ.items() if k.startswith("SG_")}}
for F in [int(x) for x in (sys.argv[1:] or [16, 32, 41, 64, 128])]:
    ld = (F + 3) // 4 * 4
    X = torch.rand((V, ld), device="cuda")[:, :F]
    out = torch.empty((V, ld), device="cuda")[:, :F]
    for pi, name in ((grid.csc[(0, 0)], "csc"), (grid.csr[(0, 0)], "csr")):
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
        res[f"F{F}_{name}"] = round(float(np.median(ts)), 3)
print(json.dumps(res))
