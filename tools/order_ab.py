"""Edge-order A/B: the Reddit layer-1 GCN gather (CSC fwd / CSR bwd) on the R-MAT edge list in
generation order vs the same multiset sorted by (dst, src) and by (src, dst).

    python tools/order_ab.py [F ...]
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
g0 = sg.rmat_graph(V, E, seed=0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ws = K.Workspace(torch.device("cuda"))
Fs = [int(x) for x in sys.argv[1:]] or [602, 128]
for name, order in (("generation", None), ("dst_src", np.lexsort((g0.src, g0.dst))),
                    ("src_dst", np.lexsort((g0.dst, g0.src)))):
    g = g0 if order is None else sg.Graph(V, g0.src[order], g0.dst[order])
    grid = sg.ChunkGrid(g, V)
    res = {"order": name}
    for F in Fs:
        ld = (F + 3) // 4 * 4
        X = torch.rand((V, ld), device="cuda")[:, :F]
        out = torch.empty((V, ld), device="cuda")[:, :F]
        for pi, pn in ((grid.csc[(0, 0)], "csc"), (grid.csr[(0, 0)], "csr")):
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
            res[f"F{F}_{pn}"] = round(float(np.median(ts)), 3)
    print(json.dumps(res), flush=True)
    del grid
    torch.cuda.empty_cache()
