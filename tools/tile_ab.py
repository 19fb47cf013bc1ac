"""Source-interval tiling A/B: layer-1 forward gather over the P x P chunk grid (Locality
order, accumulating into A_j) for several P, on a bench workload.

    python tools/tile_ab.py reddit 1 2 4 8
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_08403_b200 as sg  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_1810_08403_b200 import _lib  # noqa: E402
from paper_1810_08403_b200 import kernels as K  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
Ps = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
V, E, F = cfg["V"], cfg["E"], cfg["F"]
g = (sg.rmat_graph if cfg["graph"] == "rmat" else sg.uniform_graph)(V, E, seed=0)
ld = (F + 3) // 4 * 4
X = torch.from_numpy(sg.synthetic_features(V, F, seed=1, ld=ld)).cuda()[:, :F]
out = torch.zeros((V, ld), device="cuda")[:, :F]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ws = K.Workspace(torch.device("cuda"))
res = {"config": sys.argv[1], "F": F}
for P in Ps:
    t0 = time.perf_counter()
    grid = sg.ChunkGrid(g, -(-V // P))
    setup = time.perf_counter() - t0

    def run():
        for j in range(grid.P):
            chain = [i for i in range(grid.P) if (i, j) in grid.csc]
            rows = slice(grid.begin(j), grid.begin(j) + grid.size(j))
            for k, i in enumerate(chain):
                K.propagate(grid.csc[(i, j)], _lib.PROP_GCN, X[grid.begin(i): grid.begin(i) + grid.size(i)],
                            out[rows], F, accumulate=k > 0, ws=ws)
    run()
    ts = []
    for _ in range(5):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    res[f"P{P}"] = round(float(np.median(ts)), 3)
    del grid
    torch.cuda.empty_cache()
print(json.dumps(res), flush=True)
