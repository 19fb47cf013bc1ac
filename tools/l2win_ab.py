"""A/B: an L2 persisting access-policy window over the first rows of the gathered feature
matrix (R-MAT concentrates degree at low vertex ids) for one layer-1 GCN pass (F = 602).

    python tools/l2win_ab.py [MB ...]
"""
import ctypes
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

cu = ctypes.CDLL("libcuda.so.1")


class Window(ctypes.Structure):
    _fields_ = [("base", ctypes.c_void_p), ("nbytes", ctypes.c_size_t), ("hit", ctypes.c_float),
                ("hitp", ctypes.c_int), ("missp", ctypes.c_int), ("pad", ctypes.c_char * 32)]


def attr(a):
    v = ctypes.c_int()
    cu.cuDeviceGetAttribute(ctypes.byref(v), a, 0)
    return v.value


V, E, F = 232965, 114615892, 602
g = sg.rmat_graph(V, E, seed=0)
grid = sg.ChunkGrid(g, V)
src = g.src if hasattr(g, "src") else None
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ws = K.Workspace(torch.device("cuda"))
ld = (F + 3) // 4 * 4
X = torch.rand((V, ld), device="cuda")[:, :F]
out = torch.empty((V, ld), device="cuda")[:, :F]
pi = grid.csc[(0, 0)]
stream = torch.cuda.current_stream().cuda_stream
res = {"max_persist_MB": attr(108) / 2**20, "max_window_MB": attr(109) / 2**20}
if src is not None:
    deg = np.bincount(np.asarray(src), minlength=V)
for i, mb in enumerate([float(x) for x in (sys.argv[1:] or [0, 16, 32, 48, 64, 96])]):
    nbytes = int(mb * 2**20)
    if nbytes:
        lim = min(nbytes, attr(108))
        assert cu.cuCtxSetLimit(6, ctypes.c_size_t(lim)) == 0
        w = Window(X.data_ptr(), min(nbytes, attr(109)), min(1.0, lim / nbytes), 2, 1)
    else:
        w = Window(0, 0, 0.0, 0, 0)
    rc = cu.cuStreamSetAttribute(ctypes.c_void_p(stream), 1, ctypes.byref(w))
    assert rc == 0, rc
    for _ in range(2):
        K.propagate(pi, _lib.PROP_GCN, X, out, F, ws=ws)
    ts = []
    for _ in range(7):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        K.propagate(pi, _lib.PROP_GCN, X, out, F, ws=ws)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    rows = nbytes // (ld * 4)
    share = float(deg[:rows].sum() / E) if src is not None else None
    res[f"{i}:{mb:g}MB"] = {"ms": round(float(np.median(ts)), 3), "rows": rows, "edge_share": share}
    cu.cuCtxResetPersistingL2Cache()
print(json.dumps(res))
