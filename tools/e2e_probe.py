"""Where the end-to-end overhead goes: Reddit GCN epochs as CUDA-graph replays with
(a) no input copies, (b) per-step H2D staging on the copy stream but no move into place,
(c) the bench's full e2e loop (H2D staging + D2D move + loss read)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_08403_b200 as sg  # noqa: E402

V, E, F, H, C = 232965, 114615892, 602, 128, 41
g = sg.rmat_graph(V, E, seed=0)
grid = sg.ChunkGrid(g, V)
m = sg.gcn_model(grid, [F, H, C])
X_host = torch.from_numpy(sg.synthetic_features(V, F, seed=1)).pin_memory()
lab = torch.from_numpy(np.random.default_rng(3).integers(0, C, V)).pin_memory()
m.load_features(X_host)
m.load_labels(lab)
m.capture(0.01)
torch.cuda.synchronize()
n = 10


def run(mode):
    torch.cuda.synchronize()
    t = time.perf_counter()
    if mode != "a":
        m.prefetch_inputs(X_host, lab)
    for k in range(n):
        if mode == "b":
            m._staged = None          # staged copy is never moved into place
            m.graph.replay()
        else:
            m.replay()
        if mode != "a" and k + 1 < n:
            m.prefetch_inputs(X_host, lab)
        float(m.loss.item())
    return (time.perf_counter() - t) / n * 1e3


for mode in ("a", "b", "c", "a", "c"):
    print(mode, round(run(mode), 3), flush=True)


def dev(fn, k=10):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


print("device ms, graph replay", round(dev(lambda: m.graph.replay()), 3))
print("device ms, eager train_step", round(dev(lambda: m.train_step(0.01)), 3))
print("device ms, graph replay", round(dev(lambda: m.graph.replay()), 3))
