"""Out-of-core GCN / G-GCN epoch on the Reddit-shaped graph (host-resident features,
activations and chunk index).

    python tools/stream_bench.py [--parts 4] [--steps 3] [--model gcn|ggcn]

Prints one JSON line: epoch ms (device events), H2D / D2H GB per epoch, device working set.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_08403_b200 as sg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", type=int, default=4)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--model", choices=["gcn", "ggcn"], default="gcn")
    a = ap.parse_args()
    V, E, dims = 232965, 114615892, [602, 128, 41]
    t0 = time.time()
    g = sg.rmat_graph(V, E, seed=0)
    grid = sg.HostGrid(g, -(-V // a.parts), gcn_weights=a.model == "gcn")
    m = (sg.StreamingGCN if a.model == "gcn" else sg.StreamingGGCN)(grid, dims)
    m.load_features(torch.from_numpy(sg.synthetic_features(V, dims[0], seed=1)))
    m.load_labels(np.random.default_rng(3).integers(0, dims[-1], V))
    setup = time.time() - t0
    m.train_step(0.01)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m.train_step(0.01)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    print(json.dumps({"workload": f"out-of-core 2-layer {a.model.upper()} epoch, Reddit-shaped",
                      "parts": a.parts,
                      "epoch_ms": round(ms, 2), "edges_per_s": E / (ms / 1e3),
                      "h2d_gb": round(m.h2d_bytes / 1e9, 3), "d2h_gb": round(m.d2h_bytes / 1e9, 3),
                      "h2d_gbs": round(m.h2d_bytes / 1e6 / ms, 1),
                      "device_working_set_gb": round(m.working_set / 1e9, 3),
                      "loss": float(m.loss.item()), "setup_s": round(setup, 1)}))


if __name__ == "__main__":
    main()
