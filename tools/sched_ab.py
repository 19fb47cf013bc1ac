"""A/B of the propagation schedule on the bench workload: one JSON line of stage times.

    SG_LIB_PATH=... SG_PLAN_ORDER=row|src python tools/sched_ab.py [config] [dtype]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_08403_b200 as sg  # noqa: E402
from bench import CONFIGS, timed_epochs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
dtype = sys.argv[2] if len(sys.argv) > 2 else "f32"
cfg = CONFIGS[name]
V, E, F, H, C = cfg["V"], cfg["E"], cfg["F"], cfg["H"], cfg["C"]
g = (sg.rmat_graph if cfg["graph"] == "rmat" else sg.uniform_graph)(V, E, seed=0)
grid = sg.ChunkGrid(g, V, gcn_weights=cfg["model"] == "gcn")
kw = {"dtype": dtype} if dtype != "f32" else {}
m = (sg.gcn_model if cfg["model"] == "gcn" else sg.ggcn_model)(grid, [F, H, C], **kw)
m.load_features(torch.from_numpy(sg.synthetic_features(V, F, seed=1)))
m.load_labels(np.random.default_rng(3).integers(0, C, V))


class A:
    warmup, steps, lr = 3, 10, 0.01


flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ms, st = timed_epochs(m, A, flush)
print(json.dumps({"lib": os.path.basename(os.environ.get("SG_LIB_PATH", "libsagann.so")),
                  "order": os.environ.get("SG_PLAN_ORDER", "src"), "config": name, "dtype": dtype,
                  "epoch_ms": round(ms, 3), "loss": m.loss.item(),
                  "stages": {k: round(v, 3) for k, v in st.items()}}), flush=True)
